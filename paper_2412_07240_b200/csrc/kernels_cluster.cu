// kernels_cluster.cu -- one 2-D 256 x 256 fp64 filter epoch (BASELINE configs[1], C2) in
// ONE launch: a thread-block cluster (16 CTAs = B200's non-portable maximum, else 8)
// holds the filter's 129 x 256 complex half spectrum (528 KB) in distributed shared
// memory and exchanges it over DSMEM between the column and row passes instead of
// through HBM and kernel boundaries.
//
// CTA c of the cluster owns the columns j0 in [c N/NCTA, (c+1) N/NCTA) (column pairs):
//   prep  each CTA redundantly: regrid target (R12 / R28), grid motion (eq:gridMov
//         P:142-148), Euler-factor coefficients of the l substeps (Alg. 3, R3/R4)
//   P1    [multilinear regrid gather of the previous posterior from global memory]; the
//         column pair packed as one complex column, forward DFT along axis 1 (Alg. 1);
//         the two real columns' half spectra (k1 = 0..128) into its slab X[k1][32]
//   P2    rows k1 = c, c + NCTA, ... (of the 129): gathered from all slabs over
//         DSMEM, forward DFT along axis 0, x s Psi / N^2 (Alg. 3-4), inverse, scattered back
//   P3    column pairs: Hermitian rebuild, inverse DFT along axis 1 (Alg. 5), likelihood
//         at the moved points (eq:filt P:46), store, index-space moment sums; the sums of
//         the CTAs reduced over DSMEM -> normaliser C, closed-form predict scale
//         (Alg. 6: sum w' = s DC), mean and covariance (R14) by CTA 0.
// The shared-memory FFT is fft_any<256> (compile-time Stockham, radix 8-8-4).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "device_common.cuh"
#include "fft_smem.cuh"

namespace cg = cooperative_groups;

namespace pmf {
namespace clu {

constexpr int N = 256;
constexpr int H = N / 2 + 1;          // 129 half-spectrum rows
constexpr int NT = 256;
// cluster of NCTA CTAs (8 = portable maximum, 16 = B200's non-portable maximum)
template <int NCTA> struct CCfg {
    static constexpr int COLS = N / NCTA;                 // columns per CTA
    static constexpr int PAIRS = COLS / 2;                // column pairs per CTA
    static constexpr int RMAX = (H + NCTA - 1) / NCTA;    // rows per CTA at most
};
constexpr int LMAX = 64;              // substeps held in shared memory
constexpr int PS = N + N / 8 + 1;     // pencil stride of fft_any<256>

struct Args {
    double* W;                        // weights [filter][j1][j0]
    FilterState* st;
    const SubstepEntry* sub;
    const double* z;
    const double2* tw;                // e^{-2 pi i m / 256}
    ModelParams mp;
    LikParams lp;
    Dims d;
    double ks;                        // > 0: regrid first
};

template <int NCTA>
constexpr size_t smem_bytes() {
    using C = CCfg<NCTA>;
    return sizeof(double2) * ((size_t)H * C::COLS + 2 * (size_t)C::RMAX * PS) + sizeof(double) * (3 * LMAX + 128);
}

// bilinear interpolation (R12) of the old weights at old index coordinates (v0, v1),
// zero ghost nodes: node i contributes when 0 <= i <= N-1
__device__ __forceinline__ double gather2(const double* __restrict__ Wf, double v0, double v1) {
    const double f0 = floor(v0), f1 = floor(v1);
    const int i0 = __double2int_rz(f0), i1 = __double2int_rz(f1);
    const double a0 = v0 - f0, a1 = v1 - f1;
    const bool lo0 = i0 >= 0 && i0 <= N - 1, hi0 = i0 >= -1 && i0 <= N - 2;
    const bool lo1 = i1 >= 0 && i1 <= N - 1, hi1 = i1 >= -1 && i1 <= N - 2;
    double val = 0.0;
    if (lo0 && lo1) val = fma((1.0 - a0) * (1.0 - a1), Wf[(long long)i1 * N + i0], val);
    if (hi0 && lo1) val = fma(a0 * (1.0 - a1), Wf[(long long)i1 * N + i0 + 1], val);
    if (lo0 && hi1) val = fma((1.0 - a0) * a1, Wf[(long long)(i1 + 1) * N + i0], val);
    if (hi0 && hi1) val = fma(a0 * a1, Wf[(long long)(i1 + 1) * N + i0 + 1], val);
    return val;
}

template <bool UPDATE, bool RG, int NCTA>
__global__ void __launch_bounds__(NT, 1) k_cluster_epoch(Args a) {
    using V = double2;
    constexpr int COLS = CCfg<NCTA>::COLS, PAIRS = CCfg<NCTA>::PAIRS, RMAX = CCfg<NCTA>::RMAX;
    cg::cluster_group cluster = cg::this_cluster();
    const int c = (int)cluster.block_rank();
    const int filt = blockIdx.x / NCTA;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* X = reinterpret_cast<V*>(smem_raw);                   // [H][COLS] this CTA's slab
    V* A = X + H * COLS;                                      // [RMAX][PS] FFT buffers
    V* Bf = A + RMAX * PS;
    double* cfs = reinterpret_cast<double*>(Bf + RMAX * PS);  // [LMAX][3] h D00, h D11, h (D01 + D10)
    double* sh = cfs + 3 * LMAX;                              // scalars (below)
    double* red = sh + 40;                                    // [8 warps][8] -> CTA sums [8]
    // sh: 0..3 M, 4..5 o, 6..7 c_l, 8..11 B_l, 12 vol_l, 13 skip, 14..15 c0, 16..19 B0,
    //     24..29 linear-Gaussian exponent e(u) = q0 + q1 u0 + q2 u1 + q3 u0^2 + q4 u0 u1 + q5 u1^2
    //     in the moved grid's index coordinates (R13), 30 log normalising constant
    FilterState& f = a.st[filt];
    double* Wf = a.W + (long long)filt * N * N;
    const double* zf = a.z + (long long)filt * a.lp.nz;
    const int l = a.mp.l;

    // ---------------------------------------------------------------- prep (every CTA)
    if (tid == 0) {
        double cn[4] = {f.c[0], f.c[1], 0, 0}, Bn[16] = {f.B[0], f.B[1], 0, 0, f.B[4], f.B[5]};
        bool ok = f.status == 0;
        if (RG) {
            ok = ok && regrid_target(2, a.d.ng, f, a.ks, cn, Bn, a.d.grid);
            const double det = f.B[0] * f.B[5] - f.B[1] * f.B[4];
            const double Bi[4] = {f.B[5] / det, -f.B[1] / det, -f.B[4] / det, f.B[0] / det};
            sh[0] = fma(Bi[0], Bn[0], Bi[1] * Bn[4]);
            sh[1] = fma(Bi[0], Bn[1], Bi[1] * Bn[5]);
            sh[2] = fma(Bi[2], Bn[0], Bi[3] * Bn[4]);
            sh[3] = fma(Bi[2], Bn[1], Bi[3] * Bn[5]);
            const double d0 = cn[0] - f.c[0], d1 = cn[1] - f.c[1];
            sh[4] = fma(Bi[0], d0, fma(Bi[1], d1, 0.5 * (N - 1)));
            sh[5] = fma(Bi[2], d0, fma(Bi[3], d1, 0.5 * (N - 1)));
        }
        const double* Mt = a.mp.Mtau;
        const double Bl[4] = {fma(Mt[0], Bn[0], Mt[1] * Bn[4]), fma(Mt[0], Bn[1], Mt[1] * Bn[5]),
                              fma(Mt[4], Bn[0], Mt[5] * Bn[4]), fma(Mt[4], Bn[1], Mt[5] * Bn[5])};
        const double cl[2] = {fma(Mt[0], cn[0], Mt[1] * cn[1]), fma(Mt[4], cn[0], Mt[5] * cn[1])};
        sh[14] = cn[0];
        sh[15] = cn[1];
        sh[16] = Bn[0];
        sh[17] = Bn[1];
        sh[18] = Bn[4];
        sh[19] = Bn[5];
        sh[6] = cl[0];
        sh[7] = cl[1];
        sh[8] = Bl[0];
        sh[9] = Bl[1];
        sh[10] = Bl[2];
        sh[11] = Bl[3];
        sh[12] = fabs(Bl[0] * Bl[3] - Bl[1] * Bl[2]);
        sh[13] = ok ? 0.0 : 1.0;
        if (UPDATE && a.lp.kind == 0) {
            // r(u) = (z - H c_l) - (H B_l) u, e = r^T R^-1 r expanded in u (as the resident prep)
            double r0[4] = {0, 0, 0, 0}, G0[4] = {0, 0, 0, 0}, G1[4] = {0, 0, 0, 0};
            const int nz = a.lp.nz;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (i >= nz) break;
                const double h0 = a.lp.H[i * 4], h1 = a.lp.H[i * 4 + 1];
                r0[i] = zf[i] - fma(h0, cl[0], h1 * cl[1]);
                G0[i] = fma(h0, Bl[0], h1 * Bl[2]);
                G1[i] = fma(h0, Bl[1], h1 * Bl[3]);
            }
            double qa = 0, qb0 = 0, qb1 = 0, g00 = 0, g01 = 0, g11 = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    if (i >= nz || j >= nz) continue;
                    const double R = a.lp.Rinv[i * 4 + j];
                    qa = fma(r0[i] * R, r0[j], qa);
                    qb0 = fma(-2.0 * G0[i] * R, r0[j], qb0);
                    qb1 = fma(-2.0 * G1[i] * R, r0[j], qb1);
                    g00 = fma(G0[i] * R, G0[j], g00);
                    g01 = fma(G0[i] * R, G1[j], g01);
                    g11 = fma(G1[i] * R, G1[j], g11);
                }
            sh[24] = qa;
            sh[25] = qb0;
            sh[26] = qb1;
            sh[27] = g00;
            sh[28] = 2.0 * g01;
            sh[29] = g11;
            sh[30] = a.lp.lognorm;
        }
    }
    __syncthreads();
    if (sh[13] != 0.0) {                  // failed filter / degenerate target (uniform per cluster)
        if (c == 0 && tid == 0 && RG && f.status == 0) f.status = -6;
        return;
    }
    {
        double B0[16] = {sh[16], sh[17], 0, 0, sh[18], sh[19]}, Bi0[16];
        mat_inv4(2, B0, Bi0);
        for (int n = tid; n < l; n += NT) {
            double o[10];
            substep_coefs(2, B0, Bi0, a.mp, a.sub[n], o);
            cfs[3 * n] = o[0];
            cfs[3 * n + 1] = o[1];
            cfs[3 * n + 2] = o[2];
        }
    }
    // ---------------------------------------------------------------- P1: columns, axis 1
    double dc = 0.0;
    {
        const double M0 = sh[0], M1 = sh[1], M2 = sh[2], M3 = sh[3], o0 = sh[4], o1 = sh[5];
#pragma unroll 4
        for (int e = tid; e < PAIRS * N; e += NT) {
            const int m = e / N, j1 = e - m * N;
            const int j0 = c * COLS + 2 * m;
            double w0, w1;
            if (RG) {
                const double u1 = j1 - 0.5 * (N - 1);
                const double ua = j0 - 0.5 * (N - 1), ub = ua + 1.0;
                w0 = gather2(Wf, fma(M0, ua, fma(M1, u1, o0)), fma(M2, ua, fma(M3, u1, o1)));
                w1 = gather2(Wf, fma(M0, ub, fma(M1, u1, o0)), fma(M2, ub, fma(M3, u1, o1)));
            } else {
                w0 = Wf[j1 * N + j0];
                w1 = Wf[j1 * N + j0 + 1];
            }
            dc += w0 + w1;
            A[m * PS + sx<N>(j1)] = V{w0, w1};
        }
    }
    __syncthreads();
    {
        V* r = fft_any<N, false>(A, Bf, PAIRS, PS, FFTPlan{}, a.tw);
        // unpack the two real columns: Wa = (Z(k) + conj Z(-k))/2, Wb = (Z(k) - conj Z(-k))/(2i)
        for (int e = tid; e < PAIRS * H; e += NT) {
            const int m = e / H, k1 = e - m * H;
            const V zk = r[m * PS + sx<N>(k1)], zp = r[m * PS + sx<N>((N - k1) & (N - 1))];
            X[k1 * COLS + 2 * m] = V{0.5 * (zk.x + zp.x), 0.5 * (zk.y - zp.y)};
            X[k1 * COLS + 2 * m + 1] = V{0.5 * (zk.y + zp.y), 0.5 * (zp.x - zk.x)};
        }
    }
    cluster.sync();                       // every slab holds its columns' half spectra
    // ---------------------------------------------------------------- P2: rows, axis 0, Psi
    const int nr = (H - 1 - c) / NCTA + 1;                    // rows k1 = c + NCTA q
    for (int e = tid; e < nr * N; e += NT) {
        const int q = e / N, j0 = e - q * N;
        const V* src = cluster.map_shared_rank(X, j0 / COLS);
        A[q * PS + sx<N>(j0)] = src[(c + NCTA * q) * COLS + (j0 % COLS)];
    }
    __syncthreads();
    {
        V* r = fft_any<N, false>(A, Bf, nr, PS, FFTPlan{}, a.tw);
        const double mult = a.mp.s / ((double)N * N), ks2 = 2.0 * PMF_PI / N;
        for (int e = tid; e < nr * N; e += NT) {
            const int q = e / N, k0 = e - q * N, k1 = c + NCTA * q;
            const double kap0 = ks2 * (k0 < N / 2 ? k0 : k0 - N), kap1 = ks2 * k1;
            const double kx0 = (2 * k0 == N) ? 0.0 : kap0, kx1 = (2 * k1 == N) ? 0.0 : kap1;
            const double kk0 = kap0 * kap0, kk1 = kap1 * kap1, kxx = kx0 * kx1;
            double den = 1.0;
            for (int n = 0; n < l; ++n) den *= fma(cfs[3 * n], kk0, fma(cfs[3 * n + 1], kk1, fma(cfs[3 * n + 2], kxx, 1.0)));
            const double ps = mult / den;
            const V v = r[q * PS + sx<N>(k0)];
            r[q * PS + sx<N>(k0)] = V{v.x * ps, v.y * ps};
        }
        __syncthreads();
        V* r2 = fft_any<N, true>(r, (r == A) ? Bf : A, nr, PS, FFTPlan{}, a.tw);
        for (int e = tid; e < nr * N; e += NT) {
            const int q = e / N, j0 = e - q * N;
            V* dst = cluster.map_shared_rank(X, j0 / COLS);
            dst[(c + NCTA * q) * COLS + (j0 % COLS)] = r2[q * PS + sx<N>(j0)];
        }
    }
    cluster.sync();                       // every slab holds its columns' row-transformed values
    // ---------------------------------------------------------------- P3: columns, inverse axis 1
    for (int e = tid; e < PAIRS * N; e += NT) {
        const int m = e / N, k1 = e - m * N;
        V zz;
        if (k1 <= N / 2) {
            const V wa = X[k1 * COLS + 2 * m], wb = X[k1 * COLS + 2 * m + 1];
            zz = V{wa.x - wb.y, wa.y + wb.x};
        } else {
            const int kp = N - k1;
            const V wa = X[kp * COLS + 2 * m], wb = X[kp * COLS + 2 * m + 1];
            zz = V{wa.x + wb.y, wb.x - wa.y};
        }
        A[m * PS + sx<N>(k1)] = zz;
    }
    __syncthreads();
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    {
        V* r = fft_any<N, true>(A, Bf, PAIRS, PS, FFTPlan{}, a.tw);
        const double cl0 = sh[6], cl1 = sh[7], B00 = sh[8], B01 = sh[9], B10 = sh[10], B11 = sh[11];
        const bool quad = a.lp.kind == 0;
        const double q0 = sh[24], q1 = sh[25], q2 = sh[26], q3 = sh[27], q4 = sh[28], q5 = sh[29], lgn = sh[30];
        for (int e = tid; e < PAIRS * N; e += NT) {
            const int m = e / N, j1 = e - m * N;
            const int j0 = c * COLS + 2 * m;
            const V v = r[m * PS + sx<N>(j1)];
            const double u1 = j1 - 0.5 * (N - 1);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double u0 = (j0 + h) - 0.5 * (N - 1);
                double w = h ? v.y : v.x;
                if (UPDATE) {
                    if (quad) {
                        const double ee = fma(u0, fma(q3, u0, fma(q4, u1, q1)), fma(u1, fma(q5, u1, q2), q0));
                        w *= exp_fast(fma(-0.5, ee, lgn));
                    } else {
                        const double x[2] = {fma(B00, u0, fma(B01, u1, cl0)), fma(B10, u0, fma(B11, u1, cl1))};
                        w *= exp_fast(log_lik(a.lp, x, zf));
                    }
                    const double wu0 = w * u0;
                    acc[0] += w;
                    acc[1] += wu0;
                    acc[2] = fma(w, u1, acc[2]);
                    acc[3] = fma(wu0, u0, acc[3]);
                    acc[4] = fma(wu0, u1, acc[4]);
                    acc[5] = fma(w * u1, u1, acc[5]);
                }
                Wf[j1 * N + j0 + h] = w;
            }
        }
    }
    // ---------------------------------------------------------------- sums: warps -> CTA -> cluster
    acc[6] = dc;
#pragma unroll
    for (int i = 0; i < 7; ++i)
        for (int o = 16; o > 0; o >>= 1) acc[i] += __shfl_down_sync(0xffffffffu, acc[i], o);
    if (lane == 0)
        for (int i = 0; i < 7; ++i) red[warp * 8 + i] = acc[i];
    __syncthreads();
    if (tid < 7) {
        double s = 0.0;
        for (int w = 0; w < NT / 32; ++w) s += red[w * 8 + tid];
        red[64 + tid] = s;                                    // this CTA's sums
    }
    cluster.sync();                       // all CTA sums visible; all P3 reads of slabs done
    if (c == 0 && tid == 0) {
        double tot[7] = {0, 0, 0, 0, 0, 0, 0};
        for (int r = 0; r < NCTA; ++r) {
            const double* src = cluster.map_shared_rank(red, r);
            for (int i = 0; i < 7; ++i) tot[i] += src[64 + i];
        }
        const double vol = sh[12], s = a.mp.s, DC = tot[6];
        f.c[0] = sh[6];
        f.c[1] = sh[7];
        f.B[0] = sh[8];
        f.B[1] = sh[9];
        f.B[4] = sh[10];
        f.B[5] = sh[11];
        if (!UPDATE) {
            f.scale = 1.0 / (vol * s * DC);                   // Alg. 6 closed form
        } else {
            const double C = tot[0] / (s * DC);
            f.mass = tot[0];
            f.has_moments = 1;
            if (!(C > 0.0) || !isfinite(C) || !(tot[0] > 0.0)) {
                f.status = -6;
                f.logC = -INFINITY;
            } else {
                f.status = 0;
                f.logC = log(C);
                f.scale = 1.0 / (vol * tot[0]);
                double am[NMOM];
                for (int i = 0; i < NMOM; ++i) am[i] = 0.0;
                for (int i = 0; i < 6; ++i) am[i] = tot[i];
                finish_moments(2, am, f.c, f.B, f.mean, f.cov);
            }
        }
    }
    cluster.sync();                       // CTA 0 read the others' sums before they exit
}

}  // namespace clu

using namespace clu;

bool cluster_epoch_supported(const Dims& d, int dtype, const ModelParams& mp) {
    return d.nx == 2 && d.n[0] == N && d.n[1] == N && dtype == 0 && mp.step == 0 && mp.l <= LMAX &&
           d.ng[0] == N && d.ng[1] == N;
}

template <int NCTA, bool UPDATE, bool RG>
static cudaError_t cluster_go(const Args& a, int batch, const PencilBufs& b, cudaStream_t s) {
    auto kern = k_cluster_epoch<UPDATE, RG, NCTA>;
    const size_t smem = smem_bytes<NCTA>();
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess && NCTA > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(batch * NCTA);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = NCTA;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
    if (e != cudaSuccess || ncl < 1) return cudaErrorInvalidConfiguration;
    if (b.ev0) cudaEventRecordWithFlags(b.ev0, s, cudaEventRecordExternal);
    e = cudaLaunchKernelEx(&cfg, kern, a);
    if (b.ev1) cudaEventRecordWithFlags(b.ev1, s, cudaEventRecordExternal);
    return e != cudaSuccess ? e : cudaGetLastError();
}

template <int NCTA>
static cudaError_t cluster_n(const Args& a, int batch, const PencilBufs& b, bool up, bool rg, cudaStream_t s) {
    if (up && rg) return cluster_go<NCTA, true, true>(a, batch, b, s);
    if (up) return cluster_go<NCTA, true, false>(a, batch, b, s);
    if (rg) return cluster_go<NCTA, false, true>(a, batch, b, s);
    return cluster_go<NCTA, false, false>(a, batch, b, s);
}

cudaError_t launch_cluster_epoch(const Dims& d, PencilBufs& b, const Twiddles& tw, const ModelParams& mp,
                                 const LikParams* lp, double ks, cudaStream_t s, int64_t* launches) {
    Args a;
    a.W = (double*)b.W;
    a.st = b.st;
    a.sub = b.sub;
    a.z = b.z;
    a.tw = (const double2*)tw.tw[0];
    a.mp = mp;
    a.lp = lp ? *lp : LikParams{};
    a.d = d;
    a.ks = ks;
    // 16 CTAs per filter (non-portable cluster) when the device schedules it, else 8
    static int n16 = -1;
    cudaError_t e = cudaErrorInvalidConfiguration;
    if (n16 != 0) {
        e = cluster_n<16>(a, d.batch, b, lp != nullptr, ks > 0.0, s);
        if (n16 < 0) n16 = e == cudaSuccess ? 1 : 0;
        if (e != cudaSuccess) cudaGetLastError();            // clear, fall back
    }
    if (n16 == 0) e = cluster_n<8>(a, d.batch, b, lp != nullptr, ks > 0.0, s);
    ++*launches;
    return e;
}

}  // namespace pmf
