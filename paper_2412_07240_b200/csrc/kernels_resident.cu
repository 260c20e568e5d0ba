// kernels_resident.cu -- the fused filter-epoch kernel for batches of 2-D
// 128 x 128 filters (BASELINE configs[4], C5): ONE launch per epoch, a
// persistent CTA per SM walking the filters, each filter's whole half spectrum
// resident in shared memory.
//
// Per filter (R15 epoch order, regrid of the previous epoch fused in front):
//   P0  warp 0: grid constants -- regrid target (R12), grid motion
//       B_l = e^{A tau} B0 (eq:gridMov P:142-148), Euler-factor coefficients of
//       the l substeps (Alg. 3, R3/R4), likelihood residual plan.
//   P1  64 teams x 8 threads, team m owns the column pair j0 = 2m, 2m+1: load (or
//       multilinear regrid-gather, R12) the pair, pack it as one complex column
//       z = w(2m,.) + i w(2m+1,.), 128-point FFT along axis 1 (16 x 8, registers +
//       one shared-memory exchange), unpack the two real columns' half spectra
//       (k1 = 0..64) into X[k1][j0].                       (Alg. 1, eq:fourtrsf)
//   P2  team m owns row k1 = m (team 0: rows 0 and 64 packed as one complex row):
//       FFT along axis 0, multiply by s Psi / N^2 (Alg. 3-4), inverse FFT.
//   P3  team m: inverse FFT along axis 1 of the column pair (Hermitian rebuild),
//       normalise by the DC coefficient (Alg. 6: sum w' = s sum w), likelihood
//       (eq:filt P:46), store, moments -> normaliser C, mean and cov.
// HBM traffic: read + write each weight once (16 B/point fp64).
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "device_common.cuh"

namespace pmf {

namespace res {

constexpr int N = 128;            // points per axis
constexpr int H = N / 2 + 1;      // 65 rows of the half spectrum (k1 = 0..64)
constexpr int PITCH = 130;        // row pitch in complex elements (= 2 mod 8: conflict-free exchanges)
constexpr int NT = 512;           // threads: 64 teams x 8

template <typename T> struct K {
    static constexpr T C1 = T(0.92387953251128675613);   // cos(pi/8)
    static constexpr T S1 = T(0.38268343236508977173);   // sin(pi/8)
    static constexpr T R2 = T(0.70710678118654752440);   // 1/sqrt(2)
};

// multiply by W16^e (forward: e^{-2 pi i e/16}; inverse: conjugate)
template <int E, bool INV, typename V>
__device__ __forceinline__ V w16(V a) {
    using T = decltype(a.x);
    constexpr int e = E & 15;
    if constexpr (e == 0) return a;
    else if constexpr (e == 4) return mul_mi<INV>(a);
    else if constexpr (e == 8) return V{-a.x, -a.y};
    else if constexpr (e == 12) return mul_mi<!INV>(a);
    else if constexpr (e == 2 || e == 6 || e == 10 || e == 14) {
        // (1 - i)/sqrt2 rotated by multiples of -i
        V b = a;
        if constexpr (e == 6) b = mul_mi<INV>(a);
        else if constexpr (e == 10) b = V{-a.x, -a.y};
        else if constexpr (e == 14) b = mul_mi<!INV>(a);
        const T r = K<T>::R2;
        if (INV) return V{(b.x - b.y) * r, (b.x + b.y) * r};
        return V{(b.x + b.y) * r, (b.y - b.x) * r};
    } else {
        const double ang = 2.0 * 3.14159265358979323846 * e / 16.0;
        // compile-time constants for e = 1,3,5,7,9,11,13,15
        T c, s;
        if constexpr (e == 1 || e == 15) { c = K<T>::C1; s = K<T>::S1; }
        else if constexpr (e == 3 || e == 13) { c = K<T>::S1; s = K<T>::C1; }
        else if constexpr (e == 5 || e == 11) { c = -K<T>::S1; s = K<T>::C1; }
        else { c = -K<T>::C1; s = K<T>::S1; }
        (void)ang;
        if constexpr (e > 8) s = -s;     // sin(2 pi e/16) < 0 for e > 8
        // forward multiplier (c, -s); inverse (c, s)
        const T si = INV ? s : -s;
        return V{fma(a.x, c, -a.y * si), fma(a.x, si, a.y * c)};
    }
}

template <bool INV, typename V>
__device__ __forceinline__ void r4(V& a0, V& a1, V& a2, V& a3) {
    V s02 = cadd(a0, a2), d02 = csub(a0, a2);
    V s13 = cadd(a1, a3), d13 = mul_mi<INV>(csub(a1, a3));
    a0 = cadd(s02, s13);
    a2 = csub(s02, s13);
    a1 = cadd(d02, d13);
    a3 = csub(d02, d13);
}

// in-place 16-point DFT, natural order in and out
template <bool INV, typename V>
__device__ __forceinline__ void dft16(V* x) {
    // radix-4 over r2 for each r1: x[r1 + 4 r2] -> Y(r1, s2) at x[r1 + 4 s2]
#pragma unroll
    for (int r1 = 0; r1 < 4; ++r1) r4<INV>(x[r1], x[r1 + 4], x[r1 + 8], x[r1 + 12]);
    x[5] = w16<1, INV>(x[5]);
    x[9] = w16<2, INV>(x[9]);
    x[13] = w16<3, INV>(x[13]);
    x[6] = w16<2, INV>(x[6]);
    x[10] = w16<4, INV>(x[10]);
    x[14] = w16<6, INV>(x[14]);
    x[7] = w16<3, INV>(x[7]);
    x[11] = w16<6, INV>(x[11]);
    x[15] = w16<9, INV>(x[15]);
    // radix-4 over r1 for each s2: (x[4 s2 + r1]) -> X(s2 + 4 s1)
    V y[16];
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) {
        V a0 = x[4 * s2], a1 = x[4 * s2 + 1], a2 = x[4 * s2 + 2], a3 = x[4 * s2 + 3];
        r4<INV>(a0, a1, a2, a3);
        y[s2] = a0;
        y[s2 + 4] = a1;
        y[s2 + 8] = a2;
        y[s2 + 12] = a3;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = y[i];
}

// in-place 8-point DFT, natural order in and out
template <bool INV, typename V>
__device__ __forceinline__ void dft8(V* x) {
    using T = decltype(x[0].x);
    // radix-4 over r2 for r1 = 0, 1: x[r1 + 2 r2]
    V a0 = x[0], a1 = x[2], a2 = x[4], a3 = x[6];
    V b0 = x[1], b1 = x[3], b2 = x[5], b3 = x[7];
    r4<INV>(a0, a1, a2, a3);
    r4<INV>(b0, b1, b2, b3);
    const T r = K<T>::R2;
    // twiddle W8^{s2} on the r1 = 1 branch
    if (INV) {
        b1 = V{(b1.x - b1.y) * r, (b1.x + b1.y) * r};
        b2 = mul_mi<true>(b2);
        b3 = V{-(b3.x + b3.y) * r, (b3.x - b3.y) * r};
    } else {
        b1 = V{(b1.x + b1.y) * r, (b1.y - b1.x) * r};
        b2 = mul_mi<false>(b2);
        b3 = V{(b3.y - b3.x) * r, -(b3.x + b3.y) * r};
    }
    x[0] = cadd(a0, b0);
    x[4] = csub(a0, b0);
    x[1] = cadd(a1, b1);
    x[5] = csub(a1, b1);
    x[2] = cadd(a2, b2);
    x[6] = csub(a2, b2);
    x[3] = cadd(a3, b3);
    x[7] = csub(a3, b3);
}

// exchange slot of element (s, t) inside a row (128 consecutive complex)
__device__ __forceinline__ int rslot(int s, int t) { return s * 8 + (t ^ (s & 7)); }
// exchange slot of element (s, t) inside the column pair of a team: (row, col)
__device__ __forceinline__ int cslot(int s, int t, int m) {
    const int row = 4 * s + ((t >> 1) ^ (s & 3));
    const int col = (t & 1) ^ ((s >> 2) & 1);
    return row * PITCH + 2 * m + col;
}

struct Shared {              // per-filter constants (shared memory)
    double cl[2], Bl[4];     // moved grid
    double M[4], o[2];       // regrid map v = o + M u'
    double qa, qb[2], qG[3]; // linear-Gauss: e(u) = qa + qb.u + u^T [qG0 qG1; qG1 qG2] u
    double zr;               // range likelihood: z
    double lognorm, inv_sigma;
    double vol_l, s_over_n2;
    double dc;
    int skip;
};

}  // namespace res

using namespace res;

template <typename T>
struct ResArgs {
    T* W;
    FilterState* st;
    const double* z;
    const SubstepEntry* sub;
    ModelParams mp;
    LikParams lp;
    double ks;
    int batch;
};

template <typename T, bool REGRID, bool UPDATE>
__global__ void __launch_bounds__(NT, 1) k_resident_epoch(ResArgs<T> a) {
    using V = typename C2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* X = reinterpret_cast<V*>(smem_raw);                          // [H][PITCH]
    V* tw = X + H * PITCH;                                          // [16][8]  W128^{ts}
    Shared* sh = reinterpret_cast<Shared*>(tw + 128);
    double* red = reinterpret_cast<double*>(sh + 1);                // [16 warps][6]
    T* cf = reinterpret_cast<T*>(red + 16 * 6);                      // [l][3]

    const int tid = threadIdx.x;
    const int m = tid >> 3, t = tid & 7;
    const int lane = tid & 31, warp = tid >> 5;
    // own s pair for the 8-point stages: {t, 16 - t}, thread 0 takes {0, 8}
    const int sa = t, sb = (t == 0) ? 8 : 16 - t;
    const int l = a.mp.l;
    const int nx = 2;

    for (int i = tid; i < 128; i += NT) {
        const int s = i >> 3, tt = i & 7;
        const double ang = 2.0 * 3.14159265358979323846 * (double)(tt * s) / 128.0;
        double sn, cs;
        sincos(ang, &sn, &cs);
        tw[i] = V{(T)cs, (T)(-sn)};
    }

    for (int filt = blockIdx.x; filt < a.batch; filt += gridDim.x) {
        const long long off = (long long)filt * (N * N);
        T* Wf = a.W + off;
        // ---------------------------------------------------------------- P0
        if (warp == 0) {
            const FilterState& f = a.st[filt];
            double B[4] = {f.B[0], f.B[1], f.B[4], f.B[5]};
            double c[2] = {f.c[0], f.c[1]};
            double B0[4] = {B[0], B[1], B[2], B[3]}, c0[2] = {c[0], c[1]};
            int skip = f.status != 0;
            double detB = B[0] * B[3] - B[1] * B[2];
            double Bi[4] = {B[3] / detB, -B[1] / detB, -B[2] / detB, B[0] / detB};
            if (REGRID) {
                const double v0 = f.cov[0], v1 = f.cov[5];
                if (!(v0 > 0.0) || !(v1 > 0.0) || !isfinite(v0) || !isfinite(v1)) skip = 1;
                c0[0] = f.mean[0];
                c0[1] = f.mean[1];
                B0[0] = 2.0 * a.ks * sqrt(v0) / N;
                B0[1] = 0.0;
                B0[2] = 0.0;
                B0[3] = 2.0 * a.ks * sqrt(v1) / N;
            }
            if (lane == 0) {
                sh->skip = skip;
                if (REGRID) {
                    // v = B^-1 (c0 + B0 u' - c) + (N-1)/2
                    sh->M[0] = Bi[0] * B0[0] + Bi[1] * B0[2];
                    sh->M[1] = Bi[0] * B0[1] + Bi[1] * B0[3];
                    sh->M[2] = Bi[2] * B0[0] + Bi[3] * B0[2];
                    sh->M[3] = Bi[2] * B0[1] + Bi[3] * B0[3];
                    const double d0 = c0[0] - c[0], d1 = c0[1] - c[1];
                    sh->o[0] = fma(Bi[0], d0, fma(Bi[1], d1, 0.5 * (N - 1)));
                    sh->o[1] = fma(Bi[2], d0, fma(Bi[3], d1, 0.5 * (N - 1)));
                }
                const double* Mt = a.mp.Mtau;      // stride 4
                double Bl[4], cl[2];
                Bl[0] = fma(Mt[0], B0[0], Mt[1] * B0[2]);
                Bl[1] = fma(Mt[0], B0[1], Mt[1] * B0[3]);
                Bl[2] = fma(Mt[4], B0[0], Mt[5] * B0[2]);
                Bl[3] = fma(Mt[4], B0[1], Mt[5] * B0[3]);
                cl[0] = fma(Mt[0], c0[0], Mt[1] * c0[1]);
                cl[1] = fma(Mt[4], c0[0], Mt[5] * c0[1]);
                for (int q = 0; q < 4; ++q) sh->Bl[q] = Bl[q];
                sh->cl[0] = cl[0];
                sh->cl[1] = cl[1];
                sh->vol_l = fabs(Bl[0] * Bl[3] - Bl[1] * Bl[2]);
                sh->s_over_n2 = a.mp.s / (double)(N * N);
                // likelihood: residual r(u) = (z - H c_l) - (H B_l) u relative to the moved grid
                // centre; e(u) = r^T R^-1 r expanded as a quadratic form in u (eq:meas P:36, R13)
                const LikParams& lp = a.lp;
                sh->lognorm = lp.lognorm;
                sh->inv_sigma = lp.inv_sigma;
                if (UPDATE && lp.kind == 0) {
                    const double* zf = a.z + (long long)filt * lp.nz;
                    double r0[4], G0[4], G1[4];
                    for (int i = 0; i < lp.nz; ++i) {
                        const double h0 = lp.H[i * 4], h1 = lp.H[i * 4 + 1];
                        r0[i] = zf[i] - fma(h0, cl[0], h1 * cl[1]);
                        G0[i] = fma(h0, Bl[0], h1 * Bl[2]);
                        G1[i] = fma(h0, Bl[1], h1 * Bl[3]);
                    }
                    double qa = 0, qb0 = 0, qb1 = 0, g00 = 0, g01 = 0, g11 = 0;
                    for (int i = 0; i < lp.nz; ++i)
                        for (int j = 0; j < lp.nz; ++j) {
                            const double R = lp.Rinv[i * 4 + j];
                            qa = fma(r0[i] * R, r0[j], qa);
                            qb0 = fma(-2.0 * G0[i] * R, r0[j], qb0);
                            qb1 = fma(-2.0 * G1[i] * R, r0[j], qb1);
                            g00 = fma(G0[i] * R, G0[j], g00);
                            g01 = fma(G0[i] * R, G1[j], g01);
                            g11 = fma(G1[i] * R, G1[j], g11);
                        }
                    sh->qa = qa;
                    sh->qb[0] = qb0;
                    sh->qb[1] = qb1;
                    sh->qG[0] = g00;
                    sh->qG[1] = g01;
                    sh->qG[2] = g11;
                } else if (UPDATE) {
                    sh->zr = a.z[filt];
                }
            }
            // Euler-factor coefficients on the start-of-interval grid B0 (R3/R4)
            const double det0 = B0[0] * B0[3] - B0[1] * B0[2];
            const double Bi0[4] = {B0[3] / det0, -B0[1] / det0, -B0[2] / det0, B0[0] / det0};
            for (int n = lane; n < l; n += 32) {
                double D00, D01, D11;
                if (a.mp.diff_mode == 0) {
                    const double* E = a.sub[n].E;
                    // T1 = Bi0 E, D = T1 Bi0^T
                    const double t00 = fma(Bi0[0], E[0], Bi0[1] * E[4]);
                    const double t01 = fma(Bi0[0], E[1], Bi0[1] * E[5]);
                    const double t10 = fma(Bi0[2], E[0], Bi0[3] * E[4]);
                    const double t11 = fma(Bi0[2], E[1], Bi0[3] * E[5]);
                    D00 = fma(t00, Bi0[0], t01 * Bi0[1]);
                    const double D01a = fma(t00, Bi0[2], t01 * Bi0[3]);
                    const double D10a = fma(t10, Bi0[0], t11 * Bi0[1]);
                    D01 = 0.5 * (D01a + D10a);
                    D11 = fma(t10, Bi0[2], t11 * Bi0[3]);
                } else {
                    const double* P = a.sub[n].P;
                    const double b00 = fma(P[0], B0[0], P[1] * B0[2]);
                    const double b01 = fma(P[0], B0[1], P[1] * B0[3]);
                    const double b10 = fma(P[4], B0[0], P[5] * B0[2]);
                    const double b11 = fma(P[4], B0[1], P[5] * B0[3]);
                    D00 = a.mp.Q[0] / fma(b00, b00, b10 * b10);
                    D11 = a.mp.Q[5] / fma(b01, b01, b11 * b11);
                    D01 = 0.0;
                }
                cf[3 * n] = (T)(0.5 * a.mp.dt * D00);
                cf[3 * n + 1] = (T)(0.5 * a.mp.dt * D11);
                cf[3 * n + 2] = (T)(a.mp.dt * D01);
            }
        }
        __syncthreads();
        if (sh->skip) {
            if (tid == 0) a.st[filt].status = -6;
            __syncthreads();
            continue;
        }
        // prefetch the next filter into L2 while this one computes
        if (tid < 8) {
            const int nf = filt + gridDim.x;
            if (nf < a.batch) {
                const char* p = reinterpret_cast<const char*>(a.W + (long long)nf * (N * N)) + tid * (N * N * sizeof(T) / 8);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((unsigned)(N * N * sizeof(T) / 8))
                             : "memory");
            }
        }

        // ---------------------------------------------------------------- P1: load / regrid, FFT along axis 1
        {
            V z[16];
            if (!REGRID) {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const int j1 = t + 8 * r;
                    z[r] = *reinterpret_cast<const V*>(Wf + j1 * N + 2 * m);
                }
            } else {
                const double M0 = sh->M[0], M1 = sh->M[1], M2 = sh->M[2], M3 = sh->M[3];
                const double o0 = sh->o[0], o1 = sh->o[1];
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const double u1 = (t + 8 * r) - 0.5 * (N - 1);
                    T val[2];
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const double u0 = (2 * m + e) - 0.5 * (N - 1);
                        const double v0 = fma(M0, u0, fma(M1, u1, o0));
                        const double v1 = fma(M2, u0, fma(M3, u1, o1));
                        const double f0 = floor(v0), f1 = floor(v1);
                        const double a0 = v0 - f0, a1 = v1 - f1;
                        const int i0 = (int)fmax(fmin(f0, 4096.0), -4096.0);
                        const int i1 = (int)fmax(fmin(f1, 4096.0), -4096.0);
                        double acc = 0.0;
                        const bool x0 = (unsigned)i0 < (unsigned)N, x1 = (unsigned)(i0 + 1) < (unsigned)N;
                        const bool y0 = (unsigned)i1 < (unsigned)N, y1 = (unsigned)(i1 + 1) < (unsigned)N;
                        const T* row0 = Wf + i1 * N;
                        if (y0) {
                            if (x0) acc = fma((1.0 - a0) * (1.0 - a1), (double)row0[i0], acc);
                            if (x1) acc = fma(a0 * (1.0 - a1), (double)row0[i0 + 1], acc);
                        }
                        if (y1) {
                            if (x0) acc = fma((1.0 - a0) * a1, (double)row0[N + i0], acc);
                            if (x1) acc = fma(a0 * a1, (double)row0[N + i0 + 1], acc);
                        }
                        val[e] = (T)acc;
                    }
                    z[r] = V{val[0], val[1]};
                }
            }
            dft16<false>(z);                       // over r: Y_t(s)
#pragma unroll
            for (int s = 1; s < 16; ++s) z[s] = cmul(z[s], tw[s * 8 + t]);
#pragma unroll
            for (int s = 0; s < 16; ++s) X[cslot(s, t, m)] = z[s];
            __syncwarp();
            V pa[8], pb[8];
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) {
                pa[tt] = X[cslot(sa, tt, m)];
                pb[tt] = X[cslot(sb, tt, m)];
            }
            dft8<false>(pa);                       // Z(sa + 16 q)
            dft8<false>(pb);                       // Z(sb + 16 q)
            __syncwarp();
            // unpack the two real columns: Wa = (Z(k) + conj Z(-k))/2, Wb = (Z(k) - conj Z(-k))/(2i)
            auto store_pair = [&](int k1, V zk, V zp) {
                const V wa = V{T(0.5) * (zk.x + zp.x), T(0.5) * (zk.y - zp.y)};
                const V wb = V{T(0.5) * (zk.y + zp.y), T(0.5) * (zp.x - zk.x)};
                X[k1 * PITCH + 2 * m] = wa;
                X[k1 * PITCH + 2 * m + 1] = wb;
            };
            if (t == 0) {
                // s = 0: k = 16 q, partner 16 (8 - q) mod 128;  s = 8: k = 8 + 16 q, partner 8 + 16 (7 - q)
#pragma unroll
                for (int q = 0; q <= 4; ++q) store_pair(16 * q, pa[q], pa[(8 - q) & 7]);
#pragma unroll
                for (int q = 0; q < 4; ++q) store_pair(8 + 16 * q, pb[q], pb[7 - q]);
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    store_pair(sa + 16 * q, pa[q], pb[7 - q]);
                    store_pair(sb + 16 * q, pb[q], pa[7 - q]);
                }
            }
        }
        __syncthreads();

        // ---------------------------------------------------------------- P2: rows, FFT axis 0, Psi, inverse
        {
            V x[16];
            V* row = X + m * PITCH;
            if (m == 0) {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const int j0 = t + 8 * r;
                    x[r] = V{X[j0].x, X[64 * PITCH + j0].x};
                }
            } else {
#pragma unroll
                for (int r = 0; r < 16; ++r) x[r] = row[t + 8 * r];
            }
            dft16<false>(x);
#pragma unroll
            for (int s = 1; s < 16; ++s) x[s] = cmul(x[s], tw[s * 8 + t]);
            __syncwarp();
#pragma unroll
            for (int s = 0; s < 16; ++s) row[rslot(s, t)] = x[s];
            __syncwarp();
            V pa[8], pb[8];
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) {
                pa[tt] = row[rslot(sa, tt)];
                pb[tt] = row[rslot(sb, tt)];
            }
            dft8<false>(pa);                       // F(sa + 16 q)
            dft8<false>(pb);
            // ---- spectral multiplier s Psi(k0, k1) / N^2  (Alg. 3-4)
            const T sn2 = (T)sh->s_over_n2;
            const T kscale = (T)(2.0 * 3.14159265358979323846 / N);
            // ps[q] = s Psi(k0 = sv + 16 q, k1) / N^2; kappa = 2 pi k / N (signed k), the
            // cross term uses kx = kappa with the Nyquist wavenumber zeroed (R7)
            auto psi8 = [&](int k1, int sv, T* ps) {
                const int k1s = k1 < N / 2 ? k1 : k1 - N;
                const T kap1 = kscale * (T)k1s;
                const T kx1 = (k1 == N / 2) ? T(0) : kap1;
                const T k1sq = kap1 * kap1;
                T kk[8], kx[8], den[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int k0 = sv + 16 * q;
                    const int k0s = k0 < N / 2 ? k0 : k0 - N;
                    const T kap0 = kscale * (T)k0s;
                    kk[q] = kap0 * kap0;
                    kx[q] = (k0 == N / 2) ? T(0) : kap0;
                    den[q] = T(1);
                }
                for (int n = 0; n < l; ++n) {
                    const T ca = cf[3 * n], cb = cf[3 * n + 1], cc = cf[3 * n + 2];
                    const T gam = fma(cb, k1sq, T(1));
                    const T bet = cc * kx1;
#pragma unroll
                    for (int q = 0; q < 8; ++q) den[q] *= fma(ca, kk[q], fma(bet, kx[q], gam));
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) ps[q] = sn2 / den[q];
            };
            // packed rows k1 = 0 (A) and 64 (B): R(k) = A(k) + i B(k) with A, B Hermitian;
            // A(k) = (R(k) + conj R(-k))/2, B(k) = (R(k) - conj R(-k))/(2i). After the
            // multiply R'(k) = A'(k) + i B'(k), R'(-k) = conj A'(k) + i conj B'(k).
            auto packed = [&](V& rk, V& rm, bool self, T pA, T pB, bool is_dc) {
                const V R = rk, Rm = rm;
                V A = V{T(0.5) * (R.x + Rm.x), T(0.5) * (R.y - Rm.y)};
                V Bv = V{T(0.5) * (R.y + Rm.y), T(0.5) * (Rm.x - R.x)};
                if (is_dc) sh->dc = (double)A.x;           // sum of the input weights (k = 0)
                A = V{A.x * pA, A.y * pA};
                Bv = V{Bv.x * pB, Bv.y * pB};
                rk = V{A.x - Bv.y, A.y + Bv.x};
                if (!self) rm = V{A.x + Bv.y, Bv.x - A.y};
            };
            if (m != 0) {
                T ps[8];
                psi8(m, sa, ps);
#pragma unroll
                for (int q = 0; q < 8; ++q) pa[q] = V{pa[q].x * ps[q], pa[q].y * ps[q]};
                psi8(m, sb, ps);
#pragma unroll
                for (int q = 0; q < 8; ++q) pb[q] = V{pb[q].x * ps[q], pb[q].y * ps[q]};
            } else if (t != 0) {
                T pA[8], pB[8];
                psi8(0, sa, pA);
                psi8(N / 2, sa, pB);
#pragma unroll
                for (int q = 0; q < 8; ++q) packed(pa[q], pb[7 - q], false, pA[q], pB[q], false);
            } else {
                T pA[8], pB[8];
                psi8(0, 0, pA);                    // s = 0: k0 = 16 q, partner 16 (8 - q) mod 128
                psi8(N / 2, 0, pB);
#pragma unroll
                for (int q = 0; q <= 4; ++q) packed(pa[q], pa[(8 - q) & 7], q == 0 || q == 4, pA[q], pB[q], q == 0);
                psi8(0, 8, pA);                    // s = 8: k0 = 8 + 16 q, partner 8 + 16 (7 - q)
                psi8(N / 2, 8, pB);
#pragma unroll
                for (int q = 0; q < 4; ++q) packed(pb[q], pb[7 - q], false, pA[q], pB[q], false);
            }
            dft8<true>(pa);                        // G_s(t'')
            dft8<true>(pb);
            __syncwarp();
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) {
                row[rslot(sa, tt)] = pa[tt];
                row[rslot(sb, tt)] = pb[tt];
            }
            __syncwarp();
#pragma unroll
            for (int s = 0; s < 16; ++s) x[s] = row[rslot(s, t)];
#pragma unroll
            for (int s = 1; s < 16; ++s) {
                V w = tw[s * 8 + t];
                w.y = -w.y;
                x[s] = cmul(x[s], w);
            }
            dft16<true>(x);
            __syncwarp();
            if (m == 0) {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const int j0 = t + 8 * r;
                    X[j0] = V{x[r].x, T(0)};
                    X[64 * PITCH + j0] = V{x[r].y, T(0)};
                }
            } else {
#pragma unroll
                for (int r = 0; r < 16; ++r) row[t + 8 * r] = x[r];
            }
        }
        __syncthreads();

        // ---------------------------------------------------------------- P3: inverse axis 1, normalise, update
        {
            V pa[8], pb[8];
            auto ld = [&](int k1, int col) -> V { return X[k1 * PITCH + 2 * m + col]; };
            // Z(k) = Wa(k) + i Wb(k); for k > 64: Wa(k) = conj Wa(128 - k)
            auto zdir = [&](int k1) -> V {
                const V wa = ld(k1, 0), wb = ld(k1, 1);
                return V{wa.x - wb.y, wa.y + wb.x};
            };
            auto zmir = [&](int kp) -> V {     // Z(128 - kp) from the stored kp <= 64
                const V wa = ld(kp, 0), wb = ld(kp, 1);
                return V{wa.x + wb.y, wb.x - wa.y};
            };
            if (t == 0) {
#pragma unroll
                for (int q = 0; q < 8; ++q) pa[q] = (q <= 4) ? zdir(16 * q) : zmir(16 * (8 - q));
#pragma unroll
                for (int q = 0; q < 8; ++q) pb[q] = (q < 4) ? zdir(8 + 16 * q) : zmir(8 + 16 * (7 - q));
            } else {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    pa[q] = (q < 4) ? zdir(sa + 16 * q) : zmir(sb + 16 * (7 - q));
                    pb[q] = (q < 4) ? zdir(sb + 16 * q) : zmir(sa + 16 * (7 - q));
                }
            }
            dft8<true>(pa);
            dft8<true>(pb);
            __syncwarp();
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) {
                X[cslot(sa, tt, m)] = pa[tt];
                X[cslot(sb, tt, m)] = pb[tt];
            }
            __syncwarp();
            V x[16];
#pragma unroll
            for (int s = 0; s < 16; ++s) x[s] = X[cslot(s, t, m)];
#pragma unroll
            for (int s = 1; s < 16; ++s) {
                V w = tw[s * 8 + t];
                w.y = -w.y;
                x[s] = cmul(x[s], w);
            }
            dft16<true>(x);                        // x[r] = w(2m, t+8r) + i w(2m+1, t+8r)
            // Alg. 6: sum of the predicted weights = s * DC  ->  normalised = w / (vol_l s DC)
            const double scale_pred = 1.0 / (sh->vol_l * a.mp.s * sh->dc);
            double acc[6] = {0, 0, 0, 0, 0, 0};
            const double Bl0 = sh->Bl[0], Bl1 = sh->Bl[1], Bl2 = sh->Bl[2], Bl3 = sh->Bl[3];
            const double cl0 = sh->cl[0], cl1 = sh->cl[1];
            const bool range = a.lp.kind == 1;
            const double lgn = sh->lognorm;
            // linear-Gauss exponent along this thread's two columns: e = p_e + u1 (q_e + G11 u1)
            double pe[2], qe[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const double u0 = (2 * m + e) - 0.5 * (N - 1);
                pe[e] = fma(u0, fma(sh->qG[0], u0, sh->qb[0]), sh->qa);
                qe[e] = fma(2.0 * sh->qG[1], u0, sh->qb[1]);
            }
            const double g11 = sh->qG[2];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const int j1 = t + 8 * r;
                const double u1 = j1 - 0.5 * (N - 1);
                T outv[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const double u0 = (2 * m + e) - 0.5 * (N - 1);
                    double w = (double)(e == 0 ? x[r].x : x[r].y);
                    if (UPDATE) {
                        double ee;
                        if (!range) {
                            ee = fma(u1, fma(g11, u1, qe[e]), pe[e]);
                        } else {
                            const double x0 = fma(Bl0, u0, fma(Bl1, u1, cl0));
                            const double x1 = fma(Bl2, u0, fma(Bl3, u1, cl1));
                            const double d = (sh->zr - sqrt(fma(x0, x0, x1 * x1))) * sh->inv_sigma;
                            ee = d * d;
                        }
                        w = w * scale_pred * exp(fma(-0.5, ee, lgn));
                        const T wt = (T)w;
                        outv[e] = wt;
                        const double wd = (double)wt;
                        acc[0] += wd;
                        const double wu0 = wd * u0, wu1 = wd * u1;
                        acc[1] += wu0;
                        acc[2] += wu1;
                        acc[3] = fma(wu0, u0, acc[3]);
                        acc[4] = fma(wu0, u1, acc[4]);
                        acc[5] = fma(wu1, u1, acc[5]);
                    } else {
                        outv[e] = (T)w;
                    }
                }
                *reinterpret_cast<V*>(Wf + j1 * N + 2 * m) = V{outv[0], outv[1]};
            }
            if (UPDATE) {
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                    double v = acc[i];
                    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
                    acc[i] = v;
                }
                if (lane == 0)
                    for (int i = 0; i < 6; ++i) red[warp * 6 + i] = acc[i];
            }
            __syncthreads();
            if (tid == 0) {
                FilterState& f = a.st[filt];
                f.c[0] = sh->cl[0];
                f.c[1] = sh->cl[1];
                f.B[0] = sh->Bl[0];
                f.B[1] = sh->Bl[1];
                f.B[4] = sh->Bl[2];
                f.B[5] = sh->Bl[3];
                if (UPDATE) {
                    double s6[6];
                    for (int i = 0; i < 6; ++i) {
                        double s = 0.0;
                        for (int w = 0; w < NT / 32; ++w) s += red[w * 6 + i];
                        s6[i] = s;
                    }
                    const double C = sh->vol_l * s6[0];
                    f.mass = s6[0];
                    f.has_moments = 1;
                    if (!(C > 0.0) || !isfinite(C)) {
                        f.status = -6;
                        f.logC = -INFINITY;
                    } else {
                        f.status = 0;
                        f.logC = log(C);
                        f.scale = 1.0 / C;
                        double acc15[NMOM];
                        for (int i = 0; i < NMOM; ++i) acc15[i] = 0.0;
                        for (int i = 0; i < 6; ++i) acc15[i] = s6[i];
                        finish_moments(nx, acc15, f.c, f.B, f.mean, f.cov);
                    }
                } else {
                    f.scale = scale_pred;
                }
            }
            __syncthreads();
        }
    }
}

bool resident_supported(const Dims& d, int dtype) {
    (void)dtype;
    return d.nx == 2 && d.n[0] == N && d.n[1] == N;
}

template <typename T, bool RG, bool UP>
static cudaError_t launch_t(ResArgs<T> a, cudaStream_t s, int64_t* launches) {
    using V = typename C2<T>::type;
    const size_t smem = sizeof(V) * (H * PITCH + 128) + sizeof(Shared) + 16 * 6 * sizeof(double) +
                        3 * sizeof(T) * (size_t)a.mp.l + 64;
    auto kern = k_resident_epoch<T, RG, UP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) { fprintf(stderr, "[pmf] resident setattr smem=%zu: %s\n", smem, cudaGetErrorString(e)); return e; }
    int dev = 0, nsm = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (e != cudaSuccess) { fprintf(stderr, "[pmf] resident occupancy: %s\n", cudaGetErrorString(e)); return e; }
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const int grid = std::min(a.batch, nsm * occ);
    kern<<<grid, NT, smem, s>>>(a);
    ++*launches;
    e = cudaGetLastError();
    if (e != cudaSuccess) {
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, kern);
        fprintf(stderr, "[pmf] resident launch grid=%d occ=%d smem=%zu regs=%d local=%zu maxthr=%d: %s\n", grid, occ, smem,
                fa.numRegs, fa.localSizeBytes, fa.maxThreadsPerBlock, cudaGetErrorString(e));
    }
    return e;
}

template <typename T>
static cudaError_t launch_dt(const Dims& d, PencilBufs& b, const ModelParams* mp, const LikParams* lp, double ks,
                             cudaStream_t s, int64_t* launches) {
    ResArgs<T> a;
    a.W = (T*)b.W;
    a.st = b.st;
    a.z = b.z;
    a.sub = b.sub;
    a.mp = *mp;
    a.lp = lp ? *lp : LikParams{};
    a.ks = ks;
    a.batch = d.batch;
    const bool rg = ks > 0.0;
    if (rg && lp) return launch_t<T, true, true>(a, s, launches);
    if (rg) return launch_t<T, true, false>(a, s, launches);
    if (lp) return launch_t<T, false, true>(a, s, launches);
    return launch_t<T, false, false>(a, s, launches);
}

cudaError_t launch_resident(const Dims& d, int dtype, PencilBufs& b, const Twiddles& tw, const ModelParams* mp,
                            const LikParams* lp, double ks, cudaStream_t s, int64_t* launches) {
    (void)tw;
    if (!mp) return cudaErrorInvalidValue;      // the host routes update-/regrid-only work to the point kernels
    if (dtype == 0) return launch_dt<double>(d, b, mp, lp, ks, s, launches);
    return launch_dt<float>(d, b, mp, lp, ks, s, launches);
}

}  // namespace pmf
