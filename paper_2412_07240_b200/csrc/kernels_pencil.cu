// kernels_pencil.cu -- the general multi-pass path (any nx <= 4, any
// N with factors 2, 3, 5, 7, 11, 13, 17 per axis, any batch), plus the per-filter kernels shared with the
// resident path: initial density, standalone likelihood update, reductions
// into per-filter moments, and the multilinear regrid.
//
// Predict (Alg. 1-6) for nx >= 2 runs as
//   prep  -> axis-0 R2C (half spectrum) -> forward C2C along axes
//   1..nx-2 -> last axis: forward, x s*Psi (Alg. 3-4), inverse -> inverse C2C
//   axes nx-2..1 -> axis-0 C2R fused with the measurement update (eq:filt P:46)
// and for nx = 1 as one fused line kernel. Each pass stages a tile of pencils in
// shared memory (coalesced: contiguous inner index across threads) and runs the
// Stockham FFT of fft_smem.cuh. Kernels that touch points are templated on nx so
// every per-point loop is static (no local-memory arrays).
#include <algorithm>
#include <type_traits>
#include <cmath>
#include <vector>

#include "device_common.cuh"
#include "fft_smem.cuh"

namespace pmf {

static constexpr int kThreads = 256;
static constexpr int LCAP = 64;       // substeps kept per pencil in shared memory (Psi pass)

static FFTPlan make_plan(int N) {
    FFTPlan p{};
    p.N = N;
    int m = N, k = 0;
    while (m % 4 == 0) { p.r[k++] = 4; m /= 4; }
    if (m % 2 == 0) { p.r[k++] = 2; m /= 2; }
    while (m % 3 == 0) { p.r[k++] = 3; m /= 3; }
    for (int q : {5, 7, 11, 13, 17})
        while (m % q == 0) { p.r[k++] = q; m /= q; }
    p.nst = k;
    return p;
}

// rows per CTA for axis-0 passes: power of two dividing rows_per_filter, P*N ~ 2048
static int rows_per_cta(int N, long long rows_per_filter) {
    int P = std::max(1, 2048 / N);
    int p2 = 1;
    while (p2 * 2 <= P) p2 *= 2;
    while (p2 > 1 && rows_per_filter % p2) p2 /= 2;
    return p2;
}

static int pstride_host(int N) {
    const bool ct = N == 34 || N == 64 || N == 96 || N == 128 || N == 256;   // with_nc's compile-time sizes
    return ct ? N + N / 8 + 1 : N + 1;
}

static int pencils_per_cta(int N) {
    int P = std::max(1, 2048 / N);
    int p2 = 1;
    while (p2 * 2 <= P) p2 *= 2;
    return std::min(p2, 32);
}

// unsigned division by a runtime constant d (1 <= d, x < 2^32): q = umulhi64(x, ceil(2^64/d))
struct FastDiv {
    unsigned long long m;
    unsigned d;
};
static FastDiv make_div(unsigned d) {
    FastDiv f;
    f.d = d;
    f.m = d == 1 ? 0ull : (~0ull / d) + 1ull;
    return f;
}
__device__ __forceinline__ unsigned fdiv(unsigned x, const FastDiv& f) {
    return f.d == 1 ? x : (unsigned)__umul64hi((unsigned long long)x, f.m);
}

struct DivSet {
    FastDiv n[4];   // per axis
};
static DivSet make_divs(const Dims& d) {
    DivSet s;
    for (int a = 0; a < 4; ++a) s.n[a] = make_div((unsigned)d.n[a]);
    return s;
}

// index offsets u of point pt (axis 0 fastest) of one filter
template <int NX>
__device__ __forceinline__ void point_u(const Dims& d, const DivSet& dv, unsigned pt, double* u) {
#pragma unroll
    for (int a = 0; a < NX; ++a) {
        const unsigned q = (a < NX - 1) ? fdiv(pt, dv.n[a]) : 0u;
        const unsigned j = (a < NX - 1) ? pt - q * (unsigned)d.n[a] : pt;
        u[a] = (double)(j + d.lo[a]) - 0.5 * (d.ng[a] - 1);
        pt = q;
    }
}

template <int NX>
__device__ __forceinline__ void phys(const FilterState& f, const double* u, double* x) {
#pragma unroll
    for (int a = 0; a < NX; ++a) {
        double s = f.c[a];
#pragma unroll
        for (int b = 0; b < NX; ++b) s = fma(f.B[a * 4 + b], u[b], s);
        x[a] = s;
    }
}

// moment accumulators: acc[0] = sum w, acc[1..NX] = sum w u_a, then sum w u_a u_b (a <= b)
template <int NX>
__device__ __forceinline__ void acc_mom(double w, const double* u, double* acc) {
    acc[0] += w;
    int k = 1 + NX;
#pragma unroll
    for (int a = 0; a < NX; ++a) {
        const double wu = w * u[a];
        acc[1 + a] += wu;
#pragma unroll
        for (int b = a; b < NX; ++b) {
            acc[k] = fma(wu, u[b], acc[k]);
            ++k;
        }
    }
}

// coefficient block per filter: [0] input scale, [4 .. 4+10l) Euler factors (epoch_coefs),
// [lq(l) .. +16) likelihood exponent as a quadratic form in the moved grid's index
// coordinates: e(u) = q[0] + sum_a q[1+a] u_a + sum_{a<=b} q[5+tri(a,b)] u_a u_b
__host__ __device__ __forceinline__ int lq_off(int l) { return 4 + 10 * (l + 1); }   // room for CN's l + 1 sets


// ============================================================================ prep
// One thread per filter: Euler-factor coefficients (epoch_coefs), the input
// scale, then move the grid (c <- M c, B <- M B, eq:gridMov) and set the
// closed-form normalisation of Alg. 6: scale' = vol_0 / (vol_l s)  (R9; the DC
// coefficient is multiplied by exactly s because psi(0) = 1). With an update
// pending, the linear-Gaussian exponent is expanded around the moved grid
// (r(u) = (z - H c_l) - (H B_l) u; e = r^T R^-1 r, R13).
// One warp per filter: lane n computes substep n's coefficients (n = lane, lane + 32, ...),
// lane 0 the rest (was one serial thread: 30-80 us per epoch for a single filter).
__global__ void k_predict_prep(FilterState* st, double* coef, int cstride, ModelParams mp,
                               const SubstepEntry* __restrict__ sub, int batch, LikParams lp,
                               const double* __restrict__ z, int update) {
    const int b = blockIdx.x, lane = threadIdx.x;
    if (b >= batch) return;
    FilterState& f = st[b];
    double* cf = coef + (long long)b * cstride;
    {
        double B0[16], Bi[16];
        for (int i = 0; i < 16; ++i) B0[i] = f.B[i];
        mat_inv4(mp.nx, B0, Bi);
        const int nsets = mp.l + (mp.step ? 1 : 0);
        for (int n = lane; n < nsets; n += 32) substep_coefs(mp.nx, B0, Bi, mp, sub[n], cf + 4 + 10 * n);
    }
    __syncwarp();
    if (lane != 0) return;
    cf[0] = f.scale;
    const int nx = mp.nx;
    double vol0 = fabs(det4(nx, f.B));
    double Bn[16], cn[4];
    for (int i = 0; i < 16; ++i) Bn[i] = 0.0;
    mat_mul4(nx, mp.Mtau, f.B, Bn);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < nx) s = fma(mp.Mtau[a * 4 + k], f.c[k], s);
        cn[a] = s;
    }
    double voll = fabs(det4(nx, Bn));
    for (int i = 0; i < 16; ++i) f.B[i] = Bn[i];
    for (int a = 0; a < nx; ++a) f.c[a] = cn[a];
    f.scale = vol0 / (voll * mp.s);
    double* q = cf + lq_off(mp.l);
    for (int i = 0; i < 16; ++i) q[i] = 0.0;
    if (update && lp.kind == 0) lik_quadform(nx, lp, cn, Bn, z + (long long)b * lp.nz, q);
}

// ============================================================================ spectral multiplier helpers
__device__ __forceinline__ void wavenum(int k, int N, double& kap, double& kx) {
    int ks = signed_k(k, N);
    kap = 2.0 * PMF_PI * ks / N;
    kx = (2 * k == N) ? 0.0 : kap;
}

// ============================================================================ axis-0 R2C
template <typename T, int NC>
__global__ void __launch_bounds__(kThreads, 2) k_axis0_r2c(const T* __restrict__ W, typename C2<T>::type* __restrict__ S,
                                                         const double* __restrict__ coef, int cstride, Dims d,
                                                         FFTPlan pl, const typename C2<T>::type* __restrict__ tw,
                                                         int P) {
    using V = typename C2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = NC > 0 ? NC : d.n[0], PS = pencil_stride<NC>(N);
    V* a = reinterpret_cast<V*>(smem_raw);
    V* b = a + P * PS;
    const long long rpf = d.ntot / N;
    const long long row0 = (long long)blockIdx.x * P;
    const int filt = (int)(row0 / rpf);
    const T sc = (T)coef[(long long)filt * cstride];
    const T* src = W + row0 * N;
    const float invN = 1.0f / N;
    {
        constexpr int UNR = 8;                       // loads in flight per thread (see k_axis_c2c)
        const int PN = P * N;
        for (int i0 = threadIdx.x; i0 < PN; i0 += UNR * blockDim.x) {
            T v[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int i = i0 + u * blockDim.x;
                v[u] = i < PN ? src[i] : T(0);
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int i = i0 + u * blockDim.x;
                if (i < PN) {
                    const int p = (int)((i + 0.5f) * invN), j = i - p * N;
                    a[p * PS + sx<NC>(j)] = V{v[u] * sc, T(0)};
                }
            }
        }
    }
    __syncthreads();
    V* r = fft_any<NC, false>(a, b, P, PS, pl, tw);
    V* dst = S + row0 * d.H0;
    const float invH = 1.0f / d.H0;
    for (int i = threadIdx.x; i < P * d.H0; i += blockDim.x) {
        const int p = (int)((i + 0.5f) * invH), k = i - p * d.H0;
        dst[i] = r[p * PS + sx<NC>(k)];
    }
}

// ============================================================================ strided C2C (+ optional Psi)
// Pencils along axis m of the half-spectrum buffer: element (i, j, o) at
// S[o*Nm*I + j*I + i], i < I = H0*N_1*..*N_{m-1}, o < O. A CTA takes P
// consecutive i (coalesced rows of P complex) of one o.
// MODE 2 (last axis m = NX-1): forward, x s Psi(k) / N_total, inverse. Psi is
// factored per pencil: for substep n, f_n = gam_n + bet_n kx_L + alp_n kap_L^2 with
// (gam_n, bet_n) depending only on the pencil's other wavenumbers (Alg. 3, R3, R7).
template <typename T, int MODE, int NX, int NC>
__global__ void __launch_bounds__(kThreads, 2) k_axis_c2c(typename C2<T>::type* __restrict__ S, Dims d, int m,
                                                        long long I, FFTPlan pl,
                                                        const typename C2<T>::type* __restrict__ tw, int P,
                                                        const double* __restrict__ coef, int cstride,
                                                        ModelParams mp, long long inner_off) {
    using V = typename C2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = NC > 0 ? NC : pl.N, PS = pencil_stride<NC>(N);
    V* a = reinterpret_cast<V*>(smem_raw);
    V* b = a + P * PS;
    const long long ntile = (I + P - 1) / P;
    const long long o = blockIdx.x / ntile;
    const long long i0 = (blockIdx.x - o * ntile) * P;
    V* base = S + o * (long long)N * I;
    {
        // UNR independent loads in flight per thread before the shared stores (the
        // one-load-per-iteration loop serialised on the L2 / HBM latency)
        constexpr int UNR = 8;
        const int PN = P * N, lp2 = __ffs(P) - 1;    // P is a power of two
        for (int t0 = threadIdx.x; t0 < PN; t0 += UNR * blockDim.x) {
            V v[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int t = t0 + u * blockDim.x;
                const int j = t >> lp2, p = t & (P - 1);
                const long long i = i0 + p;
                v[u] = (t < PN && i < I) ? base[(long long)j * I + i] : V{T(0), T(0)};
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const int t = t0 + u * blockDim.x;
                if (t < PN) a[(t & (P - 1)) * PS + sx<NC>(t >> lp2)] = v[u];
            }
        }
    }
    __syncthreads();
    V* r;
    if (MODE == 1) {
        r = fft_any<NC, true>(a, b, P, PS, pl, tw);
    } else {
        r = fft_any<NC, false>(a, b, P, PS, pl, tw);
        if (MODE == 2) {
            const double* cf = coef + o * cstride + 4;   // o is the filter index on the last axis
            double ntot = 1.0;
#pragma unroll
            for (int q = 0; q < NX; ++q) ntot *= d.ng[q];
            const double mult = mp.s / ntot;
            const int l = mp.l, nsets = l + (mp.step ? 1 : 0);
            const bool cached = nsets <= LCAP;
            double* pg = reinterpret_cast<double*>(b + P * PS);    // [P][l][2]: gam, bet
            constexpr int L = NX - 1;
            auto pencil_k = [&](long long i, double* kap, double* kx) {
                long long rem = i + inner_off;          // global inner index (sharded: my range)
                const int k0 = (int)(rem % d.H0);
                rem /= d.H0;
                wavenum(k0, d.n[0], kap[0], kx[0]);
#pragma unroll
                for (int q = 1; q < L; ++q) {
                    const int kq = (int)(rem % d.n[q]);
                    rem /= d.n[q];
                    wavenum(kq, d.n[q], kap[q], kx[q]);
                }
            };
            auto gam_bet = [&](const double* kap, const double* kx, int n, double& gam, double& bet) {
                const double* c = cf + 10 * n;
                double g = 1.0, bb = 0.0;
#pragma unroll
                for (int a2 = 0; a2 < L; ++a2) {
                    g = fma(c[a2], kap[a2] * kap[a2], g);
#pragma unroll
                    for (int b2 = a2 + 1; b2 < L; ++b2) g = fma(c[pair_index(NX, a2, b2)], kx[a2] * kx[b2], g);
                    bb = fma(c[pair_index(NX, a2, L)], kx[a2], bb);
                }
                gam = g;
                bet = bb;
            };
            if (cached) {
                for (int t = threadIdx.x; t < P * nsets; t += blockDim.x) {
                    const int p = t / nsets, n = t - p * nsets;
                    const long long i = i0 + p;
                    double kap[4] = {0, 0, 0, 0}, kx[4] = {0, 0, 0, 0};
                    if (i < I) pencil_k(i, kap, kx);
                    double g, bb;
                    gam_bet(kap, kx, n, g, bb);
                    pg[2 * t] = g;
                    pg[2 * t + 1] = bb;
                }
                __syncthreads();
            }
            for (int t = threadIdx.x; t < P * N; t += blockDim.x) {
                const int p = t / N, j = t - p * N;
                const long long i = i0 + p;
                if (i >= I) continue;
                double kapL, kxL;
                wavenum(j, N, kapL, kxL);
                const double kL2 = kapL * kapL;
                // Euler: 1 / prod_{n<l} f_n; Crank-Nicolson: prod_{n<l} (2 - f_n) / prod_{n=1..l} f_n
                double prod = 1.0, num = 1.0;
                const double* g = pg + 2 * p * nsets;
                double kap[4] = {0, 0, 0, 0}, kx[4] = {0, 0, 0, 0};
                if (!cached) pencil_k(i, kap, kx);
                for (int n = 0; n < nsets; ++n) {
                    double gg, bb;
                    if (cached) {
                        gg = g[2 * n];
                        bb = g[2 * n + 1];
                    } else {
                        gam_bet(kap, kx, n, gg, bb);
                    }
                    const double fn = fma(cf[10 * n + L], kL2, fma(bb, kxL, gg));
                    if (!mp.step) {
                        prod *= fn;
                    } else {
                        if (n < l) num *= 2.0 - fn;
                        if (n > 0) prod *= fn;
                    }
                }
                const T ps = (T)(mult * num / prod);
                V v = r[p * PS + sx<NC>(j)];
                r[p * PS + sx<NC>(j)] = V{v.x * ps, v.y * ps};
            }
            __syncthreads();
            V* other = (r == a) ? b : a;
            r = fft_any<NC, true>(r, other, P, PS, pl, tw);
        }
    }
    for (int t = threadIdx.x; t < P * N; t += blockDim.x) {
        const int j = t / P, p = t - j * P;
        long long i = i0 + p;
        if (i < I) base[(long long)j * I + i] = r[p * PS + sx<NC>(j)];
    }
}

// ============================================================================ axis-0 C2R (+ update)
// Per row the likelihood exponent is a quadratic in u0: e = A_p + u0 (B_p + G00 u0).
template <typename T, bool UPDATE, int NX, int NC>
__global__ void __launch_bounds__(kThreads, 2) k_axis0_c2r(const typename C2<T>::type* __restrict__ S, T* __restrict__ W,
                                                         const FilterState* __restrict__ st, Dims d, DivSet dv,
                                                         FFTPlan pl, const typename C2<T>::type* __restrict__ tw,
                                                         int P, LikParams lp, const double* __restrict__ z,
                                                         const double* __restrict__ coef, int cstride, int lqo,
                                                         double* __restrict__ partials, int cpf, int tpc) {
    // CTA (filter, q) processes tiles [q tpc, (q+1) tpc) of P rows of its filter and
    // writes ONE set of moment partials (cpf CTAs per filter).
    using V = typename C2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = NC > 0 ? NC : d.n[0], PS = pencil_stride<NC>(N);
    V* a = reinterpret_cast<V*>(smem_raw);
    V* b = a + P * PS;
    double* red = reinterpret_cast<double*>(b + P * PS);            // 32 * NMOM
    double* rowu = red + 32 * NMOM;                                  // [P][6]: u_1..u_3, A_p, B_p
    const long long rpf = d.ntot / N;
    const int tiles = (int)(rpf / P);
    const int filt = blockIdx.x / cpf, qc = blockIdx.x - filt * cpf;
    const int t_end = min(tiles, (qc + 1) * tpc);
    const FilterState& f = st[filt];
    const double* q = coef + (long long)filt * cstride + lqo;
    const double scale = f.scale;
    const double g00 = q[5];
    const double* zf = z + (long long)filt * lp.nz;
    const float invN = 1.0f / N;
    double acc[NMOM];
#pragma unroll
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    for (int tile = qc * tpc; tile < t_end; ++tile) {
        const long long rloc = (long long)tile * P;                  // first row of the tile in the filter
        const long long row0 = (long long)filt * rpf + rloc;
        const V* src = S + row0 * d.H0;
        {
            constexpr int UNR = 8;                   // loads in flight per thread (see k_axis_c2c)
            const int PN = P * N;
            for (int i0 = threadIdx.x; i0 < PN; i0 += UNR * blockDim.x) {
                V v[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const int i = i0 + u * blockDim.x;
                    const int p = (int)((i + 0.5f) * invN), k = i - p * N;
                    v[u] = i < PN ? src[p * d.H0 + (k < d.H0 ? k : N - k)] : V{T(0), T(0)};
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    const int i = i0 + u * blockDim.x;
                    if (i < PN) {
                        const int p = (int)((i + 0.5f) * invN), k = i - p * N;
                        a[p * PS + sx<NC>(k)] = k < d.H0 ? v[u] : V{v[u].x, -v[u].y};
                    }
                }
            }
        }
        if (UPDATE) {
            for (int p = threadIdx.x; p < P; p += blockDim.x) {
                double u[4] = {0, 0, 0, 0};
                unsigned rr = (unsigned)(rloc + p);
#pragma unroll
                for (int a2 = 1; a2 < NX; ++a2) {
                    const unsigned qq = (a2 < NX - 1) ? fdiv(rr, dv.n[a2]) : 0u;
                    const unsigned j = (a2 < NX - 1) ? rr - qq * (unsigned)d.n[a2] : rr;
                    u[a2] = (double)(j + d.lo[a2]) - 0.5 * (d.ng[a2] - 1);
                    rr = qq;
                }
                double A = q[0], Bc = q[1];
#pragma unroll
                for (int a2 = 1; a2 < NX; ++a2) {
                    A = fma(q[1 + a2], u[a2], A);
                    Bc = fma(q[5 + tri(0, a2)], u[a2], Bc);
#pragma unroll
                    for (int b2 = a2; b2 < NX; ++b2) A = fma(q[5 + tri(a2, b2)] * u[a2], u[b2], A);
                }
                double* ru = rowu + 6 * p;
                ru[0] = u[1];
                ru[1] = u[2];
                ru[2] = u[3];
                ru[3] = A;
                ru[4] = Bc;
            }
        }
        __syncthreads();
        V* r = fft_any<NC, true>(a, b, P, PS, pl, tw);
        T* dst = W + row0 * N;
        for (int i = threadIdx.x; i < P * N; i += blockDim.x) {
            const int p = (int)((i + 0.5f) * invN), j = i - p * N;
            double w = (double)r[p * PS + sx<NC>(j)].x;
            if (UPDATE) {
                const double* ru = rowu + 6 * p;
                double u[4];
                u[0] = j - 0.5 * (N - 1);
#pragma unroll
                for (int a2 = 1; a2 < NX; ++a2) u[a2] = ru[a2 - 1];
                double ll;
                if (lp.kind == 0) {
                    const double e = fma(u[0], fma(g00, u[0], ru[4]), ru[3]);
                    ll = fma(-0.5, e, lp.lognorm);
                } else {
                    double x[4];
                    phys<NX>(f, u, x);
                    ll = log_lik(lp, x, zf);
                }
                const T wt = (T)(w * scale * exp_fast(ll));
                dst[i] = wt;
                acc_mom<NX>((double)wt, u, acc);
            } else {
                dst[i] = (T)w;
            }
        }
        __syncthreads();                     // the tile's shared memory is reused by the next tile
    }
    if (UPDATE) {
        block_sum<NMOM>(acc, red);
        if (threadIdx.x == 0)
            for (int q2 = 0; q2 < NMOM; ++q2) partials[(long long)blockIdx.x * NMOM + q2] = acc[q2];
    }
}

// ============================================================================ nx = 1 fused line
template <typename T, bool UPDATE, int NC>
__global__ void __launch_bounds__(kThreads, 2) k_line_psi(T* __restrict__ W, FilterState* __restrict__ st, Dims d,
                                                        FFTPlan pl, const typename C2<T>::type* __restrict__ tw,
                                                        const double* __restrict__ coef, int cstride,
                                                        ModelParams mp, LikParams lp, const double* __restrict__ z,
                                                        double* __restrict__ partials) {
    using V = typename C2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = NC > 0 ? NC : d.n[0], PS = pencil_stride<NC>(N);
    V* a = reinterpret_cast<V*>(smem_raw);
    V* b = a + PS;
    double* red = reinterpret_cast<double*>(b + PS);
    const int filt = blockIdx.x;
    const double* cf = coef + (long long)filt * cstride;
    const T sc = (T)cf[0];
    T* row = W + (long long)filt * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) a[sx<NC>(j)] = V{row[j] * sc, T(0)};
    __syncthreads();
    V* r = fft_any<NC, false>(a, b, 1, PS, pl, tw);
    const double mult = mp.s / N;
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double kap, kx;
        wavenum(k, N, kap, kx);
        double prod = 1.0, num = 1.0;
        if (!mp.step) {
            for (int n = 0; n < mp.l; ++n) prod *= fma(cf[4 + 10 * n], kap * kap, 1.0);
        } else {          // Crank-Nicolson (R27)
            for (int n = 0; n < mp.l; ++n) num *= 1.0 - cf[4 + 10 * n] * kap * kap;
            for (int n = 1; n <= mp.l; ++n) prod *= fma(cf[4 + 10 * n], kap * kap, 1.0);
        }
        const T ps = (T)(mult * num / prod);
        V v = r[sx<NC>(k)];
        r[sx<NC>(k)] = V{v.x * ps, v.y * ps};
    }
    __syncthreads();
    r = fft_any<NC, true>(r, (r == a) ? b : a, 1, PS, pl, tw);
    const FilterState& f = st[filt];
    double acc[NMOM];
#pragma unroll
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    const double scale = f.scale;
    const double* zf = z + (long long)filt * lp.nz;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        double w = (double)r[sx<NC>(j)].x;
        if (UPDATE) {
            double u = j - 0.5 * (N - 1), x;
            phys<1>(f, &u, &x);
            w = w * scale * exp_fast(log_lik(lp, &x, zf));
            T wt = (T)w;
            row[j] = wt;
            acc_mom<1>((double)wt, &u, acc);
        } else {
            row[j] = (T)w;
        }
    }
    if (UPDATE) {
        block_sum<NMOM>(acc, red);
        if (threadIdx.x == 0)
            for (int q = 0; q < NMOM; ++q) partials[(long long)blockIdx.x * NMOM + q] = acc[q];
    }
}

// ============================================================================ per-filter point kernels
// grid: batch * nbpf blocks; block (filt, q) covers points q*blockDim + k*nbpf*blockDim
static int blocks_per_filter(long long ntot) {
    long long nb = (ntot + kThreads * 8 - 1) / (kThreads * 8);
    return (int)std::max(1LL, std::min(nb, 1024LL));
}

// blocks per filter for the grid-stride point passes: at most one wave of the device
// (a partial second or third wave made the tail; C6: 653 blocks on 296 slots)
template <typename K>
static int wave_bpf(K kern, int threads, size_t smem, long long ntot, int batch) {
    int occ = 0, dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        sms = 148;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem) != cudaSuccess || occ < 1) occ = 1;
    const long long per = std::max(1LL, (long long)occ * sms / std::max(1, batch));
    return (int)std::max(1LL, std::min((long long)blocks_per_filter(ntot), per));
}

template <typename T, int MODE, int NX>   // 0: standalone update, 1: init gaussian, 2: plain sum
__global__ void __launch_bounds__(kThreads, 2) k_points(T* __restrict__ W, const FilterState* __restrict__ st, Dims d,
                                                      DivSet dv, int nbpf, LikParams lp,
                                                      const double* __restrict__ z, const double* __restrict__ gauss,
                                                      double* __restrict__ partials) {
    __shared__ double red[32 * NMOM];
    const int filt = blockIdx.x / nbpf, qb = blockIdx.x - filt * nbpf;
    const FilterState& f = st[filt];
    T* Wf = W + (long long)filt * d.ntot;
    double acc[NMOM];
#pragma unroll
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    const double* zf = z ? z + (long long)filt * lp.nz : nullptr;
    const double* g = gauss ? gauss + (long long)filt * 21 : nullptr;
    for (long long pt = (long long)qb * blockDim.x + threadIdx.x; pt < d.ntot; pt += (long long)nbpf * blockDim.x) {
        double u[4], x[4];
        if (MODE != 2) {
            point_u<NX>(d, dv, (unsigned)pt, u);
            phys<NX>(f, u, x);
        }
        if (MODE == 0) {
            const double lk = lp.kind == 2 ? lik_terrain_gm(lp, x, zf) : exp_fast(log_lik(lp, x, zf));
            const double w = (double)Wf[pt] * f.scale * lk;
            const T wt = (T)w;
            Wf[pt] = wt;
            acc_mom<NX>((double)wt, u, acc);
        } else if (MODE == 1) {
            double rr[4], e = 0.0;
#pragma unroll
            for (int a = 0; a < NX; ++a) rr[a] = x[a] - g[a];
#pragma unroll
            for (int a = 0; a < NX; ++a) {
                double t = 0.0;
#pragma unroll
                for (int b = 0; b < NX; ++b) t = fma(g[4 + a * 4 + b], rr[b], t);
                e = fma(rr[a], t, e);
            }
            const T wt = (T)exp(fma(-0.5, e, g[20]));
            Wf[pt] = wt;
            acc[0] += (double)wt;
        } else {
            acc[0] += (double)Wf[pt];
        }
    }
    block_sum<NMOM>(acc, red);
    if (threadIdx.x == 0)
        for (int i = 0; i < NMOM; ++i) partials[(long long)blockIdx.x * NMOM + i] = acc[i];
}

// ============================================================================ finalisers (1 block per filter)
// Fixed-order sums of the per-CTA partials: thread k sums partials k, k+256, ...,
// then a fixed tree (block_sum) -- deterministic for a given launch geometry.
__device__ inline void block_sum_partials(const double* __restrict__ partials, long long first, int nb, double* acc,
                                          double* red) {
#pragma unroll
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    for (int k = threadIdx.x; k < nb; k += blockDim.x)
#pragma unroll
        for (int i = 0; i < NMOM; ++i) acc[i] += partials[(first + k) * NMOM + i];
    block_sum<NMOM>(acc, red);
}

// Scalar tail of every reduction (sums acc[] over the whole filter):
// MODE 0: update -> normaliser C = vol * sum, log C, scale = 1/C, moments.
// MODE 1: renormalise (init/set_state): scale = 1/(vol * sum).
// MODE 2: commit a regrid: new grid (R12), scale = 1/(vol' * sum).
// NX a compile-time constant: the small matrix loops unroll into registers (with a
// runtime nx they ran from a 700-byte stack frame in one thread: C6's finaliser 16.8 us)
template <int NX>
__device__ __forceinline__ void finalize_from_t(FilterState& f, const double* acc, const Dims& d, int mode, double ks) {
    constexpr int nx = NX;
    if (mode == 2) {
        double cn[4], Bn[16];
        bool ok = regrid_target(nx, d.ng, f, ks, cn, Bn, d.grid);
        for (int a = 0; a < nx; ++a) f.c[a] = cn[a];
        for (int i = 0; i < 16; ++i) f.B[i] = Bn[i];
        double C = fabs(det4(nx, Bn)) * acc[0];
        if (!ok || !(C > 0.0) || !isfinite(C)) { f.status = -6; return; }
        f.scale = 1.0 / C;
        return;
    }
    double vol = fabs(det4(nx, f.B));
    double C = vol * acc[0];
    if (mode == 0) {
        f.mass = acc[0];
        f.has_moments = 1;
        if (!(C > 0.0) || !isfinite(C)) {
            f.status = -6;
            f.logC = -INFINITY;
            return;
        }
        f.status = 0;
        f.logC = log(C);
        f.scale = 1.0 / C;
        finish_moments(nx, acc, f.c, f.B, f.mean, f.cov);
    } else {
        if (!(C > 0.0) || !isfinite(C)) { f.status = -6; return; }
        f.scale = 1.0 / C;
    }
}

__device__ __forceinline__ void finalize_from(FilterState& f, const double* acc, const Dims& d, int mode, double ks) {
    switch (d.nx) {
        case 1: finalize_from_t<1>(f, acc, d, mode, ks); break;
        case 2: finalize_from_t<2>(f, acc, d, mode, ks); break;
        case 3: finalize_from_t<3>(f, acc, d, mode, ks); break;
        default: finalize_from_t<4>(f, acc, d, mode, ks); break;
    }
}

__global__ void k_finalize(FilterState* st, const double* __restrict__ partials, int nbpf, Dims d, int mode) {
    __shared__ double red[32 * NMOM];
    const int filt = blockIdx.x;
    double acc[NMOM];
    block_sum_partials(partials, (long long)filt * nbpf, nbpf, acc, red);
    if (threadIdx.x != 0) return;
    finalize_from(st[filt], acc, d, mode, 0.0);
}

// sharded path: per-rank totals (partials -> tot), then after the all-reduce the tail
__global__ void k_reduce_partials(const double* __restrict__ partials, int nbpf, double* __restrict__ tot) {
    __shared__ double red[32 * NMOM];
    const int filt = blockIdx.x;
    double acc[NMOM];
    block_sum_partials(partials, (long long)filt * nbpf, nbpf, acc, red);
    if (threadIdx.x == 0)
        for (int i = 0; i < NMOM; ++i) tot[(long long)filt * NMOM + i] = acc[i];
}

__global__ void k_finalize_tot(FilterState* st, const double* __restrict__ tot, Dims d, int mode, double ks, int batch) {
    const int filt = blockIdx.x * blockDim.x + threadIdx.x;
    if (filt >= batch) return;
    finalize_from(st[filt], tot + (long long)filt * NMOM, d, mode, ks);
}

// all-to-all packing of the half spectrum [planes][I] into per-destination blocks
// [d][planes][I_d] (x in I_d starts at inner offset off_d), and the inverse.
template <typename V>
__global__ void k_pack_blocks(const V* __restrict__ S, V* __restrict__ send, long long I, int planes,
                              const long long* __restrict__ off, int world, int unpack) {
    // off[0..world]: inner-range boundaries; block d holds planes x (off[d+1]-off[d]) values
    const long long total = (long long)planes * I;
    for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long pl = e / I, x = e - pl * I;
        int dd = 0;
        while (dd + 1 < world && x >= off[dd + 1]) ++dd;
        const long long Id = off[dd + 1] - off[dd];
        const long long boff = (long long)planes * off[dd];     // block start in the packed buffer
        const long long pe = boff + pl * Id + (x - off[dd]);
        if (unpack) const_cast<V*>(S)[e] = send[pe];
        else send[pe] = S[e];
    }
}

// ============================================================================ nx = 1: one launch per epoch
// The whole epoch of a 1-D filter in one CTA (BASELINE C1 is launch-latency bound):
// [regrid of the previous posterior (R12): target grid, linear interpolation of the stored
// weights with zero ghosts, renormalisation by summation] -> per-substep Euler (or CN)
// coefficients on the start grid (Alg. 3, R3/R4) -> grid motion (eq:gridMov) and the
// closed-form predict normalisation (Alg. 6) -> forward DFT, s Psi / N, inverse (Alg. 1-5)
// -> likelihood at the moved points (eq:filt P:46) -> normaliser, moments.
// Same arithmetic as k_regrid_gather + k_finalize_regrid + k_predict_prep + k_line_psi +
// k_finalize, without the four kernel boundaries. cfs: nsets coefficients in shared memory.
template <typename T, bool UPDATE, bool RG, int NC>
__global__ void __launch_bounds__(kThreads, 2) k_line_epoch(T* __restrict__ W, FilterState* st, Dims d,
                                                          FFTPlan pl, const typename C2<T>::type* __restrict__ tw,
                                                          ModelParams mp, const SubstepEntry* __restrict__ sub,
                                                          LikParams lp, const double* __restrict__ z, double ks) {
    using V = typename C2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = NC > 0 ? NC : d.n[0], PS = pencil_stride<NC>(N);
    V* a = reinterpret_cast<V*>(smem_raw);
    V* b = a + PS;
    double* red = reinterpret_cast<double*>(b + PS);
    double* cfs = red + 32 * NMOM;                          // [nsets] h D_n (nx = 1)
    // M, o, input scale, skip flag, moved grid c_l, B_l, closed-form scale: written by thread
    // 0, read by all through shared memory
    __shared__ double sh[8];
    const int filt = blockIdx.x, tid = threadIdx.x;
    FilterState& f = st[filt];
    T* row = W + (long long)filt * N;
    double acc[NMOM];
    if (RG) {
        // ------------------------------------------------------------ regrid (R12)
        // scalar tails (nx = 1): thread 0 only, no local arrays on the critical path
        double cn1 = 0.0, Bn1 = 0.0;
        bool ok = true;
        if (tid == 0) {
            double cn[4], Bn[16];
            ok = regrid_target(1, d.ng, f, ks, cn, Bn, d.grid);
            cn1 = cn[0];
            Bn1 = Bn[0];
            const double Bi = 1.0 / f.B[0];
            sh[0] = Bi * Bn1;                                  // M = B^-1 B'
            sh[1] = fma(Bi, cn1 - f.c[0], 0.5 * (d.ng[0] - 1));  // o = B^-1 (c' - c) + (N-1)/2
        }
        for (int j = tid; j < N; j += blockDim.x) b[j] = V{row[j], T(0)};
        __syncthreads();
        const double M0 = sh[0], o0 = sh[1];
#pragma unroll
        for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
        for (int j = tid; j < N; j += blockDim.x) {
            const double v = fma(M0, (double)j - 0.5 * (N - 1), o0), fl = floor(v);
            const int i0 = __double2int_rz(fl);
            const double fr = v - fl;
            double val = 0.0;
            if (i0 >= 0 && i0 <= N - 1) val = fma(1.0 - fr, (double)b[i0].x, val);
            if (i0 >= -1 && i0 <= N - 2) val = fma(fr, (double)b[i0 + 1].x, val);
            const T vt = (T)val;
            a[sx<NC>(j)] = V{vt, T(0)};
            acc[0] += (double)vt;
        }
        block_sum<NMOM>(acc, red);                          // ends with a barrier
        if (tid == 0) {
            // commit the regrid (finalize_from mode 2): new grid, scale = 1 / (vol' sum)
            const double C = fabs(Bn1) * acc[0];
            f.c[0] = cn1;
            f.B[0] = Bn1;
            if (!ok || !(C > 0.0) || !isfinite(C)) f.status = -6;
            else f.scale = 1.0 / C;
            sh[3] = f.status != 0 ? 1.0 : 0.0;
        }
        __syncthreads();
        if (sh[3] != 0.0) {                                 // degenerate target: weights kept
            return;
        }
    }
    // ---------------------------------------------------------------- prep (k_predict_prep)
    const int nsets = mp.l + (mp.step ? 1 : 0);
    {
        double B0[16], Bi[16];
        for (int i = 0; i < 16; ++i) B0[i] = f.B[i];
        mat_inv4(1, B0, Bi);
        for (int n = tid; n < nsets; n += blockDim.x) {
            double o[10];
            substep_coefs(1, B0, Bi, mp, sub[n], o);
            cfs[n] = o[0];
        }
    }
    __syncthreads();                                        // every thread has read f.B
    if (tid == 0) {
        sh[2] = f.scale;                                    // input scale
        const double vol0 = fabs(f.B[0]);
        const double Bn = mp.Mtau[0] * f.B[0], cn = mp.Mtau[0] * f.c[0];
        f.B[0] = Bn;
        f.c[0] = cn;
        f.scale = vol0 / (fabs(Bn) * mp.s);
        sh[4] = cn;
        sh[5] = Bn;
        sh[6] = f.scale;
    }
    if (!RG)
        for (int j = tid; j < N; j += blockDim.x) a[sx<NC>(j)] = V{row[j], T(0)};
    __syncthreads();
    // ---------------------------------------------------------------- predict (k_line_psi)
    const T sc = (T)sh[2];
    for (int j = tid; j < N; j += blockDim.x) {
        const V v = a[sx<NC>(j)];
        a[sx<NC>(j)] = V{v.x * sc, T(0)};
    }
    __syncthreads();
    V* r = fft_any<NC, false>(a, b, 1, PS, pl, tw);
    const double mult = mp.s / N;
    for (int k = tid; k < N; k += blockDim.x) {
        double kap, kx;
        wavenum(k, N, kap, kx);
        double prod = 1.0, num = 1.0;
        if (!mp.step) {
            for (int n = 0; n < mp.l; ++n) prod *= fma(cfs[n], kap * kap, 1.0);
        } else {          // Crank-Nicolson (R27)
            for (int n = 0; n < mp.l; ++n) num *= 1.0 - cfs[n] * kap * kap;
            for (int n = 1; n <= mp.l; ++n) prod *= fma(cfs[n], kap * kap, 1.0);
        }
        const T ps = (T)(mult * num / prod);
        V v = r[sx<NC>(k)];
        r[sx<NC>(k)] = V{v.x * ps, v.y * ps};
    }
    __syncthreads();
    r = fft_any<NC, true>(r, (r == a) ? b : a, 1, PS, pl, tw);
#pragma unroll
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    const double scale = sh[6], cl = sh[4], Bl = sh[5];
    const double* zf = z + (long long)filt * lp.nz;
    for (int j = tid; j < N; j += blockDim.x) {
        double w = (double)r[sx<NC>(j)].x;
        if (UPDATE) {
            double u = j - 0.5 * (N - 1);
            double x = fma(Bl, u, cl);                      // the moved point (R13)
            w = w * scale * exp_fast(log_lik(lp, &x, zf));
            T wt = (T)w;
            row[j] = wt;
            acc_mom<1>((double)wt, &u, acc);
        } else {
            row[j] = (T)w;
        }
    }
    if (UPDATE) {
        block_sum<NMOM>(acc, red);
        if (tid == 0) {
            // normaliser C = vol sum, log C, scale, moments (R14): finalize_from mode 0
            const double C = fabs(Bl) * acc[0];
            f.mass = acc[0];
            f.has_moments = 1;
            if (!(C > 0.0) || !isfinite(C)) {
                f.status = -6;
                f.logC = -INFINITY;
            } else {
                f.status = 0;
                f.logC = log(C);
                f.scale = 1.0 / C;
                const double ub = acc[1] / acc[0];
                const double su = acc[2] / acc[0] - ub * ub;
                f.mean[0] = fma(Bl, ub, cl);
                f.cov[0] = fma(fma(Bl, su, 0.0), Bl, 0.0);
            }
        }
    }
}

// ============================================================================ regrid
// Multilinear interpolation with zero ghost nodes at the points of the new grid
// (R12). v = B^-1 (x' - c) + (N-1)/2 = o + M u' with M = B^-1 B', o = B^-1(c'-c)+(N-1)/2.
template <typename T, int NX>
__global__ void __launch_bounds__(kThreads, 2) k_regrid_gather(const T* __restrict__ Wold, T* __restrict__ Wnew,
                                                             const FilterState* __restrict__ st, Dims d, DivSet dv,
                                                             int nbpf, double ks, double* __restrict__ partials) {
    __shared__ double red[32 * NMOM];
    __shared__ double Msh[16], osh[4];
    const int filt = blockIdx.x / nbpf, qb = blockIdx.x - filt * nbpf;
    const FilterState& f = st[filt];
    if (threadIdx.x == 0) {
        double cn[4], Bn[16], Bi[16];
        regrid_target(NX, d.ng, f, ks, cn, Bn, d.grid);
        mat_inv4(NX, f.B, Bi);
        double M[16];
        for (int i = 0; i < 16; ++i) M[i] = 0.0;
        mat_mul4(NX, Bi, Bn, M);
        for (int i = 0; i < 16; ++i) Msh[i] = M[i];
        for (int a = 0; a < NX; ++a) {
            double s = 0.5 * (d.ng[a] - 1);
            for (int b = 0; b < NX; ++b) s = fma(Bi[a * 4 + b], cn[b] - f.c[b], s);
            osh[a] = s;
        }
    }
    __syncthreads();
    double M[16], o[4];
#pragma unroll
    for (int i = 0; i < NX; ++i) {
        o[i] = osh[i];
#pragma unroll
        for (int j = 0; j < NX; ++j) M[i * 4 + j] = Msh[i * 4 + j];
    }
    long long stride[4];
    stride[0] = 1;
#pragma unroll
    for (int a = 1; a < NX; ++a) stride[a] = stride[a - 1] * d.n[a - 1];
    const T* Wo = Wold + (long long)filt * (d.ntot / d.n[NX - 1] * d.src_n);   // regrid source window
    T* Wn = Wnew + (long long)filt * d.ntot;
    double acc[NMOM];
#pragma unroll
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    for (long long pt = (long long)qb * blockDim.x + threadIdx.x; pt < d.ntot; pt += (long long)nbpf * blockDim.x) {
        double u[4];
        point_u<NX>(d, dv, (unsigned)pt, u);
        double fr[4];
        long long base = 0;
        bool lo_ok[4], hi_ok[4];
#pragma unroll
        for (int a = 0; a < NX; ++a) {
            double s = o[a];
#pragma unroll
            for (int b = 0; b < NX; ++b) s = fma(M[a * 4 + b], u[b], s);
            const double fl = floor(s);
            const int i0 = __double2int_rz(fl);           // saturating
            fr[a] = s - fl;
            // global bounds (zero ghosts); the last axis is addressed inside the source window
            const int w0 = (a == NX - 1) ? i0 - d.src_lo : i0;
            const int wn = (a == NX - 1) ? d.src_n : d.n[a];
            lo_ok[a] = i0 >= 0 && i0 <= d.ng[a] - 1 && w0 >= 0 && w0 <= wn - 1;
            hi_ok[a] = i0 >= -1 && i0 <= d.ng[a] - 2 && w0 >= -1 && w0 <= wn - 2;
            base += (long long)w0 * stride[a];
        }
        double val = 0.0;
#pragma unroll
        for (int corner = 0; corner < (1 << NX); ++corner) {
            double wt = 1.0;
            long long off = base;
            bool ok = true;
#pragma unroll
            for (int a = 0; a < NX; ++a) {
                const bool bit = (corner >> a) & 1;
                wt *= bit ? fr[a] : (1.0 - fr[a]);
                ok = ok && (bit ? hi_ok[a] : lo_ok[a]);
                if (bit) off += stride[a];
            }
            if (ok) val = fma(wt, (double)Wo[off], val);
        }
        const T vt = (T)val;
        Wn[pt] = vt;
        acc[0] += (double)vt;
    }
    block_sum<NMOM>(acc, red);
    if (threadIdx.x == 0)
        for (int i = 0; i < NMOM; ++i) partials[(long long)blockIdx.x * NMOM + i] = acc[i];
}

// Row-separable regrid: when the old index coordinates v_a, a >= 1, do not depend on
// the new u'_0 (M[a][0] == 0 for a >= 1 -- exactly the case after an axis-aligned
// regrid followed by a CV-type drift, whose e^{A tau} is block upper triangular),
// every point of a new axis-0 row interpolates between the SAME 2^(nx-1) old rows
// with the SAME weights: blend those rows once (coalesced), then interpolate
// linearly along axis 0 (zero ghosts at both ends). Identical to the 2^nx-tap
// multilinear formula of R12 up to rounding order. Otherwise the kernel falls back
// to the per-point gather (k_regrid_gather's arithmetic).
template <typename T, int NX, int CH = 8>               // CH: new rows per chunk (shared memory CH x N0 doubles)
__global__ void __launch_bounds__(128, 4) k_regrid_rows(const T* __restrict__ Wold, T* __restrict__ Wnew,
                                                       const FilterState* __restrict__ st, Dims d, DivSet dv,
                                                       int nbpf, double ks, double* __restrict__ partials) {
    constexpr int NC = 1 << (NX - 1);                  // old rows blended per new row
    __shared__ double red[32 * NMOM];
    __shared__ double Msh[16], osh[4];
    __shared__ int sep_sh;
    __shared__ double rw[CH][NC];                      // corner weights (0 for invalid rows)
    __shared__ long long roff[CH][NC];                 // old row offsets
    __shared__ double rv0[CH];                         // v0 at u'_0 = 0 for the row
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* tmp = reinterpret_cast<double*>(smem_raw); // [CH][N0]
    const int filt = blockIdx.x / nbpf, qb = blockIdx.x - filt * nbpf;
    const FilterState& f = st[filt];
    const int N0 = d.n[0];
    if (threadIdx.x == 0) {
        double cn[4], Bn[16], Bi[16];
        regrid_target(NX, d.ng, f, ks, cn, Bn, d.grid);
        mat_inv4(NX, f.B, Bi);
        double M[16];
        for (int i = 0; i < 16; ++i) M[i] = 0.0;
        mat_mul4(NX, Bi, Bn, M);
        int sep = 1;
        for (int a2 = 1; a2 < NX; ++a2) sep &= (M[a2 * 4] == 0.0);
        sep_sh = sep;
        for (int i = 0; i < 16; ++i) Msh[i] = M[i];
        for (int a2 = 0; a2 < NX; ++a2) {
            double sacc = 0.5 * (d.ng[a2] - 1);
            for (int b2 = 0; b2 < NX; ++b2) sacc = fma(Bi[a2 * 4 + b2], cn[b2] - f.c[b2], sacc);
            osh[a2] = sacc;
        }
    }
    __syncthreads();
    const T* Wo = Wold + (long long)filt * (d.ntot / d.n[NX - 1] * d.src_n);   // regrid source window
    T* Wn = Wnew + (long long)filt * d.ntot;
    double acc[NMOM];
#pragma unroll
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    long long stride[4];
    stride[0] = 1;
#pragma unroll
    for (int a2 = 1; a2 < NX; ++a2) stride[a2] = stride[a2 - 1] * d.n[a2 - 1];
    if (sep_sh) {
        // chunks of CH rows interleaved over the filter's blocks: the blocks running together
        // sweep one contiguous region of rows, so the old rows a chunk shares with its
        // neighbours along axes 1.. (the +1 corners: N_1 and N_1 N_2 rows ahead) are still in
        // L2 when those chunks come up. (A contiguous range per block put the concurrent
        // blocks ~rows/blocks apart: at 96^4 every corner row came from DRAM again, 2.66 GB
        // read for 0.68 GB of weights.)
        const long long rpf = d.ntot / N0;
        const float invN0 = 1.0f / N0;
        for (long long c0 = (long long)qb * CH; c0 < rpf; c0 += (long long)nbpf * CH) {
            const int nr = (int)((rpf - c0) < CH ? (rpf - c0) : CH);
            // per-row constants: old-row corners and weights, v0 offset
            if (threadIdx.x < nr) {
                const int rl = threadIdx.x;
                unsigned rr = (unsigned)(c0 + rl);
                double u[4] = {0, 0, 0, 0};
#pragma unroll
                for (int a2 = 1; a2 < NX; ++a2) {
                    const unsigned qq = (a2 < NX - 1) ? fdiv(rr, dv.n[a2]) : 0u;
                    const unsigned j = (a2 < NX - 1) ? rr - qq * (unsigned)d.n[a2] : rr;
                    u[a2] = (double)(j + d.lo[a2]) - 0.5 * (d.ng[a2] - 1);
                    rr = qq;
                }
                double fr[4] = {0, 0, 0, 0};
                int i0[4] = {0, 0, 0, 0};
                double v0 = osh[0];
#pragma unroll
                for (int b2 = 1; b2 < NX; ++b2) v0 = fma(Msh[b2], u[b2], v0);
                rv0[rl] = v0;
#pragma unroll
                for (int a2 = 1; a2 < NX; ++a2) {
                    double v = osh[a2];
#pragma unroll
                    for (int b2 = 1; b2 < NX; ++b2) v = fma(Msh[a2 * 4 + b2], u[b2], v);
                    const double fl = floor(v);
                    i0[a2] = __double2int_rz(fl);
                    fr[a2] = v - fl;
                }
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    double wt = 1.0;
                    long long off = 0;
                    bool ok = true;
#pragma unroll
                    for (int a2 = 1; a2 < NX; ++a2) {
                        const int bit = (c >> (a2 - 1)) & 1;
                        const int ia = i0[a2] + bit;
                        wt *= bit ? fr[a2] : (1.0 - fr[a2]);
                        const int wa = (a2 == NX - 1) ? ia - d.src_lo : ia;
                        const int wn = (a2 == NX - 1) ? d.src_n : d.n[a2];
                        ok = ok && ia >= 0 && ia <= d.ng[a2] - 1 && wa >= 0 && wa <= wn - 1;
                        off += (long long)wa * stride[a2];
                    }
                    rw[rl][c] = ok ? wt : 0.0;
                    roff[rl][c] = ok ? off : 0;
                }
            }
            __syncthreads();
            for (int e = threadIdx.x; e < nr * N0; e += blockDim.x) {
                const int rl = (int)((e + 0.5f) * invN0), i = e - rl * N0;
                double v = 0.0;
#pragma unroll
                for (int c = 0; c < NC; ++c) v = fma(rw[rl][c], (double)Wo[roff[rl][c] + i], v);
                tmp[rl * N0 + i] = v;
            }
            __syncthreads();
            const double M00 = Msh[0];
            for (int e = threadIdx.x; e < nr * N0; e += blockDim.x) {
                const int rl = (int)((e + 0.5f) * invN0), j = e - rl * N0;
                const double v0 = fma(M00, (double)j - 0.5 * (N0 - 1), rv0[rl]);
                const double fl = floor(v0);
                const int ia = __double2int_rz(fl);
                const double fa = v0 - fl;
                const double lo = (ia >= 0 && ia <= N0 - 1) ? tmp[rl * N0 + ia] : 0.0;
                const double hi = (ia >= -1 && ia <= N0 - 2) ? tmp[rl * N0 + ia + 1] : 0.0;
                const T vt = (T)fma(fa, hi - lo, lo);
                Wn[(c0 + rl) * N0 + j] = vt;
                acc[0] += (double)vt;
            }
            __syncthreads();
        }
    } else {
        double M[16], o[4];
#pragma unroll
        for (int i = 0; i < NX; ++i) {
            o[i] = osh[i];
#pragma unroll
            for (int j = 0; j < NX; ++j) M[i * 4 + j] = Msh[i * 4 + j];
        }
        for (long long pt = (long long)qb * blockDim.x + threadIdx.x; pt < d.ntot;
             pt += (long long)nbpf * blockDim.x) {
            double u[4];
            point_u<NX>(d, dv, (unsigned)pt, u);
            double fr[4];
            long long base = 0;
            bool lo_ok[4], hi_ok[4];
#pragma unroll
            for (int a2 = 0; a2 < NX; ++a2) {
                double sv = o[a2];
#pragma unroll
                for (int b2 = 0; b2 < NX; ++b2) sv = fma(M[a2 * 4 + b2], u[b2], sv);
                const double fl = floor(sv);
                const int ia = __double2int_rz(fl);
                fr[a2] = sv - fl;
                const int w0 = (a2 == NX - 1) ? ia - d.src_lo : ia;
                const int wn = (a2 == NX - 1) ? d.src_n : d.n[a2];
                lo_ok[a2] = ia >= 0 && ia <= d.ng[a2] - 1 && w0 >= 0 && w0 <= wn - 1;
                hi_ok[a2] = ia >= -1 && ia <= d.ng[a2] - 2 && w0 >= -1 && w0 <= wn - 2;
                base += (long long)w0 * stride[a2];
            }
            double val = 0.0;
#pragma unroll
            for (int corner = 0; corner < (1 << NX); ++corner) {
                double wt = 1.0;
                long long off = base;
                bool ok = true;
#pragma unroll
                for (int a2 = 0; a2 < NX; ++a2) {
                    const bool bit = (corner >> a2) & 1;
                    wt *= bit ? fr[a2] : (1.0 - fr[a2]);
                    ok = ok && (bit ? hi_ok[a2] : lo_ok[a2]);
                    if (bit) off += stride[a2];
                }
                if (ok) val = fma(wt, (double)Wo[off], val);
            }
            const T vt = (T)val;
            Wn[pt] = vt;
            acc[0] += (double)vt;
        }
    }
    block_sum<NMOM>(acc, red);
    if (threadIdx.x == 0)
        for (int i = 0; i < NMOM; ++i) partials[(long long)blockIdx.x * NMOM + i] = acc[i];
}

__global__ void k_finalize_regrid(FilterState* st, const double* __restrict__ partials, int nbpf, Dims d, double ks) {
    __shared__ double red[32 * NMOM];
    const int filt = blockIdx.x;
    double acc[NMOM];
    block_sum_partials(partials, (long long)filt * nbpf, nbpf, acc, red);
    if (threadIdx.x != 0) return;
    finalize_from(st[filt], acc, d, 2, ks);
}

template <typename T>
__global__ void k_scale_out(const T* __restrict__ W, T* __restrict__ dst, const FilterState* __restrict__ st,
                            long long ntot, long long total) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        long long filt = i / ntot;
        dst[i] = (T)((double)W[i] * st[filt].scale);
    }
}

// ============================================================================ compact moments for the host
// out[b] = {mean (nx), cov (nx*nx, row-major), log C, status}
__global__ void k_pack_moments(const FilterState* __restrict__ st, double* __restrict__ out, int nx, int batch) {
    const int stride = nx + nx * nx + 2;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < batch * stride; i += gridDim.x * blockDim.x) {
        const int b = i / stride, k = i - b * stride;
        const FilterState& f = st[b];
        double v;
        if (k < nx) v = f.mean[k];
        else if (k < nx + nx * nx) { const int q = k - nx; v = f.cov[(q / nx) * 4 + q % nx]; }
        else if (k == nx + nx * nx) v = f.logC;
        else v = (double)f.status;
        out[i] = v;
    }
}

cudaError_t launch_pack_moments(const Dims& d, const FilterState* st, double* out, cudaStream_t s,
                                int64_t* launches) {
    const int n = d.batch * (d.nx + d.nx * d.nx + 2);
    k_pack_moments<<<std::min((n + 255) / 256, 1184), 256, 0, s>>>(st, out, d.nx, d.batch);
    ++*launches;
    return cudaGetLastError();
}

// ============================================================================ launchers
#define PMF_TRY(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return e_; } while (0)

template <typename K>
static cudaError_t smem_attr(K kernel, size_t bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

// dispatch a launch lambda on the compile-time FFT length (0 = runtime plan)
template <typename F>
static cudaError_t with_nc(int N, F&& f) {
    switch (N) {
        case 34: return f(std::integral_constant<int, 34>{});   // the paper's N_pa = 34
        case 64: return f(std::integral_constant<int, 64>{});
        case 96: return f(std::integral_constant<int, 96>{});
        case 128: return f(std::integral_constant<int, 128>{});
        case 256: return f(std::integral_constant<int, 256>{});
        default: return f(std::integral_constant<int, 0>{});
    }
}

// Phases of the nx >= 2 predict (so the sharded path can insert its transposes):
//   PH_FWD: axis-0 R2C + forward C2C along axes 1..L-1 (L = nx-1)
//   PH_PSI: last axis forward * s Psi * inverse on `psibuf` (I x N_L pencils, inner offset)
//   PH_INV: inverse C2C axes L-1..1 + axis-0 C2R (+ update); moment partials reduced to
//           `tot` (sharded) or finalised into the state (tot == nullptr)
enum { PH_FWD = 1, PH_PSI = 2, PH_INV = 4, PH_ALL = 7 };

template <typename T, int NX>
static cudaError_t predict_nd(const Dims& d, PencilBufs& b, const Twiddles& tw, const ModelParams& mp,
                              const LikParams* lp, const LikParams& lpv, int cs, cudaStream_t s, int64_t* launches,
                              int phases = PH_ALL, void* psibuf = nullptr, long long psiI = -1,
                              long long inner_off = 0, double* tot = nullptr) {
    using V = typename C2<T>::type;
    const DivSet dv = make_divs(d);
    const int N0 = d.n[0];
    const long long rpf = d.ntot / N0;
    const int P0 = rows_per_cta(N0, rpf);
    FFTPlan pl0 = make_plan(N0);
    size_t sm0 = 2 * (size_t)P0 * pstride_host(N0) * sizeof(V);
    long long nrow_blocks = (long long)d.batch * rpf / P0;
    // strided axes
    auto strided = [&](int m, int mode, V* buf, long long Iov, long long Oov, long long ioff) -> cudaError_t {
        long long I = d.H0;
        for (int q = 1; q < m; ++q) I *= d.n[q];
        long long O = d.batch;
        for (int q = m + 1; q < d.nx; ++q) O *= d.n[q];
        if (Iov >= 0) { I = Iov; O = Oov; }
        const int N = (Iov >= 0) ? d.ng[m] : d.n[m];
        const int P = pencils_per_cta(N);
        FFTPlan pl = make_plan(N);
        size_t sm = 2 * (size_t)P * pstride_host(N) * sizeof(V);
        if (mode == 2) sm += sizeof(double) * 2 * P * std::min(mp.l + (mp.step ? 1 : 0), LCAP);
        long long nblk = O * ((I + P - 1) / P);
        if (nblk == 0) return cudaSuccess;
        cudaError_t e = with_nc(N, [&](auto nc) -> cudaError_t {
            constexpr int NC = decltype(nc)::value;
            if (mode == 0) {
                PMF_TRY(smem_attr(k_axis_c2c<T, 0, 2, NC>, sm));
                k_axis_c2c<T, 0, 2, NC><<<(unsigned)nblk, kThreads, sm, s>>>(buf, d, m, I, pl, (const V*)tw.tw[m], P,
                                                                              b.coef, cs, mp, ioff);
            } else if (mode == 1) {
                PMF_TRY(smem_attr(k_axis_c2c<T, 1, 2, NC>, sm));
                k_axis_c2c<T, 1, 2, NC><<<(unsigned)nblk, kThreads, sm, s>>>(buf, d, m, I, pl, (const V*)tw.tw[m], P,
                                                                              b.coef, cs, mp, ioff);
            } else {
                PMF_TRY(smem_attr(k_axis_c2c<T, 2, NX, NC>, sm));
                k_axis_c2c<T, 2, NX, NC><<<(unsigned)nblk, kThreads, sm, s>>>(buf, d, m, I, pl, (const V*)tw.tw[m],
                                                                               P, b.coef, cs, mp, ioff);
            }
            return cudaGetLastError();
        });
        ++*launches;
        return e;
    };
    if (phases & PH_FWD) {
        // axis 0 forward (R2C)
        PMF_TRY(with_nc(N0, [&](auto nc) -> cudaError_t {
            constexpr int NC = decltype(nc)::value;
            PMF_TRY(smem_attr(k_axis0_r2c<T, NC>, sm0));
            k_axis0_r2c<T, NC><<<(unsigned)nrow_blocks, kThreads, sm0, s>>>((const T*)b.W, (V*)b.S, b.coef, cs, d,
                                                                            pl0, (const V*)tw.tw[0], P0);
            return cudaGetLastError();
        }));
        ++*launches;
        for (int m = 1; m < d.nx - 1; ++m) PMF_TRY(strided(m, 0, (V*)b.S, -1, -1, 0));
    }
    if (phases & PH_PSI) {
        if (psibuf) PMF_TRY(strided(d.nx - 1, 2, (V*)psibuf, psiI, 1, inner_off));
        else PMF_TRY(strided(d.nx - 1, 2, (V*)b.S, -1, -1, 0));
    }
    if (phases & PH_INV) {
        for (int m = d.nx - 2; m >= 1; --m) PMF_TRY(strided(m, 1, (V*)b.S, -1, -1, 0));
        // axis 0 inverse (C2R) + update: cpf CTAs per filter, tpc tiles each
        const int tiles_pf = (int)(rpf / P0);
        const int cpf = std::max(1, std::min(tiles_pf, 2048 / std::max(1, d.batch)));
        const int tpc = (tiles_pf + cpf - 1) / cpf;
        const int cpf_used = (tiles_pf + tpc - 1) / tpc;
        size_t smc = sm0 + 32 * NMOM * sizeof(double) + 6 * sizeof(double) * P0;
        PMF_TRY(with_nc(N0, [&](auto nc) -> cudaError_t {
            constexpr int NC = decltype(nc)::value;
            if (lp) {
                PMF_TRY(smem_attr(k_axis0_c2r<T, true, NX, NC>, smc));
                k_axis0_c2r<T, true, NX, NC><<<(unsigned)(cpf_used * d.batch), kThreads, smc, s>>>(
                    (const V*)b.S, (T*)b.W, b.st, d, dv, pl0, (const V*)tw.tw[0], P0, lpv, b.z, b.coef, cs,
                    lq_off(mp.l), b.partials, cpf_used, tpc);
            } else {
                PMF_TRY(smem_attr(k_axis0_c2r<T, false, NX, NC>, smc));
                k_axis0_c2r<T, false, NX, NC><<<(unsigned)(cpf_used * d.batch), kThreads, smc, s>>>(
                    (const V*)b.S, (T*)b.W, b.st, d, dv, pl0, (const V*)tw.tw[0], P0, lpv, b.z, b.coef, cs,
                    lq_off(mp.l), b.partials, cpf_used, tpc);
            }
            return cudaGetLastError();
        }));
        ++*launches;
        if (lp) {
            if (tot) k_reduce_partials<<<d.batch, kThreads, 0, s>>>(b.partials, cpf_used, tot);
            else k_finalize<<<d.batch, kThreads, 0, s>>>(b.st, b.partials, cpf_used, d, 0);
            ++*launches;
        }
    }
    return cudaGetLastError();
}

template <typename T>
static cudaError_t predict_pencil_t(const Dims& d, PencilBufs& b, const Twiddles& tw, const ModelParams& mp,
                                    const LikParams* lp, cudaStream_t s, int64_t* launches) {
    using V = typename C2<T>::type;
    const int cs = coef_stride(mp.l);
    LikParams lpv{};
    if (lp) lpv = *lp;
    if (b.ev0) cudaEventRecordWithFlags(b.ev0, s, cudaEventRecordExternal);
    k_predict_prep<<<d.batch, 32, 0, s>>>(b.st, b.coef, cs, mp, b.sub, d.batch, lpv, b.z,
                                                         lp ? 1 : 0);
    ++*launches;
    PMF_TRY(cudaGetLastError());
    cudaError_t e = cudaSuccess;
    if (d.nx == 1) {
        FFTPlan pl = make_plan(d.n[0]);
        size_t sm = 2 * pstride_host(d.n[0]) * sizeof(V) + 32 * NMOM * sizeof(double);
        PMF_TRY(with_nc(d.n[0], [&](auto nc) -> cudaError_t {
            constexpr int NC = decltype(nc)::value;
            PMF_TRY(smem_attr(k_line_psi<T, true, NC>, sm));
            PMF_TRY(smem_attr(k_line_psi<T, false, NC>, sm));
            if (lp)
                k_line_psi<T, true, NC><<<d.batch, kThreads, sm, s>>>((T*)b.W, b.st, d, pl, (const V*)tw.tw[0],
                                                                      b.coef, cs, mp, lpv, b.z, b.partials);
            else
                k_line_psi<T, false, NC><<<d.batch, kThreads, sm, s>>>((T*)b.W, b.st, d, pl, (const V*)tw.tw[0],
                                                                       b.coef, cs, mp, lpv, b.z, b.partials);
            return cudaGetLastError();
        }));
        ++*launches;
        if (lp) {
            k_finalize<<<d.batch, kThreads, 0, s>>>(b.st, b.partials, 1, d, 0);
            ++*launches;
        }
        e = cudaGetLastError();
    } else if (d.nx == 2) {
        e = predict_nd<T, 2>(d, b, tw, mp, lp, lpv, cs, s, launches);
    } else if (d.nx == 3) {
        e = predict_nd<T, 3>(d, b, tw, mp, lp, lpv, cs, s, launches);
    } else {
        e = predict_nd<T, 4>(d, b, tw, mp, lp, lpv, cs, s, launches);
    }
    if (b.ev1) cudaEventRecordWithFlags(b.ev1, s, cudaEventRecordExternal);
    return e;
}

template <typename T>
static cudaError_t line_epoch_t(const Dims& d, PencilBufs& b, const Twiddles& tw, const ModelParams& mp,
                                const LikParams* lp, double ks, cudaStream_t s, int64_t* launches) {
    using V = typename C2<T>::type;
    const int nsets = mp.l + (mp.step ? 1 : 0);
    FFTPlan pl = make_plan(d.n[0]);
    const size_t sm = 2 * pstride_host(d.n[0]) * sizeof(V) + 32 * NMOM * sizeof(double) + nsets * sizeof(double);
    LikParams lpv{};
    if (lp) lpv = *lp;
    if (b.ev0) cudaEventRecordWithFlags(b.ev0, s, cudaEventRecordExternal);
    PMF_TRY(with_nc(d.n[0], [&](auto nc) -> cudaError_t {
        constexpr int NC = decltype(nc)::value;
        auto go = [&](auto kern) -> cudaError_t {
            PMF_TRY(smem_attr(kern, sm));
            // one thread per point up to kThreads: short lines keep their reductions and
            // barriers cheap
            const int nt = std::min(kThreads, std::max(64, (d.n[0] + 31) / 32 * 32));
            kern<<<d.batch, nt, sm, s>>>((T*)b.W, b.st, d, pl, (const V*)tw.tw[0], mp, b.sub, lpv, b.z, ks);
            return cudaGetLastError();
        };
        if (lp && ks > 0.0) return go(k_line_epoch<T, true, true, NC>);
        if (lp) return go(k_line_epoch<T, true, false, NC>);
        if (ks > 0.0) return go(k_line_epoch<T, false, true, NC>);
        return go(k_line_epoch<T, false, false, NC>);
    }));
    ++*launches;
    if (b.ev1) cudaEventRecordWithFlags(b.ev1, s, cudaEventRecordExternal);
    return cudaGetLastError();
}

// nx = 1 whole epoch in one launch; nsets coefficients must fit next to the two lines
bool line_epoch_supported(const Dims& d, int nsets) {
    return d.nx == 1 && nsets <= 4096 && d.n[0] <= 4096;
}

cudaError_t launch_line_epoch(const Dims& d, int dtype, PencilBufs& b, const Twiddles& tw, const ModelParams& mp,
                              const LikParams* lp, double ks, cudaStream_t s, int64_t* launches) {
    if (dtype == 0) return line_epoch_t<double>(d, b, tw, mp, lp, ks, s, launches);
    return line_epoch_t<float>(d, b, tw, mp, lp, ks, s, launches);
}

cudaError_t launch_predict_pencil(const Dims& d, int dtype, PencilBufs& b, const Twiddles& tw,
                                  const ModelParams& mp, const LikParams* lp, cudaStream_t s, int64_t* launches) {
    if (dtype == 0) return predict_pencil_t<double>(d, b, tw, mp, lp, s, launches);
    return predict_pencil_t<float>(d, b, tw, mp, lp, s, launches);
}

template <typename T, int MODE, int NX>
static cudaError_t points_nd(const Dims& d, PencilBufs& b, const LikParams& lp, cudaStream_t s, int64_t* launches,
                             int fin_mode) {
    const int nbpf = wave_bpf(k_points<T, MODE, NX>, kThreads, 0, d.ntot, d.batch);
    k_points<T, MODE, NX><<<(unsigned)((long long)nbpf * d.batch), kThreads, 0, s>>>(
        (T*)b.W, b.st, d, make_divs(d), nbpf, lp, b.z, b.gauss, b.partials);
    ++*launches;
    PMF_TRY(cudaGetLastError());
    k_finalize<<<d.batch, kThreads, 0, s>>>(b.st, b.partials, nbpf, d, fin_mode);
    ++*launches;
    return cudaGetLastError();
}

template <typename T, int MODE>
static cudaError_t points_t(const Dims& d, PencilBufs& b, const LikParams& lp, cudaStream_t s, int64_t* launches,
                            int fin_mode) {
    switch (d.nx) {
        case 1: return points_nd<T, MODE, 1>(d, b, lp, s, launches, fin_mode);
        case 2: return points_nd<T, MODE, 2>(d, b, lp, s, launches, fin_mode);
        case 3: return points_nd<T, MODE, 3>(d, b, lp, s, launches, fin_mode);
        default: return points_nd<T, MODE, 4>(d, b, lp, s, launches, fin_mode);
    }
}

cudaError_t launch_update(const Dims& d, int dtype, PencilBufs& b, const LikParams& lp, cudaStream_t s,
                          int64_t* launches) {
    if (dtype == 0) return points_t<double, 0>(d, b, lp, s, launches, 0);
    return points_t<float, 0>(d, b, lp, s, launches, 0);
}

cudaError_t launch_init_gaussian(const Dims& d, int dtype, PencilBufs& b, cudaStream_t s, int64_t* launches) {
    LikParams lp{};
    if (dtype == 0) return points_t<double, 1>(d, b, lp, s, launches, 1);
    return points_t<float, 1>(d, b, lp, s, launches, 1);
}

cudaError_t launch_normalise_state(const Dims& d, int dtype, PencilBufs& b, cudaStream_t s, int64_t* launches) {
    LikParams lp{};
    if (dtype == 0) return points_t<double, 2>(d, b, lp, s, launches, 1);
    return points_t<float, 2>(d, b, lp, s, launches, 1);
}

template <typename T, int NX>
static cudaError_t regrid_nd(const Dims& d, PencilBufs& b, double ks, cudaStream_t s, int64_t* launches) {
    int nbpf = blocks_per_filter(d.ntot);
    if (NX >= 2) {
        // row-separable path (falls back to the per-point gather inside when M is not)
        const size_t sm = sizeof(double) * 8 * (size_t)d.n[0];
        PMF_TRY(smem_attr(k_regrid_rows<T, NX>, sm));
        nbpf = wave_bpf(k_regrid_rows<T, NX>, 128, sm, d.ntot, d.batch);
        k_regrid_rows<T, NX><<<(unsigned)((long long)nbpf * d.batch), 128, sm, s>>>(
            (const T*)b.W, (T*)b.W2, b.st, d, make_divs(d), nbpf, ks, b.partials);
    } else {
        k_regrid_gather<T, NX><<<(unsigned)((long long)nbpf * d.batch), kThreads, 0, s>>>(
            (const T*)b.W, (T*)b.W2, b.st, d, make_divs(d), nbpf, ks, b.partials);
    }
    ++*launches;
    PMF_TRY(cudaGetLastError());
    k_finalize_regrid<<<d.batch, kThreads, 0, s>>>(b.st, b.partials, nbpf, d, ks);
    ++*launches;
    std::swap(b.W, b.W2);
    return cudaGetLastError();
}

template <typename T>
static cudaError_t regrid_t(const Dims& d, PencilBufs& b, double ks, cudaStream_t s, int64_t* launches) {
    switch (d.nx) {
        case 1: return regrid_nd<T, 1>(d, b, ks, s, launches);
        case 2: return regrid_nd<T, 2>(d, b, ks, s, launches);
        case 3: return regrid_nd<T, 3>(d, b, ks, s, launches);
        default: return regrid_nd<T, 4>(d, b, ks, s, launches);
    }
}

cudaError_t launch_regrid(const Dims& d, int dtype, PencilBufs& b, double ks, cudaStream_t s, int64_t* launches) {
    if (dtype == 0) return regrid_t<double>(d, b, ks, s, launches);
    return regrid_t<float>(d, b, ks, s, launches);
}

// ============================================================================ sharded building blocks
template <typename T>
static cudaError_t sh_phase_t(const Dims& d, PencilBufs& b, const Twiddles& tw, const ModelParams& mp,
                              const LikParams* lp, int phase, void* psibuf, long long psiI, long long ioff,
                              double* tot, cudaStream_t s, int64_t* launches) {
    const int cs = coef_stride(mp.l);
    LikParams lpv{};
    if (lp) lpv = *lp;
    if (d.nx == 2) return predict_nd<T, 2>(d, b, tw, mp, lp, lpv, cs, s, launches, phase, psibuf, psiI, ioff, tot);
    if (d.nx == 3) return predict_nd<T, 3>(d, b, tw, mp, lp, lpv, cs, s, launches, phase, psibuf, psiI, ioff, tot);
    return predict_nd<T, 4>(d, b, tw, mp, lp, lpv, cs, s, launches, phase, psibuf, psiI, ioff, tot);
}

cudaError_t sh_prep(const Dims& d, PencilBufs& b, const ModelParams& mp, const LikParams* lp, cudaStream_t s,
                    int64_t* launches) {
    LikParams lpv{};
    if (lp) lpv = *lp;
    k_predict_prep<<<d.batch, 32, 0, s>>>(b.st, b.coef, coef_stride(mp.l), mp, b.sub, d.batch, lpv,
                                                         b.z, lp ? 1 : 0);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t sh_phase(const Dims& d, int dtype, PencilBufs& b, const Twiddles& tw, const ModelParams& mp,
                     const LikParams* lp, int phase, void* psibuf, long long psiI, long long ioff, double* tot,
                     cudaStream_t s, int64_t* launches) {
    if (dtype == 0) return sh_phase_t<double>(d, b, tw, mp, lp, phase, psibuf, psiI, ioff, tot, s, launches);
    return sh_phase_t<float>(d, b, tw, mp, lp, phase, psibuf, psiI, ioff, tot, s, launches);
}

cudaError_t sh_pack(int dtype, void* S, void* send, long long I, int planes, const long long* d_off, int world,
                    int unpack, cudaStream_t s, int64_t* launches) {
    const long long total = (long long)planes * I;
    const unsigned nb = (unsigned)std::max(1LL, std::min((total + 255) / 256, 148LL * 32));
    if (dtype == 0)
        k_pack_blocks<double2><<<nb, 256, 0, s>>>((const double2*)S, (double2*)send, I, planes, d_off, world, unpack);
    else
        k_pack_blocks<float2><<<nb, 256, 0, s>>>((const float2*)S, (float2*)send, I, planes, d_off, world, unpack);
    ++*launches;
    return cudaGetLastError();
}

template <typename T, int MODE>
static cudaError_t sh_points_t(const Dims& d, PencilBufs& b, const LikParams& lp, double* tot, cudaStream_t s,
                               int64_t* launches) {
    int nbpf = blocks_per_filter(d.ntot);
    const unsigned g = (unsigned)((long long)nbpf * d.batch);
    switch (d.nx) {
        case 2: k_points<T, MODE, 2><<<g, kThreads, 0, s>>>((T*)b.W, b.st, d, make_divs(d), nbpf, lp, b.z, b.gauss,
                                                             b.partials); break;
        case 3: k_points<T, MODE, 3><<<g, kThreads, 0, s>>>((T*)b.W, b.st, d, make_divs(d), nbpf, lp, b.z, b.gauss,
                                                             b.partials); break;
        default: k_points<T, MODE, 4><<<g, kThreads, 0, s>>>((T*)b.W, b.st, d, make_divs(d), nbpf, lp, b.z, b.gauss,
                                                              b.partials); break;
    }
    ++*launches;
    PMF_TRY(cudaGetLastError());
    k_reduce_partials<<<d.batch, kThreads, 0, s>>>(b.partials, nbpf, tot);
    ++*launches;
    return cudaGetLastError();
}

// mode: 0 likelihood update, 1 init gaussian, 2 plain sum (set_state)
cudaError_t sh_points(const Dims& d, int dtype, PencilBufs& b, int mode, const LikParams& lp, double* tot,
                      cudaStream_t s, int64_t* launches) {
    if (dtype == 0) {
        if (mode == 0) return sh_points_t<double, 0>(d, b, lp, tot, s, launches);
        if (mode == 1) return sh_points_t<double, 1>(d, b, lp, tot, s, launches);
        return sh_points_t<double, 2>(d, b, lp, tot, s, launches);
    }
    if (mode == 0) return sh_points_t<float, 0>(d, b, lp, tot, s, launches);
    if (mode == 1) return sh_points_t<float, 1>(d, b, lp, tot, s, launches);
    return sh_points_t<float, 2>(d, b, lp, tot, s, launches);
}

template <typename T>
static cudaError_t sh_regrid_t(const Dims& d, const void* src, void* dst, PencilBufs& b, double ks, double* tot,
                               cudaStream_t s, int64_t* launches) {
    int nbpf = blocks_per_filter(d.ntot);
    const unsigned g = (unsigned)((long long)nbpf * d.batch);
    // large slabs (many chunks per block): 32-row chunks -- the per-row setup runs on a full
    // warp and the two barriers per chunk are amortised over 4x the points
    const bool big = d.ntot / d.n[0] / nbpf >= 128 && d.n[0] <= 128;
    const size_t sm = sizeof(double) * (big ? 32 : 8) * (size_t)d.n[0];
#define PMF_RG_ROWS(NX_)                                                                                              \
    if (big) {                                                                                                         \
        PMF_TRY(smem_attr(k_regrid_rows<T, NX_, 32>, sm));                                                             \
        k_regrid_rows<T, NX_, 32><<<g, 128, sm, s>>>((const T*)src, (T*)dst, b.st, d, make_divs(d), nbpf, ks,          \
                                                     b.partials);                                                      \
    } else {                                                                                                           \
        PMF_TRY(smem_attr(k_regrid_rows<T, NX_>, sm));                                                                 \
        k_regrid_rows<T, NX_><<<g, 128, sm, s>>>((const T*)src, (T*)dst, b.st, d, make_divs(d), nbpf, ks, b.partials); \
    }
    switch (d.nx) {
        case 2: PMF_RG_ROWS(2) break;
        case 3: PMF_RG_ROWS(3) break;
        default: PMF_RG_ROWS(4) break;
    }
#undef PMF_RG_ROWS
    ++*launches;
    PMF_TRY(cudaGetLastError());
    k_reduce_partials<<<d.batch, kThreads, 0, s>>>(b.partials, nbpf, tot);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t sh_regrid(const Dims& d, int dtype, const void* src, void* dst, PencilBufs& b, double ks, double* tot,
                      cudaStream_t s, int64_t* launches) {
    if (dtype == 0) return sh_regrid_t<double>(d, src, dst, b, ks, tot, s, launches);
    return sh_regrid_t<float>(d, src, dst, b, ks, tot, s, launches);
}

// sum over ranks in rank order (virtual-rank all-reduce)
__global__ void k_sum_ranks(const double* __restrict__ in, double* __restrict__ out, int world, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    for (int r = 0; r < world; ++r) s += in[r * n + i];
    out[i] = s;
}

cudaError_t launch_sum_ranks(const double* in, double* out, int world, int n, cudaStream_t s, int64_t* launches) {
    k_sum_ranks<<<(n + 127) / 128, 128, 0, s>>>(in, out, world, n);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_finalize_tot(const Dims& d, FilterState* st, const double* tot, int mode, double ks,
                                cudaStream_t s, int64_t* launches) {
    k_finalize_tot<<<(d.batch + 127) / 128, 128, 0, s>>>(st, tot, d, mode, ks, d.batch);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_scale_out(const Dims& d, int dtype, const PencilBufs& b, void* dst, cudaStream_t s,
                             int64_t* launches) {
    long long total = d.ntot * d.batch;
    unsigned nb = (unsigned)std::min<long long>((total + 255) / 256, 148LL * 16);
    if (dtype == 0) k_scale_out<double><<<nb, 256, 0, s>>>((const double*)b.W, (double*)dst, b.st, d.ntot, total);
    else k_scale_out<float><<<nb, 256, 0, s>>>((const float*)b.W, (float*)dst, b.st, d.ntot, total);
    ++*launches;
    return cudaGetLastError();
}

}  // namespace pmf
