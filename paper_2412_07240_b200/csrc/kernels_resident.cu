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
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>

#include "device_common.cuh"
#include "fft_reg.cuh"

namespace pmf {

// Phase cycle counters of the resident kernel (debug builds with -DPMF_QPROF only; thread 0
// of every CTA adds its clock64() deltas; read with pmf_debug_counters index 16..).
__device__ unsigned long long g_rprof[12];
#ifdef PMF_QPROF
#define RPROF_T(v) \
    __syncthreads();  \
    const long long v = clock64()
#define RPROF_ADD(i, a, b) \
    if (threadIdx.x == 0) atomicAdd(&g_rprof[i], (unsigned long long)((b) - (a)))
#define RPROF_SET(v) \
    __syncthreads();   \
    v = clock64()
#else
#define RPROF_SET(v)
#define RPROF_T(v)
#define RPROF_ADD(i, a, b)
#endif

namespace res {

constexpr int N = 128;            // points per axis
constexpr int H = N / 2 + 1;      // 65 rows of the half spectrum (k1 = 0..64)
constexpr int PITCH = 130;        // row pitch in complex elements (= 2 mod 8: conflict-free exchanges)
constexpr int NT = 512;           // threads: 64 teams x 8

using namespace reg;

// x[s] *= W_128^{ts} (conjugated for INV), s = 1..15, as W^{ta} W^{4tb} (s = a + 4b, a < 4):
// six 16-byte table loads and nine complex products instead of fifteen loads
template <bool INV, typename V>
__device__ __forceinline__ void tw16(V* x, const V* tw, int t) {
    V wa[4];
#pragma unroll
    for (int a = 1; a < 4; ++a) {
        wa[a] = tw[a * 8 + t];
        if (INV) wa[a].y = -wa[a].y;
        x[a] = cmul(x[a], wa[a]);
    }
#pragma unroll
    for (int b = 1; b < 4; ++b) {
        V wb = tw[4 * b * 8 + t];
        if (INV) wb.y = -wb.y;
        x[4 * b] = cmul(x[4 * b], wb);
#pragma unroll
        for (int a = 1; a < 4; ++a) x[a + 4 * b] = cmul(x[a + 4 * b], cmul(wa[a], wb));
    }
}

// Spectrum element (k1, j0) lives at X[k1 * PITCH + xcol(k1, j0)]: the two columns of a
// pair swap places in rows with (k1 & 4), so the 8 threads of a team touching rows
// t + 16 q of one column hit 8 distinct 16-byte bank groups (PITCH = 2 mod 8).
__device__ __forceinline__ int xcol(int k1, int j0) { return j0 ^ ((k1 >> 2) & 1); }
// exchange slot of element (s, t) inside a row (128 consecutive complex)
__device__ __forceinline__ int rslot(int s, int t) { return s * 8 + (t ^ (s & 7)); }
// exchange slot of element (s, t) inside the column pair of a team: (row, col)
__device__ __forceinline__ int cslot(int s, int t, int m) {
    const int row = 4 * s + ((t >> 1) ^ (s & 3));
    const int col = (t & 1) ^ ((s >> 2) & 1);
    return row * PITCH + 2 * m + col;
}

// ---------------------------------------------------------------------------
// Per-filter constants of one epoch, written by k_res_prep (one warp per
// filter) into a global table and staged into shared memory by TMA together
// with the filter's weights. Layout (doubles), stride PRM_FIXED + 3 l (even):
enum {
    P_M = 0,        // 4: regrid map v = o + M u' (old index coordinates of new point u')
    P_O = 4,        // 2
    P_CL = 6,       // 2: moved grid centre c_l = e^{A tau} c0
    P_BL = 8,       // 4: moved grid matrix B_l = e^{A tau} B0 (row-major 2x2)
    P_VOL = 12,     // |det B_l|
    P_QA = 13,      // linear-Gauss exponent e(u) = qa + qb.u + u^T G u (G = [g0 g1; g1 g2])
    P_QB = 14,      // 2
    P_QG = 16,      // 3
    P_ZR = 19,      // range measurement z
    P_SKIP = 20,    // 1.0: skip this filter (failed earlier / degenerate regrid)
    P_S = 21,       // s / N^2 (trace factor and the transform scales)
    P_LGN = 22,     // log normalising constant of the likelihood
    P_ISG = 23,     // 1 / sigma (range likelihood)
    PRM_FIXED = 24  // then 3 doubles per coefficient set: h D00, h D11, 2h D01 with h = dt/2 (Euler,
                    // l sets) or dt/4 (Crank-Nicolson, R27: l + 1 sets, grids t_0 .. t_l)
};
inline int prm_stride(int nsets) { return (PRM_FIXED + 3 * nsets + 1) & ~1; }

}  // namespace res

using namespace res;

// ============================================================================ prep (one warp per filter)
// Grid constants of the epoch: regrid target (R12), start-of-interval grid
// (c0, B0), moved grid B_l = e^{A tau} B0 (eq:gridMov P:142-148), Euler-factor
// coefficients on B0 for the l substeps (Alg. 3, R3/R4), and the
// likelihood exponent as a quadratic form in the moved grid's index
// coordinates (eq:meas P:36, R13). The state's grid becomes (c_l, B_l).
// One warp per filter: the lanes share the substeps, lane 0 does the rest.
__global__ void k_res_prep(FilterState* st, double* prm, int pstride, ModelParams mp,
                           const SubstepEntry* __restrict__ sub, LikParams lp, const double* __restrict__ z,
                           double ks, int update, int batch, int grid) {
    const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (b >= batch) return;
    FilterState& f = st[b];
    double* P = prm + (long long)b * pstride;
    const double B[4] = {f.B[0], f.B[1], f.B[4], f.B[5]};
    const double c[2] = {f.c[0], f.c[1]};
    double B0[4] = {B[0], B[1], B[2], B[3]}, c0[2] = {c[0], c[1]};
    bool skip = f.status != 0;
    if (ks > 0.0) {
        const double v0 = f.cov[0], v1 = f.cov[5];
        if (!(v0 > 0.0) || !(v1 > 0.0) || !isfinite(v0) || !isfinite(v1)) skip = true;
        c0[0] = f.mean[0];
        c0[1] = f.mean[1];
        if (grid == 1) {                      // R28: eigen-aligned target
            const int nn[2] = {N, N};
            double Be[16];
            if (!eigen_grid(2, nn, f.cov, ks, Be)) skip = true;
            B0[0] = Be[0];
            B0[1] = Be[1];
            B0[2] = Be[4];
            B0[3] = Be[5];
        } else {                              // R12: axis-aligned target
            B0[0] = 2.0 * ks * sqrt(v0) / N;
            B0[1] = 0.0;
            B0[2] = 0.0;
            B0[3] = 2.0 * ks * sqrt(v1) / N;
        }
        const double det = B[0] * B[3] - B[1] * B[2];
        const double Bi[4] = {B[3] / det, -B[1] / det, -B[2] / det, B[0] / det};
        if (lane == 0) {
            P[P_M + 0] = Bi[0] * B0[0] + Bi[1] * B0[2];
            P[P_M + 1] = Bi[0] * B0[1] + Bi[1] * B0[3];
            P[P_M + 2] = Bi[2] * B0[0] + Bi[3] * B0[2];
            P[P_M + 3] = Bi[2] * B0[1] + Bi[3] * B0[3];
            const double d0 = c0[0] - c[0], d1 = c0[1] - c[1];
            P[P_O + 0] = fma(Bi[0], d0, fma(Bi[1], d1, 0.5 * (N - 1)));
            P[P_O + 1] = fma(Bi[2], d0, fma(Bi[3], d1, 0.5 * (N - 1)));
        }
    }
    __syncwarp();                            // every lane has read the state
    if (lane == 0) P[P_SKIP] = skip ? 1.0 : 0.0;
    if (skip) {
        if (lane == 0) f.status = -6;
        return;
    }
    const double det0 = B0[0] * B0[3] - B0[1] * B0[2];
    const double Bi0[4] = {B0[3] / det0, -B0[1] / det0, -B0[2] / det0, B0[0] / det0};
    const double h = mp.step ? 0.25 * mp.dt : 0.5 * mp.dt;
    for (int n = lane; n < mp.l + (mp.step ? 1 : 0); n += 32) {
        double D00, D01, D11;
        if (mp.diff_mode == 0) {           // R3: D_n = B0^-1 E_n B0^-T
            const double* E = sub[n].E;
            const double t00 = fma(Bi0[0], E[0], Bi0[1] * E[4]);
            const double t01 = fma(Bi0[0], E[1], Bi0[1] * E[5]);
            const double t10 = fma(Bi0[2], E[0], Bi0[3] * E[4]);
            const double t11 = fma(Bi0[2], E[1], Bi0[3] * E[5]);
            D00 = fma(t00, Bi0[0], t01 * Bi0[1]);
            D01 = 0.5 * (fma(t00, Bi0[2], t01 * Bi0[3]) + fma(t10, Bi0[0], t11 * Bi0[1]));
            D11 = fma(t10, Bi0[2], t11 * Bi0[3]);
        } else {                           // Alg. 3 literally: per-axis L^(m) = N ||B_n[:,m]||
            const double* Pn = sub[n].P;
            const double b00 = fma(Pn[0], B0[0], Pn[1] * B0[2]);
            const double b01 = fma(Pn[0], B0[1], Pn[1] * B0[3]);
            const double b10 = fma(Pn[4], B0[0], Pn[5] * B0[2]);
            const double b11 = fma(Pn[4], B0[1], Pn[5] * B0[3]);
            D00 = mp.Q[0] / fma(b00, b00, b10 * b10);
            D11 = mp.Q[5] / fma(b01, b01, b11 * b11);
            D01 = 0.0;
        }
        P[PRM_FIXED + 3 * n] = h * D00;
        P[PRM_FIXED + 3 * n + 1] = h * D11;
        P[PRM_FIXED + 3 * n + 2] = 2.0 * h * D01;
    }
    if (lane != 0) return;
    const double* Mt = mp.Mtau;      // stride 4
    double Bl[4], cl[2];
    Bl[0] = fma(Mt[0], B0[0], Mt[1] * B0[2]);
    Bl[1] = fma(Mt[0], B0[1], Mt[1] * B0[3]);
    Bl[2] = fma(Mt[4], B0[0], Mt[5] * B0[2]);
    Bl[3] = fma(Mt[4], B0[1], Mt[5] * B0[3]);
    cl[0] = fma(Mt[0], c0[0], Mt[1] * c0[1]);
    cl[1] = fma(Mt[4], c0[0], Mt[5] * c0[1]);
    for (int q = 0; q < 4; ++q) P[P_BL + q] = Bl[q];
    P[P_CL] = cl[0];
    P[P_CL + 1] = cl[1];
    P[P_VOL] = fabs(Bl[0] * Bl[3] - Bl[1] * Bl[2]);
    P[P_S] = mp.s / (double)(N * N);
    P[P_LGN] = lp.lognorm;
    P[P_ISG] = lp.inv_sigma;
    if (update && lp.kind == 0) {
        const double* zf = z + (long long)b * lp.nz;
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
        P[P_QA] = qa;
        P[P_QB] = qb0;
        P[P_QB + 1] = qb1;
        P[P_QG] = g00;
        P[P_QG + 1] = g01;
        P[P_QG + 2] = g11;
    } else if (update) {
        P[P_ZR] = z[b];
    }
    f.c[0] = cl[0];
    f.c[1] = cl[1];
    f.B[0] = Bl[0];
    f.B[1] = Bl[1];
    f.B[4] = Bl[2];
    f.B[5] = Bl[3];
}

// ============================================================================ finalize (1 thread per filter)
// out[b] = {sum w, sum w u0, sum w u1, sum w u0^2, sum w u0 u1, sum w u1^2, DC}.
// Update: C = sum w / (s DC), log C, scale = 1/(vol_l sum w), moments (R14).
// Predict only: closed-form normalisation scale = 1 / (vol_l s DC) (Alg. 6).
__global__ void k_res_finalize(FilterState* st, const double* __restrict__ out, const double* __restrict__ prm,
                               int pstride, double s, int update, int batch) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    const double* P = prm + (long long)b * pstride;
    if (P[P_SKIP] != 0.0) return;
    FilterState& f = st[b];
    const double* o = out + (long long)b * 8;
    const double vol = P[P_VOL];
    if (!update) {
        f.scale = 1.0 / (vol * s * o[6]);
        return;
    }
    // stored weights are the unnormalised prior (sum = s DC) times the likelihood:
    // normaliser C = vol sum(prior_normalised lik) = o[0] / (s DC)
    const double C = o[0] / (s * o[6]);
    f.mass = o[0];
    f.has_moments = 1;
    if (!(C > 0.0) || !isfinite(C) || !(o[0] > 0.0)) {
        f.status = -6;
        f.logC = -INFINITY;
        return;
    }
    f.status = 0;
    f.logC = log(C);
    f.scale = 1.0 / (vol * o[0]);
    double acc[NMOM];
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    for (int i = 0; i < 6; ++i) acc[i] = o[i];
    finish_moments(2, acc, f.c, f.B, f.mean, f.cov);
}

// ============================================================================ TMA helpers
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <typename T>
struct ResArgs {
    T* W;
    const double* prm;
    double* out;
    int pstride;
    int l;
    int batch;
    int range;        // likelihood kind 1
};

// Staging row pitch in bytes for the weights (padded so the regrid gather's 8
// rows per team hit distinct banks; 16-byte aligned for the bulk copies).
// Staged weights: row j1 in [-1, 129] at byte (j1 + 1) * B, column j0 in [-1, 129] at
// byte (j0 + OFF) * sizeof(T). The ring j = -1, 128, 129 is zero (the zero ghost nodes
// of R12), the pitch B makes the 8 rows a team gathers from fall in distinct banks, and
// (OFF * sizeof(T)) keeps every interior row 16-byte aligned for the bulk copies.
template <typename T> struct StagePitch;
template <> struct StagePitch<double> { static constexpr unsigned B = 134 * 8; static constexpr int OFF = 2; };
template <> struct StagePitch<float> { static constexpr unsigned B = 140 * 4; static constexpr int OFF = 4; };
constexpr int STAGE_ROWS = N + 3;
template <typename T> __host__ __device__ constexpr unsigned stage_bytes() { return STAGE_ROWS * StagePitch<T>::B; }

// zero the ghost ring of the staging area (called by all threads)
template <typename T>
__device__ __forceinline__ void zero_ring(void* Xr, int tid) {
    char* base = reinterpret_cast<char*>(Xr);
    constexpr int W = N + 3;                       // columns j0 = -1 .. 129 (+1 alignment slot)
    // rows -1, 128, 129: all columns; rows 0..127: columns -1, 128, 129
    for (int i = tid; i < 3 * W + 3 * N; i += NT) {
        int row, col;
        if (i < 3 * W) {
            const int rr = i / W;
            row = rr == 0 ? -1 : N - 1 + rr;
            col = i - rr * W - 1;
        } else {
            const int k = i - 3 * W;
            row = k / 3;
            const int cc = k - 3 * row;
            col = cc == 0 ? -1 : N - 1 + cc;
        }
        *reinterpret_cast<T*>(base + (row + 1) * StagePitch<T>::B + (col + StagePitch<T>::OFF) * sizeof(T)) = T(0);
    }
}

// Stage filter `filt` (called by ALL threads of the CTA): its 128 weight rows into
// the X region at pitch StagePitch (one bulk copy per thread of the first 128), and its
// constants into pbuf, completing on `bar`. Thread 0 arrives with the expected byte
// count; the mbarrier phase cannot complete before that arrival, whatever the order.
template <typename T>
__device__ __forceinline__ void stage(const ResArgs<T>& a, int filt, void* Xr, double* pbuf,
                                      unsigned long long* bar, int tid) {
    constexpr unsigned RB = N * sizeof(T);
    const unsigned pbytes = a.pstride * sizeof(double);
    if (tid < N) {
        fence_proxy_async();
        if (tid == 0) {
            mbar_expect_tx(bar, N * RB + pbytes);
            bulk_g2s(pbuf, a.prm + (long long)filt * a.pstride, pbytes, bar);
        }
        const char* src = reinterpret_cast<const char*>(a.W + (long long)filt * (N * N));
        bulk_g2s(reinterpret_cast<char*>(Xr) + (tid + 1) * StagePitch<T>::B + StagePitch<T>::OFF * sizeof(T),
                 src + tid * RB, RB, bar);
    }
}

// Warp reduce-scatter of 8 doubles per lane: halving exchanges at offsets 16, 8, 4 (each
// lane keeps half of its values, adds the partner's matching half), then a 2-level sum.
// Returns, in lane L, the warp-wide sum of value 4 b16 + 2 b8 + b4 (b_k = bit k of L), so
// lane 4v holds the sum of value v. Fixed order: deterministic.
__device__ __forceinline__ double warp_sum8(const double* v, int lane) {
    const bool b16 = (lane >> 4) & 1, b8 = (lane >> 3) & 1, b4 = (lane >> 2) & 1;
    double h[4], q[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double keep = b16 ? v[4 + i] : v[i], send = b16 ? v[i] : v[4 + i];
        h[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double keep = b8 ? h[2 + i] : h[i], send = b8 ? h[i] : h[2 + i];
        q[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    double r = (b4 ? q[1] : q[0]) + __shfl_xor_sync(0xffffffffu, b4 ? q[0] : q[1], 4);
    r += __shfl_xor_sync(0xffffffffu, r, 2);
    r += __shfl_xor_sync(0xffffffffu, r, 1);
    return r;
}

// ============================================================================ the fused epoch kernel
// weight staging rows for the TMA store: 128 values + padding (16-byte rows; the padding lies
// beyond j0 = 127 of the box and is not written)
template <typename T> struct WsPitch;
template <> struct WsPitch<double> { static constexpr int P = 130; };
template <> struct WsPitch<float> { static constexpr int P = 132; };
template <typename T> __host__ __device__ constexpr size_t ws_bytes() { return (size_t)64 * WsPitch<T>::P * sizeof(T); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

template <typename T, bool REGRID, bool UPDATE, bool CN>
__global__ void __launch_bounds__(NT, 1) k_resident_epoch(ResArgs<T> a, const __grid_constant__ CUtensorMap wmap) {
    using V = typename C2<T>::type;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    V* X = reinterpret_cast<V*>(smem_raw);                          // [H][PITCH]; also the dense staging area
    // staged weights: element (j0, j1) at Xs + j1 * StagePitch + j0 * sizeof(T), j0, j1 in [-1, 129]
    const char* Xs = reinterpret_cast<const char*>(smem_raw) + StagePitch<T>::B + StagePitch<T>::OFF * sizeof(T);
    constexpr unsigned XBYTES = (sizeof(V) * H * PITCH > stage_bytes<T>()) ? sizeof(V) * H * PITCH : stage_bytes<T>();
    V* tw = reinterpret_cast<V*>(smem_raw + XBYTES);                // [16][8]  W128^{ts}
    double* red = reinterpret_cast<double*>(tw + 128);              // [16 warps][6]
    double* dcs = red + 16 * 6;                                     // DC of the current filter
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(dcs + 2);
    double* pb0 = reinterpret_cast<double*>(bar + 2);               // 2 x pstride parameter buffers
    T* Ws = reinterpret_cast<T*>(smem_raw + ((XBYTES + sizeof(V) * 128 + 16 * 6 * sizeof(double) + 2 * sizeof(double) +
                                             2 * sizeof(unsigned long long) + 2 * sizeof(double) * a.pstride + 127) /
                                            128 * 128));            // 64 x WsPitch staged weight rows

    const int tid = threadIdx.x;
    const int m = tid >> 3, t = tid & 7;
    const int lane = tid & 31, warp = tid >> 5;
    const int sa = t, sb = (t == 0) ? 8 : 16 - t;   // own s pair of the 8-point stages
    const int l = a.l;

    for (int i = tid; i < 128; i += NT) {
        const int s = i >> 3, tt = i & 7;
        const double ang = 2.0 * 3.14159265358979323846 * (double)(tt * s) / 128.0;
        double sn, cs;
        sincos(ang, &sn, &cs);
        tw[i] = V{(T)cs, (T)(-sn)};
    }
    if (tid == 0) mbar_init(bar, 1);
    zero_ring<T>(smem_raw, tid);
    __syncthreads();
    if ((int)blockIdx.x < a.batch) stage(a, blockIdx.x, smem_raw, pb0, bar, tid);

    int it = 0;
    for (int filt = blockIdx.x; filt < a.batch; filt += gridDim.x, ++it) {
        T* Wf = a.W + (long long)filt * (N * N);
        const double* P = pb0 + (it & 1) * a.pstride;
        double* Pn = pb0 + ((it + 1) & 1) * a.pstride;
        const int nxt = filt + gridDim.x;
        RPROF_T(c0);
        mbar_wait(bar, it & 1);                 // weights + constants of this filter are in shared memory
        RPROF_T(c1);
        RPROF_ADD(0, c0, c1);
#ifdef PMF_QPROF
        long long c2 = 0;
#endif

        if (warp == 0 && lane < 8 && nxt < a.batch) {
            // pull the next filter's weights into L2 now; its TMA staging (issued late in P3,
            // once X is free) then reads L2 instead of HBM
            const char* p = reinterpret_cast<const char*>(a.W + (long long)nxt * (N * N)) + lane * (N * N * sizeof(T) / 8);
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"((unsigned)(N * N * sizeof(T) / 8))
                         : "memory");
        }
        if (P[P_SKIP] != 0.0) {                 // failed filter: leave it untouched
            __syncthreads();
            if (nxt < a.batch) stage(a, nxt, smem_raw, Pn, bar, tid);
            continue;
        }
        // ---------------------------------------------------------------- P1: (regrid-)load, FFT along axis 1
        {
            V z[16];
            if (!REGRID) {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const int j1 = t + 8 * r;
                    z[r] = *reinterpret_cast<const V*>(Xs + j1 * (int)StagePitch<T>::B + 2 * m * (int)sizeof(T));
                }
            } else {
                // multilinear interpolation of the old weights at the new points (R12), zero ghosts.
                // v = o + M u' is affine in r: v(r) = v(0) + r * 8 M[:,1].
                const double M0 = P[P_M], M1 = P[P_M + 1], M2 = P[P_M + 2], M3 = P[P_M + 3];
                const double o0 = P[P_O], o1 = P[P_O + 1];
                const double u10 = t - 0.5 * (N - 1);
                const double s0 = 8.0 * M1, s1 = 8.0 * M3;
                double b0[2], b1[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const double u0 = (2 * m + e) - 0.5 * (N - 1);
                    b0[e] = fma(M0, u0, fma(M1, u10, o0));
                    b1[e] = fma(M2, u0, fma(M3, u10, o1));
                }
                // integer clamp to [-1, 128]: beyond it every tap is a zero ghost or has weight 0
                auto split = [&](double v, int& i, double& a) {
                    const double f = floor(v);
                    const int fi = __double2int_rz(f);          // saturating
                    i = min(max(fi, -1), N);
                    a = (fi == i) ? v - f : 0.0;
                };
                // upper-triangular map (CV drift after an axis-aligned regrid): v1 does not
                // depend on the column, one split per row serves both columns
                const bool tri = M2 == 0.0;
                // odd teams gather their second column first: the 4 teams of a warp then read
                // columns of both parities in each load, which halves the bank conflicts of
                // the even staging pitch (4 -> 2 wavefronts per 8-byte gather)
                const bool sw = m & 1;
                const double b0a = sw ? b0[1] : b0[0], b0b = sw ? b0[0] : b0[1];
                const double b1a = sw ? b1[1] : b1[0], b1b = sw ? b1[0] : b1[1];
                if (tri && M0 >= 0.0 && M0 < 1.0) {
                    // one row split serves both columns and 0 <= M0 < 1: their taps lie in one
                    // 3-wide window of the staged rows i1, i1 + 1 (6 loads instead of 8)
#pragma unroll
                    for (int r = 0; r < 16; ++r) {
                        int i1, i0a, i0b;
                        double a1, a0a, a0b;
                        split(fma((double)r, s1, b1[0]), i1, a1);
                        split(fma((double)r, s0, b0[0]), i0a, a0a);
                        split(fma((double)r, s0, b0[1]), i0b, a0b);
                        const T* row0 = reinterpret_cast<const T*>(Xs + i1 * (int)StagePitch<T>::B) + i0a;
                        const T* row1 = reinterpret_cast<const T*>(reinterpret_cast<const char*>(row0) + StagePitch<T>::B);
                        const double w0 = (double)row0[0], w1 = (double)row0[1], w2 = (double)row0[2];
                        const double v0 = (double)row1[0], v1 = (double)row1[1], v2 = (double)row1[2];
                        const bool d = i0b != i0a;
                        const double x0 = d ? w1 : w0, x1 = d ? w2 : w1, y0 = d ? v1 : v0, y1 = d ? v2 : v1;
                        const double loa = fma(a0a, w1 - w0, w0), hia = fma(a0a, v1 - v0, v0);
                        const double lob = fma(a0b, x1 - x0, x0), hib = fma(a0b, y1 - y0, y0);
                        z[r] = V{(T)fma(a1, hia - loa, loa), (T)fma(a1, hib - lob, lob)};
                    }
                } else
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    T val[2];
                    int i1r;
                    double a1r;
                    split(fma((double)r, s1, b1a), i1r, a1r);
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        int i0, i1 = i1r;
                        double a0, a1 = a1r;
                        split(fma((double)r, s0, q ? b0b : b0a), i0, a0);
                        if (q == 1 && !tri) split(fma((double)r, s1, b1b), i1, a1);
                        const T* row0 = reinterpret_cast<const T*>(Xs + i1 * (int)StagePitch<T>::B) + i0;
                        const T* row1 = reinterpret_cast<const T*>(reinterpret_cast<const char*>(row0) + StagePitch<T>::B);
                        const double w00 = (double)row0[0], w01 = (double)row0[1];
                        const double w10 = (double)row1[0], w11 = (double)row1[1];
                        const double lo = fma(a0, w01 - w00, w00);
                        const double hi = fma(a0, w11 - w10, w10);
                        val[q] = (T)fma(a1, hi - lo, lo);
                    }
                    z[r] = sw ? V{val[1], val[0]} : V{val[0], val[1]};
                }
            }
            __syncthreads();                      // the staged weights are consumed: X is free
            RPROF_SET(c2);
            RPROF_ADD(1, c1, c2);
            dft16<false>(z);                      // over r: Y_t(s)
            tw16<false>(z, tw, t);
#pragma unroll
            for (int s = 0; s < 16; ++s) X[cslot(s, t, m)] = z[s];
            __syncwarp();
            V pa[8], pb[8];
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) {
                pa[tt] = X[cslot(sa, tt, m)];
                pb[tt] = X[cslot(sb, tt, m)];
            }
            dft8<false>(pa);                      // Z(sa + 16 q)
            dft8<false>(pb);                      // Z(sb + 16 q)
            __syncwarp();
            // unpack the two real columns: Wa = (Z(k) + conj Z(-k))/2, Wb = (Z(k) - conj Z(-k))/(2i)
            auto store_pair = [&](int k1, V zk, V zp) {
                X[k1 * PITCH + xcol(k1, 2 * m)] = V{T(0.5) * (zk.x + zp.x), T(0.5) * (zk.y - zp.y)};
                X[k1 * PITCH + xcol(k1, 2 * m + 1)] = V{T(0.5) * (zk.y + zp.y), T(0.5) * (zp.x - zk.x)};
            };
            // k1 = sa + 16q and sb + 16q (q < 4) on every thread; only the mirror partner
            // differs on t = 0 (its pairs are s = 0 and 8, both self-mirrored): register
            // selects instead of a divergent branch. t = 0 also owns the Nyquist row 64.
            const bool t0 = t == 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const V ma = t0 ? pa[(8 - q) & 7] : pb[7 - q];
                const V mb = t0 ? pb[7 - q] : pa[7 - q];
                store_pair(sa + 16 * q, pa[q], ma);
                store_pair(sb + 16 * q, pb[q], mb);
            }
            if (t0) store_pair(64, pa[4], pa[4]);
        }
        __syncthreads();

        RPROF_T(c3);
        RPROF_ADD(2, c2, c3);
        // ---------------------------------------------------------------- P2: rows, FFT axis 0, s Psi / N^2, inverse
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
                for (int r = 0; r < 16; ++r) x[r] = row[xcol(m, t + 8 * r)];
            }
            dft16<false>(x);
            tw16<false>(x, tw, t);
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
            dft8<false>(pa);                      // F(sa + 16 q)
            dft8<false>(pb);
            const T sn2 = (T)P[P_S];
            const T kscale = (T)(2.0 * 3.14159265358979323846 / N);
            const double* cfp = P + PRM_FIXED;
            // ps[q] = s Psi(k0[q], k1) / N^2 with kappa = 2 pi k / N (signed k) and the
            // cross term's kx = kappa with the Nyquist wavenumber zeroed (R7)
            auto psi8 = [&](int k1, const int* k0, T* ps) {
                const int k1s = k1 < N / 2 ? k1 : k1 - N;
                const T kap1 = kscale * (T)k1s;
                const T kx1 = (k1 == N / 2) ? T(0) : kap1;
                const T k1sq = kap1 * kap1;
                T kk[8], kx[8], den[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int k0s = k0[q] < N / 2 ? k0[q] : k0[q] - N;
                    const T kap0 = kscale * (T)k0s;
                    kk[q] = kap0 * kap0;
                    kx[q] = (k0[q] == N / 2) ? T(0) : kap0;
                    den[q] = T(1);
                }
                T num[8];
                if constexpr (!CN) {
                    for (int n = 0; n < l; ++n) {
                        const T ca = (T)cfp[3 * n], cb = (T)cfp[3 * n + 1], cc = (T)cfp[3 * n + 2];
                        const T gam = fma(cb, k1sq, T(1));
                        const T bet = cc * kx1;
#pragma unroll
                        for (int q = 0; q < 8; ++q) den[q] *= fma(ca, kk[q], fma(bet, kx[q], gam));
                    }
                } else {
                    // Crank-Nicolson (R27): prod_{n<l} (2 - f_n) / prod_{n=1..l} f_n, f_n on the
                    // grid at t_n (l + 1 coefficient sets scaled dt/4)
#pragma unroll
                    for (int q = 0; q < 8; ++q) num[q] = T(1);
                    for (int n = 0; n <= l; ++n) {
                        const T ca = (T)cfp[3 * n], cb = (T)cfp[3 * n + 1], cc = (T)cfp[3 * n + 2];
                        const T gam = fma(cb, k1sq, T(1));
                        const T bet = cc * kx1;
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const T fq = fma(ca, kk[q], fma(bet, kx[q], gam));
                            if (n > 0) den[q] *= fq;
                            if (n < l) num[q] *= T(2) - fq;
                        }
                    }
                }
                if constexpr (sizeof(T) == 8) {
                    // one division for the 8 values (prefix products), unless the product leaves range
                    T pre[8];
                    pre[0] = den[0];
#pragma unroll
                    for (int q = 1; q < 8; ++q) pre[q] = pre[q - 1] * den[q];
                    if (pre[7] < T(1e300)) {
                        T inv = sn2 / pre[7];
#pragma unroll
                        for (int q = 7; q > 0; --q) {
                            ps[q] = inv * pre[q - 1];
                            inv *= den[q];
                        }
                        ps[0] = inv;
                        if constexpr (CN) {
#pragma unroll
                            for (int q = 0; q < 8; ++q) ps[q] *= num[q];
                        }
                        return;
                    }
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) ps[q] = sn2 / den[q];
                if constexpr (CN) {
#pragma unroll
                    for (int q = 0; q < 8; ++q) ps[q] *= num[q];
                }
            };
            // packed rows k1 = 0 (A) and 64 (B): R = A + i B with A, B Hermitian in k0.
            // A(k) = (R(k) + conj R(-k))/2, B(k) = (R(k) - conj R(-k))/(2i); after the multiply
            // R'(k) = A'(k) + i B'(k), R'(-k) = conj A'(k) + i conj B'(k).
            auto packed = [&](V& rk, V& rm, bool self, T pA, T pB, bool is_dc) {
                const V R = rk, Rm = rm;
                V A = V{T(0.5) * (R.x + Rm.x), T(0.5) * (R.y - Rm.y)};
                V Bv = V{T(0.5) * (R.y + Rm.y), T(0.5) * (Rm.x - R.x)};
                if (is_dc) *dcs = (double)A.x;    // sum of the input weights (k = 0)
                A = V{A.x * pA, A.y * pA};
                Bv = V{Bv.x * pB, Bv.y * pB};
                rk = V{A.x - Bv.y, A.y + Bv.x};
                if (!self) rm = V{A.x + Bv.y, Bv.x - A.y};
            };
            // every thread evaluates the multiplier on two lists of 8 wavenumbers:
            //   rows m > 0: (k1 = m, k0 = sa + 16 q) and (k1 = m, k0 = sb + 16 q);
            //   team 0 (rows 0 and 64 packed): one k0 per Hermitian pair -- thread t > 0 owns
            //   k0 = t + 16 q, thread 0 owns 16 q and 8 + 16 q (q < 4) + the Nyquist k0 = 64 below.
            int kx_[8], ky_[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int kl = (t == 0) ? ((q < 4) ? 16 * q : 8 + 16 * (q - 4)) : sa + 16 * q;
                kx_[q] = (m != 0) ? sa + 16 * q : kl;
                ky_[q] = (m != 0) ? sb + 16 * q : kl;
            }
            T px[8], py[8];
            psi8(m, kx_, px);                        // team 0: row k1 = 0
            psi8(m != 0 ? m : N / 2, ky_, py);       // team 0: row k1 = 64
            if (m != 0) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    pa[q] = V{pa[q].x * px[q], pa[q].y * px[q]};
                    pb[q] = V{pb[q].x * py[q], pb[q].y * py[q]};
                }
            } else if (t != 0) {
#pragma unroll
                for (int q = 0; q < 8; ++q) packed(pa[q], pb[7 - q], false, px[q], py[q], false);
            } else {
                // k0 = 64 (self-paired, both rows): scalar product (kx = 0 at the Nyquist
                // wavenumbers: no cross term)
                T dA = T(1), dB = T(1), nA = T(1), nB = T(1);
                const T kN = kscale * (T)(-N / 2);
                for (int n = 0; n < (CN ? l + 1 : l); ++n) {
                    const T ca = (T)cfp[3 * n], cb = (T)cfp[3 * n + 1];
                    const T fA = fma(ca, kN * kN, T(1)), fB = fma(ca, kN * kN, fma(cb, kN * kN, T(1)));
                    if (!CN || n > 0) {
                        dA *= fA;
                        dB *= fB;
                    }
                    if (CN && n < l) {
                        nA *= T(2) - fA;
                        nB *= T(2) - fB;
                    }
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) packed(pa[q], pa[(8 - q) & 7], q == 0, px[q], py[q], q == 0);
                packed(pa[4], pa[4], true, sn2 * nA / dA, sn2 * nB / dB, false);
#pragma unroll
                for (int q = 0; q < 4; ++q) packed(pb[q], pb[7 - q], false, px[4 + q], py[4 + q], false);
            }
            dft8<true>(pa);                       // G_s(t'')
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
            tw16<true>(x, tw, t);
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
                for (int r = 0; r < 16; ++r) row[xcol(m, t + 8 * r)] = x[r];
            }
        }
        __syncthreads();

        RPROF_T(c4);
        RPROF_ADD(3, c3, c4);
        // ---------------------------------------------------------------- P3: inverse axis 1, normalise, update
        {
            V pa[8], pb[8];
            auto ld = [&](int k1, int col) -> V { return X[k1 * PITCH + xcol(k1, 2 * m + col)]; };
            // Z(k) = Wa(k) + i Wb(k); for k > 64, Wa(k) = conj Wa(128 - k)
            auto zdir = [&](int k1) -> V {
                const V wa = ld(k1, 0), wb = ld(k1, 1);
                return V{wa.x - wb.y, wa.y + wb.x};
            };
            auto zmir = [&](int kp) -> V {
                const V wa = ld(kp, 0), wb = ld(kp, 1);
                return V{wa.x + wb.y, wb.x - wa.y};
            };
            // one index formula for every thread (no divergent branch): the mirrored halves
            // start at 16 - t (pa; t = 0: 16 (8 - q), with zmir(64) = zdir(64) since the
            // Nyquist row is real) and at t, or 8 on t = 0 (pb)
            const int ma = 16 - t, mb = (t == 0) ? 8 : t;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                pa[q] = (q < 4) ? zdir(sa + 16 * q) : zmir(ma + 16 * (7 - q));
                pb[q] = (q < 4) ? zdir(sb + 16 * q) : zmir(mb + 16 * (7 - q));
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
            const double lgn = P[P_LGN];
            double pe[2], qe[2];
            const double g11 = P[P_QG + 2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const double u0 = (2 * m + e) - 0.5 * (N - 1);
                pe[e] = fma(u0, fma(P[P_QG], u0, P[P_QB]), P[P_QA]);
                qe[e] = fma(2.0 * P[P_QG + 1], u0, P[P_QB + 1]);
            }
            __syncthreads();                      // X is consumed
            RPROF_T(c5);
            RPROF_ADD(4, c4, c5);
            zero_ring<T>(smem_raw, tid);          // visible to the gather after the end-of-filter barrier
            if (nxt < a.batch) stage(a, nxt, smem_raw, Pn, bar, tid);   // overlaps the rest of P3
            tw16<true>(x, tw, t);
            dft16<true>(x);                       // x[r] = w(2m, t+8r) + i w(2m+1, t+8r) (unnormalised)
            RPROF_T(d1);
            RPROF_ADD(7, c5, d1);
            // Likelihood (linear Gauss): along this thread's column e the exponent is a quadratic
            // in r (u1 = u1_0 + 8 r): E(r) = E0 + E1 r + E2 r^2, so L(r+1) = L(r) R(r) and
            // R(r+1) = R(r) exp(2 E2) -- two multiplies per point. Used when every partial
            // exponent stays inside the fp64 range (|E0| + 15|E1| + 225|E2| < 650; each step
            // adds at most one rounding, < 16 ulp in total); otherwise exp per point.
            double Lr[2], Rr[2], Gr[2];
            bool rec = UPDATE && !a.range;
            if (UPDATE && !a.range) {
                const double u10 = t - 0.5 * (N - 1);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const double base = fma(-0.5, pe[e], lgn);
                    const double E0 = fma(-0.5, u10 * fma(g11, u10, qe[e]), base);
                    const double E1 = -0.5 * (8.0 * qe[e] + 16.0 * g11 * u10);
                    const double E2 = -32.0 * g11;
                    rec = rec && (fabs(E0) + 15.0 * fabs(E1) + 225.0 * fabs(E2) < 650.0);
                    Lr[e] = exp_fast(E0);
                    Rr[e] = exp_fast(E1 + E2);
                    Gr[e] = exp_fast(2.0 * E2);
                }
            }
            // moments per column: S = sum w, Tm = sum w u1, U = sum w u1^2 (u0 is fixed per column)
            double S[2] = {0, 0}, Tm[2] = {0, 0}, U[2] = {0, 0};
            auto emit = [&](int r, int e, double w) -> T {
                const T wt = (T)w;
                if (UPDATE) {
                    const double u1 = (t + 8 * r) - 0.5 * (N - 1);
                    const double wd = (double)wt;
                    const double wu = wd * u1;
                    S[e] += wd;
                    Tm[e] += wu;
                    U[e] = fma(wu, u1, U[e]);
                }
                return wt;
            };
            // the filter's new weights leave through shared memory (rows of pitch WSP, two halves of
            // 64 rows) and a tensor-map TMA store each -- 1 KB rows instead of per-thread 64-byte
            // row pieces (measured: the strided stores cost ~15 % of the kernel) -- whenever every
            // thread has its outputs in registers (CTA-uniform); the generic likelihood path stores
            // directly
            const bool staged = __syncthreads_and(!UPDATE || rec);
            if (!UPDATE) {
            } else if (rec) {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const T o0 = emit(r, 0, (double)x[r].x * Lr[0]);
                    const T o1 = emit(r, 1, (double)x[r].y * Lr[1]);
                    Lr[0] *= Rr[0];
                    Rr[0] *= Gr[0];
                    Lr[1] *= Rr[1];
                    Rr[1] *= Gr[1];
                    if (staged) x[r] = V{o0, o1};
                    else *reinterpret_cast<V*>(Wf + (t + 8 * r) * N + 2 * m) = V{o0, o1};
                }
            } else {
#pragma unroll 1
                for (int rr = 0; rr < 16; rr += 4) {
                    // generic path (range likelihood or extreme exponents): exp per point; the
                    // register array is indexed statically through the inner unrolled switch
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        V xv;
                        switch (rr + q) {
#define PMF_X(i) case i: xv = x[i]; break;
                            PMF_X(0) PMF_X(1) PMF_X(2) PMF_X(3) PMF_X(4) PMF_X(5) PMF_X(6) PMF_X(7)
                            PMF_X(8) PMF_X(9) PMF_X(10) PMF_X(11) PMF_X(12) PMF_X(13) PMF_X(14) PMF_X(15)
#undef PMF_X
                        }
                        const int r = rr + q;
                        const double u1 = (t + 8 * r) - 0.5 * (N - 1);
                        T o[2];
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            double ee;
                            if (!a.range) {
                                ee = fma(u1, fma(g11, u1, qe[e]), pe[e]);
                            } else {
                                // range likelihood: constants re-read from shared memory (P stays
                                // valid: the next filter is staged into the other parameter buffer)
                                const double u0 = (2 * m + e) - 0.5 * (N - 1);
                                const double y0 = fma(P[P_BL], u0, fma(P[P_BL + 1], u1, P[P_CL]));
                                const double y1 = fma(P[P_BL + 2], u0, fma(P[P_BL + 3], u1, P[P_CL + 1]));
                                const double d = (P[P_ZR] - sqrt(fma(y0, y0, y1 * y1))) * P[P_ISG];
                                ee = d * d;
                            }
                            const double w = (double)(e == 0 ? xv.x : xv.y);
                            o[e] = emit(r, e, w * exp_fast(fma(-0.5, ee, lgn)));
                        }
                        *reinterpret_cast<V*>(Wf + (t + 8 * r) * N + 2 * m) = V{o[0], o[1]};
                    }
                }
            }
            RPROF_T(d2);
            RPROF_ADD(8, d1, d2);
            if (staged) {
                constexpr int WSP = WsPitch<T>::P;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (tid == 0) bulk_wait_read0();                 // the previous half's store has read Ws
                    __syncthreads();
#pragma unroll
                    for (int r = 8 * h; r < 8 * h + 8; ++r)
                        *reinterpret_cast<V*>(Ws + (t + 8 * (r - 8 * h)) * WSP + 2 * m) = x[r];
                    __syncthreads();
                    if (tid == 0) {
                        fence_proxy_async();
                        asm volatile(
                            "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&wmap),
                            "r"(0), "r"(64 * h), "r"(filt), "r"(smem_u32(Ws))
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                }
            }
            double acc[6];
            {
                const double ua = (2 * m) - 0.5 * (N - 1), ub = ua + 1.0;
                acc[0] = S[0] + S[1];
                acc[1] = fma(ua, S[0], ub * S[1]);
                acc[2] = Tm[0] + Tm[1];
                acc[3] = fma(ua * ua, S[0], ub * ub * S[1]);
                acc[4] = fma(ua, Tm[0], ub * Tm[1]);
                acc[5] = U[0] + U[1];
            }
            if (UPDATE) {
                // transposed warp reduction (reduce-scatter): 9 double shuffles instead of 30;
                // afterwards lane 4v holds the warp sum of accumulator v (fixed order)
                double v8[8] = {acc[0], acc[1], acc[2], acc[3], acc[4], acc[5], 0.0, 0.0};
                const double ws = warp_sum8(v8, lane);
                if ((lane & 3) == 0 && (lane >> 2) < 6) red[warp * 6 + (lane >> 2)] = ws;
            }
            __syncthreads();
            if (warp == 0) {
                // per-filter sums in a fixed order (deterministic); the scalar work is in k_res_finalize
                double v = 0.0;
                if (UPDATE && lane < 6)
                    for (int w = 0; w < NT / 32; ++w) v += red[w * 6 + lane];
                if (lane == 6) v = *dcs;
                if (lane < 7) a.out[(long long)filt * 8 + lane] = v;
            }
            RPROF_T(c6);
            RPROF_ADD(5, c5, c6);
            RPROF_ADD(6, 0, 1);
        }
    }
    if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int resident_debug_counters(double* out, int n, int reset) {
    unsigned long long h[12];
    if (cudaMemcpyFromSymbol(h, g_rprof, sizeof(h)) != cudaSuccess) return -1;
    for (int i = 0; i < n && i < 12; ++i) out[i] = (double)h[i];
    if (reset) {
        std::fill(h, h + 12, 0ull);
        cudaMemcpyToSymbol(g_rprof, h, sizeof(h));
    }
    return 0;
}

bool resident_supported(const Dims& d, int dtype) {
    (void)dtype;
    return d.nx == 2 && d.n[0] == N && d.n[1] == N;
}

size_t resident_param_bytes(int l, int batch) { return sizeof(double) * (size_t)prm_stride(l) * batch; }

// Tensor map of the weights [batch][128][128] for the kernel's row stores: box
// WsPitch x 64 x 1 -- the staged rows' padding lies beyond j0 = 127 and is not written
template <typename T>
static cudaError_t w_map(T* W, int batch, CUtensorMap* m) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !encode) {
            encode = nullptr;
            return cudaErrorNotSupported;
        }
    }
    cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)batch};
    cuuint64_t str[2] = {sizeof(T) * (cuuint64_t)N, sizeof(T) * (cuuint64_t)N * N};
    cuuint32_t box[3] = {(cuuint32_t)WsPitch<T>::P, 64, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode(m, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)W,
                        dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <typename T, bool RG, bool UP, bool CN>
static cudaError_t launch_t(ResArgs<T> a, cudaStream_t s, int64_t* launches, cudaEvent_t ev0, cudaEvent_t ev1) {
    using V = typename C2<T>::type;
    const size_t xbytes = std::max<size_t>(sizeof(V) * H * PITCH, stage_bytes<T>());
    const size_t base = xbytes + sizeof(V) * 128 + 16 * 6 * sizeof(double) + 2 * sizeof(double) +
                        2 * sizeof(unsigned long long) + 2 * sizeof(double) * (size_t)a.pstride;
    const size_t smem = (base + 127) / 128 * 128 + ws_bytes<T>();
    CUtensorMap wmap;
    cudaError_t e = w_map<T>(a.W, a.batch, &wmap);
    if (e != cudaSuccess) return e;
    auto kern = k_resident_epoch<T, RG, UP, CN>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    const int grid = std::min(a.batch, nsm * occ);
    if (ev0) cudaEventRecordWithFlags(ev0, s, cudaEventRecordExternal);
    kern<<<grid, NT, smem, s>>>(a, wmap);
    if (ev1) cudaEventRecordWithFlags(ev1, s, cudaEventRecordExternal);
    ++*launches;
    return cudaGetLastError();
}

template <typename T>
static cudaError_t launch_dt(const Dims& d, PencilBufs& b, const ModelParams& mp, const LikParams* lp, double ks,
                             cudaStream_t s, int64_t* launches) {
    const int ps = prm_stride(mp.l + (mp.step ? 1 : 0));
    LikParams lpv = lp ? *lp : LikParams{};
    k_res_prep<<<(d.batch + 3) / 4, 128, 0, s>>>(b.st, b.coef, ps, mp, b.sub, lpv, b.z, ks, lp ? 1 : 0, d.batch,
                                                d.grid);
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    ResArgs<T> a;
    a.W = (T*)b.W;
    a.prm = b.coef;
    a.out = b.partials;
    a.pstride = ps;
    a.l = mp.l;
    a.batch = d.batch;
    a.range = lpv.kind == 1;
    const bool rg = ks > 0.0;
    if (mp.step) {
        if (rg && lp) e = launch_t<T, true, true, true>(a, s, launches, b.ev0, b.ev1);
        else if (rg) e = launch_t<T, true, false, true>(a, s, launches, b.ev0, b.ev1);
        else if (lp) e = launch_t<T, false, true, true>(a, s, launches, b.ev0, b.ev1);
        else e = launch_t<T, false, false, true>(a, s, launches, b.ev0, b.ev1);
    } else {
        if (rg && lp) e = launch_t<T, true, true, false>(a, s, launches, b.ev0, b.ev1);
        else if (rg) e = launch_t<T, true, false, false>(a, s, launches, b.ev0, b.ev1);
        else if (lp) e = launch_t<T, false, true, false>(a, s, launches, b.ev0, b.ev1);
        else e = launch_t<T, false, false, false>(a, s, launches, b.ev0, b.ev1);
    }
    if (e != cudaSuccess) return e;
    k_res_finalize<<<(d.batch + 127) / 128, 128, 0, s>>>(b.st, b.partials, b.coef, ps, mp.s, lp ? 1 : 0, d.batch);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_resident(const Dims& d, int dtype, PencilBufs& b, const Twiddles& tw, const ModelParams* mp,
                            const LikParams* lp, double ks, cudaStream_t s, int64_t* launches) {
    (void)tw;
    if (!mp) return cudaErrorInvalidValue;      // the host routes update-/regrid-only work to the point kernels
    if (dtype == 0) return launch_dt<double>(d, b, *mp, lp, ks, s, launches);
    return launch_dt<float>(d, b, *mp, lp, ks, s, launches);
}

}  // namespace pmf
