// kernels_quad.cu -- the three-pass ("transposed spectrum") time update for nx = 4
// grids (BASELINE configs[3], C4: 96^4 fp64).
//
//   K1 k_plane_fwd (kernels_plane.cu)  per (j0, j1)-plane: [split regrid, in-plane part,
//                R12] -> forward DFT along axes 1 and 0 (Alg. 1, eq:fourtrsf P:221) -> the
//                plane's half spectrum S[filter][j3][j2][k1][k0] (contiguous rows)
//   K2 k_q_mid   per (filter, k1, k0): its (j3, j2)-plane gathered from S by tensor-map TMA
//                loads (16-byte elements, the row pitch padded by an out-of-range column)
//                -> [split regrid, axes-2/3 part] -> forward DFT along axes 2, 3 -> s Psi /
//                N_tot (Alg. 3-4) -> inverse DFT along axes 3, 2 (Alg. 5) -> contiguous rows
//                of S2[filter][k1][k0][j3][j2] (the transposed layout)
//   K3 k_q_inv   per (j0, j1)-plane: its coefficients gathered from S2 by one TMA load ->
//                inverse DFT along axes 0, 1 -> likelihood at the moved points (eq:filt
//                P:46, R13) -> weights staged in shared memory, one TMA store; index-space
//                moment partials
//
// Three passes over HBM (K1 reads the weights and writes S, K2 reads S and writes S2, K3
// reads S2 and writes the weights) against five on the per-plane layout of
// kernels_plane.cu: the transposition rides on the TMA gathers, whose 16-byte element
// rate is hidden behind each kernel's arithmetic. fp64 only; N_0 = N_1 in {32, 64, 96},
// n2 = n3 in {16, .., 96}.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "device_common.cuh"
#include "fft_reg.cuh"
#include "plane_common.cuh"
#include "tma.cuh"

namespace pmf {
namespace pln {

using V = double2;

#ifndef PMF_K2_TEAMS96
#define PMF_K2_TEAMS96 48    // K2's 8-thread teams at NQ = 96 (a divisor of 96; 48 measured best)
#endif

// Phase cycle counters (debug builds with -DPMF_QPROF only): thread 0 of every CTA adds the
// clock64() deltas of its phases; read with pmf_debug_counters (tools/qprof.py).
__device__ unsigned long long g_qprof[16];
#ifdef PMF_QPROF
#define QPROF_T(v) \
    __syncthreads();  \
    const long long v = clock64()
#define QPROF_ADD(i, a, b) \
    if (threadIdx.x == 0) atomicAdd(&g_qprof[i], (unsigned long long)((b) - (a)))
#else
#define QPROF_T(v)
#define QPROF_ADD(i, a, b)
#endif

struct QArgs {
    double* W;               // weights written by K3
    const V* Yin;            // K1's spectrum S[filter][j3][j2][k1][k0] (K2's input)
    V* Y;                    // S2[filter][k0][k1][j3][j2] (K2's output, K3's input)
    const double* coef;
    int cs;
    double* dc3;             // [filter][n3] the regridded sums (split maps; K2)
    double* part;            // [filter][K3 CTAs][NMOM]
    int batch;
    int n2, n3;              // plane sizes (n2 == n3 == NQ) of this block (K3: its j3 slab)
    int l, step;
    int range;               // likelihood kind 1 (range), else linear Gauss
    // slab sharding over G ranks (unsharded: G = 1, koff = 0, j3off = 0, slab = n3g = n3):
    // K2 runs the k0 range [koff, koff + N0/G) and writes output row j3 to rank j3 / slab's
    // block; K3 runs the planes j3 in [j3off, j3off + slab) of n3g
    int N0f;                 // N_0 (wavenumbers)
    int koff;
    int G, slab, j3off, n3g;
    // K2 over a k0 sub-range (pipelined back exchange): items (k1, k0 in [kbeg, kbeg + N0)) of the
    // input's N0blk k0 columns; the output blocks keep their full k0 extent N0blk
    int kbeg = 0, N0blk = 0;
    // S2 layout: G == 1 -> [filter][k1][k0][j3][j2]; G > 1 -> per destination block
    // [k0][k1][j3 % slab][j2] (k0 outermost, so the back exchange stacks the blocks into k0)
};

// ============================================================================ K2: contiguous (j3, j2)-planes
// Work item = (filter, k1, k0); its plane Y[f][k1][k0][.][.] (NQ rows of NQ complex) is
// staged row by row (bulk copies completing on one mbarrier) into rows of pitch NQ + 1
// (conflict-free along rows and columns). Team q owns rows / columns q + TEAMS j.
//   F2  [split regrid (R12): each output row u3' bilinear from old rows ja, ja + 1 (per-item
//       tap table) at v2 = o2 + M22 u2' + M23 u3', into registers; CTA barrier] forward DFT
//       along axis 2 of every row
//   F3  per column k2: forward DFT along axis 3, x s Psi / N_tot (Alg. 3-4), inverse
//   I2  inverse DFT along axis 2 of every row, stored back in place from registers;
//       each freed row is refilled at once with the next item's row (its bulk copy
//       overlaps the rest of this item)
// shared memory: X [NQ][P] complex, the item's s Psi / N_tot table [NQ (k2)][PSP (k3)],
// the axis-3 regrid taps per output row (split maps), twiddles, one mbarrier.
template <int NQ> struct Q2 {
    static constexpr int PSP = NQ + 1;                       // Psi table pitch (doubles)
    static constexpr int R3 = (NQ + 31) / 32;                // k3 values per lane in the table phase
    static constexpr int QTW = 6;                            // doubles per substep in the item's table
    static constexpr int TEAMS = NQ == 96 ? PMF_K2_TEAMS96 : (NQ >= 64 ? 32 : NQ / 2);   // K2's teams (8 threads)
    static constexpr int RP = TEAMS;                         // rows per TMA part of the gathered plane
    static constexpr size_t SMEM = sizeof(V) * NQ * QCfg<NQ>::P + sizeof(double) * NQ * PSP +
                                   2 * (sizeof(double) + sizeof(int)) * NQ + sizeof(V) * NQ + 16 +
                                   sizeof(double) * QTW * (LCAP + 1) + sizeof(double) * PL_EU;
};

// The item's Euler-factor table (Alg. 3 with R3's D_n): for substep n the factor at
// (k0, k1, k2, k3) is f_n = gb_n + c2_n kap2^2 + d_n kx2 + (e_n + c9_n kx2) kx3 + a_n kap3^2,
// where gb_n = 1 + c0 kap0^2 + c1 kap1^2 + c4 kx0 kx1, d_n = c5 kx0 + c7 kx1, e_n = c6 kx0 + c8 kx1
// collect the (k0, k1) terms once per item (cf = the coefficients of substep_coefs, packed
// order diag 0..3, (0,1) (0,2) (0,3) (1,2) (1,3) (2,3)); row n = {gb, d, e, c2, c9, a}.
__device__ __forceinline__ void q_item_table(const double* cf, int nsets, const double* kap, const double* kx,
                                             double* qt) {
    for (int n = threadIdx.x; n < nsets; n += blockDim.x) {
        const double* c = cf + 10 * n;
        double* o = qt + 6 * n;
        o[0] = fma(c[4], kx[0] * kx[1], fma(c[1], kap[1] * kap[1], fma(c[0], kap[0] * kap[0], 1.0)));
        o[1] = fma(c[7], kx[1], c[5] * kx[0]);
        o[2] = fma(c[8], kx[1], c[6] * kx[0]);
        o[3] = c[2];
        o[4] = c[9];
        o[5] = c[3];
    }
}

// pair j of list `list` as a quartic in kap3 (psi_pair's output layout) from the item table
__device__ __forceinline__ void q_pair(const double* qt, int l, int cn, int list, int j, double kap2sq, double kx2,
                                       double2* q) {
    const int base = (list == 0 && cn) ? 1 : 0;        // CN den: f_1 .. f_l
    auto gba = [&](int n, double& g, double& b, double& a) {
        const double* r = qt + 6 * n;
        g = fma(r[3], kap2sq, fma(r[1], kx2, r[0]));
        b = fma(r[4], kx2, r[2]);
        a = r[5];
    };
    double g0, b0, a0, g1 = 1.0, b1 = 0.0, a1 = 0.0;
    gba(base + 2 * j, g0, b0, a0);
    const bool two = 2 * j + 1 < l;
    if (two) gba(base + 2 * j + 1, g1, b1, a1);
    if (list == 1) {                                   // 2 - f = (2 - g) - b k - a k^2
        g0 = 2.0 - g0;
        b0 = -b0;
        a0 = -a0;
        if (two) {
            g1 = 2.0 - g1;
            b1 = -b1;
            a1 = -a1;
        }
    }
    constexpr double kn2 = PMF_PI * PMF_PI;
    q[0] = double2{g0 * g1, fma(g0, b1, b0 * g1)};
    q[1] = double2{fma(g0, a1, fma(b0, b1, a0 * g1)), fma(b0, a1, a0 * b1)};
    q[2] = double2{a0 * a1, fma(a0, kn2, g0) * fma(a1, kn2, g1)};
}

// acc[r] *= product of list `list`'s pair quartics at kap3 = kp[r]; every thread forms the
// quartics itself from the item table (no shuffles: the 12 Horner chains per pair overlap
// the next pair's coefficients)
template <int NQ, int R = NQ / 8>
__device__ __forceinline__ void q_psi_prod(double (&acc)[R], const double* kp, const double* qt, int l,
                                           int cn, int list, double kap2sq, double kx2, int t) {
    static_assert((NQ / 2) >> 3 < R, "the Nyquist value k3 = NQ/2 must be among the thread's values");
    const int nq = (l + 1) >> 1;
    double nyq = 1.0;
    // (measured: software-pipelining pair j + 1's quartic under pair j's Horner chains, or
    // computing Psi inside the F3 loop instead of this table, both run K2 7-9 % slower)
#pragma unroll 1
    for (int j = 0; j < nq; ++j) {
        double2 c[3];
        q_pair(qt, l, cn, list, j, kap2sq, kx2, c);
        nyq *= c[2].y;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double x1 = kp[r];
            acc[r] *= fma(fma(fma(fma(c[2].x, x1, c[1].y), x1, c[1].x), x1, c[0].y), x1, c[0].x);
        }
    }
    if (t == ((NQ / 2) & 7)) acc[(NQ / 2) >> 3] = nyq;
}

template <int NQ>
static size_t qmid_smem() { return Q2<NQ>::SMEM; }

template <int NQ, int TM>
__global__ void __launch_bounds__(QCfg<NQ, TM>::NT, 1) k_q_mid(QArgs a, int I, int N0, int H1,
                                                                const __grid_constant__ CUtensorMap smap) {
    using C = QCfg<NQ, TM>;
    constexpr int R = C::R, TEAMS = C::TEAMS, P = C::P;
    constexpr int PSP = Q2<NQ>::PSP;
    constexpr int RP = Q2<NQ>::RP, NPART = NQ / RP;          // rows per TMA part, parts per item
    constexpr unsigned PLANE = NQ * P * sizeof(V);            // incl. the zero-filled padding column
    extern __shared__ __align__(128) unsigned char smem_raw[];
    V* X = reinterpret_cast<V*>(smem_raw);                    // [NQ][P]: row j3
    double* psi = reinterpret_cast<double*>(X + NQ * P);      // [k2][PSP]
    double* w3t = psi + NQ * PSP;                             // [u3'][2] axis-3 tap weights (split regrid)
    int* j3t = reinterpret_cast<int*>(w3t + 2 * NQ);          // [u3'][2] axis-3 tap rows (clamped)
    V* tw = reinterpret_cast<V*>(j3t + 2 * NQ);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(tw + NQ);
    double* qt = reinterpret_cast<double*>(bar + 2);          // [nsets][6] the item's factor table
    double* hd = qt + Q2<NQ>::QTW * (LCAP + 1);               // the filter's coefficient head (PL_*)
    int curf = -1;
    const int tid = threadIdx.x, q = tid >> 3, t = tid & 7;
    init_tw<NQ>(tw);
    if (tid == 0) tma::mbar_init(bar, 1);
    const int items = a.batch * I;
    __syncthreads();
    auto rs = [](int s2, int tt) { return rslot(s2, tt); };
    auto cs = [](int s2, int tt) { return rslot(s2, tt) * P; };
    // rows [c RP, (c + 1) RP) of item `it`'s (j3, j2)-plane: one TMA load (thread 0; the caller
    // has ordered the rows' earlier reads before it); 128-byte aligned (P RP = 0 mod 8)
    auto load_part = [&](int it, int c) {
        const unsigned fi = (unsigned)it / (unsigned)I, ii = (unsigned)it - fi * (unsigned)I;
        const unsigned k1 = ii / (unsigned)N0, k0 = ii - k1 * (unsigned)N0 + (unsigned)a.kbeg;
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
            "%6}], [%7];" ::"r"(tma::smem_u32(X + c * RP * P)),
            "l"(&smap), "r"(0), "r"((int)k0), "r"((int)k1), "r"(0), "r"((int)(fi * NQ + c * RP)),
            "r"(tma::smem_u32(bar))
            : "memory");
    };
    if (tid == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&smap) : "memory");
    if ((int)blockIdx.x < items && tid == 0) {
        tma::mbar_expect_tx(bar, PLANE);
        for (int c = 0; c < NPART; ++c) load_part(blockIdx.x, c);
    }
    int k = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++k) {
        QPROF_T(q0);
        const int nxt = item + gridDim.x;
        const unsigned f = (unsigned)item / (unsigned)I, i = (unsigned)item - f * (unsigned)I;
        if ((int)f != curf) {                                 // uniform: cache the filter's head
            if (tid < PL_EU) hd[tid] = a.coef[(long long)f * a.cs + tid];
            curf = (int)f;
            __syncthreads();
        }
        const double* Pg = a.coef + (long long)f * a.cs;      // (the substep coefficients stay global)
        const double* Pc = hd;
        const bool skip = Pc[PL_SKIP] != 0.0;
        const int flag = (int)Pc[PL_FLAG];
        if (!skip) {
            // ------------------------------------------------------------ tables (while the plane loads)
            // s Psi / N_tot at every (k2, k3) of this (k0, k1) (Alg. 3-4): Euler factors
            // f_n = gam_n + bet_n kx3 + alp_n kap3^2 multiplied in pairs as quartics in kap3;
            // warp w owns columns k2 = w + NW j, lane owns k3 = lane + 32 r; pair j's quartic is
            // computed by lane j % 32 and broadcast
            const double* cf = Pg + PL_EU;
            const int cn = a.step, l = a.l;
            const unsigned k1 = i / (unsigned)N0;
            const int N0f = a.N0f, k0 = a.koff + a.kbeg + (int)(i - k1 * (unsigned)N0);   // global k0
            const int N1 = 2 * (H1 - 1);
            double kap[3], kx[3];
            kap[0] = (2.0 * PMF_PI / N0f) * (k0 < N0f / 2 ? k0 : k0 - N0f);
            kx[0] = (2 * k0 == N0f) ? 0.0 : kap[0];
            kap[1] = (2.0 * PMF_PI / N1) * (int)k1;
            kx[1] = (2 * (int)k1 == N1) ? 0.0 : kap[1];
            const double mult = Pc[PL_SN];
            q_item_table(cf, l + cn, kap, kx, qt);
            __syncthreads();
            double kp[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int kk = t + 8 * r;
                kp[r] = (2.0 * PMF_PI / NQ) * (kk < NQ / 2 ? kk : kk - NQ);
            }
            // Point symmetry: when no Euler factor couples (k0, k1) with (k2, k3) (d_n = e_n = 0 in
            // the item table -- the two independent CV blocks of C4), f_n(k2, k3) = f_n(-k2, -k3)
            // (R7: kx = 0 and kap^2 = pi^2 at the Nyquist index either way), so each thread
            // evaluates its values with k3 = t + 8r <= NQ/2 + 7 only and writes every value twice,
            // at (k2, k3) and (-k2, -k3): 7 of the 12 Horner sweeps at NQ = 96. The mirrored
            // entries are covered by the owner of column -k2 (bitwise-equal values where two
            // threads write the same entry: k3 = 0, NQ/2).
            bool sym = true;
            for (int n = 0; n < l + cn; ++n) sym = sym && qt[6 * n + 1] == 0.0 && qt[6 * n + 2] == 0.0;
            constexpr int RH = NQ % 16 == 0 ? NQ / 16 + 1 : R;
            if (sym && RH < R) {
#pragma unroll 1
                for (int k2 = q; k2 < NQ; k2 += TEAMS) {
                    const double kap2 = (2.0 * PMF_PI / NQ) * (k2 < NQ / 2 ? k2 : k2 - NQ);
                    const double kx2 = (2 * k2 == NQ) ? 0.0 : kap2;
                    double den[RH], ps[RH];
#pragma unroll
                    for (int r = 0; r < RH; ++r) den[r] = 1.0;
                    q_psi_prod<NQ, RH>(den, kp, qt, l, cn, 0, kap2 * kap2, kx2, t);
                    psi_div<RH>(den, mult, ps);
                    if (cn) {                                 // Crank-Nicolson numerators (R27)
#pragma unroll
                        for (int r = 0; r < RH; ++r) den[r] = 1.0;
                        q_psi_prod<NQ, RH>(den, kp, qt, l, cn, 1, kap2 * kap2, kx2, t);
#pragma unroll
                        for (int r = 0; r < RH; ++r) ps[r] *= den[r];
                    }
                    const int m2 = k2 ? NQ - k2 : 0;
#pragma unroll
                    for (int r = 0; r < RH; ++r) {
                        const int k3 = t + 8 * r;
                        psi[k2 * PSP + k3] = ps[r];
                        psi[m2 * PSP + (k3 ? NQ - k3 : 0)] = ps[r];
                    }
                }
            } else
            // team q: columns k2 = q + TEAMS j; thread t: k3 = t + 8 r
#pragma unroll 1
            for (int k2 = q; k2 < NQ; k2 += TEAMS) {
                const double kap2 = (2.0 * PMF_PI / NQ) * (k2 < NQ / 2 ? k2 : k2 - NQ);
                const double kx2 = (2 * k2 == NQ) ? 0.0 : kap2;
                double den[R], ps[R];
#pragma unroll
                for (int r = 0; r < R; ++r) den[r] = 1.0;
#if !defined(QDBG) || (QDBG != 1 && QDBG != 3)
                q_psi_prod<NQ>(den, kp, qt, l, cn, 0, kap2 * kap2, kx2, t);
#endif
#if !defined(QDBG) || QDBG < 2
                psi_div<R>(den, mult, ps);
#else
#pragma unroll
                for (int r = 0; r < R; ++r) ps[r] = den[r] * mult;
#endif
                if (cn) {                                     // Crank-Nicolson numerators (R27)
#pragma unroll
                    for (int r = 0; r < R; ++r) den[r] = 1.0;
                    q_psi_prod<NQ>(den, kp, qt, l, cn, 1, kap2 * kap2, kx2, t);
#pragma unroll
                    for (int r = 0; r < R; ++r) ps[r] *= den[r];
                }
#pragma unroll
                for (int r = 0; r < R; ++r) psi[k2 * PSP + t + 8 * r] = ps[r];
            }
            if (flag == 4 && tid < NQ) {
                // axis-3 part of the split regrid (R12): output row u3' = (1 - w3) old row ja +
                // w3 old row ja + 1, zero ghosts: taps outside the grid get weight 0 (row clamped)
                const double v3 = fma(Pc[PL_M + 15], (double)tid - 0.5 * (NQ - 1), Pc[PL_O + 3]), f3 = floor(v3);
                const int fi3 = __double2int_rz(f3);
                const int ja = min(max(fi3, -2), NQ);
                const double w3 = (ja == fi3) ? v3 - f3 : 0.0;
                const bool va = ja >= 0 && ja < NQ, vb = ja + 1 >= 0 && ja + 1 < NQ;
                j3t[2 * tid] = va ? ja : 0;
                j3t[2 * tid + 1] = vb ? ja + 1 : 0;
                w3t[2 * tid] = va ? 1.0 - w3 : 0.0;
                w3t[2 * tid + 1] = vb ? w3 : 0.0;
            }
        }
        QPROF_T(q1);
        tma::mbar_wait(bar, (unsigned)(k & 1));               // the plane is in shared memory
        __syncthreads();                                      // (and the tables are written)
        QPROF_T(q2);
        QPROF_ADD(0, q0, q1);
        QPROF_ADD(1, q1, q2);
        if (!skip) {
            // ------------------------------------------------------------ [split regrid] + F2
            const bool rg = flag == 4;
            static_assert(NQ == 2 * TEAMS, "two rows per team");
            if (rg) {
                // both of the team's output rows u3' (q, q + TEAMS): the bilinear value (axis 3 by the
                // per-row taps, then axis 2 at v2 = o2 + M22 u2' + M23 u3', zero ghosts) straight
                // into registers; every read precedes every write (CTA barrier), then the forward
                // DFT along axis 2 continues from registers (one pass over the plane, not two)
                const double M22 = Pc[PL_M + 10], M23 = Pc[PL_M + 11], o2 = Pc[PL_O + 2];
                V xr[2][R];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int u3 = q + h * TEAMS;
                    const int2 ij = reinterpret_cast<const int2*>(j3t)[u3];
                    const double2 w = reinterpret_cast<const double2*>(w3t)[u3];
                    const V* ra = X + ij.x * P;
                    const V* rb = X + ij.y * P;
                    const double vb2 = fma(M23, (double)u3 - 0.5 * (NQ - 1), o2);
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const double v2 = fma(M22, (t + 8 * r) - 0.5 * (NQ - 1), vb2), fl = floor(v2);
                        const int fi = min(max(__double2int_rz(fl), -2), NQ);
                        const double fr = v2 - fl;
                        const bool vl = fi >= 0 && fi < NQ, vh = fi + 1 >= 0 && fi + 1 < NQ;
                        const V la = vl ? ra[fi] : V{0.0, 0.0}, ha = vh ? ra[fi + 1] : V{0.0, 0.0};
                        const V lb = vl ? rb[fi] : V{0.0, 0.0}, hb = vh ? rb[fi + 1] : V{0.0, 0.0};
                        const double ax = fma(fr, ha.x - la.x, la.x), ay = fma(fr, ha.y - la.y, la.y);
                        const double bx = fma(fr, hb.x - lb.x, lb.x), by = fma(fr, hb.y - lb.y, lb.y);
                        xr[h][r] = V{fma(w.y, bx, w.x * ax), fma(w.y, by, w.x * ay)};
                    }
                    dftR<R, false>(xr[h]);
                    apply_tw<R, false>(xr[h], tw, t);
                }
                __syncthreads();
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    V* row = X + (q + h * TEAMS) * P;
#pragma unroll
                    for (int s2 = 0; s2 < R; ++s2) row[rs(s2, t)] = xr[h][s2];
                }
                __syncwarp();
#pragma unroll 1
                for (int h = 0; h < 2; ++h)
                    tdft_s2<R>(X + (q + h * TEAMS) * P, t, rs, [](int, V* p) { reg::dft8<false>(p); });
            } else
            {
#pragma unroll 1
                for (int j3 = q; j3 < NQ; j3 += TEAMS) {
                    V x[R];
#pragma unroll
                    for (int r = 0; r < R; ++r) x[r] = X[j3 * P + t + 8 * r];
                    // forward DFT along axis 2; the row's spectrum stays in exchange-slot order
                    // (X(k2) at slot(k2 % R, k2 / R))
                    V* row = X + j3 * P;
                    __syncwarp();
                    tdft_s1<R, false>(x, row, tw, t, rs);
                    __syncwarp();
                    tdft_s2<R>(row, t, rs, [](int, V* p) { reg::dft8<false>(p); });
                }
            }
            __syncthreads();
            QPROF_T(q3);
            QPROF_ADD(2, q2, q3);
            // ------------------------------------------------------------ F3: axis 3, x table, inverse
#pragma unroll 1
            for (int k2 = q; k2 < NQ; k2 += TEAMS) {
                V* col = X + rslot(k2 % R, k2 / R);           // logical column k2 (slot order)
                const double* pr = psi + k2 * PSP;
                V x[R];
#pragma unroll
                for (int r = 0; r < R; ++r) x[r] = col[(t + 8 * r) * P];
                __syncwarp();
                tdft_s1<R, false>(x, col, tw, t, cs);
                __syncwarp();
                const bool dc = flag == 4 && i == 0 && a.koff + a.kbeg == 0 && k2 == 0;
                tdft_s2<R>(col, t, cs, [&](int s3, V* p) {
                    reg::dft8<false>(p);                      // X(k2, k3 = s3 + R qq)
                    if (dc && s3 == 0) {
                        // (k0, k1, k2, k3) = 0: the sum of the regridded weights
                        a.dc3[(long long)f * a.n3] = p[0].x;
                        for (int j = 1; j < a.n3; ++j) a.dc3[(long long)f * a.n3 + j] = 0.0;
                    }
#pragma unroll
                    for (int qq = 0; qq < 8; ++qq) {
                        const double fq = pr[s3 + R * qq];
                        p[qq] = V{p[qq].x * fq, p[qq].y * fq};
                    }
                    reg::dft8<true>(p);
                });
                __syncwarp();
                tdft_s1_dif<R, true>(x, col, tw, t, cs);
                __syncwarp();
#pragma unroll
                for (int r = 0; r < R; ++r) col[(t + 8 * r) * P] = x[r];
            }
        }
        if (tid == 0 && nxt < items) tma::mbar_expect_tx(bar, PLANE);   // the next phase's bytes
        __syncthreads();
        QPROF_T(q4);
        QPROF_ADD(3, q2, q4);
        // ---------------------------------------------------------------- I2: inverse axis 2, store, refill
        // by parts of RP rows: once every team has finished a part, its rows take the next
        // item's part (one TMA load), which then overlaps the rest of this item and the next
        // item's tables
        // output row j3 of this item: G == 1: S2[f][k1][k0][j3][j2]; G > 1: S2 (rank j3 / slab's
        // block)[k0][k1][j3 % slab][j2]. (Measured: the k0-major order for G == 1 doubles K3's
        // DRAM reads of S2 -- the same sectors, gathered in a different order, miss L2.)
        const unsigned ok1 = i / (unsigned)N0, ok0 = i - ok1 * (unsigned)N0 + (unsigned)a.kbeg;
        const int NB = a.N0blk ? a.N0blk : N0;                            // k0 extent of an output block
        V* dst = a.Y + (long long)f * ((long long)a.G * NB * H1 * a.slab * NQ) +
                 (a.G == 1 ? (long long)i : ((long long)ok0 * H1 + ok1)) * ((long long)a.slab * NQ);
        const long long rstride = (long long)NB * H1 * a.slab * NQ;      // between destination blocks
#pragma unroll 1
        for (int c = 0; c < NPART; ++c) {
#pragma unroll 1
            for (int j3 = c * RP + q; j3 < (c + 1) * RP; j3 += TEAMS) {
                V* row = X + j3 * P;
                if (!skip) {
                    V x[R];
                    // inverse DFT along axis 2 from the slot-order spectrum: x[r] = element j2 = t + 8r
                    tdft_s2<R>(row, t, rs, [](int, V* p) { reg::dft8<true>(p); });
                    __syncwarp();
                    tdft_s1_dif<R, true>(x, row, tw, t, rs);
                    {
                        const int rk = j3 / a.slab, j3l = j3 - rk * a.slab;
                        V* o = dst + rk * rstride + j3l * NQ + t;
#pragma unroll
                        for (int r = 0; r < R; ++r) __stcg(o + 8 * r, x[r]);
                    }
                }
            }
            if (nxt < items) {
                tma::fence_proxy_async();                     // this thread's reads of the part's rows
                __syncthreads();                              // ... and everyone's precede the load
                if (tid == 0) load_part(nxt, c);
            }
        }
        QPROF_T(q5);
        QPROF_ADD(4, q4, q5);
        QPROF_ADD(5, 0, 1);
    }
}

// ============================================================================ K3: inverse plane pass (+ update)
// Plane p's coefficients Y[f][k1][k0][j3][j2] arrive by ONE tensor-map TMA load (box
// 2 x 1 x 1 x (N + 2) x H doubles over the map (re/im, j2, j3, k0, filter*k1)): the two
// out-of-range k0 per row are zero-filled, so the box lands as [H][PITCH = N + 2] -- the
// conflict-free pitch of the transforms. Two buffers: the next plane's load overlaps this
// plane's work. The rest is k_plane_inv's arithmetic; the filter's coefficient block is
// cached in shared memory.
template <int N> struct Q3 {
    static constexpr size_t XS = (sizeof(V) * Cfg<N>::H * Cfg<N>::PITCH + 127) / 128 * 128;   // TMA: 128-B aligned
    static constexpr size_t SMEM = 2 * XS + sizeof(V) * N + sizeof(double) * NMOM * (Cfg<N>::NT / 32) + 16 +
                                   sizeof(double) * NMOM * Cfg<N>::NT + sizeof(double) * PL_EU;
};
template <int N>
static size_t qinv_smem() { return Q3<N>::SMEM; }

template <int N, bool UP>
__global__ void __launch_bounds__(Cfg<N>::NT, 1) k_q_inv(QArgs a, const __grid_constant__ CUtensorMap ymap,
                                                       const __grid_constant__ CUtensorMap wmap) {
    using C = Cfg<N>;
    constexpr int R1 = C::R1, H = C::H, PITCH = C::PITCH, NT = C::NT, NW = NT / 32, NX = 4;
    constexpr int XSV = (int)(Q3<N>::XS / sizeof(V));
    extern __shared__ __align__(128) unsigned char smem_raw[];
    V* X0 = reinterpret_cast<V*>(smem_raw);
    V* tw = X0 + 2 * XSV;
    double* red = reinterpret_cast<double*>(tw + N);          // [NW][NMOM]
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(red + NMOM * NW);
    double* cfs = reinterpret_cast<double*>(bar + 2) + NMOM * NT;   // the current filter's coefficients
    const int tid = threadIdx.x, m = tid >> 3, t = tid & 7, lane = tid & 31, warp = tid >> 5;
    init_tw<N>(tw);
    if (tid == 0) {
        tma::mbar_init(&bar[0], 1);
        tma::mbar_init(&bar[1], 1);
        asm volatile("prefetch.tensormap [%0];" ::"l"(&ymap) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&wmap) : "memory");
    }
    const int n2 = a.n2, n3 = a.n3, ppf = n2 * n3;
    const long long ntot = (long long)N * N * ppf, nq = (long long)n2 * n3;
    const int nplanes = a.batch * ppf;
    __syncthreads();
    constexpr int NM = 1 + NX + NX * (NX + 1) / 2;
    double* mom = reinterpret_cast<double*>(bar + 2) + tid;  // this thread's sums, stride NT (shared)
#pragma unroll
    for (int q = 0; q < NM; ++q) mom[q * NT] = 0.0;
    int curf = -1;
    auto flush = [&]() {
        if (curf < 0) return;
#pragma unroll
        for (int q = 0; q < NM; ++q) {
            double v = mom[q * NT];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
            if (lane == 0) red[warp * NM + q] = v;
            mom[q * NT] = 0.0;
        }
        __syncthreads();
        if (tid < NM) {
            double v = 0.0;
            for (int w = 0; w < NW; ++w) v += red[w * NM + tid];
            a.part[((long long)curf * gridDim.x + blockIdx.x) * NMOM + tid] = v;
        }
        __syncthreads();
    };
    // plane p (filter f, (j2, j3)) into buffer buf: one TMA tensor load
    auto issue = [&](int p, int buf) {
        if (p >= nplanes || tid != 0) return;
        const int f = p / ppf, pl = p - f * ppf, j3 = pl / n2, j2 = pl - j3 * n2;
        tma::fence_proxy_async();
        tma::mbar_expect_tx(&bar[buf], (unsigned)(H * PITCH * sizeof(V)));
        asm volatile(
            "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
            "%6}], [%7];" ::"r"(tma::smem_u32(X0 + buf * XSV)),
            "l"(&ymap), "r"(0), "r"(a.G == 1 ? 0 : f * N), "r"(a.G == 1 ? f * H : 0), "r"(j2), "r"(j3),
            "r"(tma::smem_u32(&bar[buf]))
            : "memory");
    };
    issue(blockIdx.x, 0);
    int k = 0;
    for (int p = blockIdx.x; p < nplanes; p += gridDim.x, ++k) {
        const int buf = k & 1;
        QPROF_T(r0);
        tma::mbar_wait(&bar[buf], (unsigned)((k >> 1) & 1));
        QPROF_T(r1);
        QPROF_ADD(11, r0, r1);
        V* X = X0 + buf * XSV;
        const int filt = p / ppf, pl = p - filt * ppf;
        if (filt != curf) {                                   // uniform
            if (UP) flush();
            curf = filt;
            if (tid < PL_EU) cfs[tid] = a.coef[(long long)filt * a.cs + tid];
            __syncthreads();
        }
        const double* P = cfs;
        if (P[PL_SKIP] != 0.0) {                              // uniform: failed filter, left untouched
            if (tid == 0) tma::bulk_wait_read<0>();
            issue(p + gridDim.x, buf ^ 1);
            __syncthreads();
            continue;
        }
        // ------------------------------------------------------------ inverse axis 0 of row k1 = m
        // split team DFT: the row's spectrum is left in (swizzled) slot order, read as such below
        {
            V x[R1];
            V* row = X + m * PITCH;
            const bool m0 = m == 0;
            const int sw = (m >> 2) & 1;
            auto slot = [sw](int s, int tt) { return rslot(s, tt) ^ sw; };
#pragma unroll
            for (int r = 0; r < R1; ++r) {
                const V A = row[t + 8 * r];
                const V B = m0 ? X[(N / 2) * PITCH + t + 8 * r] : V{0.0, 0.0};
                x[r] = V{A.x - B.y, A.y + B.x};
            }
            __syncwarp();
            tdft_s1<R1, true>(x, row, tw, t, slot);
            __syncwarp();
            tdft_s2<R1>(row, t, slot, [&](int s, V* p) {
                reg::dft8<true>(p);
                if (m0) {                                     // rows 0 and N/2 were packed as one
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        X[(N / 2) * PITCH + rslot(s, q)] = V{p[q].y, 0.0};
                        p[q] = V{p[q].x, 0.0};
                    }
                }
            });
        }
        __syncthreads();
        // the next plane into the other buffer, once that buffer's weight store has read it
        if (tid == 0) tma::bulk_wait_read<0>();
        issue(p + gridDim.x, buf ^ 1);
        QPROF_T(r2);
        QPROF_ADD(12, r1, r2);
        // ------------------------------------------------------------ inverse axis 1 of the column pair
        V x[R1];
        {
            V pa[8], pb[8];
            const int oc0 = rslot((2 * m) % R1, (2 * m) / R1), oc1 = rslot((2 * m + 1) % R1, (2 * m + 1) / R1);
            auto ld = [&](int k1, int col) -> V { return X[k1 * PITCH + ((col ? oc1 : oc0) ^ ((k1 >> 2) & 1))]; };
            auto zdir = [&](int k1) -> V {
                const V wa = ld(k1, 0), wb = ld(k1, 1);
                return V{wa.x - wb.y, wa.y + wb.x};
            };
            auto zmir = [&](int kp) -> V {
                const V wa = ld(kp, 0), wb = ld(kp, 1);
                return V{wa.x + wb.y, wb.x - wa.y};
            };
            if (s_on<R1>(t)) {
                const int sa = s_a<R1>(t), sb = s_b<R1>(t), ma = R1 - t, mb = (t == 0) ? R1 / 2 : t;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    pa[q] = (q < 4) ? zdir(sa + R1 * q) : zmir(ma + R1 * (7 - q));
                    pb[q] = (q < 4) ? zdir(sb + R1 * q) : zmir(mb + R1 * (7 - q));
                }
            }
            // exchange inside this team's own two column homes (the other teams' are still being read)
            team_dft_dif<R1, true>(pa, pb, x, X, tw, t, [&](int s, int tt) {
                const int r = 4 * s + ((tt >> 1) ^ (s & 3)), cb = (tt & 1) ^ ((s >> 2) & 1);
                return r * PITCH + ((cb ? oc1 : oc0) ^ (s & 1));
            });
        }
        QPROF_T(r3);
        QPROF_ADD(13, r2, r3);
        int j2, j3;
        plane_j(pl, n2, j2, j3);
        // the plane's weights are staged in X (rows of pitch N + 2 doubles: conflict-free) and
        // leave by one TMA tensor store (768-byte rows) instead of per-thread strided stores
        __syncthreads();                                      // X is consumed by the transforms
        double* Ws = reinterpret_cast<double*>(X);
        auto store_plane = [&]() {
            __syncthreads();                                  // the staged rows are complete
            if (tid == 0) {
                tma::fence_proxy_async();
                asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];"
                             ::"l"(&wmap), "r"(0), "r"(0), "r"(p), "r"(tma::smem_u32(Ws))
                             : "memory");
                tma::bulk_commit();
            }
        };
        if (!UP) {
#pragma unroll
            for (int r = 0; r < R1; ++r) *reinterpret_cast<V*>(Ws + (t + 8 * r) * (N + 2) + 2 * m) = x[r];
            store_plane();
            continue;
        }
        const double u2 = j2 - 0.5 * (n2 - 1), u3 = (a.j3off + j3) - 0.5 * (a.n3g - 1);   // global j3
        const double u10 = t - 0.5 * (N - 1);
        const double lgn = P[PL_LGN];
        double S[2] = {0, 0}, Tm[2] = {0, 0}, U[2] = {0, 0};
        auto emit = [&](int r, int e, double w) -> double {
            const double u1 = fma(8.0, (double)r, u10);
            const double wu = w * u1;
            S[e] += w;
            Tm[e] += wu;
            U[e] = fma(wu, u1, U[e]);
            return w;
        };
        bool rec = !a.range;
        double Lr[2], Rr[2], Gr[2];
        if (!a.range) {
            const double* q = P + PL_LQ;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const double u0 = (2 * m + e) - 0.5 * (N - 1);
                const double c2 = q[5 + tri(1, 1)];
                double c1 = fma(q[5 + tri(0, 1)], u0, q[2]);
                double c0 = fma(u0, fma(q[5 + tri(0, 0)], u0, q[1]), q[0]);
                c1 = fma(q[5 + tri(1, 2)], u2, c1);
                c0 = fma(u2, fma(q[5 + tri(2, 2)], u2, fma(q[5 + tri(0, 2)], u0, q[3])), c0);
                c1 = fma(q[5 + tri(1, 3)], u3, c1);
                c0 = fma(u3, fma(q[5 + tri(3, 3)], u3, fma(q[5 + tri(2, 3)], u2, fma(q[5 + tri(0, 3)], u0, q[4]))),
                         c0);
                const double E0 = fma(-0.5, fma(u10, fma(c2, u10, c1), c0), lgn);
                const double E1 = -0.5 * (8.0 * c1 + 16.0 * c2 * u10);
                const double E2 = -32.0 * c2;
                rec = rec && (fabs(E0) + (R1 - 1) * fabs(E1) + (R1 - 1) * (R1 - 1) * fabs(E2) < 650.0);
                Lr[e] = exp_fast(E0);
                Rr[e] = exp_fast(E1 + E2);
                Gr[e] = exp_fast(2.0 * E2);
            }
        }
        if (rec) {
#pragma unroll
            for (int r = 0; r < R1; ++r) {
                const double o0 = emit(r, 0, x[r].x * Lr[0]);
                const double o1 = emit(r, 1, x[r].y * Lr[1]);
                Lr[0] *= Rr[0];
                Rr[0] *= Gr[0];
                Lr[1] *= Rr[1];
                Rr[1] *= Gr[1];
                *reinterpret_cast<V*>(Ws + (t + 8 * r) * (N + 2) + 2 * m) = V{o0, o1};
            }
        } else {
            const double* q = P + PL_LQ;
#pragma unroll
            for (int r = 0; r < R1; ++r) {
                const double u1 = fma(8.0, (double)r, u10);
                const double uu[4] = {0.0, u1, u2, u3};
                double o[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    double uv[4] = {(2 * m + e) - 0.5 * (N - 1), uu[1], uu[2], uu[3]};
                    double ll;
                    if (!a.range) {
                        double ee = q[0];
#pragma unroll
                        for (int a2 = 0; a2 < NX; ++a2) {
                            ee = fma(q[1 + a2], uv[a2], ee);
#pragma unroll
                            for (int b2 = a2; b2 < NX; ++b2) ee = fma(q[5 + tri(a2, b2)] * uv[a2], uv[b2], ee);
                        }
                        ll = fma(-0.5, ee, lgn);
                    } else {
                        double r2 = 0.0;
#pragma unroll
                        for (int a2 = 0; a2 < NX; ++a2) {
                            double y = P[PL_CL + a2];
#pragma unroll
                            for (int b2 = 0; b2 < NX; ++b2) y = fma(P[PL_BL + a2 * 4 + b2], uv[b2], y);
                            r2 = fma(y, y, r2);
                        }
                        const double d = (P[PL_ZR] - sqrt(r2)) * P[PL_ISG];
                        ll = fma(-0.5 * d, d, lgn);
                    }
                    const double w = e == 0 ? x[r].x : x[r].y;
                    o[e] = emit(r, e, w * exp_fast(ll));
                }
                *reinterpret_cast<V*>(Ws + (t + 8 * r) * (N + 2) + 2 * m) = V{o[0], o[1]};
            }
        }
        {
            const double ua = (2 * m) - 0.5 * (N - 1), ub = ua + 1.0;
            const double s0 = S[0] + S[1], su0 = fma(ua, S[0], ub * S[1]), st = Tm[0] + Tm[1];
            const double m1[4] = {su0, st, u2 * s0, u3 * s0};
            mom[0] += s0;
#pragma unroll
            for (int a2 = 0; a2 < NX; ++a2) mom[(1 + a2) * NT] += m1[a2];
            int kk = 1 + NX;
            const double uu[4] = {0.0, 0.0, u2, u3};
#pragma unroll
            for (int a2 = 0; a2 < NX; ++a2)
#pragma unroll
                for (int b2 = a2; b2 < NX; ++b2) {
                    double v;
                    if (a2 >= 2) v = uu[a2] * uu[b2] * s0;
                    else if (b2 >= 2) v = uu[b2] * m1[a2];
                    else if (a2 == 0 && b2 == 0) v = fma(ua * ua, S[0], ub * ub * S[1]);
                    else if (a2 == 0) v = fma(ua, Tm[0], ub * Tm[1]);
                    else v = U[0] + U[1];
                    mom[(kk++) * NT] += v;
                }
        }
        store_plane();                    // (its barrier: the moment sums are also complete)
        QPROF_T(r4);
        QPROF_ADD(14, r3, r4);
        QPROF_ADD(15, 0, 1);
    }
    if (UP) flush();
    if (tid == 0) tma::bulk_wait_all();
    (void)lane;
    (void)warp;
}

}  // namespace pln

using namespace pln;

// sharded route: one shard's totals tot[16] = {K3's 15 index-space moment sums over its CTAs,
// the DC (sum of K1's per-plane input sums)} in a fixed order (block tree), all-reduced next
__global__ void k_shard_sum(const double* __restrict__ dcpart, int nplanes, const double* __restrict__ part, int ginv,
                            int update, double* tot) {
    __shared__ double red[32 * 16];
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
    for (int p = threadIdx.x; p < nplanes; p += blockDim.x) acc[15] += dcpart[p];
    if (update)
        for (int c = threadIdx.x; c < ginv; c += blockDim.x)
#pragma unroll
            for (int i = 0; i < NMOM; ++i) acc[i] += part[(long long)c * NMOM + i];
    block_sum<16>(acc, red);
    if (threadIdx.x == 0)
        for (int i = 0; i < 16; ++i) tot[i] = acc[i];
}

cudaError_t launch_shard_sum(const double* dcpart, int nplanes, const double* part, int ginv, int update, double* tot,
                             cudaStream_t s, int64_t* launches) {
    k_shard_sum<<<1, 256, 0, s>>>(dcpart, nplanes, part, ginv, update, tot);
    ++*launches;
    return cudaGetLastError();
}

// debug: read (and optionally reset) the phase counters of -DPMF_QPROF builds
int quad_debug_counters(double* out, int n, int reset) {
    unsigned long long h[16];
    if (cudaMemcpyFromSymbol(h, g_qprof, sizeof(h)) != cudaSuccess) return -1;
    for (int i = 0; i < n && i < 16; ++i) out[i] = (double)h[i];
    if (reset) {
        std::fill(h, h + 16, 0ull);
        cudaMemcpyToSymbol(g_qprof, h, sizeof(h));
    }
    return 0;
}

bool quad_supported(const Dims& d, int dtype) {
    if (dtype != 0 || d.nx != 4 || d.n[0] != d.n[1] || d.n[2] != d.n[3]) return false;
    const int N = d.n[0], NQ = d.n[2];
    if (N != 32 && N != 64 && N != 96) return false;
    if (NQ != 16 && NQ != 32 && NQ != 64 && NQ != 96) return false;
    const char* e = std::getenv("PMF_NO_QUAD");
    return !(e && e[0] == '1');
}

template <typename K>
static cudaError_t q_grid(K kern, int nt, size_t smem, long long work, int* grid) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nt, smem);
    if (e != cudaSuccess) return e;
    if (occ < 1) return cudaErrorInvalidConfiguration;
    *grid = (int)std::max(1LL, std::min(work, (long long)nsm * occ));
    return cudaSuccess;
}

// Tensor map of the spectrum for K3's plane loads: doubles, dims (innermost first)
// re/im 2, j2 n2, j3 n3, k0 N, (filter, k1) batch*H; box 2 x 1 x 1 x (N + 2) x H -- the
// two k0 beyond N are out of range (zero-filled) and pad each shared-memory row to N + 2.
static cudaError_t y_map(const QArgs& qa, int N, int H, CUtensorMap* m) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !encode) {
            encode = nullptr;
            return cudaErrorNotSupported;
        }
    }
    // S2 = [filter, k0][k1][j3 (this block's slab)][j2] (filter and k0 merged: adjacent); the dims
    // are listed innermost-first as re/im, (filter, k0), k1, j2, j3 -- the box (2, N + 2, H, 1, 1)
    // lands as [k1][k0 + 2 padding] (the padding reads beyond k0 = N - 1: out of range for the
    // last filter, the next filter's first k0 otherwise -- never used)
    const cuuint64_t n2 = qa.n2, sl = qa.n3;
    cuuint64_t dims[5] = {2, (cuuint64_t)qa.batch * N, (cuuint64_t)H, n2, sl};
    cuuint64_t str[4] = {16 * (cuuint64_t)H * sl * n2, 16 * sl * n2, 16, 16 * n2};
    if (qa.G == 1) {
        // S2 = [filter][k1][k0][j3][j2]: dims re/im, k0, (filter, k1) merged, j2, j3
        dims[1] = (cuuint64_t)N;
        dims[2] = (cuuint64_t)qa.batch * H;
        str[0] = 16 * sl * n2;
        str[1] = 16 * sl * n2 * (cuuint64_t)N;
    }
    cuuint32_t box[5] = {2, (cuuint32_t)(N + 2), (cuuint32_t)H, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)qa.Y, dims, str, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Tensor map of the weights for K3's plane stores: doubles, dims j0 N, j1 N, planes
// batch * n2 * n3; box (N + 2) x N x 1 -- the staged rows' two padding doubles fall beyond
// j0 = N - 1 and are not written.
static cudaError_t w_map(const QArgs& qa, int N, CUtensorMap* m) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !encode) {
            encode = nullptr;
            return cudaErrorNotSupported;
        }
    }
    cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)qa.batch * qa.n2 * qa.n3};
    cuuint64_t str[2] = {8 * (cuuint64_t)N, 8 * (cuuint64_t)N * N};
    cuuint32_t box[3] = {(cuuint32_t)(N + 2), (cuuint32_t)N, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, (void*)qa.W, dims, str, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Tensor map of K1's spectrum S for K2's plane gathers: doubles, dims (innermost first) re/im 2,
// k0 N, k1 H, j2 n2, (filter, j3) batch*n3; box 2 x 1 x 1 x (n2 + 1) x RP -- the j2 beyond n2 - 1 is
// out of range (zero-filled) and pads each shared-memory row to n2 + 1 (conflict-free columns)
static cudaError_t s_map(const QArgs& qa, int N, int H, CUtensorMap* m) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !encode) {
            encode = nullptr;
            return cudaErrorNotSupported;
        }
    }
    const cuuint64_t n2 = qa.n2, n3 = qa.n3;
    const cuuint32_t rp = qa.n2 == 96 ? PMF_K2_TEAMS96 : (qa.n2 >= 64 ? 32 : (cuuint32_t)qa.n2 / 2);   // Q2<NQ>::RP
    cuuint64_t dims[5] = {2, (cuuint64_t)N, (cuuint64_t)H, n2, (cuuint64_t)qa.batch * n3};
    cuuint64_t str[4] = {16, 16 * (cuuint64_t)N, 16 * (cuuint64_t)N * H, 16 * (cuuint64_t)N * H * n2};
    cuuint32_t box[5] = {2, 1, 1, (cuuint32_t)(qa.n2 + 1), rp};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)qa.Yin, dims, str, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int NQ, int TM>
static cudaError_t qmid_tm(const QArgs& qa, int I, int N0, int H1, const CUtensorMap& smap, cudaStream_t s) {
    using Cq = QCfg<NQ, TM>;
    const size_t smem = qmid_smem<NQ>();
    int grid = 1;
    cudaError_t e = q_grid(k_q_mid<NQ, TM>, Cq::NT, smem, (long long)qa.batch * I, &grid);
    if (e != cudaSuccess) return e;
    k_q_mid<NQ, TM><<<grid, Cq::NT, smem, s>>>(qa, I, N0, H1, smap);
    return cudaGetLastError();
}

// (48 teams at NQ = 96: 12 warps, no spills with the split team DFT)
template <int NQ>
static cudaError_t qmid_launch(const QArgs& qa, int I, int N0, int H1, const CUtensorMap& smap, cudaStream_t s) {
    return qmid_tm<NQ, Q2<NQ>::TEAMS>(qa, I, N0, H1, smap, s);
}

// K1 -> K2 -> K3 (prep, the general-map pre-pass and the finaliser are the plane path's;
// launch_plane calls this between them). Returns the K3 grid (its partials per filter).
template <int N>
static cudaError_t quad_mid_n(const Dims& d, QArgs qa, int N0c, cudaStream_t s, int nk = -1) {
    using Cf = Cfg<N>;
    CUtensorMap smap;
    cudaError_t e = s_map(qa, N0c, Cf::H, &smap);
    if (e != cudaSuccess) return e;
    if (nk < 0) nk = N0c;                   // k0 columns [kbeg, kbeg + nk) of the N0c in the input
    const int I = Cf::H * nk;
    switch (d.n[2]) {
        case 16: return qmid_launch<16>(qa, I, nk, Cf::H, smap, s);
        case 32: return qmid_launch<32>(qa, I, nk, Cf::H, smap, s);
        case 64: return qmid_launch<64>(qa, I, nk, Cf::H, smap, s);
        case 96: return qmid_launch<96>(qa, I, nk, Cf::H, smap, s);
        default: return cudaErrorInvalidValue;
    }
}

template <int N>
static cudaError_t quad_inv_n(QArgs qa, bool up, cudaStream_t s, int* ginv) {
    using Cf = Cfg<N>;
    CUtensorMap ymap, wmap;
    cudaError_t e;
    if ((e = y_map(qa, N, Cf::H, &ymap)) != cudaSuccess) return e;
    if ((e = w_map(qa, N, &wmap)) != cudaSuccess) return e;
    const size_t smem = qinv_smem<N>();
    const long long nplanes = (long long)qa.batch * qa.n2 * qa.n3;
    if (up) {
        e = q_grid(k_q_inv<N, true>, Cf::NT, smem, nplanes, ginv);
        if (e == cudaSuccess && qa.batch > 1)
            e = cudaMemsetAsync(qa.part, 0, sizeof(double) * NMOM * (*ginv) * (size_t)qa.batch, s);
        if (e == cudaSuccess) k_q_inv<N, true><<<*ginv, Cf::NT, smem, s>>>(qa, ymap, wmap);
    } else {
        e = q_grid(k_q_inv<N, false>, Cf::NT, smem, nplanes, ginv);
        if (e == cudaSuccess) k_q_inv<N, false><<<*ginv, Cf::NT, smem, s>>>(qa, ymap, wmap);
    }
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

static QArgs make_qargs(const Dims& d, PencilBufs& b, const ModelParams& mp, int range, double* dc3, double* part) {
    QArgs qa;
    qa.W = (double*)b.W;
    qa.Yin = (const V*)b.S;
    qa.Y = (V*)b.S2;
    qa.coef = b.coef;
    qa.cs = coef_stride(mp.l);
    qa.dc3 = dc3;
    qa.part = part;
    qa.batch = d.batch;
    qa.n2 = d.n[2];
    qa.n3 = d.n[3];
    qa.l = mp.l;
    qa.step = mp.step;
    qa.range = range;
    qa.N0f = d.ng[0];
    qa.koff = 0;
    qa.G = 1;
    qa.slab = d.n[3];
    qa.j3off = 0;
    qa.n3g = d.n[3];
    return qa;
}

cudaError_t launch_quad(const Dims& d, PencilBufs& b, const ModelParams& mp, int range, bool up, double* dcpart,
                        double* dc3, double* part, cudaStream_t s, int64_t* launches, int* ginv) {
    (void)dcpart;
    QArgs qa = make_qargs(d, b, mp, range, dc3, part);
    cudaError_t e;
    if (b.ev0) cudaEventRecordWithFlags(b.ev0, s, cudaEventRecordExternal);
    switch (d.n[0]) {
        case 32: e = quad_mid_n<32>(d, qa, 32, s); break;
        case 64: e = quad_mid_n<64>(d, qa, 64, s); break;
        case 96: e = quad_mid_n<96>(d, qa, 96, s); break;
        default: e = cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    ++*launches;
    if (b.ev1) cudaEventRecordWithFlags(b.ev1, s, cudaEventRecordExternal);
    switch (d.n[0]) {
        case 32: e = quad_inv_n<32>(qa, up, s, ginv); break;
        case 64: e = quad_inv_n<64>(qa, up, s, ginv); break;
        case 96: e = quad_inv_n<96>(qa, up, s, ginv); break;
        default: e = cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    ++*launches;
    return cudaSuccess;
}

// Sharded (slab over j3, G ranks; pmf_sharded.cpp): K2 of rank q over the k0 range
// [q N0/G, (q+1) N0/G) reading the all-to-all receive buffer `in` = [j3][j2][k1][k0 - q N0/G]
// (K1's blocks of every rank, stacked in rank order) and writing `out` = [dest rank][k0][k1]
// [j3 % slab][j2]; K3 of rank r over its slab's planes reading `in` = [k0][k1][j3 % slab][j2]
// (the back exchange, source blocks stacked in rank order) and writing the shard's weights.
cudaError_t launch_quad_mid_shard(const Dims& d, PencilBufs& b, const ModelParams& mp, int rank, int world,
                                  const void* in, void* out, int kbeg, int kend, cudaStream_t s, int64_t* launches) {
    QArgs qa = make_qargs(d, b, mp, 0, nullptr, nullptr);
    qa.Yin = (const V*)in;
    qa.Y = (V*)out;
    qa.n3 = d.ng[3];                        // K2 sees whole (j3, j2)-planes
    qa.G = world;
    qa.slab = d.n[3];
    qa.koff = rank * (d.ng[0] / world);
    qa.n3g = d.ng[3];
    const int N0c = d.ng[0] / world;
    if (kend < 0) {
        kbeg = 0;
        kend = N0c;
    }
    if (kend <= kbeg) return cudaSuccess;
    qa.kbeg = kbeg;
    qa.N0blk = N0c;
    cudaError_t e;
    switch (d.n[0]) {
        case 32: e = quad_mid_n<32>(d, qa, N0c, s, kend - kbeg); break;
        case 64: e = quad_mid_n<64>(d, qa, N0c, s, kend - kbeg); break;
        case 96: e = quad_mid_n<96>(d, qa, N0c, s, kend - kbeg); break;
        default: e = cudaErrorInvalidValue;
    }
    if (e == cudaSuccess) ++*launches;
    return e;
}

cudaError_t launch_quad_inv_shard(const Dims& d, PencilBufs& b, const ModelParams& mp, const LikParams* lp, int rank,
                                  int world, const void* in, double* part, cudaStream_t s, int64_t* launches,
                                  int* ginv) {
    QArgs qa = make_qargs(d, b, mp, lp ? (lp->kind == 1) : 0, nullptr, part);
    qa.Y = (V*)in;
    qa.G = world;
    qa.j3off = rank * d.n[3];
    qa.n3g = d.ng[3];
    cudaError_t e;
    switch (d.n[0]) {
        case 32: e = quad_inv_n<32>(qa, lp != nullptr, s, ginv); break;
        case 64: e = quad_inv_n<64>(qa, lp != nullptr, s, ginv); break;
        case 96: e = quad_inv_n<96>(qa, lp != nullptr, s, ginv); break;
        default: e = cudaErrorInvalidValue;
    }
    if (e == cudaSuccess) ++*launches;
    return e;
}

}  // namespace pmf
