// plane_common.cuh -- helpers shared by the plane-path kernels (kernels_plane.cu) and the
// transposed-layout nx = 4 path (kernels_quad.cu): team-of-8 register FFTs, the per-filter
// coefficient block, the Psi evaluation (Alg. 3-4) and the split regrid steps (R12).
#pragma once
#include <cmath>
#include "device_common.cuh"
#include "fft_reg.cuh"
#include "tma.cuh"

namespace pmf {
namespace pln {

template <int N>
struct Cfg {
    static constexpr int R1 = N / 8;           // stage-1 radix
    static constexpr int H = N / 2 + 1;        // rows of a plane's half spectrum (k1 = 0..N/2)
    static constexpr int PITCH = N + 2;        // complex per shared-memory row (= 2 mod 8: conflict-free)
    static constexpr int TEAMS = N / 2;        // column pairs (P1, P3) = rows (P2)
    static constexpr int NT = 8 * TEAMS;
    static constexpr int SP = N + 2;           // real staging pitch (separable regrid)
    static constexpr int MINB = N >= 96 ? 1 : (N == 64 ? 2 : 4);
};

constexpr int LCAP = 64;                       // substeps held per pencil (mid pass, Psi)

// per-filter coefficient block (doubles), stride >= PL_EU + 10 l (coef_stride)
enum {
    PL_M = 0,       // 16: regrid map v = o + M u' (old index coordinates of new point u'), row stride 4
    PL_O = 16,      // 4
    PL_FLAG = 20,   // 0: no regrid, 2: general map (gather pre-pass), 4: split map (nx = 4 CV structure)
    PL_SKIP = 21,   // 1: filter failed (status) or degenerate regrid target: leave untouched
    PL_SN = 22,     // s / N_tot (trace factor and the transform scales, folded into Psi)
    PL_VOL = 23,    // |det B_l|
    PL_CL = 24,     // 4: moved grid centre c_l
    PL_BL = 28,     // 16: moved grid matrix B_l
    PL_LQ = 44,     // 16: linear-Gauss exponent e(u) = q0 + q_a u_a + sum_{a<=b} q_ab u_a u_b (tri order)
    PL_LGN = 60,    // log normalising constant of the likelihood
    PL_ISG = 61,    // 1 / sigma (range likelihood)
    PL_ZR = 62,     // range measurement
    PL_S = 63,      // s
    PL_EU = 64      // 10 per substep: Euler-factor coefficients (substep_coefs order)
};

__device__ __forceinline__ int xcol(int k1, int j0) { return j0 ^ ((k1 >> 2) & 1); }
__device__ __forceinline__ int rslot(int s, int t) { return s * 8 + (t ^ (s & 7)); }
template <int N>
__device__ __forceinline__ int cslot(int s, int t, int m) {
    const int row = 4 * s + ((t >> 1) ^ (s & 3));
    const int col = (t & 1) ^ ((s >> 2) & 1);
    return row * Cfg<N>::PITCH + 2 * m + col;
}

// stage-2 ownership (R1 >= 2)
template <int R1> __device__ __forceinline__ bool s_on(int t) { return t < R1 / 2; }
template <int R1> __device__ __forceinline__ int s_a(int t) { return t; }
template <int R1> __device__ __forceinline__ int s_b(int t) { return t == 0 ? R1 / 2 : R1 - t; }

template <int R1, bool INV, typename V>
__device__ __forceinline__ void dftR(V* x) {
    if constexpr (R1 == 16) reg::dft16<INV>(x);
    else if constexpr (R1 == 12) reg::dft12<INV>(x);
    else if constexpr (R1 == 8) reg::dft8<INV>(x);
    else if constexpr (R1 == 4) reg::r4<INV>(x[0], x[1], x[2], x[3]);
    else if constexpr (R1 == 2) {
        const V a = x[0];
        x[0] = cadd(a, x[1]);
        x[1] = csub(a, x[1]);
    }
}

// W_N^{ts} for s < R1, t < 8 at tw[s * 8 + t]
template <int N, typename V>
__device__ __forceinline__ void init_tw(V* tw) {
    using T = decltype(tw[0].x);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const int s = i >> 3, t = i & 7;
        double sn, cs;
        sincospi(2.0 * (double)(t * s) / (double)N, &sn, &cs);
        tw[i] = V{(T)cs, (T)(-sn)};
    }
}

template <bool INV, typename V>
__device__ __forceinline__ V twid(V a, V w) {
    if (INV) w.y = -w.y;
    return cmul(a, w);
}

// x[s] *= W_N^{ts} (conjugated for INV), s = 1 .. R1-1. With s = a + 4b (a < 4) the twiddle is
// W^{ta} W^{4tb}: R1/4 + 2 table loads and one complex product each for the rest, instead of
// R1 - 1 loads (16-byte shared loads cost 4 wavefronts per warp: the twiddles were 10 % of
// the plane kernels' shared-memory traffic).
template <int R1, bool INV, typename V>
__device__ __forceinline__ void apply_tw(V* x, const V* tw, int t) {
    if constexpr (R1 <= 4) {
#pragma unroll
        for (int s = 1; s < R1; ++s) x[s] = twid<INV>(x[s], tw[s * 8 + t]);
    } else {
        V wa[4];
#pragma unroll
        for (int a = 1; a < 4; ++a) {
            wa[a] = tw[a * 8 + t];
            x[a] = twid<INV>(x[a], wa[a]);
        }
#pragma unroll
        for (int b = 1; b < R1 / 4; ++b) {
            const V wb = tw[4 * b * 8 + t];
            x[4 * b] = twid<INV>(x[4 * b], wb);
#pragma unroll
            for (int a = 1; a < 4; ++a) x[a + 4 * b] = twid<INV>(x[a + 4 * b], cmul(wa[a], wb));
        }
    }
}

// Team DFT, DIT order: in x[r] = element t + 8r (registers), out pa[q] = X[sa + R1 q],
// pb[q] = X[sb + R1 q] on the threads with s_on(t). `ex` is the team's exchange area,
// `slot(s, t)` its conflict-free layout.
template <int R1, bool INV, typename V, typename SLOT>
__device__ __forceinline__ void team_dft(V* x, V* pa, V* pb, V* ex, const V* tw, int t, SLOT slot) {
    dftR<R1, INV>(x);
    apply_tw<R1, INV>(x, tw, t);
    __syncwarp();
#pragma unroll
    for (int s = 0; s < R1; ++s) ex[slot(s, t)] = x[s];
    __syncwarp();
    if (s_on<R1>(t)) {
        const int sa = s_a<R1>(t), sb = s_b<R1>(t);
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) {
            pa[tt] = ex[slot(sa, tt)];
            pb[tt] = ex[slot(sb, tt)];
        }
        reg::dft8<INV>(pa);
        reg::dft8<INV>(pb);
    }
    __syncwarp();
}

// Team DFT, DIF order (the inverse of team_dft's layout): in pa[q] = X[sa + R1 q],
// pb[q] = X[sb + R1 q] (threads with s_on), out x[r] = element t + 8r.
template <int R1, bool INV, typename V, typename SLOT>
__device__ __forceinline__ void team_dft_dif(V* pa, V* pb, V* x, V* ex, const V* tw, int t, SLOT slot) {
    __syncwarp();
    if (s_on<R1>(t)) {
        const int sa = s_a<R1>(t), sb = s_b<R1>(t);
        reg::dft8<INV>(pa);
        reg::dft8<INV>(pb);
#pragma unroll
        for (int tt = 0; tt < 8; ++tt) {
            ex[slot(sa, tt)] = pa[tt];
            ex[slot(sb, tt)] = pb[tt];
        }
    }
    __syncwarp();
#pragma unroll
    for (int s = 0; s < R1; ++s) x[s] = ex[slot(s, t)];
    apply_tw<R1, INV>(x, tw, t);
    dftR<R1, INV>(x);
    __syncwarp();
}

// ---------------------------------------------------------------------------- split team DFT
// The team DFT in two halves with an exchange area that doubles as the spectrum's home:
//   tdft_s1      DIT stage 1: x[r] (element t + 8r) -> ex[slot(s, t)] = DFT_R1(x)_s W_N^{ts}
//   tdft_s2      stage 2 over the thread's own s values (sa, then sb), one 8-point group at a
//                time: ex[slot(s, tt)] (tt < 8) -> f(s, p) -> back into the same slots, i.e.
//                X[s + R1 q] stays at slot(s, q)
//   tdft_s1_dif  the inverse's last stage: ex[slot(s, t)] -> twiddle -> DFT_R1 -> x[r]
// A thread only rewrites the slots it read, so stage 2 needs no second warp sync, keeps
// 8 values live instead of 16, and a spectrum left "in slot order" between passes costs no
// permutation (callers address column k as slot(k % R1, k / R1)).
template <int R1, bool INV, typename V, typename SLOT>
__device__ __forceinline__ void tdft_s1(V* x, V* ex, const V* tw, int t, SLOT slot) {
    dftR<R1, INV>(x);
    apply_tw<R1, INV>(x, tw, t);
#pragma unroll
    for (int s = 0; s < R1; ++s) ex[slot(s, t)] = x[s];
}
template <int R1, typename V, typename SLOT, typename F>
__device__ __forceinline__ void tdft_s2(V* ex, int t, SLOT slot, F f) {
    if (s_on<R1>(t)) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int s = h ? s_b<R1>(t) : s_a<R1>(t);
            V p[8];
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) p[tt] = ex[slot(s, tt)];
            f(s, p);
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) ex[slot(s, tt)] = p[tt];
        }
    }
}
template <int R1, bool INV, typename V, typename SLOT>
__device__ __forceinline__ void tdft_s1_dif(V* x, const V* ex, const V* tw, int t, SLOT slot) {
#pragma unroll
    for (int s = 0; s < R1; ++s) x[s] = ex[slot(s, t)];
    apply_tw<R1, INV>(x, tw, t);
    dftR<R1, INV>(x);
}

template <typename T>
struct PlaneArgs {
    const T* Wsrc;          // weights read by the forward pass (old grid when regridding)
    const T* W2src;         // pre-regridded weights (general regrid map, flag 2)
    T* W;                   // weights written by the inverse pass
    typename C2<T>::type* S;      // spectrum written by the forward pass
    typename C2<T>::type* Sinv;   // spectrum read by the inverse pass (S, or S2 after an out-of-place pass)
    const double* coef;
    int cs;
    double* dcpart;         // [plane] sums of the forward pass's input planes
    double* dc3;            // [filter][n3] slab sums after the split regrid (flag 4)
    double* part;           // [plane][6]
    int nplanes;            // batch * ppf
    int ppf;                // planes per filter
    int n2, n3;             // sizes of axes 2, 3 (1 if absent)
    int l;
    int range;              // likelihood kind 1
    int chunks = 1;         // forward pass: each spectrum row leaves as `chunks` pieces of N / chunks
    long long chunk_stride = 0;   // ... piece q to S + q chunk_stride + (plane H + k1) N / chunks (sharded)
    int pbeg = 0;           // forward pass: planes [pbeg, nplanes) (sharded: one chunk of the slab's planes)
};

// plane p of its filter -> (j2, j3)
__device__ __forceinline__ void plane_j(int pl, int n2, int& j2, int& j3) {
    j3 = pl / n2;
    j2 = pl - j3 * n2;
}

// ps[r] = mult / den[r] with ONE division for all R values (prefix products, kept in ps
// itself), every den >= 1; when the product of the R values leaves the range, one
// division per value
template <int R>
__device__ __forceinline__ void psi_div(const double* den, double mult, double* ps) {
    ps[0] = den[0];
#pragma unroll
    for (int r = 1; r < R; ++r) ps[r] = ps[r - 1] * den[r];
    if (ps[R - 1] < 1e300) {
        double inv = mult / ps[R - 1];
#pragma unroll
        for (int r = R - 1; r > 0; --r) {
            const double v = inv * ps[r - 1];
            inv *= den[r];
            ps[r] = v;
        }
        ps[0] = inv;
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) ps[r] = mult / den[r];
    }
}

template <int NQ, int TM = (NQ >= 64 ? 32 : NQ / 2)>
struct QCfg {
    static constexpr int R = NQ / 8;
    static constexpr int TEAMS = TM;            // team q owns rows / columns q + TEAMS j
    static constexpr int NT = 8 * TEAMS;
    static constexpr int P = NQ + 1;            // row pitch (complex)
};

// Euler factors of pair j of list `list` (0: denominators, 1: Crank-Nicolson numerators
// 2 - f_n, R27) as a quartic in kap_L: q[0] = (c0, c1), q[1] = (c2, c3), q[2] = (c4, value at
// the Nyquist wavenumber, where kx_L = 0, R7). f_n = gam_n + bet_n kx_L + alp_n kap_L^2 with
// gam_n, bet_n from the other axes' wavenumbers kap[a], kx[a] (a < L).
template <int NX, int L>
__device__ __forceinline__ void psi_pair(const double* cf, int l, int cn, int list, int j, const double* kap,
                                         const double* kx, double2* q) {
    auto gam_bet = [&](int n, double& g, double& bb) {
        const double* c = cf + 10 * n;
        g = 1.0;
        bb = 0.0;
#pragma unroll
        for (int a2 = 0; a2 < L; ++a2) {
            g = fma(c[a2], kap[a2] * kap[a2], g);
#pragma unroll
            for (int b2 = a2 + 1; b2 < L; ++b2) g = fma(c[pair_index(NX, a2, b2)], kx[a2] * kx[b2], g);
            bb = fma(c[pair_index(NX, a2, L)], kx[a2], bb);
        }
    };
    const int base = (list == 0 && cn) ? 1 : 0;        // CN den: f_1 .. f_l
    double g0, b0, g1 = 1.0, b1 = 0.0, a1 = 0.0;
    gam_bet(base + 2 * j, g0, b0);
    double a0 = cf[10 * (base + 2 * j) + L];
    const bool two = 2 * j + 1 < l;
    if (two) {
        gam_bet(base + 2 * j + 1, g1, b1);
        a1 = cf[10 * (base + 2 * j + 1) + L];
    }
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

// F2 of one row: forward DFT along axis 2 of x (element t + 8r), result in place in the row
template <int NQ, typename V>
__device__ __forceinline__ void quad_f2_row(V (&x)[NQ / 8], V* row, const V* tw, int t) {
    constexpr int R = NQ / 8;
    V pa[8], pb[8];
    team_dft<R, false>(x, pa, pb, row, tw, t, [](int s2, int tt) { return rslot(s2, tt); });
    if (s_on<R>(t)) {
        const int sa = s_a<R>(t), sb = s_b<R>(t);
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) {
            row[sa + R * qq] = pa[qq];
            row[sb + R * qq] = pb[qq];
        }
    }
}

// acc[r] *= product of list `list`'s Euler-factor pairs at kap_3 = kp[r]; pair j's quartic is
// computed by thread j % 8 of the team and broadcast by shuffles (full warp, width 8)
template <int NQ>
__device__ __forceinline__ void quad_psi_prod(double (&acc)[NQ / 8], const double (&kp)[NQ / 8], const double* cf,
                                              int l, int cn, int list, const double* kap, const double* kx, int t) {
    constexpr int R = NQ / 8;
    const int nq = (l + 1) >> 1;
    double nyq = 1.0;
    for (int jb = 0; jb < nq; jb += 8) {
        double2 c[3] = {double2{1.0, 0.0}, double2{0.0, 0.0}, double2{0.0, 1.0}};
        if (jb + t < nq) psi_pair<4, 3>(cf, l, cn, list, jb + t, kap, kx, c);
        const int cnt = min(8, nq - jb);
        for (int jj = 0; jj < cnt; ++jj) {
            const double c0 = __shfl_sync(0xffffffffu, c[0].x, jj, 8);
            const double c1 = __shfl_sync(0xffffffffu, c[0].y, jj, 8);
            const double c2 = __shfl_sync(0xffffffffu, c[1].x, jj, 8);
            const double c3 = __shfl_sync(0xffffffffu, c[1].y, jj, 8);
            const double c4 = __shfl_sync(0xffffffffu, c[2].x, jj, 8);
            nyq *= __shfl_sync(0xffffffffu, c[2].y, jj, 8);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const double x1 = kp[r];
                acc[r] *= fma(fma(fma(fma(c4, x1, c3), x1, c2), x1, c1), x1, c0);
            }
        }
    }
    if (t == ((NQ / 2) & 7)) acc[(NQ / 2) >> 3] = nyq;
}

}  // namespace pln
}  // namespace pmf
