// kernels_plane.cu -- the plane path for large single grids (nx >= 3 with
// N_0 = N_1 in {32, 64, 96, 128}: BASELINE configs[2] (C3, 128^3) and
// configs[3] (C4, 96^4)). One prediction interval + measurement update is
//
//   prep   per filter: regrid map (R12), grid motion e^{A tau} (eq:gridMov
//          P:142-148), Euler-factor coefficients of the l substeps (Alg. 3
//          P:333-336, R3/R4), likelihood quadratic form on the moved grid (R13)
//   fwd    per (i0, i1)-plane: [multilinear regrid gather of the previous
//          posterior, R12] -> forward DFT along axes 1 and 0 (Alg. 1, eq:fourtrsf
//          P:221) in registers + one shared-memory exchange per axis -> the plane's
//          half spectrum (k1 = 0..N/2) to HBM; the plane's DC (sum of its weights)
//   mid    per strided axis m >= 2: pencils of the spectrum; the last axis runs
//          forward DFT x s Psi / N_tot (Alg. 3-4) x inverse DFT (Alg. 5) in
//          registers; the others forward before / inverse after it
//   inv    per plane: inverse DFT along axes 0 and 1, likelihood at the moved
//          points (eq:filt P:46, R13), store, index-space moment partials
//   fin    per filter: DC and moment sums in a fixed order -> normaliser C
//          (P:49), closed-form predict normalisation (Alg. 6: sum w' = s DC),
//          mean and covariance (R14)
//
// HBM traffic per interval: (2 + 2 (nx - 2)) passes over the spectrum -- 3 for
// nx = 3, 5 for nx = 4 -- instead of 2 nx - 1 per-axis passes plus a regrid pass.
//
// Register FFT of length N = 8 R1 held by a team of 8 threads (element j = t + 8r
// in register r of thread t): DFT_R1 over r, twiddle W_N^{ts}, exchange, DFT_8
// over t for the s values thread t owns (s = t and R1 - t; thread 0: 0 and R1/2),
// giving X[s + R1 q]. The pairing (s, R1 - s) puts X[k] and X[-k] in the same
// thread, so Hermitian (un)packing of real data is thread-local.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "device_common.cuh"
#include "fft_reg.cuh"
#include "tma.cuh"
#include "plane_common.cuh"

namespace pmf {
namespace pln {


// ============================================================================ prep (one warp per filter)
template <int NX>
__global__ void k_plane_prep(FilterState* st, double* coef, int cs, ModelParams mp,
                             const SubstepEntry* __restrict__ sub, LikParams lp, const double* __restrict__ z,
                             double ks, int update, Dims d) {
    const int b = blockIdx.x, lane = threadIdx.x;
    FilterState& f = st[b];
    double* P = coef + (long long)b * cs;
    double c0[4] = {0, 0, 0, 0}, B0[16];
    for (int i = 0; i < 16; ++i) B0[i] = f.B[i];
    for (int a = 0; a < NX; ++a) c0[a] = f.c[a];
    bool skip = f.status != 0;
    int flag = 0;
    if (ks > 0.0) {
        double cn[4], Bn[16], Bi[16], M[16];
        if (!regrid_target(NX, d.ng, f, ks, cn, Bn, d.grid)) skip = true;
        mat_inv4(NX, B0, Bi);
        for (int i = 0; i < 16; ++i) M[i] = 0.0;
        mat_mul4(NX, Bi, Bn, M);
        // split map (nx = 4): v_0 = f(u'_0, u'_1), v_1 = f(u'_1), v_2 = f(u'_2, u'_3), v_3 = f(u'_3),
        // i.e. block-diagonal (01)(23) with zero lower entries -- the CV models after an
        // axis-aligned regrid: the in-plane part runs in the forward pass, the (2,3) part in
        // the first strided pass (flag 4). Anything else: 2^nx-tap gather pre-pass (flag 2).
        bool split = NX == 4;
        const int zero_ix[10] = {1 * 4 + 0, 0 * 4 + 2, 0 * 4 + 3, 1 * 4 + 2, 1 * 4 + 3,
                                 2 * 4 + 0, 2 * 4 + 1, 3 * 4 + 0, 3 * 4 + 1, 3 * 4 + 2};
        for (int q = 0; q < 10; ++q) split = split && M[zero_ix[q]] == 0.0;
        flag = split ? 4 : 2;
        if (lane == 0) {
            for (int i = 0; i < 16; ++i) P[PL_M + i] = M[i];
            for (int a = 0; a < NX; ++a) {
                double s = 0.5 * (d.ng[a] - 1);
                for (int k = 0; k < NX; ++k) s = fma(Bi[a * 4 + k], cn[k] - c0[k], s);
                P[PL_O + a] = s;
            }
        }
        for (int a = 0; a < NX; ++a) c0[a] = cn[a];
        for (int i = 0; i < 16; ++i) B0[i] = Bn[i];
    }
    __syncwarp();
    if (lane == 0) {
        P[PL_FLAG] = flag;
        P[PL_SKIP] = skip ? 1.0 : 0.0;
        if (skip) f.status = -6;
    }
    if (skip) return;
    double Bi0[16];
    mat_inv4(NX, B0, Bi0);
    for (int n = lane; n < mp.l + (mp.step ? 1 : 0); n += 32) substep_coefs(NX, B0, Bi0, mp, sub[n], P + PL_EU + 10 * n);
    if (lane != 0) return;
    double Bl[16], cl[4];
    for (int i = 0; i < 16; ++i) Bl[i] = 0.0;
    mat_mul4(NX, mp.Mtau, B0, Bl);
    for (int a = 0; a < NX; ++a) {
        double s = 0.0;
        for (int k = 0; k < NX; ++k) s = fma(mp.Mtau[a * 4 + k], c0[k], s);
        cl[a] = s;
    }
    double ntot = 1.0;
    for (int a = 0; a < NX; ++a) ntot *= d.ng[a];
    P[PL_SN] = mp.s / ntot;
    P[PL_S] = mp.s;
    P[PL_VOL] = fabs(det4(NX, Bl));
    for (int a = 0; a < 4; ++a) P[PL_CL + a] = a < NX ? cl[a] : 0.0;
    for (int i = 0; i < 16; ++i) P[PL_BL + i] = Bl[i];
    P[PL_LGN] = lp.lognorm;
    P[PL_ISG] = lp.inv_sigma;
    double* q = P + PL_LQ;
    for (int i = 0; i < 16; ++i) q[i] = 0.0;
    if (update && lp.kind == 0) {
        lik_quadform(NX, lp, cl, Bl, z + (long long)b * lp.nz, q);
    } else if (update) {
        P[PL_ZR] = z[b];
    }
    for (int a = 0; a < NX; ++a) f.c[a] = cl[a];
    for (int i = 0; i < 16; ++i) f.B[i] = Bl[i];
}

// ============================================================================ general regrid pre-pass
// Filters whose regrid map is neither absent nor split (flag 2): multilinear
// interpolation (R12, zero ghosts) of the old weights at every new point into W2,
// which the forward pass then reads plainly. One warp per axis-0 row (N0 is a multiple
// of 32 on the plane path): the row's (j1, j2, j3) split once per warp, v = v_row +
// M[:,0] u0 per point, the 2^nx taps loaded together (zero outside the old grid) and
// combined by nested linear interpolation, axis 0 first (2^nx - 1 lerps).
template <typename T, int NX>
__device__ __forceinline__ double gather_lerp(const T* __restrict__ Wf, const int* n, const int* st, const double* v) {
    int base = 0;
    double fr[NX];
    bool lo[NX], hi[NX];
#pragma unroll
    for (int a = 0; a < NX; ++a) {
        const double fl = floor(v[a]);
        const int i = __double2int_rz(fl);
        fr[a] = v[a] - fl;
        lo[a] = i >= 0 && i <= n[a] - 1;
        hi[a] = i >= -1 && i <= n[a] - 2;
        base += i * st[a];
    }
    double w[1 << NX];
    bool inner = true;
#pragma unroll
    for (int a = 0; a < NX; ++a) inner = inner && lo[a] && hi[a];
    if (inner) {
        // every tap inside the old grid (all but the points near its edge): one base
        // pointer, no per-tap predicates
        const T* pb = Wf + base;
#pragma unroll
        for (int c = 0; c < (1 << NX); c += 2) {
            int off = 0;
#pragma unroll
            for (int a = 1; a < NX; ++a)
                if ((c >> a) & 1) off += st[a];
            w[c] = (double)__ldg(pb + off);
            w[c + 1] = (double)__ldg(pb + off + 1);
        }
    } else {
#pragma unroll
        for (int c = 0; c < (1 << NX); ++c) {
            int off = base;
            bool ok = true;
#pragma unroll
            for (int a = 0; a < NX; ++a) {
                const bool bit = (c >> a) & 1;
                ok = ok && (bit ? hi[a] : lo[a]);
                if (bit) off += st[a];
            }
            w[c] = ok ? (double)__ldg(Wf + off) : 0.0;
        }
    }
#pragma unroll
    for (int a = 0; a < NX; ++a)
#pragma unroll
        for (int c = 0; c < (1 << (NX - 1 - a)); ++c) w[c] = fma(fr[a], w[2 * c + 1] - w[2 * c], w[2 * c]);
    return w[0];
}

template <typename T, int NX>
__global__ void __launch_bounds__(256) k_plane_pre(const T* __restrict__ W, T* __restrict__ W2,
                                                   const double* __restrict__ coef, int cs, Dims d, int bpf) {
    const int filt = blockIdx.x / bpf, qb = blockIdx.x - filt * bpf;
    const double* P = coef + (long long)filt * cs;
    if (P[PL_SKIP] != 0.0 || (int)P[PL_FLAG] != 2) return;
    const long long ntot = d.ntot;
    const T* Wf = W + filt * ntot;
    T* Wn = W2 + filt * ntot;
    const int nsz[4] = {d.n[0], d.n[1], d.n[2], NX == 4 ? d.n[3] : 1};
    const int st[4] = {1, nsz[0], nsz[0] * nsz[1], nsz[0] * nsz[1] * nsz[2]};
    double M0[NX], o[NX];
#pragma unroll
    for (int a = 0; a < NX; ++a) {
        M0[a] = P[PL_M + a * 4];
        o[a] = P[PL_O + a];
    }
    const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const int nrows = nsz[1] * nsz[2] * nsz[3], n0 = nsz[0];
    for (int row = qb * nw + (threadIdx.x >> 5); row < nrows; row += bpf * nw) {
        const int q1 = row / nsz[1], j1 = row - q1 * nsz[1];          // warp-uniform
        const int j3 = q1 / nsz[2], j2 = q1 - j3 * nsz[2];
        const double u[4] = {0.0, j1 - 0.5 * (nsz[1] - 1), j2 - 0.5 * (nsz[2] - 1), j3 - 0.5 * (nsz[3] - 1)};
        double vr[NX];
#pragma unroll
        for (int a = 0; a < NX; ++a) {
            double x = o[a];
#pragma unroll
            for (int b = 1; b < NX; ++b) x = fma(P[PL_M + a * 4 + b], u[b], x);
            vr[a] = x;
        }
        T* out = Wn + (long long)row * n0;
#pragma unroll 4
        for (int j0 = lane; j0 < n0; j0 += 32) {
            const double u0 = j0 - 0.5 * (n0 - 1);
            double v[NX];
#pragma unroll
            for (int a = 0; a < NX; ++a) v[a] = fma(M0[a], u0, vr[a]);
            out[j0] = (T)gather_lerp<T, NX>(Wf, nsz, st, v);
        }
    }
}

// ============================================================================ forward plane pass
// Staged real plane: element (j0, j1), j in [-1, N+1], at stg[(j1 + 1) * SP + j0 + OFF];
// the ring j = -1, N, N+1 is zero (the zero ghost nodes of R12). SP/2 odd (fp64) keeps
// the 8 rows a team reads in distinct 16-byte bank groups; interior rows are 16-byte
// aligned for the bulk copies.
template <typename T, int N> struct SPitch;
template <int N> struct SPitch<double, N> { static constexpr int SP = N + 6, OFF = 2; };
template <int N> struct SPitch<float, N> { static constexpr int SP = N + 12, OFF = 4; };
template <typename T, int N>
__host__ __device__ constexpr size_t stage_bytes() { return (size_t)(N + 3) * SPitch<T, N>::SP * sizeof(T); }
template <typename T, int N>
__host__ __device__ constexpr size_t xbytes() { return 2 * sizeof(T) * Cfg<N>::H * Cfg<N>::PITCH; }
// separate staging buffer (the next plane's copy overlaps this plane's FFTs) when both fit
template <typename T, int N>
__host__ __device__ constexpr bool fwd_sep() { return stage_bytes<T, N>() + xbytes<T, N>() <= 200 * 1024; }
template <typename T, int N>
static size_t fwd_smem() {
    const size_t xs = fwd_sep<T, N>() ? stage_bytes<T, N>() + xbytes<T, N>()
                                      : std::max(stage_bytes<T, N>(), xbytes<T, N>());
    return xs + 2 * sizeof(T) * N + 16;
}

template <typename T, int N>
__device__ __forceinline__ void zero_ring(T* stg, int tid, int nt) {
    constexpr int SP = SPitch<T, N>::SP, OFF = SPitch<T, N>::OFF, W = N + 3;
    for (int i = tid; i < 3 * W + 3 * N; i += nt) {
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
        stg[(row + 1) * SP + col + OFF] = T(0);
    }
}

template <typename T, int N, int NX, bool RG>
__global__ void __launch_bounds__(Cfg<N>::NT, Cfg<N>::MINB) k_plane_fwd(PlaneArgs<T> a) {
    using V = typename C2<T>::type;
    using C = Cfg<N>;
    constexpr int R1 = C::R1, H = C::H, PITCH = C::PITCH, NT = C::NT;
    constexpr int SP = SPitch<T, N>::SP, OFF = SPitch<T, N>::OFF;
    constexpr bool SEP = fwd_sep<T, N>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* X = reinterpret_cast<V*>(smem_raw);                    // [H][PITCH]
    T* stg = SEP ? reinterpret_cast<T*>(smem_raw + xbytes<T, N>()) : reinterpret_cast<T*>(smem_raw);
    constexpr size_t XS = SEP ? stage_bytes<T, N>() + xbytes<T, N>()
                              : (stage_bytes<T, N>() > xbytes<T, N>() ? stage_bytes<T, N>() : xbytes<T, N>());
    V* tw = reinterpret_cast<V*>(smem_raw + XS);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(tw + N);

    const int tid = threadIdx.x, m = tid >> 3, t = tid & 7;
    init_tw<N>(tw);
    if (tid == 0) tma::mbar_init(bar, 1);
    zero_ring<T, N>(stg, tid, NT);
    const long long ntot = (long long)N * N * a.n2 * a.n3;
    __syncthreads();
    // stage plane p (all threads call; rows issued by the first N threads)
    auto issue = [&](int p) {
        if (p >= a.nplanes || tid >= N) return;
        const int filt = p / a.ppf, pl = p - filt * a.ppf;
        const double* P = a.coef + (long long)filt * a.cs;
        const T* src = ((RG && (int)P[PL_FLAG] == 2) ? a.W2src : a.Wsrc) + filt * ntot + (long long)pl * N * N;
        tma::fence_proxy_async();
        if (tid == 0) tma::mbar_expect_tx(bar, (unsigned)(N * N * sizeof(T)));
        tma::bulk_g2s(stg + (tid + 1) * SP + OFF, src + (long long)tid * N, (unsigned)(N * sizeof(T)), bar);
    };
    if (SEP) issue(a.pbeg + blockIdx.x);
    int k = 0;
    for (int p = a.pbeg + blockIdx.x; p < a.nplanes; p += gridDim.x, ++k) {
        if (!SEP) {
            if (k > 0) {
                zero_ring<T, N>(stg, tid, NT);
                __syncthreads();
            }
            issue(p);
        }
        const int filt = p / a.ppf;
        const double* P = a.coef + (long long)filt * a.cs;
        const int flag = RG ? (int)P[PL_FLAG] : 0;
        tma::mbar_wait(bar, (unsigned)(k & 1));
        // ------------------------------------------------------------ P1 input: column pair (2m, 2m+1)
        V z[R1];
        if (RG && flag == 4) {
            // in-plane part of the split regrid map (R12): bilinear from the staged old plane,
            // v1 = o1 + M11 u1', v0 = o0 + M00 u0' + M01 u1'; zero ghosts via the staged ring
            const double M00 = P[PL_M], M01 = P[PL_M + 1], M11 = P[PL_M + 5], o0 = P[PL_O], o1 = P[PL_O + 1];
            auto split = [&](double v, int& i, double& fr) {
                const double f = floor(v);
                const int fi = __double2int_rz(f);
                i = min(max(fi, -1), N);
                fr = (fi == i) ? v - f : 0.0;
            };
            if (M00 >= 0.0 && M00 < 1.0) {
                // 0 <= M00 < 1 (the new spacing below the old one: the usual case after an update):
                // the two columns' taps lie in one 3-wide window of the staged rows i1, i1 + 1,
                // so 6 loads serve both (the second column's pair starts 0 or 1 further)
#pragma unroll
                for (int r = 0; r < R1; ++r) {
                    const double u1 = (t + 8 * r) - 0.5 * (N - 1);
                    int i1, i0a, i0b;
                    double a1, a0a, a0b;
                    split(fma(M11, u1, o1), i1, a1);
                    const double vb = fma(M01, u1, o0);
                    split(fma(M00, (2 * m) - 0.5 * (N - 1), vb), i0a, a0a);
                    split(fma(M00, (2 * m + 1) - 0.5 * (N - 1), vb), i0b, a0b);
                    const T* r0 = stg + (i1 + 1) * SP + i0a + OFF;
                    const double w0 = (double)r0[0], w1 = (double)r0[1], w2 = (double)r0[2];
                    const double v0 = (double)r0[SP], v1 = (double)r0[SP + 1], v2 = (double)r0[SP + 2];
                    const bool d = i0b != i0a;
                    const double x0 = d ? w1 : w0, x1 = d ? w2 : w1, y0 = d ? v1 : v0, y1 = d ? v2 : v1;
                    const double loa = fma(a0a, w1 - w0, w0), hia = fma(a0a, v1 - v0, v0);
                    const double lob = fma(a0b, x1 - x0, x0), hib = fma(a0b, y1 - y0, y0);
                    z[r] = V{(T)fma(a1, hia - loa, loa), (T)fma(a1, hib - lob, lob)};
                }
            } else
#pragma unroll
            for (int r = 0; r < R1; ++r) {
                const double u1 = (t + 8 * r) - 0.5 * (N - 1);
                int i1;
                double a1;
                split(fma(M11, u1, o1), i1, a1);
                const double vb = fma(M01, u1, o0);
                // odd teams take column 2m + 1 first: in each load instruction half the warp
                // reads even and half odd source columns (all 16 eight-byte bank slots),
                // instead of every lane the same parity (rows start 16-byte aligned)
                const int ep = m & 1;
                T val[2];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const int e = k ^ ep;
                    int i0;
                    double a0;
                    split(fma(M00, (2 * m + e) - 0.5 * (N - 1), vb), i0, a0);
                    const T* r0 = stg + (i1 + 1) * SP + i0 + OFF;
                    const double w00 = (double)r0[0], w01 = (double)r0[1];
                    const double w10 = (double)r0[SP], w11 = (double)r0[SP + 1];
                    const double lo = fma(a0, w01 - w00, w00), hi = fma(a0, w11 - w10, w10);
                    val[k] = (T)fma(a1, hi - lo, lo);
                }
                z[r] = ep ? V{val[1], val[0]} : V{val[0], val[1]};
            }
        } else {
#pragma unroll
            for (int r = 0; r < R1; ++r) z[r] = *reinterpret_cast<const V*>(stg + (t + 8 * r + 1) * SP + 2 * m + OFF);
        }
        if (tid < H) tma::bulk_wait_read();                   // the previous plane's X rows are out
        __syncthreads();                                      // staged plane consumed, X free
        if (SEP) issue(p + gridDim.x);                        // overlaps the FFTs below
        if (P[PL_SKIP] != 0.0) continue;                      // uniform; the stage ring stays intact
        // ------------------------------------------------------------ P1: axis-1 FFT of the packed pair
        {
            V pa[8], pb[8];
            team_dft<R1, false>(z, pa, pb, X, tw, t, [&](int s2, int tt) { return cslot<N>(s2, tt, m); });
            if (s_on<R1>(t)) {
                const int sa = s_a<R1>(t), sb = s_b<R1>(t);
                // unpack the two real columns: Wa = (Z(k) + conj Z(-k))/2, Wb = (Z(k) - conj Z(-k))/(2i)
                auto store_pair = [&](int k1, V zk, V zp) {
                    X[k1 * PITCH + xcol(k1, 2 * m)] = V{T(0.5) * (zk.x + zp.x), T(0.5) * (zk.y - zp.y)};
                    X[k1 * PITCH + xcol(k1, 2 * m + 1)] = V{T(0.5) * (zk.y + zp.y), T(0.5) * (zp.x - zk.x)};
                };
                // k1 = sa + R1 q and sb + R1 q on every thread; only the mirror partner differs
                // on t = 0 (s = 0 and R1/2 are self-mirrored): selects, not a divergent branch
                const bool t0 = t == 0;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const V ma = t0 ? pa[(8 - q) & 7] : pb[7 - q];
                    const V mb = t0 ? pb[7 - q] : pa[7 - q];
                    store_pair(sa + R1 * q, pa[q], ma);
                    store_pair(sb + R1 * q, pb[q], mb);
                }
                if (t0) store_pair(R1 * 4, pa[4], pa[4]);
            }
        }
        __syncthreads();
        // ------------------------------------------------------------ P2: axis-0 FFT of row k1 = m
        {
            V x[R1], pa[8], pb[8];
            V* row = X + m * PITCH;
            const bool m0 = m == 0;                 // team 0 packs rows 0 and N/2 (both real in j0)
#pragma unroll
            for (int r = 0; r < R1; ++r) {
                const V A = row[xcol(m, t + 8 * r)];
                const T B = m0 ? X[(N / 2) * PITCH + t + 8 * r].x : T(0);
                x[r] = m0 ? V{A.x, B} : A;
            }
            team_dft<R1, false>(x, pa, pb, row, tw, t, [](int s2, int tt) { return rslot(s2, tt); });
            if (s_on<R1>(t)) {
                const int sa = s_a<R1>(t), sb = s_b<R1>(t);
                if (m == 0) {
                    // rows 0 and N/2 were packed as one complex row R = A + i B (both real in j0)
                    auto unpack = [&](int kk, V rk, V rm) {
                        X[kk] = V{T(0.5) * (rk.x + rm.x), T(0.5) * (rk.y - rm.y)};
                        X[(N / 2) * PITCH + kk] = V{T(0.5) * (rk.y + rm.y), T(0.5) * (rm.x - rk.x)};
                    };
                    const bool t0 = t == 0;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        unpack(sa + R1 * q, pa[q], t0 ? pa[(8 - q) & 7] : pb[7 - q]);
                        unpack(sb + R1 * q, pb[q], t0 ? pb[7 - q] : pa[7 - q]);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        row[sa + R1 * q] = pa[q];
                        row[sb + R1 * q] = pb[q];
                    }
                }
            }
        }
        __syncthreads();
        if (tid == 0) a.dcpart[p] = (double)X[0].x;           // sum of the plane's input weights
        if (tid < H) {                                        // one bulk store per spectrum row
            tma::fence_proxy_async();
            if (a.chunks == 1) {
                tma::bulk_s2g(a.S + (long long)p * (H * N) + (long long)tid * N, X + tid * PITCH,
                              (unsigned)(N * sizeof(V)));
            } else {
                // sharded: k0 range q of the row to destination rank q's block
                const int Nc = N / a.chunks;
                for (int q = 0; q < a.chunks; ++q)
                    tma::bulk_s2g(a.S + q * a.chunk_stride + ((long long)p * H + tid) * Nc, X + tid * PITCH + q * Nc,
                                  (unsigned)(Nc * sizeof(V)));
            }
            tma::bulk_commit();
        }
        if (!SEP) {
            if (tid < H) tma::bulk_wait_read();               // the staging area aliases X
            __syncthreads();
        }
    }
    if (tid < H) tma::bulk_wait_all();
}


// ============================================================================ strided pass (axes >= 2)
// Pencils along one axis of the spectrum [o][j][i] (stride I). MODE 0 forward,
// 1 inverse, 2 forward x s Psi / N_tot x inverse (last axis; Alg. 3-5). Psi per
// substep n: f_n = gam_n + bet_n kx_L + alp_n kap_L^2, (gam_n, bet_n) per pencil.
// Persistent CTAs; a tile (TP consecutive pencils x NA rows) is staged into
// shared memory by NA bulk row copies completing on the stage's mbarrier, NS
// stages deep, so the HBM reads of the next tiles overlap this tile's FFTs. Team
// p's staged column doubles as its exchange area (pitch TP + 1: conflict-free).
template <typename T>
struct MidArgs {
    typename C2<T>::type* S;      // input spectrum
    typename C2<T>::type* Sout;   // output (== S: in place)
    const double* coef;
    int cs;
    long long I, O;          // inner stride (pencils per o) and outer count
    int ocpf;                // o values per filter (MODE 2: 1)
    int N0, H1, n2, n3;      // plane sizes, axis-2/3 sizes (wavenumber decode, split regrid)
    int l;
    int step;                // 0 Euler, 1 Crank-Nicolson (R27)
    int skip4;               // MODE 0: leave filters with a split regrid map (flag 4) to k_plane_split
    double* dc3;             // k_plane_split: [filter][n3] slab sums of the regridded weights
};

// tile shape / pipeline variants: TP pencils per tile, NS stages, MINB CTAs per SM
template <int V_> struct MidVar;
template <> struct MidVar<0> { static constexpr int TP = 32, NS = 2, MINB = 2; };   // small pencils
template <> struct MidVar<1> { static constexpr int TP = 32, NS = 4, MINB = 1; };   // 96: 4-deep ring
template <> struct MidVar<3> { static constexpr int TP = 32, NS = 3, MINB = 1; };   // 128

template <typename T, int NA, int VAR>
struct MidCfg {
    static constexpr int TP = MidVar<VAR>::TP;                      // pencils (teams) per tile
    static constexpr int PP = sizeof(T) == 8 ? TP + 1 : TP + 2;     // staged row pitch (complex), 16-B rows
    static constexpr int NS = MidVar<VAR>::NS;                      // pipeline stages
    static constexpr int MINB = MidVar<VAR>::MINB;
    static constexpr int NT = 8 * TP;
};

template <typename T, int NA, int VAR>
static size_t mid_smem(int l, int sets) {
    using C = MidCfg<T, NA, VAR>;
    return sizeof(typename C2<T>::type) * ((size_t)sets * C::NS * NA * C::PP + NA) + 16 * 4 +
           sizeof(double2) * C::TP * 3 * ((l + 1) / 2) * 2;   // den (+ CN num) quartic tables
}

template <typename T, int NA, int MODE, int NX, int VAR>
__global__ void __launch_bounds__(MidCfg<T, NA, VAR>::NT, MidCfg<T, NA, VAR>::MINB) k_plane_mid(MidArgs<T> a) {
    using V = typename C2<T>::type;
    using C = MidCfg<T, NA, VAR>;
    constexpr int R1 = NA / 8, TP = C::TP, PP = C::PP, NS = C::NS;
    constexpr int L = NX - 1;                                 // this pass's axis when MODE == 2
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* stg = reinterpret_cast<V*>(smem_raw);                  // [NS][NA][PP]
    V* tw = stg + NS * NA * PP;                               // [NA]
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(tw + NA);   // [NS] (<= 4)
    double2* psi = reinterpret_cast<double2*>(bar + 4);       // [TP][l] (gam, bet)
    const int tid = threadIdx.x, p = tid >> 3, t = tid & 7;
    init_tw<NA>(tw);
    if (tid == 0)
        for (int q = 0; q < NS; ++q) tma::mbar_init(&bar[q], 1);
    __syncthreads();
    const long long tiles = (a.I + TP - 1) / TP, ntile = a.O * tiles;
    // does this pass transform the tiles of filter f? (MODE 0 / 3 split the filters by regrid kind)
    long long act_f = -1;                                     // one-filter cache (filters span many tiles)
    bool act_v = true;
    auto active = [&](long long f) -> bool {
        if (!(MODE == 0 && a.skip4)) return true;
        if (f != act_f) {
            const double* P = a.coef + f * a.cs;
            const bool split = P[PL_SKIP] == 0.0 && (int)P[PL_FLAG] == 4;   // handled by k_plane_split
            act_v = !split;
            act_f = f;
        }
        return act_v;
    };
    // tiles of inactive filters are neither staged nor waited for (their stage's phase is not used)
    auto issue = [&](long long blk, int st) {
        if (blk >= ntile || tid >= NA) return;
        const long long o = (unsigned)blk / (unsigned)tiles, i0 = ((unsigned)blk - (unsigned)o * (unsigned)tiles) * TP;
        const long long cnt = a.I - i0 < TP ? a.I - i0 : TP;
        const unsigned bytes = ((unsigned)(cnt * sizeof(V)) + 15u) & ~15u;
        const long long filt = (unsigned)o / (unsigned)a.ocpf;
        if (!active(filt)) return;
        tma::fence_proxy_async();
        if (tid == 0) tma::mbar_expect_tx(&bar[st], bytes * NA);
        tma::bulk_g2s(stg + (st * NA + tid) * PP, a.S + (o * NA + tid) * a.I + i0, bytes, &bar[st]);
    };
    if (MODE == 0 && a.skip4 && a.O / a.ocpf <= 64) {         // every filter left to the split pass: done
        bool any = false;
        for (long long f = 0; f < a.O / a.ocpf && !any; ++f) any = active(f);
        if (!any) return;
    }
#pragma unroll
    for (int j = 0; j < NS - 1; ++j) issue(blockIdx.x + (long long)j * gridDim.x, j);
    auto slot = [](int s2, int tt) { return rslot(s2, tt) * PP; };
    int k = 0;
    unsigned phase = 0;                                       // bit q: parity of stage q's next wait
    for (long long blk = blockIdx.x; blk < ntile; blk += gridDim.x, ++k) {
        const int st = k % NS;
        issue(blk + (long long)(NS - 1) * gridDim.x, (k + NS - 1) % NS);
        const long long o = (unsigned)blk / (unsigned)tiles;   // 32-bit: ntile < 2^31
        const long long i = ((unsigned)blk - (unsigned)o * (unsigned)tiles) * TP + p;
        const bool valid = i < a.I;
        const long long filt = (unsigned)o / (unsigned)a.ocpf;
        if (!active(filt)) continue;                          // uniform; nothing was staged
        tma::mbar_wait(&bar[st], (phase >> st) & 1u);
        phase ^= 1u << st;
        V* base = a.Sout + o * (long long)NA * a.I + (valid ? i : 0);
        V* col = stg + st * NA * PP + p;
        V x[R1], pa[8], pb[8];
#pragma unroll
        for (int r = 0; r < R1; ++r) x[r] = col[(t + 8 * r) * PP];
        team_dft<R1, MODE == 1>(x, pa, pb, col, tw, t, slot);
        if (MODE != 2) {
            if (valid && s_on<R1>(t)) {
                const int sa = s_a<R1>(t), sb = s_b<R1>(t);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    __stcg(base + (long long)(sa + R1 * q) * a.I, pa[q]);
                    __stcg(base + (long long)(sb + R1 * q) * a.I, pb[q]);
                }
            }
        } else {
            // ------------------------------------------------------------ s Psi / N_tot (Alg. 3-4)
            // Euler factors f_n(kap) = gam_n + bet_n kx + alp_n kap^2 (kx = kap but 0 at the Nyquist
            // wavenumber, R7), multiplied in pairs: f_n f_{n+1} is a quartic in kap (Horner, 4 FMA)
            // whose per-pencil coefficients the team tabulates first. Every factor is >= 1 (D_n is
            // PSD), so the quartic evaluation is well conditioned.
            const double* P = a.coef + filt * a.cs;
            const double* cf = P + PL_EU;
            // Euler: den factors f_n, n < l. Crank-Nicolson (R27): den f_n, n = 1..l, and num
            // (2 - f_n), n < l -- each list paired into quartics
            const int nq = (a.l + 1) >> 1, cn = a.step;
            double2* qt = psi + p * 3 * nq * (1 + cn);         // [1+cn][nq][3]: (c0,c1) (c2,c3) (c4,nyq)
            {
                // wavenumbers of the pencil's other axes: inner i = (j2 *) H1 N0 + k1 N0 + k0
                double kap[3] = {0, 0, 0}, kx[3] = {0, 0, 0};
                const long long ii = valid ? i : 0;
                const unsigned r1 = (unsigned)ii / (unsigned)a.N0;      // I < 2^31
                const int k0 = (int)((unsigned)ii - r1 * (unsigned)a.N0);
                const unsigned r2 = r1 / (unsigned)a.H1;
                const int k1 = (int)(r1 - r2 * (unsigned)a.H1);
                const int k2 = (int)r2;
                const int N1 = 2 * (a.H1 - 1);
                const int ks0 = k0 < a.N0 / 2 ? k0 : k0 - a.N0;
                kap[0] = (2.0 * PMF_PI / a.N0) * ks0;
                kx[0] = (2 * k0 == a.N0) ? 0.0 : kap[0];
                kap[1] = (2.0 * PMF_PI / N1) * k1;              // k1 in [0, N1/2]: the half axis
                kx[1] = (2 * k1 == N1) ? 0.0 : kap[1];
                if (L == 3) {
                    const int ks2 = k2 < a.n2 / 2 ? k2 : k2 - a.n2;
                    kap[2] = (2.0 * PMF_PI / a.n2) * ks2;
                    kx[2] = (2 * k2 == a.n2) ? 0.0 : kap[2];
                }
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
                for (int jj = t; jj < nq * (1 + cn); jj += 8) {
                    const int list = jj / nq, j = jj - list * nq;       // list 0: den, 1: num
                    const int base = (list == 0 && cn) ? 1 : 0;       // CN den: f_1 .. f_l
                    double g0, b0, g1 = 1.0, b1 = 0.0, a1 = 0.0;
                    gam_bet(base + 2 * j, g0, b0);
                    double a0 = cf[10 * (base + 2 * j) + L];
                    const bool two = 2 * j + 1 < a.l;
                    if (two) {
                        gam_bet(base + 2 * j + 1, g1, b1);
                        a1 = cf[10 * (base + 2 * j + 1) + L];
                    }
                    if (list == 1) {                                  // 2 - f = (2 - g) - b k - a k^2
                        g0 = 2.0 - g0;
                        b0 = -b0;
                        a0 = -a0;
                        if (two) {
                            g1 = 2.0 - g1;
                            b1 = -b1;
                            a1 = -a1;
                        }
                    }
                    // the Nyquist wavenumber has kx = 0 in the first-order terms (R7): its pair value
                    constexpr double kn2 = PMF_PI * PMF_PI;
                    double2* q = qt + 3 * jj;
                    q[0] = double2{g0 * g1, fma(g0, b1, b0 * g1)};
                    q[1] = double2{fma(g0, a1, fma(b0, b1, a0 * g1)), fma(b0, a1, a0 * b1)};
                    q[2] = double2{a0 * a1, fma(a0, kn2, g0) * fma(a1, kn2, g1)};
                }
            }
            __syncwarp();
            {
                // Psi at k = t + 8r on all 8 threads of the team, then to the owners via the
                // (now free) staged column
                double kp[R1], den[R1];
#pragma unroll
                for (int r = 0; r < R1; ++r) {
                    const int k = t + 8 * r;
                    kp[r] = (2.0 * PMF_PI / NA) * (k < NA / 2 ? k : k - NA);
                    den[r] = 1.0;
                }
                auto prodq = [&](const double2* tb, double* acc) {
                    for (int j = 0; j < nq; ++j) {
                        const double2 q01 = tb[3 * j], q23 = tb[3 * j + 1], q4 = tb[3 * j + 2];
#pragma unroll
                        for (int r = 0; r < R1; ++r) {
                            const double x1 = kp[r];
                            acc[r] *= fma(fma(fma(fma(q4.x, x1, q23.y), x1, q23.x), x1, q01.y), x1, q01.x);
                        }
                    }
                    if (t == ((NA / 2) & 7)) {
                        constexpr int rn = (NA / 2) >> 3;
                        double d = 1.0;
                        for (int j = 0; j < nq; ++j) d *= tb[3 * j + 2].y;
                        acc[rn] = d;
                    }
                };
                prodq(qt, den);
                double numr[R1];
#pragma unroll
                for (int r = 0; r < R1; ++r) numr[r] = 1.0;
                if (cn) prodq(qt + 3 * nq, numr);
                const double mult = P[PL_SN];
                double ps[R1];
                psi_div<R1>(den, mult, ps);
#pragma unroll
                for (int r = 0; r < R1; ++r) reinterpret_cast<double*>(col + (t + 8 * r) * PP)[0] = ps[r] * numr[r];
            }
            __syncwarp();
            if (s_on<R1>(t)) {
                const int sa = s_a<R1>(t), sb = s_b<R1>(t);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const double fa = reinterpret_cast<const double*>(col + (sa + R1 * q) * PP)[0];
                    const double fb = reinterpret_cast<const double*>(col + (sb + R1 * q) * PP)[0];
                    pa[q] = V{(T)(pa[q].x * fa), (T)(pa[q].y * fa)};
                    pb[q] = V{(T)(pb[q].x * fb), (T)(pb[q].y * fb)};
                }
            }
            team_dft_dif<R1, true>(pa, pb, x, col, tw, t, slot);
            if (valid) {
#pragma unroll
                for (int r = 0; r < R1; ++r) __stcg(base + (long long)(t + 8 * r) * a.I, x[r]);
            }
        }
        __syncthreads();                  // stage st is consumed: it is refilled next iteration
    }
}

// ============================================================================ split regrid, axes 3 -> 2 (nx = 4)
// For filters with a split regrid map (flag 4): Y(k0, k1, u2', u3') = linear interpolation
// along axis 2 (v2 = o2 + M22 u2' + M23 u3') of Z(j2) = (1 - w3) S(j2, j3) + w3 S(j2, j3 + 1)
// (v3 = o3 + M33 u3'), zero ghosts (R12), then the forward DFT along axis 2, into S2.
// Each CTA owns TP pencils (k0, k1) of one filter and walks u3' = 0..n3-1; the old slabs
// j3 stream once through a ring of RS staged row sets (v3 is monotone in u3').
template <typename T, int NA>
struct SplitCfg {
    static constexpr int TP = NA >= 96 ? 16 : 32;
    static constexpr int PP = sizeof(T) == 8 ? TP + 1 : TP + 2;
    static constexpr int RS = 3;
    static constexpr int NT = 8 * TP;
};
template <typename T, int NA>
static size_t split_smem() {
    using C = SplitCfg<T, NA>;
    return sizeof(typename C2<T>::type) * ((size_t)(C::RS + 1) * NA * C::PP + NA) + 8 * C::RS + 16;
}

template <typename T, int NA>
__global__ void __launch_bounds__(SplitCfg<T, NA>::NT, 1) k_plane_split(MidArgs<T> a) {
    using V = typename C2<T>::type;
    using C = SplitCfg<T, NA>;
    constexpr int R1 = NA / 8, TP = C::TP, PP = C::PP, RS = C::RS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* ring = reinterpret_cast<V*>(smem_raw);                 // [RS][NA][PP]
    V* scr = ring + RS * NA * PP;                             // [NA][PP] blended Z, then the exchange
    V* tw = scr + NA * PP;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(tw + NA);
    const int tid = threadIdx.x, p = tid >> 3, t = tid & 7;
    const long long tiles = (a.I + TP - 1) / TP;
    const long long filt = blockIdx.x / (unsigned)tiles, i0 = (blockIdx.x - (unsigned)filt * (unsigned)tiles) * TP;
    const double* P = a.coef + filt * a.cs;
    if (P[PL_SKIP] != 0.0 || (int)P[PL_FLAG] != 4) return;   // uniform
    init_tw<NA>(tw);
    if (tid == 0)
        for (int q = 0; q < RS; ++q) tma::mbar_init(&bar[q], 1);
    __syncthreads();
    const long long i = i0 + p;
    const bool valid = i < a.I;
    const long long cnt = a.I - i0 < TP ? a.I - i0 : TP;
    const unsigned bytes = ((unsigned)(cnt * sizeof(V)) + 15u) & ~15u;
    const int n3 = a.n3;
    const double M33 = P[PL_M + 15], o3 = P[PL_O + 3], M22 = P[PL_M + 10], M23 = P[PL_M + 11], o2 = P[PL_O + 2];
    auto row_of = [&](int u3) {                               // first old slab of output slab u3
        const double v3 = fma(M33, (double)u3 - 0.5 * (n3 - 1), o3);
        const double f = floor(v3);
        const int fi = __double2int_rz(f);
        return min(max(fi, -2), n3);
    };
    // rows r0, r0+1, ... are loaded in order into slot (r - r0) % RS, none skipped
    const int r0 = max(row_of(0), 0);
    int next = r0;
    auto issue = [&](int r) {
        if (tid >= NA) return;
        const int sl = (r - r0) % RS;
        tma::fence_proxy_async();
        if (tid == 0) tma::mbar_expect_tx(&bar[sl], bytes * NA);
        tma::bulk_g2s(ring + (sl * NA + tid) * PP, a.S + ((filt * n3 + r) * (long long)NA + tid) * a.I + i0, bytes,
                      &bar[sl]);
    };
    auto slab = [&](int r) -> const V* { return ring + ((r - r0) % RS) * NA * PP + p; };
    auto wait_row = [&](int r) { tma::mbar_wait(&bar[(r - r0) % RS], (unsigned)(((r - r0) / RS) & 1)); };
    V* col = scr + p;
    auto slot = [](int s2, int tt) { return rslot(s2, tt) * PP; };
    for (int u3 = 0; u3 < n3; ++u3) {
        const int ja = row_of(u3);
        const double v3 = fma(M33, (double)u3 - 0.5 * (n3 - 1), o3);
        const double w3 = (ja == __double2int_rz(floor(v3))) ? v3 - floor(v3) : 0.0;
        // rows below ja are never needed again: their slots take the rows ahead
        const int lim = min(max(ja, r0) + RS, n3);
        while (next < lim) issue(next++);
        const bool va = ja >= 0 && ja < n3, vb = ja + 1 >= 0 && ja + 1 < n3;
        if (va) wait_row(ja);
        if (vb) wait_row(ja + 1);
#pragma unroll
        for (int r = 0; r < R1; ++r) {
            const int j2 = t + 8 * r;
            double zx = 0.0, zy = 0.0;
            if (va) {
                const V v = slab(ja)[j2 * PP];
                zx = (1.0 - w3) * (double)v.x;
                zy = (1.0 - w3) * (double)v.y;
            }
            if (vb) {
                const V v = slab(ja + 1)[j2 * PP];
                zx = fma(w3, (double)v.x, zx);
                zy = fma(w3, (double)v.y, zy);
            }
            col[j2 * PP] = V{(T)zx, (T)zy};
        }
        __syncwarp();
        const double vb2 = fma(M23, (double)u3 - 0.5 * (n3 - 1), o2);
        V x[R1], pa[8], pb[8];
        double dcs = 0.0;
#pragma unroll
        for (int r = 0; r < R1; ++r) {
            const double v2 = fma(M22, (t + 8 * r) - 0.5 * (NA - 1), vb2);
            const double f = floor(v2);
            const int fi = __double2int_rz(f);
            const double fr = v2 - f;
            const V lo = (fi >= 0 && fi < NA) ? col[fi * PP] : V{T(0), T(0)};
            const V hi = (fi + 1 >= 0 && fi + 1 < NA) ? col[(fi + 1) * PP] : V{T(0), T(0)};
            x[r] = V{(T)fma(fr, (double)hi.x - (double)lo.x, (double)lo.x),
                     (T)fma(fr, (double)hi.y - (double)lo.y, (double)lo.y)};
            dcs += (double)x[r].x;
        }
        if (i == 0) {      // pencil k0 = k1 = 0: sum of this slab's regridded weights
            const unsigned tm = 0xFFu << ((tid & 31) & ~7);
            dcs += __shfl_xor_sync(tm, dcs, 1);
            dcs += __shfl_xor_sync(tm, dcs, 2);
            dcs += __shfl_xor_sync(tm, dcs, 4);
            if (t == 0) a.dc3[filt * n3 + u3] = dcs;
        }
        team_dft<R1, false>(x, pa, pb, col, tw, t, slot);
        if (valid && s_on<R1>(t)) {
            V* base = a.Sout + (filt * n3 + u3) * (long long)NA * a.I + i;
            const int sa = s_a<R1>(t), sb = s_b<R1>(t);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                __stcg(base + (long long)(sa + R1 * q) * a.I, pa[q]);
                __stcg(base + (long long)(sb + R1 * q) * a.I, pb[q]);
            }
        }
        __syncthreads();                  // ring slots below the next ja may be refilled
    }
}

// ============================================================================ inverse plane pass (+ update)
template <typename T, int N>
__host__ __device__ constexpr bool inv_dbl() { return 2 * xbytes<T, N>() <= 200 * 1024; }
template <typename T, int N>
static size_t inv_smem() {
    return (inv_dbl<T, N>() ? 2 : 1) * xbytes<T, N>() + 2 * sizeof(T) * N +
           sizeof(double) * NMOM * (Cfg<N>::NT / 32) + 16 + sizeof(double) * NMOM * Cfg<N>::NT;
}

// The plane's spectrum rows are staged by H bulk copies; with two buffers (N <= 96)
// the next plane's copy overlaps this plane's transforms and likelihood.
template <typename T, int N, int NX, bool UP>
__global__ void __launch_bounds__(Cfg<N>::NT, Cfg<N>::MINB) k_plane_inv(PlaneArgs<T> a) {
    using V = typename C2<T>::type;
    using C = Cfg<N>;
    constexpr int R1 = C::R1, H = C::H, PITCH = C::PITCH, NT = C::NT, NW = NT / 32;
    constexpr bool DBL = inv_dbl<T, N>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* X0 = reinterpret_cast<V*>(smem_raw);
    V* tw = X0 + (DBL ? 2 : 1) * H * PITCH;
    double* red = reinterpret_cast<double*>(tw + N);          // [NW][NMOM]
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(red + NMOM * NW);
    const int tid = threadIdx.x, m = tid >> 3, t = tid & 7, lane = tid & 31, warp = tid >> 5;
    init_tw<N>(tw);
    if (tid == 0) {
        tma::mbar_init(&bar[0], 1);
        tma::mbar_init(&bar[1], 1);
    }
    const long long ntot = (long long)N * N * a.n2 * a.n3;
    __syncthreads();
    constexpr int NM = 1 + NX + NX * (NX + 1) / 2;           // moment sums of a filter
    double* mom = reinterpret_cast<double*>(bar + 2) + tid;  // this thread's sums, stride NT (shared)
#pragma unroll
    for (int q = 0; q < NM; ++q) mom[q * NT] = 0.0;
    int curf = -1;
    // one CTA reduction per (filter, CTA): fixed order (warp tree, then warps in order)
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
    auto issue = [&](int p, int buf) {
        if (p >= a.nplanes || tid >= H) return;
        tma::fence_proxy_async();
        if (tid == 0) tma::mbar_expect_tx(&bar[buf], (unsigned)(H * N * sizeof(V)));
        tma::bulk_g2s(X0 + (buf * H + tid) * PITCH, a.Sinv + (long long)p * (H * N) + (long long)tid * N,
                      (unsigned)(N * sizeof(V)), &bar[buf]);
    };
    issue(blockIdx.x, 0);
    int k = 0;
    for (int p = blockIdx.x; p < a.nplanes; p += gridDim.x, ++k) {
        const int buf = DBL ? (k & 1) : 0;
        if (DBL) issue(p + gridDim.x, buf ^ 1);
        else if (k > 0) issue(p, 0);
        tma::mbar_wait(&bar[buf], (unsigned)(DBL ? ((k >> 1) & 1) : (k & 1)));
        V* X = X0 + buf * H * PITCH;
        const int filt = p / a.ppf, pl = p - filt * a.ppf;
        if (UP && filt != curf) {                             // uniform
            flush();
            curf = filt;
        }
        const double* P = a.coef + (long long)filt * a.cs;
        if (P[PL_SKIP] != 0.0) {
            __syncthreads();
            continue;
        }
        // ------------------------------------------------------------ P2: inverse axis 0 of row k1 = m
        {
            V x[R1], pa[8], pb[8];
            V* row = X + m * PITCH;
            // rows 0 and N/2 are Hermitian in k0: team 0 packs R = A + i B (its inverse is
            // a + i b); every other team has B = 0. One instruction stream for all teams
            // (no divergent branch in warp 0); rows 0 and N/2 are unswizzled (xcol = id).
            const bool m0 = m == 0;
#pragma unroll
            for (int r = 0; r < R1; ++r) {
                const V A = row[t + 8 * r];
                const V B = m0 ? X[(N / 2) * PITCH + t + 8 * r] : V{T(0), T(0)};
                x[r] = V{A.x - B.y, A.y + B.x};
            }
            team_dft<R1, true>(x, pa, pb, row, tw, t, [](int s, int tt) { return rslot(s, tt); });
            if (s_on<R1>(t)) {
                const int sa = s_a<R1>(t), sb = s_b<R1>(t);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    row[xcol(m, sa + R1 * q)] = m0 ? V{pa[q].x, T(0)} : pa[q];
                    row[xcol(m, sb + R1 * q)] = m0 ? V{pb[q].x, T(0)} : pb[q];
                    if (m0) {
                        X[(N / 2) * PITCH + sa + R1 * q] = V{pa[q].y, T(0)};
                        X[(N / 2) * PITCH + sb + R1 * q] = V{pb[q].y, T(0)};
                    }
                }
            }
        }
        __syncthreads();
        // ------------------------------------------------------------ P3: inverse axis 1 of the column pair
        V x[R1];
        {
            V pa[8], pb[8];
            auto ld = [&](int k1, int col) -> V { return X[k1 * PITCH + xcol(k1, 2 * m + col)]; };
            auto zdir = [&](int k1) -> V {
                const V wa = ld(k1, 0), wb = ld(k1, 1);
                return V{wa.x - wb.y, wa.y + wb.x};
            };
            auto zmir = [&](int kp) -> V {      // Z(N - kp) = conj Wa(kp) + i conj Wb(kp)
                const V wa = ld(kp, 0), wb = ld(kp, 1);
                return V{wa.x + wb.y, wb.x - wa.y};
            };
            if (s_on<R1>(t)) {
                // one index formula for every thread: the mirrored halves start at R1 - t
                // (t = 0: k1 = N/2 for q = 4, where zmir = zdir since that row is real) and
                // at t, or R1/2 on t = 0
                const int sa = s_a<R1>(t), sb = s_b<R1>(t), ma = R1 - t, mb = (t == 0) ? R1 / 2 : t;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    pa[q] = (q < 4) ? zdir(sa + R1 * q) : zmir(ma + R1 * (7 - q));
                    pb[q] = (q < 4) ? zdir(sb + R1 * q) : zmir(mb + R1 * (7 - q));
                }
            }
            team_dft_dif<R1, true>(pa, pb, x, X, tw, t, [&](int s, int tt) { return cslot<N>(s, tt, m); });
        }
        // x[r] = w(2m, t + 8r) + i w(2m+1, t + 8r), unnormalised
        int j2, j3;
        plane_j(pl, a.n2, j2, j3);
        T* Wp = a.W + filt * ntot + (long long)pl * N * N;
        if (!UP) {
#pragma unroll
            for (int r = 0; r < R1; ++r) *reinterpret_cast<V*>(Wp + (long long)(t + 8 * r) * N + 2 * m) = x[r];
            __syncthreads();
            continue;
        }
        const double u2 = j2 - 0.5 * (a.n2 - 1), u3 = (NX == 4) ? j3 - 0.5 * (a.n3 - 1) : 0.0;
        const double u10 = t - 0.5 * (N - 1);
        const double lgn = P[PL_LGN];
        double S[2] = {0, 0}, Tm[2] = {0, 0}, U[2] = {0, 0};
        auto emit = [&](int r, int e, double w) -> T {
            const T wt = (T)w;
            const double u1 = fma(8.0, (double)r, u10);
            const double wd = (double)wt, wu = wd * u1;
            S[e] += wd;
            Tm[e] += wu;
            U[e] = fma(wu, u1, U[e]);
            return wt;
        };
        bool rec = !a.range;
        double Lr[2], Rr[2], Gr[2];
        if (!a.range) {
            // linear Gauss: along a column the exponent is quadratic in r (u1 = u10 + 8 r):
            // E(r) = E0 + E1 r + E2 r^2, L(r+1) = L(r) R(r), R(r+1) = R(r) exp(2 E2)
            const double* q = P + PL_LQ;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const double u0 = (2 * m + e) - 0.5 * (N - 1);
                const double c2 = q[5 + tri(1, 1)];
                double c1 = fma(q[5 + tri(0, 1)], u0, q[2]);
                double c0 = fma(u0, fma(q[5 + tri(0, 0)], u0, q[1]), q[0]);
                c1 = fma(q[5 + tri(1, 2)], u2, c1);
                c0 = fma(u2, fma(q[5 + tri(2, 2)], u2, fma(q[5 + tri(0, 2)], u0, q[3])), c0);
                if (NX == 4) {
                    c1 = fma(q[5 + tri(1, 3)], u3, c1);
                    c0 = fma(u3, fma(q[5 + tri(3, 3)], u3,
                                     fma(q[5 + tri(2, 3)], u2, fma(q[5 + tri(0, 3)], u0, q[4]))), c0);
                }
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
                const T o0 = emit(r, 0, (double)x[r].x * Lr[0]);
                const T o1 = emit(r, 1, (double)x[r].y * Lr[1]);
                Lr[0] *= Rr[0];
                Rr[0] *= Gr[0];
                Lr[1] *= Rr[1];
                Rr[1] *= Gr[1];
                *reinterpret_cast<V*>(Wp + (long long)(t + 8 * r) * N + 2 * m) = V{o0, o1};
            }
        } else if (a.range) {
            // range likelihood: along the column the moved point is linear in r,
            // y(r) = y0 + r (8 B[:,1]); coefficients held in registers (the stores to W may
            // alias P, so per-point reads of P would be reloaded)
            const double zr = P[PL_ZR], isg = P[PL_ISG];
            double y0[2][NX], dy[NX];
#pragma unroll
            for (int a2 = 0; a2 < NX; ++a2) {
                const double b0 = P[PL_BL + a2 * 4], b1 = P[PL_BL + a2 * 4 + 1], b2 = P[PL_BL + a2 * 4 + 2];
                double yc = fma(b1, u10, P[PL_CL + a2]);
                yc = fma(b2, u2, yc);
                if (NX == 4) yc = fma(P[PL_BL + a2 * 4 + 3], u3, yc);
                dy[a2] = 8.0 * b1;
#pragma unroll
                for (int e = 0; e < 2; ++e) y0[e][a2] = fma(b0, (2 * m + e) - 0.5 * (N - 1), yc);
            }
#pragma unroll
            for (int r = 0; r < R1; ++r) {
                T o[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    double r2 = 0.0;
#pragma unroll
                    for (int a2 = 0; a2 < NX; ++a2) {
                        const double y = fma((double)r, dy[a2], y0[e][a2]);
                        r2 = fma(y, y, r2);
                    }
                    const double dd = (zr - sqrt(r2)) * isg;
                    const double w = (double)(e == 0 ? x[r].x : x[r].y);
                    o[e] = emit(r, e, w * exp_fast(fma(-0.5 * dd, dd, lgn)));
                }
                *reinterpret_cast<V*>(Wp + (long long)(t + 8 * r) * N + 2 * m) = V{o[0], o[1]};
            }
        } else {
            const double* q = P + PL_LQ;
#pragma unroll
            for (int r = 0; r < R1; ++r) {
                const double u1 = fma(8.0, (double)r, u10);
                const double uu[4] = {0.0, u1, u2, u3};
                T o[2];
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
                    const double w = (double)(e == 0 ? x[r].x : x[r].y);
                    o[e] = emit(r, e, w * exp_fast(ll));
                }
                *reinterpret_cast<V*>(Wp + (long long)(t + 8 * r) * N + 2 * m) = V{o[0], o[1]};
            }
        }
        {
            // this thread's two columns of the plane -> the filter's index-space moment sums
            // (R14): u0 fixed per column, u1 = t + 8r - (N-1)/2, u2, u3 fixed per plane
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
        __syncthreads();                  // X is consumed
    }
    if (UP) flush();
    (void)lane;
    (void)warp;
}

// ============================================================================ finalise (one block per filter)
template <int NX>
__global__ void k_plane_fin(FilterState* st, const double* __restrict__ coef, int cs, const double* __restrict__ dcpart,
                            const double* __restrict__ dc3, const double* __restrict__ part, int ppf, int n3,
                            int ginv, int update) {
    __shared__ double red[32 * 16];
    const int filt = blockIdx.x;
    const double* P = coef + (long long)filt * cs;
    if (P[PL_SKIP] != 0.0) return;
    const bool split = (int)P[PL_FLAG] == 4;     // the regridded sums come from the split pass (per slab)
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
    for (int pl = threadIdx.x; pl < ppf; pl += blockDim.x) {
        if (!split) acc[15] += dcpart[(long long)filt * ppf + pl];
        else if (pl < n3) acc[15] += dc3[(long long)filt * n3 + pl];
    }
    if (update)
        for (int c = threadIdx.x; c < ginv; c += blockDim.x) {
            const double* pp = part + ((long long)filt * ginv + c) * NMOM;
#pragma unroll
            for (int i = 0; i < NMOM; ++i) acc[i] += pp[i];
        }
    block_sum<16>(acc, red);
    if (threadIdx.x != 0) return;
    FilterState& f = st[filt];
    const double s = P[PL_S], vol = P[PL_VOL], dc = acc[15];
    if (!update) {
        f.scale = 1.0 / (vol * s * dc);
        return;
    }
    // stored weights: unnormalised prior (sum = s DC) times the likelihood
    const double C = acc[0] / (s * dc);
    f.mass = acc[0];
    f.has_moments = 1;
    if (!(C > 0.0) || !isfinite(C) || !(acc[0] > 0.0)) {
        f.status = -6;
        f.logC = -INFINITY;
        return;
    }
    f.status = 0;
    f.logC = log(C);
    f.scale = 1.0 / (vol * acc[0]);
    finish_moments(NX, acc, f.c, f.B, f.mean, f.cov);
}

}  // namespace pln

using namespace pln;

bool plane_supported(const Dims& d, int l) {
    if (d.nx < 3 || d.n[0] != d.n[1] || l + 1 > LCAP) return false;
    const int N = d.n[0];
    if (N != 32 && N != 64 && N != 96 && N != 128) return false;
    for (int m = 2; m < d.nx; ++m) {
        const int n = d.n[m];
        if (n != 16 && n != 32 && n != 64 && n != 96 && n != 128) return false;
    }
    return d.nx <= 4;
}

template <typename K>
static cudaError_t occ_grid(K kern, int nt, size_t smem, long long work, int* grid) {
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

template <typename T, int NA, int NX, int VAR, int MODE>
static cudaError_t mid_launch(MidArgs<T> ma, cudaStream_t s) {
    using C = MidCfg<T, NA, VAR>;
    const size_t smem = mid_smem<T, NA, VAR>(MODE == 2 ? ma.l : 0, 1);
    const long long work = ma.O * ((ma.I + C::TP - 1) / C::TP);
    int grid = 1;
    cudaError_t e = occ_grid(k_plane_mid<T, NA, MODE, NX, VAR>, C::NT, smem, work, &grid);
    if (e != cudaSuccess) return e;
    k_plane_mid<T, NA, MODE, NX, VAR><<<grid, C::NT, smem, s>>>(ma);
    return cudaGetLastError();
}

template <typename T, int NA, int NX, int VAR>
static cudaError_t mid_var(MidArgs<T> ma, int mode, cudaStream_t s) {
    switch (mode) {
        case 0: return mid_launch<T, NA, NX, VAR, 0>(ma, s);
        case 1: return mid_launch<T, NA, NX, VAR, 1>(ma, s);
        default: return mid_launch<T, NA, NX, VAR, 2>(ma, s);
    }
}

// measured on B200 (C4 96^4): a 4-deep ring at one CTA per SM beats 2 x (2-deep) by 20 %
template <typename T, int NA, int NX>
static cudaError_t mid_na(MidArgs<T> ma, int mode, cudaStream_t s) {
    if (NA == 96) return mid_var<T, NA, NX, 1>(ma, mode, s);
    if (NA == 128) return mid_var<T, NA, NX, 3>(ma, mode, s);
    return mid_var<T, NA, NX, 0>(ma, mode, s);
}

template <typename T, int NX>
static cudaError_t mid_pass(MidArgs<T> ma, int na, int mode, cudaStream_t s) {
    switch (na) {
        case 16: return mid_na<T, 16, NX>(ma, mode, s);
        case 32: return mid_na<T, 32, NX>(ma, mode, s);
        case 64: return mid_na<T, 64, NX>(ma, mode, s);
        case 96: return mid_na<T, 96, NX>(ma, mode, s);
        case 128: return mid_na<T, 128, NX>(ma, mode, s);
        default: return cudaErrorInvalidValue;
    }
}

template <typename T, int NA>
static cudaError_t split_na(MidArgs<T> ma, long long nblk, cudaStream_t s) {
    const size_t smem = split_smem<T, NA>();
    cudaError_t e = cudaFuncSetAttribute(k_plane_split<T, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_plane_split<T, NA><<<(unsigned)nblk, SplitCfg<T, NA>::NT, smem, s>>>(ma);
    return cudaGetLastError();
}

template <typename T>
static cudaError_t split_pass(const Dims& d, PencilBufs& b, int cs, typename C2<T>::type* S,
                              typename C2<T>::type* S2, double* dc3, int l, cudaStream_t s, int64_t* launches) {
    MidArgs<T> ma{};
    ma.S = S;
    ma.Sout = S2;
    ma.coef = b.coef;
    ma.cs = cs;
    ma.I = (long long)(d.n[1] / 2 + 1) * d.n[0];
    ma.n2 = d.n[2];
    ma.n3 = d.n[3];
    ma.l = l;
    ma.dc3 = dc3;
    ++*launches;
    auto nblk = [&](int tp) { return ((ma.I + tp - 1) / tp) * d.batch; };
    switch (d.n[2]) {
        case 16: return split_na<T, 16>(ma, nblk(SplitCfg<T, 16>::TP), s);
        case 32: return split_na<T, 32>(ma, nblk(SplitCfg<T, 32>::TP), s);
        case 64: return split_na<T, 64>(ma, nblk(SplitCfg<T, 64>::TP), s);
        case 96: return split_na<T, 96>(ma, nblk(SplitCfg<T, 96>::TP), s);
        case 128: return split_na<T, 128>(ma, nblk(SplitCfg<T, 128>::TP), s);
        default: return cudaErrorInvalidValue;
    }
}

template <typename T, int N, int NX>
static cudaError_t plane_t(const Dims& d, PencilBufs& b, const ModelParams& mp, const LikParams* lp, double ks,
                           cudaStream_t s, int64_t* launches) {
    using V = typename C2<T>::type;
    using Cf = Cfg<N>;
    const int cs = coef_stride(mp.l);
    LikParams lpv = lp ? *lp : LikParams{};
    k_plane_prep<NX><<<d.batch, 32, 0, s>>>(b.st, b.coef, cs, mp, b.sub, lpv, b.z, ks, lp ? 1 : 0, d);
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int n2 = d.n[2], n3 = NX == 4 ? d.n[3] : 1;
    const int ppf = n2 * n3;
    const bool rg = ks > 0.0;
    V* S = (V*)b.S;
    V* S2 = NX == 4 ? (V*)b.S2 : S;              // nx = 4: the first strided pass runs out of place
    PlaneArgs<T> pa;
    pa.Wsrc = (const T*)b.W;
    pa.W2src = (const T*)b.W2;
    pa.W = (T*)b.W;
    pa.S = S;
    pa.Sinv = S2;
    pa.coef = b.coef;
    pa.cs = cs;
    pa.ppf = ppf;
    pa.nplanes = ppf * d.batch;
    pa.dcpart = b.partials;                                   // [nplanes]
    pa.dc3 = b.partials + pa.nplanes;                         // [batch][n3]
    pa.part = pa.dc3 + (long long)d.batch * n3;               // [batch][inverse CTAs][NMOM]
    pa.n2 = n2;
    pa.n3 = n3;
    pa.l = mp.l;
    pa.range = lpv.kind == 1;
    // general regrid maps: gather pre-pass into W2 (exits at once for the other filters)
    if (rg) {
        const long long rows = d.ntot / d.n[0];                   // one warp per axis-0 row
        const int bpf = (int)std::max(1LL, std::min(2048LL, (rows + 7) / 8));
        k_plane_pre<T, NX><<<(unsigned)(bpf * d.batch), 256, 0, s>>>((const T*)b.W, (T*)b.W2, b.coef, cs, d, bpf);
        ++*launches;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    // nx = 4, fp64: the three-pass transposed-spectrum route (kernels_quad.cu)
    const bool quad = NX == 4 && std::is_same<T, double>::value && N <= 96 && quad_supported(d, 0);
    // forward plane pass (K1 of both routes: the per-plane half spectrum S[f][j3][j2][k1][k0])
    {
        const size_t smem = fwd_smem<T, N>();
        int grid = 1;
        if (rg) {
            e = occ_grid(k_plane_fwd<T, N, NX, true>, Cf::NT, smem, pa.nplanes, &grid);
            if (e == cudaSuccess) k_plane_fwd<T, N, NX, true><<<grid, Cf::NT, smem, s>>>(pa);
        } else {
            e = occ_grid(k_plane_fwd<T, N, NX, false>, Cf::NT, smem, pa.nplanes, &grid);
            if (e == cudaSuccess) k_plane_fwd<T, N, NX, false><<<grid, Cf::NT, smem, s>>>(pa);
        }
        if (e != cudaSuccess) return e;
        ++*launches;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (quad) {
        // nx = 4, fp64: K2 (gathers (j3, j2)-planes from S, writes S2 in the transposed layout)
        // and K3 (kernels_quad.cu) replace the three strided passes and the inverse plane pass
        int ginv = 1;
        e = launch_quad(d, b, mp, pa.range, lp != nullptr, pa.dcpart, pa.dc3, pa.part, s, launches, &ginv);
        if (e != cudaSuccess) return e;
        k_plane_fin<NX><<<d.batch, 256, 0, s>>>(b.st, b.coef, cs, pa.dcpart, pa.dc3, pa.part, ppf, n3, ginv,
                                                lp ? 1 : 0);
        ++*launches;
        return cudaGetLastError();
    }
    // strided axes: forward 2..nx-2 (the first out of place, + the split regrid's (2,3) part),
    // the last axis with Psi, inverse nx-2..2
    auto mid = [&](int m, int mode, V* in, V* out, int skip4) -> cudaError_t {
        MidArgs<T> ma;
        ma.S = in;
        ma.Sout = out;
        ma.coef = b.coef;
        ma.cs = cs;
        ma.I = (long long)Cf::H * N;
        for (int q = 2; q < m; ++q) ma.I *= d.n[q];
        ma.O = d.batch;
        ma.ocpf = 1;
        for (int q = m + 1; q < NX; ++q) {
            ma.O *= d.n[q];
            ma.ocpf *= d.n[q];
        }
        ma.N0 = N;
        ma.H1 = Cf::H;
        ma.n2 = n2;
        ma.n3 = n3;
        ma.l = mp.l;
        ma.step = mp.step;
        ma.skip4 = skip4;
        ma.dc3 = pa.dc3;
        ++*launches;
        return mid_pass<T, NX>(ma, d.n[m], mode, s);
    };
    if (NX == 4) {
        if ((e = mid(2, 0, S, S2, rg ? 1 : 0)) != cudaSuccess) return e;
        if (rg && (e = split_pass<T>(d, b, cs, S, S2, pa.dc3, mp.l, s, launches)) != cudaSuccess) return e;
    }
    if (b.ev0) cudaEventRecordWithFlags(b.ev0, s, cudaEventRecordExternal);
    if ((e = mid(NX - 1, 2, S2, S2, 0)) != cudaSuccess) return e;
    if (b.ev1) cudaEventRecordWithFlags(b.ev1, s, cudaEventRecordExternal);
    if (NX == 4 && (e = mid(2, 1, S2, S2, 0)) != cudaSuccess) return e;
    // inverse plane pass (+ update)
    int ginv = 1;
    {
        const size_t smem = inv_smem<T, N>();
        int& grid = ginv;
        if (lp) {
            e = occ_grid(k_plane_inv<T, N, NX, true>, Cf::NT, smem, pa.nplanes, &grid);
            if (e == cudaSuccess && d.batch > 1)
                e = cudaMemsetAsync(pa.part, 0, sizeof(double) * NMOM * grid * (size_t)d.batch, s);
            if (e == cudaSuccess) k_plane_inv<T, N, NX, true><<<grid, Cf::NT, smem, s>>>(pa);
        } else {
            e = occ_grid(k_plane_inv<T, N, NX, false>, Cf::NT, smem, pa.nplanes, &grid);
            if (e == cudaSuccess) k_plane_inv<T, N, NX, false><<<grid, Cf::NT, smem, s>>>(pa);
        }
        if (e != cudaSuccess) return e;
        ++*launches;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    k_plane_fin<NX><<<d.batch, 256, 0, s>>>(b.st, b.coef, cs, pa.dcpart, pa.dc3, pa.part, ppf, n3, ginv,
                                            lp ? 1 : 0);
    ++*launches;
    return cudaGetLastError();
}

template <typename T, int NX>
static cudaError_t plane_n(const Dims& d, PencilBufs& b, const ModelParams& mp, const LikParams* lp, double ks,
                           cudaStream_t s, int64_t* launches) {
    switch (d.n[0]) {
        case 32: return plane_t<T, 32, NX>(d, b, mp, lp, ks, s, launches);
        case 64: return plane_t<T, 64, NX>(d, b, mp, lp, ks, s, launches);
        case 96: return plane_t<T, 96, NX>(d, b, mp, lp, ks, s, launches);
        case 128: return plane_t<T, 128, NX>(d, b, mp, lp, ks, s, launches);
        default: return cudaErrorInvalidValue;
    }
}

// sharded nx = 4 fp64 route (pmf_sharded.cpp): the plane prep without a regrid, and the forward
// plane pass over the shard's planes writing each spectrum row in `chunks` k0 pieces, piece q
// to S + q chunk_stride (the all-to-all send blocks)
cudaError_t launch_plane_prep(const Dims& d, PencilBufs& b, const ModelParams& mp, const LikParams* lp, cudaStream_t s,
                              int64_t* launches) {
    LikParams lpv = lp ? *lp : LikParams{};
    k_plane_prep<4><<<d.batch, 32, 0, s>>>(b.st, b.coef, coef_stride(mp.l), mp, b.sub, lpv, b.z, -1.0, lp ? 1 : 0, d);
    ++*launches;
    return cudaGetLastError();
}

template <int N>
static cudaError_t fwd_chunks_n(const Dims& d, PencilBufs& b, const ModelParams& mp, int chunks,
                                long long chunk_stride, double* dcpart, int pbeg, int pend, cudaStream_t s,
                                int64_t* launches) {
    using Cf = Cfg<N>;
    PlaneArgs<double> pa{};
    pa.Wsrc = (const double*)b.W;
    pa.W2src = (const double*)b.W;
    pa.W = (double*)b.W;
    pa.S = (double2*)b.S;
    pa.Sinv = (double2*)b.S;
    pa.coef = b.coef;
    pa.cs = coef_stride(mp.l);
    pa.ppf = d.n[2] * d.n[3];
    pa.nplanes = pa.ppf * d.batch;
    pa.dcpart = dcpart;
    pa.n2 = d.n[2];
    pa.n3 = d.n[3];
    pa.l = mp.l;
    pa.chunks = chunks;
    pa.chunk_stride = chunk_stride;
    if (pend >= 0) {                       // a sub-range of the planes (pipelined exchange)
        pa.pbeg = pbeg;
        pa.nplanes = pend;
    }
    if (pa.nplanes <= pa.pbeg) return cudaSuccess;
    const size_t smem = fwd_smem<double, N>();
    int grid = 1;
    cudaError_t e = occ_grid(k_plane_fwd<double, N, 4, false>, Cf::NT, smem, pa.nplanes - pa.pbeg, &grid);
    if (e != cudaSuccess) return e;
    k_plane_fwd<double, N, 4, false><<<grid, Cf::NT, smem, s>>>(pa);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_plane_fwd_chunks(const Dims& d, PencilBufs& b, const ModelParams& mp, int chunks,
                                    long long chunk_stride, double* dcpart, int pbeg, int pend, cudaStream_t s,
                                    int64_t* launches) {
    switch (d.n[0]) {
        case 32: return fwd_chunks_n<32>(d, b, mp, chunks, chunk_stride, dcpart, pbeg, pend, s, launches);
        case 64: return fwd_chunks_n<64>(d, b, mp, chunks, chunk_stride, dcpart, pbeg, pend, s, launches);
        case 96: return fwd_chunks_n<96>(d, b, mp, chunks, chunk_stride, dcpart, pbeg, pend, s, launches);
        default: return cudaErrorInvalidValue;
    }
}

// the plane finaliser from per-filter totals tot[16] = {15 index-space moment sums, DC}
// (ppf = n3 = ginv = 1: k_plane_fin then reads exactly these)
cudaError_t launch_plane_fin_tot(const Dims& d, PencilBufs& b, const ModelParams& mp, double* tot, int update,
                                 cudaStream_t s, int64_t* launches) {
    k_plane_fin<4><<<d.batch, 256, 0, s>>>(b.st, b.coef, coef_stride(mp.l), tot + NMOM, tot + NMOM, tot, 1, 1, 1,
                                           update);
    ++*launches;
    return cudaGetLastError();
}

cudaError_t launch_plane(const Dims& d, int dtype, PencilBufs& b, const ModelParams& mp, const LikParams* lp,
                         double ks, cudaStream_t s, int64_t* launches) {
    if (d.nx == 3) {
        if (dtype == 0) return plane_n<double, 3>(d, b, mp, lp, ks, s, launches);
        return plane_n<float, 3>(d, b, mp, lp, ks, s, launches);
    }
    if (dtype == 0) return plane_n<double, 4>(d, b, mp, lp, ks, s, launches);
    return plane_n<float, 4>(d, b, mp, lp, ks, s, launches);
}

size_t plane_partials_doubles(const Dims& d) {
    long long ppf = 1;
    for (int m = 2; m < d.nx; ++m) ppf *= d.n[m];
    return (size_t)((ppf + d.n[3] + 1024 * NMOM) * d.batch);
}

}  // namespace pmf
