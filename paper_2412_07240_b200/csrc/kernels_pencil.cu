// kernels_pencil.cu -- the general multi-pass path (any nx <= 4, any
// N = 2^a 3^b per axis, any batch), plus the per-filter kernels shared with the
// resident path: initial density, standalone likelihood update, reductions
// into per-filter moments, and the multilinear regrid.
//
// Predict (Alg. 1-6) for nx >= 2 runs as
//   prep  -> axis-0 R2C (half spectrum) -> forward C2C along axes
//   1..nx-2 -> last axis: forward, x s*Psi (Alg. 3-4), inverse -> inverse C2C
//   axes nx-2..1 -> axis-0 C2R fused with the measurement update (eq:filt P:46)
// and for nx = 1 as one fused line kernel. Each pass stages a tile of pencils in
// shared memory (coalesced: contiguous inner index across threads) and runs the
// Stockham FFT of fft_smem.cuh.
#include <algorithm>
#include <cmath>
#include <vector>

#include "device_common.cuh"
#include "fft_smem.cuh"

namespace pmf {

static constexpr int kThreads = 256;

static FFTPlan make_plan(int N) {
    FFTPlan p{};
    p.N = N;
    int m = N, k = 0;
    while (m % 4 == 0) { p.r[k++] = 4; m /= 4; }
    if (m % 2 == 0) { p.r[k++] = 2; m /= 2; }
    while (m % 3 == 0) { p.r[k++] = 3; m /= 3; }
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

static int pencils_per_cta(int N) {
    int P = std::max(1, 2048 / N);
    int p2 = 1;
    while (p2 * 2 <= P) p2 *= 2;
    return std::min(p2, 32);
}

// ============================================================================ prep
// One thread per filter: Euler-factor coefficients (epoch_coefs), the input
// scale, then move the grid (c <- M c, B <- M B, eq:gridMov) and set the
// closed-form normalisation of Alg. 6: scale' = vol_0 / (vol_l s)  (R9; the DC
// coefficient is multiplied by exactly s because psi(0) = 1).
__global__ void k_predict_prep(FilterState* st, double* coef, int cstride, ModelParams mp,
                               const SubstepEntry* __restrict__ sub, int batch) {
    int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    FilterState& f = st[b];
    double* cf = coef + (long long)b * cstride;
    cf[0] = f.scale;
    epoch_coefs(f.B, mp, sub, cf + 4);
    const int nx = mp.nx;
    double vol0 = fabs(det4(nx, f.B));
    double Bn[16], cn[4];
    for (int i = 0; i < 16; ++i) Bn[i] = 0.0;
    mat_mul4(nx, mp.Mtau, f.B, Bn);
    for (int a = 0; a < nx; ++a) {
        double s = 0.0;
        for (int k = 0; k < nx; ++k) s = fma(mp.Mtau[a * 4 + k], f.c[k], s);
        cn[a] = s;
    }
    double voll = fabs(det4(nx, Bn));
    for (int i = 0; i < 16; ++i) f.B[i] = Bn[i];
    for (int a = 0; a < nx; ++a) f.c[a] = cn[a];
    f.scale = vol0 / (voll * mp.s);
}

// ============================================================================ spectral multiplier
// s * Psi(k) / N_total for one spectral point (Alg. 3-4): kap[a] = 2 pi k_a / N_a
// (signed k), kx = kap with the Nyquist wavenumber zeroed (R7).
__device__ __forceinline__ double psi_point(int nx, int l, const double* __restrict__ cf,
                                            const double* kap, const double* kx, double mult) {
    double prod = 1.0;
    for (int s = 0; s < l; ++s) {
        const double* c = cf + 10 * s;
        double f = 1.0;
        int idx = nx;
        for (int a = 0; a < nx; ++a) {
            f = fma(c[a], kap[a] * kap[a], f);
            for (int b = a + 1; b < nx; ++b) f = fma(c[idx++], kx[a] * kx[b], f);
        }
        prod *= f;
    }
    return mult / prod;
}

__device__ __forceinline__ void wavenum(int k, int N, double& kap, double& kx) {
    int ks = signed_k(k, N);
    kap = 2.0 * PMF_PI * ks / N;
    kx = (2 * k == N) ? 0.0 : kap;
}

// ============================================================================ axis-0 R2C
template <typename T>
__global__ void __launch_bounds__(kThreads) k_axis0_r2c(const T* __restrict__ W, typename C2<T>::type* __restrict__ S,
                                                         const double* __restrict__ coef, int cstride, Dims d,
                                                         FFTPlan pl, const typename C2<T>::type* __restrict__ tw,
                                                         int P) {
    using V = typename C2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = d.n[0], PS = N + 1;
    V* a = reinterpret_cast<V*>(smem_raw);
    V* b = a + P * PS;
    const long long rpf = d.ntot / N;
    const long long row0 = (long long)blockIdx.x * P;
    const int filt = (int)(row0 / rpf);
    const T sc = (T)coef[(long long)filt * cstride];
    const T* src = W + row0 * N;
    for (int i = threadIdx.x; i < P * N; i += blockDim.x) {
        int p = i / N, j = i - p * N;
        a[p * PS + j] = V{src[i] * sc, T(0)};
    }
    __syncthreads();
    V* r = smem_fft<false>(a, b, P, PS, pl, tw);
    V* dst = S + row0 * d.H0;
    for (int i = threadIdx.x; i < P * d.H0; i += blockDim.x) {
        int p = i / d.H0, k = i - p * d.H0;
        dst[i] = r[p * PS + k];
    }
}

// ============================================================================ strided C2C (+ optional Psi)
// Pencils along axis m of the half-spectrum buffer: element (i, j, o) at
// S[o*Nm*I + j*I + i], i < I = H0*N_1*..*N_{m-1}, o < O. A CTA takes P
// consecutive i (coalesced rows of P complex) of one o.
template <typename T, int MODE>   // MODE 0 fwd, 1 inv, 2 fwd*Psi*inv (last axis)
__global__ void __launch_bounds__(kThreads) k_axis_c2c(typename C2<T>::type* __restrict__ S, Dims d, int m,
                                                        long long I, FFTPlan pl,
                                                        const typename C2<T>::type* __restrict__ tw, int P,
                                                        const double* __restrict__ coef, int cstride,
                                                        ModelParams mp) {
    using V = typename C2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = pl.N, PS = N + 1;
    V* a = reinterpret_cast<V*>(smem_raw);
    V* b = a + P * PS;
    const long long ntile = (I + P - 1) / P;
    const long long o = blockIdx.x / ntile;
    const long long i0 = (blockIdx.x - o * ntile) * P;
    V* base = S + o * (long long)N * I;
    for (int t = threadIdx.x; t < P * N; t += blockDim.x) {
        int p = t % P, j = t / P;
        long long i = i0 + p;
        a[p * PS + j] = (i < I) ? base[(long long)j * I + i] : V{T(0), T(0)};
    }
    __syncthreads();
    V* r;
    if (MODE == 1) {
        r = smem_fft<true>(a, b, P, PS, pl, tw);
    } else {
        r = smem_fft<false>(a, b, P, PS, pl, tw);
        if (MODE == 2) {
            // last axis: o is the filter index
            const double* cf = coef + o * cstride + 4;
            const int nx = d.nx;
            double ntot = 1.0;
            for (int q = 0; q < nx; ++q) ntot *= d.n[q];
            const double mult = mp.s / ntot;
            for (int t = threadIdx.x; t < P * N; t += blockDim.x) {
                int p = t / N, j = t - p * N;
                long long i = i0 + p;
                if (i >= I) continue;
                double kap[4], kx[4];
                long long rem = i;
                int k0 = (int)(rem % d.H0);
                rem /= d.H0;
                wavenum(k0, d.n[0], kap[0], kx[0]);
                for (int q = 1; q < m; ++q) {
                    int kq = (int)(rem % d.n[q]);
                    rem /= d.n[q];
                    wavenum(kq, d.n[q], kap[q], kx[q]);
                }
                wavenum(j, N, kap[m], kx[m]);
                T ps = (T)psi_point(nx, mp.l, cf, kap, kx, mult);
                V v = r[p * PS + j];
                r[p * PS + j] = V{v.x * ps, v.y * ps};
            }
            __syncthreads();
            V* other = (r == a) ? b : a;
            r = smem_fft<true>(r, other, P, PS, pl, tw);
        }
    }
    for (int t = threadIdx.x; t < P * N; t += blockDim.x) {
        int p = t % P, j = t / P;
        long long i = i0 + p;
        if (i < I) base[(long long)j * I + i] = r[p * PS + j];
    }
}

// ============================================================================ point helpers
__device__ __forceinline__ void point_u(const Dims& d, long long pt, double* u) {
    long long rem = pt;
    for (int q = 0; q < d.nx; ++q) {
        int j = (int)(rem % d.n[q]);
        rem /= d.n[q];
        u[q] = j - 0.5 * (d.n[q] - 1);
    }
}

__device__ __forceinline__ void phys(int nx, const FilterState& f, const double* u, double* x) {
    for (int a = 0; a < nx; ++a) {
        double s = f.c[a];
        for (int b = 0; b < nx; ++b) s = fma(f.B[a * 4 + b], u[b], s);
        x[a] = s;
    }
}

// ============================================================================ axis-0 C2R (+ update)
template <typename T, bool UPDATE>
__global__ void __launch_bounds__(kThreads) k_axis0_c2r(const typename C2<T>::type* __restrict__ S, T* __restrict__ W,
                                                         const FilterState* __restrict__ st, Dims d, FFTPlan pl,
                                                         const typename C2<T>::type* __restrict__ tw, int P,
                                                         LikParams lp, const double* __restrict__ z,
                                                         double* __restrict__ partials) {
    using V = typename C2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = d.n[0], PS = N + 1;
    V* a = reinterpret_cast<V*>(smem_raw);
    V* b = a + P * PS;
    double* red = reinterpret_cast<double*>(b + P * PS);
    const long long rpf = d.ntot / N;
    const long long row0 = (long long)blockIdx.x * P;
    const int filt = (int)(row0 / rpf);
    const V* src = S + row0 * d.H0;
    for (int i = threadIdx.x; i < P * N; i += blockDim.x) {
        int p = i / N, k = i - p * N;
        V v;
        if (k < d.H0) v = src[p * d.H0 + k];
        else { v = src[p * d.H0 + (N - k)]; v.y = -v.y; }
        a[p * PS + k] = v;
    }
    __syncthreads();
    V* r = smem_fft<true>(a, b, P, PS, pl, tw);
    const FilterState& f = st[filt];
    const double scale = f.scale;
    const double* zf = z + (long long)filt * lp.nz;
    double acc[NMOM];
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    T* dst = W + row0 * N;
    const long long pt_base = row0 * N - (long long)filt * d.ntot;
    for (int i = threadIdx.x; i < P * N; i += blockDim.x) {
        int p = i / N, j = i - p * N;
        double w = (double)r[p * PS + j].x;
        if (UPDATE) {
            double u[4], x[4];
            point_u(d, pt_base + i, u);
            phys(d.nx, f, u, x);
            w = w * scale * exp_fast(log_lik(lp, x, zf));
            T wt = (T)w;
            dst[i] = wt;
            acc_moments(d.nx, (double)wt, u, acc);
        } else {
            dst[i] = (T)w;
        }
    }
    if (UPDATE) {
        block_sum<NMOM>(acc, red);
        if (threadIdx.x == 0)
            for (int q = 0; q < NMOM; ++q) partials[(long long)blockIdx.x * NMOM + q] = acc[q];
    }
}

// ============================================================================ nx = 1 fused line
template <typename T, bool UPDATE>
__global__ void __launch_bounds__(kThreads) k_line_psi(T* __restrict__ W, FilterState* __restrict__ st, Dims d,
                                                        FFTPlan pl, const typename C2<T>::type* __restrict__ tw,
                                                        const double* __restrict__ coef, int cstride,
                                                        ModelParams mp, LikParams lp, const double* __restrict__ z,
                                                        double* __restrict__ partials) {
    using V = typename C2<T>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int N = d.n[0], PS = N + 1;
    V* a = reinterpret_cast<V*>(smem_raw);
    V* b = a + PS;
    double* red = reinterpret_cast<double*>(b + PS);
    const int filt = blockIdx.x;
    const double* cf = coef + (long long)filt * cstride;
    const T sc = (T)cf[0];
    T* row = W + (long long)filt * N;
    for (int j = threadIdx.x; j < N; j += blockDim.x) a[j] = V{row[j] * sc, T(0)};
    __syncthreads();
    V* r = smem_fft<false>(a, b, 1, PS, pl, tw);
    const double mult = mp.s / N;
    for (int k = threadIdx.x; k < N; k += blockDim.x) {
        double kap, kx;
        wavenum(k, N, kap, kx);
        T ps = (T)psi_point(1, mp.l, cf + 4, &kap, &kx, mult);
        V v = r[k];
        r[k] = V{v.x * ps, v.y * ps};
    }
    __syncthreads();
    r = smem_fft<true>(r, (r == a) ? b : a, 1, PS, pl, tw);
    const FilterState& f = st[filt];
    double acc[NMOM];
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    const double scale = f.scale;
    const double* zf = z + (long long)filt * lp.nz;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
        double w = (double)r[j].x;
        if (UPDATE) {
            double u = j - 0.5 * (N - 1), x;
            phys(1, f, &u, &x);
            w = w * scale * exp_fast(log_lik(lp, &x, zf));
            T wt = (T)w;
            row[j] = wt;
            acc_moments(1, (double)wt, &u, acc);
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
// grid: batch * nbpf blocks; block (filt, q) covers points q, q+nbpf*blockDim, ...
static int blocks_per_filter(long long ntot) {
    long long nb = (ntot + kThreads * 8 - 1) / (kThreads * 8);
    return (int)std::max(1LL, std::min(nb, 512LL));
}

template <typename T, int MODE>   // 0: standalone update, 1: init gaussian, 2: plain sum
__global__ void __launch_bounds__(kThreads) k_points(T* __restrict__ W, const FilterState* __restrict__ st, Dims d,
                                                      int nbpf, LikParams lp, const double* __restrict__ z,
                                                      const double* __restrict__ gauss,
                                                      double* __restrict__ partials) {
    __shared__ double red[32 * NMOM];
    const int filt = blockIdx.x / nbpf, q = blockIdx.x - filt * nbpf;
    const FilterState& f = st[filt];
    T* Wf = W + (long long)filt * d.ntot;
    double acc[NMOM];
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    const double* zf = z ? z + (long long)filt * lp.nz : nullptr;
    const double* g = gauss ? gauss + (long long)filt * 21 : nullptr;
    for (long long pt = (long long)q * blockDim.x + threadIdx.x; pt < d.ntot; pt += (long long)nbpf * blockDim.x) {
        double u[4], x[4];
        point_u(d, pt, u);
        if (MODE == 0) {
            phys(d.nx, f, u, x);
            double w = (double)Wf[pt] * f.scale * exp_fast(log_lik(lp, x, zf));
            T wt = (T)w;
            Wf[pt] = wt;
            acc_moments(d.nx, (double)wt, u, acc);
        } else if (MODE == 1) {
            phys(d.nx, f, u, x);
            double r[4], e = 0.0;
            for (int a = 0; a < d.nx; ++a) r[a] = x[a] - g[a];
            for (int a = 0; a < d.nx; ++a) {
                double t = 0.0;
                for (int b = 0; b < d.nx; ++b) t = fma(g[4 + a * 4 + b], r[b], t);
                e = fma(r[a], t, e);
            }
            T wt = (T)exp(fma(-0.5, e, g[20]));
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

// ============================================================================ finalisers (1 warp per filter)
__device__ inline void warp_sum_partials(const double* __restrict__ partials, long long first, int nb, double* acc) {
    const int lane = threadIdx.x & 31;
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    for (int k = lane; k < nb; k += 32)
        for (int i = 0; i < NMOM; ++i) acc[i] += partials[(first + k) * NMOM + i];
    for (int i = 0; i < NMOM; ++i) {
        double x = acc[i];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        acc[i] = x;
    }
}

// MODE 0: update -> normaliser C = vol * sum, log C, scale = 1/C, moments.
// MODE 1: renormalise (init/set_state): scale = 1/(vol * sum).
__global__ void k_finalize(FilterState* st, const double* __restrict__ partials, int nbpf, int batch, Dims d,
                           int mode) {
    const int filt = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (filt >= batch) return;
    double acc[NMOM];
    warp_sum_partials(partials, (long long)filt * nbpf, nbpf, acc);
    if ((threadIdx.x & 31) != 0) return;
    FilterState& f = st[filt];
    const int nx = d.nx;
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

// ============================================================================ regrid
// Multilinear interpolation with zero ghost nodes at the points of the new grid
// (R12). v = B^-1 (x' - c) + (N-1)/2 = o + M u' with M = B^-1 B', o = B^-1(c'-c)+(N-1)/2.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_regrid_gather(const T* __restrict__ Wold, T* __restrict__ Wnew,
                                                             const FilterState* __restrict__ st, Dims d, int nbpf,
                                                             double ks, double* __restrict__ partials) {
    __shared__ double red[32 * NMOM];
    __shared__ double Msh[16], osh[4];
    const int filt = blockIdx.x / nbpf, q = blockIdx.x - filt * nbpf;
    const FilterState& f = st[filt];
    const int nx = d.nx;
    if (threadIdx.x == 0) {
        double cn[4], Bn[16], Bi[16];
        regrid_target(nx, d.n, f, ks, cn, Bn);
        mat_inv4(nx, f.B, Bi);
        double M[16];
        for (int i = 0; i < 16; ++i) M[i] = 0.0;
        mat_mul4(nx, Bi, Bn, M);
        for (int i = 0; i < 16; ++i) Msh[i] = M[i];
        for (int a = 0; a < nx; ++a) {
            double s = 0.5 * (d.n[a] - 1);
            for (int b = 0; b < nx; ++b) s = fma(Bi[a * 4 + b], cn[b] - f.c[b], s);
            osh[a] = s;
        }
    }
    __syncthreads();
    const T* Wo = Wold + (long long)filt * d.ntot;
    T* Wn = Wnew + (long long)filt * d.ntot;
    double acc[NMOM];
    for (int i = 0; i < NMOM; ++i) acc[i] = 0.0;
    for (long long pt = (long long)q * blockDim.x + threadIdx.x; pt < d.ntot; pt += (long long)nbpf * blockDim.x) {
        double u[4], v[4], fr[4];
        int i0[4];
        point_u(d, pt, u);
        for (int a = 0; a < nx; ++a) {
            double s = osh[a];
            for (int b = 0; b < nx; ++b) s = fma(Msh[a * 4 + b], u[b], s);
            v[a] = s;
            double fl = floor(s);
            i0[a] = (int)fmax(fmin(fl, 1e9), -1e9);
            fr[a] = s - fl;
        }
        double val = 0.0;
        for (int corner = 0; corner < (1 << nx); ++corner) {
            double wt = 1.0;
            long long off = 0, stride = 1;
            bool ok = true;
            for (int a = 0; a < nx; ++a) {
                int bit = (corner >> a) & 1;
                int ia = i0[a] + bit;
                wt *= bit ? fr[a] : (1.0 - fr[a]);
                ok = ok && ia >= 0 && ia <= d.n[a] - 1;
                off += (long long)ia * stride;
                stride *= d.n[a];
            }
            if (ok) val = fma(wt, (double)Wo[off], val);
        }
        T vt = (T)val;
        Wn[pt] = vt;
        acc[0] += (double)vt;
    }
    block_sum<NMOM>(acc, red);
    if (threadIdx.x == 0)
        for (int i = 0; i < NMOM; ++i) partials[(long long)blockIdx.x * NMOM + i] = acc[i];
}

__global__ void k_finalize_regrid(FilterState* st, const double* __restrict__ partials, int nbpf, int batch,
                                  Dims d, double ks) {
    const int filt = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (filt >= batch) return;
    double acc[NMOM];
    warp_sum_partials(partials, (long long)filt * nbpf, nbpf, acc);
    if ((threadIdx.x & 31) != 0) return;
    FilterState& f = st[filt];
    double cn[4], Bn[16];
    bool ok = regrid_target(d.nx, d.n, f, ks, cn, Bn);
    for (int a = 0; a < d.nx; ++a) f.c[a] = cn[a];
    for (int i = 0; i < 16; ++i) f.B[i] = Bn[i];
    double C = fabs(det4(d.nx, Bn)) * acc[0];
    if (!ok || !(C > 0.0) || !isfinite(C)) { f.status = -6; return; }
    f.scale = 1.0 / C;
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

template <typename T>
static cudaError_t predict_pencil_t(const Dims& d, PencilBufs& b, const Twiddles& tw, const ModelParams& mp,
                                    const LikParams* lp, cudaStream_t s, int64_t* launches) {
    using V = typename C2<T>::type;
    const int cs = coef_stride(mp.l);
    if (b.ev0) cudaEventRecord(b.ev0, s);
    k_predict_prep<<<(d.batch + 127) / 128, 128, 0, s>>>(b.st, b.coef, cs, mp, b.sub, d.batch);
    ++*launches;
    PMF_TRY(cudaGetLastError());
    LikParams lpv{};
    if (lp) lpv = *lp;
    if (d.nx == 1) {
        FFTPlan pl = make_plan(d.n[0]);
        size_t sm = 2 * (d.n[0] + 1) * sizeof(V) + 32 * NMOM * sizeof(double);
        PMF_TRY(smem_attr(k_line_psi<T, true>, sm));
        PMF_TRY(smem_attr(k_line_psi<T, false>, sm));
        if (lp)
            k_line_psi<T, true><<<d.batch, kThreads, sm, s>>>((T*)b.W, b.st, d, pl, (const V*)tw.tw[0], b.coef, cs,
                                                              mp, lpv, b.z, b.partials);
        else
            k_line_psi<T, false><<<d.batch, kThreads, sm, s>>>((T*)b.W, b.st, d, pl, (const V*)tw.tw[0], b.coef, cs,
                                                               mp, lpv, b.z, b.partials);
        ++*launches;
        PMF_TRY(cudaGetLastError());
        if (lp) {
            k_finalize<<<(d.batch + 3) / 4, 128, 0, s>>>(b.st, b.partials, 1, d.batch, d, 0);
            ++*launches;
        }
        if (b.ev1) cudaEventRecord(b.ev1, s);
        return cudaGetLastError();
    }
    // axis 0 forward (R2C)
    const int N0 = d.n[0];
    const long long rpf = d.ntot / N0;
    const int P0 = rows_per_cta(N0, rpf);
    FFTPlan pl0 = make_plan(N0);
    size_t sm0 = 2 * (size_t)P0 * (N0 + 1) * sizeof(V);
    long long nrow_blocks = (long long)d.batch * rpf / P0;
    PMF_TRY(smem_attr(k_axis0_r2c<T>, sm0));
    k_axis0_r2c<T><<<(unsigned)nrow_blocks, kThreads, sm0, s>>>((const T*)b.W, (V*)b.S, b.coef, cs, d, pl0,
                                                                (const V*)tw.tw[0], P0);
    ++*launches;
    PMF_TRY(cudaGetLastError());
    // strided axes
    auto strided = [&](int m, int mode) -> cudaError_t {
        long long I = d.H0;
        for (int q = 1; q < m; ++q) I *= d.n[q];
        long long O = d.batch;
        for (int q = m + 1; q < d.nx; ++q) O *= d.n[q];
        const int N = d.n[m];
        const int P = pencils_per_cta(N);
        FFTPlan pl = make_plan(N);
        size_t sm = 2 * (size_t)P * (N + 1) * sizeof(V);
        long long nblk = O * ((I + P - 1) / P);
        PMF_TRY(smem_attr(k_axis_c2c<T, 0>, sm));
        PMF_TRY(smem_attr(k_axis_c2c<T, 1>, sm));
        PMF_TRY(smem_attr(k_axis_c2c<T, 2>, sm));
        if (mode == 0)
            k_axis_c2c<T, 0><<<(unsigned)nblk, kThreads, sm, s>>>((V*)b.S, d, m, I, pl, (const V*)tw.tw[m], P,
                                                                   b.coef, cs, mp);
        else if (mode == 1)
            k_axis_c2c<T, 1><<<(unsigned)nblk, kThreads, sm, s>>>((V*)b.S, d, m, I, pl, (const V*)tw.tw[m], P,
                                                                   b.coef, cs, mp);
        else
            k_axis_c2c<T, 2><<<(unsigned)nblk, kThreads, sm, s>>>((V*)b.S, d, m, I, pl, (const V*)tw.tw[m], P,
                                                                   b.coef, cs, mp);
        ++*launches;
        return cudaGetLastError();
    };
    for (int m = 1; m < d.nx - 1; ++m) PMF_TRY(strided(m, 0));
    PMF_TRY(strided(d.nx - 1, 2));
    for (int m = d.nx - 2; m >= 1; --m) PMF_TRY(strided(m, 1));
    // axis 0 inverse (C2R) + update
    size_t smc = sm0 + 32 * NMOM * sizeof(double);
    PMF_TRY(smem_attr(k_axis0_c2r<T, true>, smc));
    PMF_TRY(smem_attr(k_axis0_c2r<T, false>, smc));
    if (lp)
        k_axis0_c2r<T, true><<<(unsigned)nrow_blocks, kThreads, smc, s>>>((const V*)b.S, (T*)b.W, b.st, d, pl0,
                                                                          (const V*)tw.tw[0], P0, lpv, b.z,
                                                                          b.partials);
    else
        k_axis0_c2r<T, false><<<(unsigned)nrow_blocks, kThreads, smc, s>>>((const V*)b.S, (T*)b.W, b.st, d, pl0,
                                                                           (const V*)tw.tw[0], P0, lpv, b.z,
                                                                           b.partials);
    ++*launches;
    PMF_TRY(cudaGetLastError());
    if (lp) {
        k_finalize<<<(d.batch + 3) / 4, 128, 0, s>>>(b.st, b.partials, (int)(rpf / P0), d.batch, d, 0);
        ++*launches;
    }
    if (b.ev1) cudaEventRecord(b.ev1, s);
    return cudaGetLastError();
}

cudaError_t launch_predict_pencil(const Dims& d, int dtype, PencilBufs& b, const Twiddles& tw,
                                  const ModelParams& mp, const LikParams* lp, cudaStream_t s, int64_t* launches) {
    if (dtype == 0) return predict_pencil_t<double>(d, b, tw, mp, lp, s, launches);
    return predict_pencil_t<float>(d, b, tw, mp, lp, s, launches);
}

template <typename T, int MODE>
static cudaError_t points_t(const Dims& d, PencilBufs& b, const LikParams& lp, cudaStream_t s, int64_t* launches,
                            int fin_mode) {
    int nbpf = blocks_per_filter(d.ntot);
    k_points<T, MODE><<<(unsigned)((long long)nbpf * d.batch), kThreads, 0, s>>>((T*)b.W, b.st, d, nbpf, lp, b.z,
                                                                                 b.gauss, b.partials);
    ++*launches;
    PMF_TRY(cudaGetLastError());
    k_finalize<<<(d.batch + 3) / 4, 128, 0, s>>>(b.st, b.partials, nbpf, d.batch, d, fin_mode);
    ++*launches;
    return cudaGetLastError();
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

template <typename T>
static cudaError_t regrid_t(const Dims& d, PencilBufs& b, double ks, cudaStream_t s, int64_t* launches) {
    int nbpf = blocks_per_filter(d.ntot);
    k_regrid_gather<T><<<(unsigned)((long long)nbpf * d.batch), kThreads, 0, s>>>((const T*)b.W, (T*)b.W2, b.st, d,
                                                                                 nbpf, ks, b.partials);
    ++*launches;
    PMF_TRY(cudaGetLastError());
    k_finalize_regrid<<<(d.batch + 3) / 4, 128, 0, s>>>(b.st, b.partials, nbpf, d.batch, d, ks);
    ++*launches;
    std::swap(b.W, b.W2);
    return cudaGetLastError();
}

cudaError_t launch_regrid(const Dims& d, int dtype, PencilBufs& b, double ks, cudaStream_t s, int64_t* launches) {
    if (dtype == 0) return regrid_t<double>(d, b, ks, s, launches);
    return regrid_t<float>(d, b, ks, s, launches);
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
