// device_common.cuh -- small device helpers: complex arithmetic, nx<=4 linear
// algebra, per-filter epoch constants, deterministic block reductions.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include "pmf_internal.h"

namespace pmf {

#define PMF_PI 3.14159265358979323846

template <typename T> struct C2;
template <> struct C2<double> { using type = double2; };
template <> struct C2<float> { using type = float2; };

template <typename V> __device__ __forceinline__ V cadd(V a, V b) { return {a.x + b.x, a.y + b.y}; }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { return {a.x - b.x, a.y - b.y}; }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
    return {fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x)};
}
// a * conj(b)
template <typename V> __device__ __forceinline__ V cmulc(V a, V b) {
    return {fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y)};
}
// multiply by -i (fwd) / +i (inv)
template <bool INV, typename V> __device__ __forceinline__ V mul_mi(V a) {
    if (INV) return {-a.y, a.x};
    return {a.y, -a.x};
}

// ---------------------------------------------------------------- small linear algebra (stride 4)
// Every loop runs to 4 under an `nx` guard and is fully unrolled, so the 4x4 arrays stay in
// registers (no local-memory stack) whether nx is a compile-time constant or not; the
// arithmetic and its order are those of the plain nx-bounded loops.
__device__ __forceinline__ void mat_mul4(int nx, const double* A, const double* B, double* C) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i >= nx || j >= nx) continue;
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k < nx) s = fma(A[i * 4 + k], B[k * 4 + j], s);
            C[i * 4 + j] = s;
        }
}

// Gauss-Jordan inverse with partial pivoting; returns determinant (0 if singular). The pivot
// row swap is a chain of predicated exchanges over compile-time row indices.
__device__ __forceinline__ double mat_inv4(int nx, const double* A, double* Ai) {
    double M[16], I[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) { M[i] = A[i]; I[i] = 0.0; }
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (i < nx) I[i * 4 + i] = 1.0;
    double det = 1.0;
#pragma unroll
    for (int col = 0; col < 4; ++col) {
        if (col >= nx) break;
        int piv = col;
        double best = fabs(M[col * 4 + col]);
#pragma unroll
        for (int r = col + 1; r < 4; ++r)
            if (r < nx && fabs(M[r * 4 + col]) > best) { best = fabs(M[r * 4 + col]); piv = r; }
        if (best == 0.0) return 0.0;
#pragma unroll
        for (int r = col + 1; r < 4; ++r) {
            const bool sw = piv == r;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double mc = M[col * 4 + k], mr = M[r * 4 + k];
                const double ic = I[col * 4 + k], ir = I[r * 4 + k];
                M[col * 4 + k] = sw ? mr : mc;
                M[r * 4 + k] = sw ? mc : mr;
                I[col * 4 + k] = sw ? ir : ic;
                I[r * 4 + k] = sw ? ic : ir;
            }
        }
        if (piv != col) det = -det;
        double p = M[col * 4 + col];
        det *= p;
        double ip = 1.0 / p;
#pragma unroll
        for (int k = 0; k < 4; ++k) { M[col * 4 + k] *= ip; I[col * 4 + k] *= ip; }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r == col || r >= nx) continue;
            double f = M[r * 4 + col];
            if (f == 0.0) continue;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                M[r * 4 + k] = fma(-f, M[col * 4 + k], M[r * 4 + k]);
                I[r * 4 + k] = fma(-f, I[col * 4 + k], I[r * 4 + k]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) Ai[i] = I[i];
    return det;
}

// packed (a <= b) index 0..9 for nx <= 4 (row stride 4 whatever nx)
__host__ __device__ __forceinline__ int tri(int a, int b) { return a * 4 - a * (a - 1) / 2 + (b - a); }

__device__ __forceinline__ int pair_index(int nx, int a, int b) {
    // packed order: diagonal 0..nx-1, then (0,1),(0,2),(0,3),(1,2),(1,3),(2,3) restricted to nx
    int idx = nx;
    for (int i = 0; i < nx; ++i)
        for (int j = i + 1; j < nx; ++j) {
            if (i == a && j == b) return idx;
            ++idx;
        }
    return -1;
}

// Per-filter Euler-factor coefficients for the l substeps of one prediction
// interval (Alg. 3 P:333-336 with R3/R4): for substep n the factor is
//   f_n(kappa) = 1 + sum_a cf[a] kappa_a^2 + sum_{a<b} cf[pair(a,b)] kx_a kx_b
// with cf_diag = dt/2 D_n,aa and cf_pair = dt D_n,ab (the 2 of the symmetric
// cross term folded in), D_n = B^-1 E_n B^-T (FULL) or diag(Q_mm/||B_n[:,m]||^2)
// (AXIS_LITERAL). Writes 10 doubles per substep (packed as pair_index).
// One substep n (Bi = B^-1 precomputed by the caller; 10 doubles to `o`).
__device__ __forceinline__ void substep_coefs(int nx, const double* B, const double* Bi, const ModelParams& mp,
                                              const SubstepEntry& e, double* o) {
    double D[16];
    if (mp.diff_mode == 0) {
        double T1[16], BiT[16], E[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) E[i] = e.E[i];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) BiT[i * 4 + j] = Bi[j * 4 + i];
        mat_mul4(nx, Bi, E, T1);
        mat_mul4(nx, T1, BiT, D);
    } else {
        double Bn[16], Pn[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) Pn[i] = e.P[i];
        mat_mul4(nx, Pn, B, Bn);
#pragma unroll
        for (int i = 0; i < 16; ++i) D[i] = 0.0;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            if (m >= nx) continue;
            double len2 = 0.0;
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (r < nx) len2 = fma(Bn[r * 4 + m], Bn[r * 4 + m], len2);
            D[m * 4 + m] = mp.Q[m * 4 + m] / len2;
        }
    }
    double out[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) out[k] = 0.0;
    // f_n = 1 + h kappa^T D_n kappa: h = dt/2 (Euler factor 1/f_n), dt/4 (Crank-Nicolson:
    // (2 - f_n) / f_{n+1})
    const double h = mp.step ? 0.25 * mp.dt : 0.5 * mp.dt;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        if (a >= nx) continue;
        out[a] = h * D[a * 4 + a];
#pragma unroll
        for (int b = a + 1; b < 4; ++b) {
            if (b >= nx) continue;
            // packed index of (a, b): nx + the pairs before it (pair_index order)
            int idx = nx;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = i + 1; j < 4; ++j)
                    if (j < nx && (i < a || (i == a && j < b))) ++idx;
            // (idx < 10 always; selects keep `out` in registers)
#pragma unroll
            for (int k = 0; k < 10; ++k)
                if (k == idx) out[k] = h * (D[a * 4 + b] + D[b * 4 + a]);
        }
    }
    for (int k = 0; k < 10; ++k) o[k] = out[k];
}

__device__ inline void epoch_coefs(const double* B, const ModelParams& mp,
                                   const SubstepEntry* sub, double* out) {
    const int nx = mp.nx;
    double Bi[16];
    mat_inv4(nx, B, Bi);
    for (int s = 0; s < mp.l + (mp.step ? 1 : 0); ++s) substep_coefs(nx, B, Bi, mp, sub[s], out + 10 * s);
}

__device__ __forceinline__ double det4(int nx, const double* B) {
    double Bi[16];
    return mat_inv4(nx, B, Bi);
}

// signed wavenumber of transform index k (N even): [0..N/2-1] -> k, [N/2..N-1] -> k - N
__device__ __forceinline__ int signed_k(int k, int N) { return k < N / 2 ? k : k - N; }

// ---------------------------------------------------------------- exp
// exp(x) in fp64 for the likelihood: Cody-Waite reduction x = k ln2 + r, |r| <= ln2/2,
// degree-13 Taylor polynomial (truncation < 1e-17 relative), scale by 2^k through the
// exponent field. Arguments below -708 return 0 (true value < 3e-308, far below the
// 1e-10 peak-relative parity bar); the likelihood exponent never exceeds +709.
__device__ __forceinline__ double exp_fast(double x) {
    const double C = 6755399441055744.0;                    // 1.5 * 2^52: round-to-nearest trick
    const double kd0 = fma(x, 1.4426950408889634074, C);
    const int k = __double2loint(kd0);
    const double kd = kd0 - C;
    double r = fma(kd, -6.93147180559945286227e-01, x);
    r = fma(kd, -2.31904681384629955842e-17, r);
    double p = 1.6059043836821614599e-10;                   // 1/13!
    p = fma(p, r, 2.0876756987868098979e-09);               // 1/12!
    p = fma(p, r, 2.5052108385441718775e-08);
    p = fma(p, r, 2.7557319223985890653e-07);
    p = fma(p, r, 2.7557319223985890653e-06);
    p = fma(p, r, 2.4801587301587301587e-05);
    p = fma(p, r, 1.9841269841269841270e-04);
    p = fma(p, r, 1.3888888888888888889e-03);
    p = fma(p, r, 8.3333333333333333333e-03);
    p = fma(p, r, 4.1666666666666666667e-02);
    p = fma(p, r, 1.6666666666666666667e-01);
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = fma(p, r, 1.0);
    const double y = __hiloint2double(__double2hiint(p) + (int)((unsigned)k << 20), __double2loint(p));
    return x < -708.0 ? 0.0 : y;
}

// ---------------------------------------------------------------- likelihood at a physical point
// Terrain table function: bilinear between nodes, nearest edge outside (R26).
__device__ __forceinline__ double terrain_height(const LikParams& lp, double px, double py) {
    double u = (px - lp.tx0) * lp.tidx, v = (py - lp.ty0) * lp.tidy;
    u = fmin(fmax(u, 0.0), (double)(lp.tcol - 1));
    v = fmin(fmax(v, 0.0), (double)(lp.trow - 1));
    const int c = min((int)u, lp.tcol - 2), r = min((int)v, lp.trow - 2);
    const double fu = u - c, fv = v - r;
    const double* t0 = lp.terrain + (long long)r * lp.tcol + c;
    const double lo = fma(fu, t0[1] - t0[0], t0[0]);
    const double hi = fma(fu, t0[lp.tcol + 1] - t0[lp.tcol], t0[lp.tcol]);
    return fma(fv, hi - lo, lo);
}

// p(z | x) for z = h(x) + v, v ~ sum_g w_g N(mu_g, var_g) (eq:ex1_PDF P:413-418)
// Loops unrolled to their maxima with runtime guards (same operations in the same order):
// a runtime index into x[] or r[] would put the caller's arrays in local memory.
__device__ __forceinline__ double lik_terrain_gm(const LikParams& lp, const double* x, const double* z) {
    double px = x[0], py = x[0];
#pragma unroll
    for (int a = 1; a < 4; ++a) {
        px = lp.ix == a ? x[a] : px;
        py = lp.iy == a ? x[a] : py;
    }
    const double d = z[0] - terrain_height(lp, px, py);
    double s = 0.0;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        if (g < lp.ncomp) {
            const double e = d - lp.gm_mu[g];
            s += exp_fast(fma(-0.5 * e * lp.gm_ivar[g], e, lp.gm_logc[g]));
        }
    }
    return s;
}

__device__ __forceinline__ double log_lik(const LikParams& lp, const double* x, const double* z) {
    if (lp.kind == 1) {
        double r2 = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
            if (a < lp.nx) r2 = fma(x[a], x[a], r2);
        double d = (z[0] - sqrt(r2)) * lp.inv_sigma;
        return fma(-0.5 * d, d, lp.lognorm);
    }
    double r[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (i < lp.nz) {
            double hx = 0.0;
#pragma unroll
            for (int a = 0; a < 4; ++a)
                if (a < lp.nx) hx = fma(lp.H[i * 4 + a], x[a], hx);
            r[i] = z[i] - hx;
        }
    }
    double e = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        if (i < lp.nz) {
            double t = 0.0;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j < lp.nz) t = fma(lp.Rinv[i * 4 + j], r[j], t);
            e = fma(r[i], t, e);
        }
    }
    return fma(-0.5, e, lp.lognorm);
}

// ---------------------------------------------------------------- moment accumulators
// acc[0] = sum w, acc[1..nx] = sum w u_a, then sum w u_a u_b (a<=b) packed row-wise.
__device__ __forceinline__ void acc_moments(int nx, double w, const double* u, double* acc) {
    acc[0] += w;
    int k = 1 + nx;
    for (int a = 0; a < nx; ++a) {
        double wu = w * u[a];
        acc[1 + a] += wu;
        for (int b = a; b < nx; ++b) { acc[k] = fma(wu, u[b], acc[k]); ++k; }
    }
}

// Deterministic block sum of NV doubles per thread; result valid in thread 0.
// scratch: >= 32 * NV doubles of shared memory.
template <int NV>
__device__ __forceinline__ void block_sum(double* v, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        double x = v[i];
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        v[i] = x;
    }
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < NV; ++i) scratch[wid * NV + i] = v[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        // unrolled: v[] stays in registers (a runtime index put it in local memory)
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double s = 0.0;
            for (int w = 0; w < nw; ++w) s += scratch[w * NV + i];
            v[i] = s;
        }
    }
    __syncthreads();
}

// Finalise moments from accumulators (index coordinates u) into physical mean/cov:
// ubar = S1/S0, S = S2/S0 - ubar ubar^T, mean = c + B ubar, cov = B S B^T (R14).
__device__ __forceinline__ void finish_moments(int nx, const double* acc, const double* c, const double* B,
                                      double* mean, double* cov) {
    double S0 = acc[0];
    double ub[4] = {0, 0, 0, 0}, Su[16];
    for (int a = 0; a < nx; ++a) ub[a] = acc[1 + a] / S0;
    int k = 1 + nx;
    for (int a = 0; a < nx; ++a)
        for (int b = a; b < nx; ++b) {
            double v = acc[k++] / S0 - ub[a] * ub[b];
            Su[a * 4 + b] = v;
            Su[b * 4 + a] = v;
        }
    for (int a = 0; a < nx; ++a) {
        double m = c[a];
        for (int b = 0; b < nx; ++b) m = fma(B[a * 4 + b], ub[b], m);
        mean[a] = m;
    }
    double T[16];
    for (int a = 0; a < nx; ++a)
        for (int b = 0; b < nx; ++b) {
            double s = 0.0;
            for (int k2 = 0; k2 < nx; ++k2) s = fma(B[a * 4 + k2], Su[k2 * 4 + b], s);
            T[a * 4 + b] = s;
        }
    for (int a = 0; a < nx; ++a)
        for (int b = 0; b < nx; ++b) {
            double s = 0.0;
            for (int k2 = 0; k2 < nx; ++k2) s = fma(T[a * 4 + k2], B[b * 4 + k2], s);
            cov[a * 4 + b] = s;
        }
    for (int a = 0; a < nx; ++a)
        for (int b = a + 1; b < nx; ++b) {
            double v = 0.5 * (cov[a * 4 + b] + cov[b * 4 + a]);
            cov[a * 4 + b] = v;
            cov[b * 4 + a] = v;
        }
}

// New grid of the re-centring policy (R12): c' = mean, B' = diag(2 ks sqrt(cov_mm)/N_m).
// Returns false when some variance is non-finite or <= 0.
// Linear-Gaussian likelihood exponent as a quadratic form in the moved grid's index
// coordinates u (R13): r(u) = (z - H c) - (H B) u, e = r^T R^-1 r = q[0] + sum_a q[1+a] u_a +
// sum_{a<=b} q[5+tri(a,b)] u_a u_b. Loops unrolled to 4 under nx / nz guards (registers only).
__device__ __forceinline__ void lik_quadform(int nx, const LikParams& lp, const double* c, const double* B,
                                             const double* zf, double* q) {
    const int nz = lp.nz;
    double r0[4], G[16], w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        r0[i] = 0.0;
        w[i] = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a) G[i * 4 + a] = 0.0;
        if (i >= nz) continue;
        double hc = 0.0;
#pragma unroll
        for (int a = 0; a < 4; ++a)
            if (a < nx) hc = fma(lp.H[i * 4 + a], c[a], hc);
        r0[i] = zf[i] - hc;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            if (a >= nx) continue;
            double g = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (k < nx) g = fma(lp.H[i * 4 + k], B[k * 4 + a], g);
            G[i * 4 + a] = g;
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {     // R^-1 r0
        if (i >= nz) continue;
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (j < nz) s = fma(lp.Rinv[i * 4 + j], r0[j], s);
        w[i] = s;
    }
    double qa = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (i < nz) qa = fma(r0[i], w[i], qa);
    q[0] = qa;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        if (a >= nx) continue;
        double s = 0.0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (i < nz) s = fma(G[i * 4 + a], w[i], s);
        q[1 + a] = -2.0 * s;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c2 = a; c2 < 4; ++c2) {
            if (c2 >= nx) continue;
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (i < nz && j < nz) s = fma(G[i * 4 + a] * lp.Rinv[i * 4 + j], G[j * 4 + c2], s);
            q[5 + tri(a, c2)] = (a == c2) ? s : 2.0 * s;
        }
}

// (the Jacobi rotations index their arrays dynamically: kept out of line so that the
// caller's arrays stay in registers; only this branch's copy goes through local memory)
static __device__ __noinline__ bool eigen_grid_dev(int nx, const int* n, const double* cov, double ks, double* B) {
    return eigen_grid(nx, n, cov, ks, B);
}

__device__ __forceinline__ bool regrid_target(int nx, const int* n, const FilterState& st, double ks,
                                              double* cn, double* Bn, int grid = 0) {
    if (grid == 1) {                          // R28: eigen-aligned
        double Be[16];
        int ng[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) ng[a] = a < nx ? n[a] : 1;
        const bool ok = eigen_grid_dev(nx, ng, st.cov, ks, Be);
#pragma unroll
        for (int i = 0; i < 16; ++i) Bn[i] = Be[i];
#pragma unroll
        for (int a = 0; a < 4; ++a)
            if (a < nx) cn[a] = st.mean[a];
        return ok;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) Bn[i] = 0.0;
    bool ok = true;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        if (a >= nx) continue;
        double v = st.cov[a * 4 + a];
        if (!(v > 0.0) || !isfinite(v)) ok = false;
        cn[a] = st.mean[a];
        Bn[a * 4 + a] = 2.0 * ks * sqrt(v) / n[a];
    }
    return ok;
}

}  // namespace pmf
