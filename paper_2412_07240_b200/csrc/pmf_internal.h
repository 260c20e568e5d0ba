// pmf_internal.h -- structures shared by the host runtime (pmf_host.cpp) and the
// CUDA kernels. Not part of the ABI (include/pmf.h is).
#pragma once
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

namespace pmf {

constexpr int MAXNX = 4;
constexpr int NMOM = 15;           // 1 + nx + nx(nx+1)/2 accumulators for nx = 4

// Per-filter state, device resident, fp64. The stored weights W (dtype) and
// `scale` represent the normalised density scale * W on the grid (c, B):
// physical point xi_j = c + B u_j, u_j[m] = j_m - (N_m - 1)/2 (R10).
struct FilterState {
    double c[4];
    double B[16];       // row-major, row stride 4
    double scale;       // density = scale * W; invariant: vol * sum(scale W) = 1
    double logC;        // log of the last update's normaliser
    double mean[4];     // posterior moments of the last update (physical)
    double cov[16];     // row stride 4
    double mass;        // sum of the stored weights after the last update
    int status;         // 0, or PMF_E_NO_SUPPORT when the last update/regrid failed
    int has_moments;
};

// Model constants of one prediction interval (host computed, kernel param).
struct ModelParams {
    int nx, l, diff_mode, step;   // step: 0 semi-implicit Euler, 1 Crank-Nicolson (R27):
                                  // then l + 1 coefficient sets (grids t_0 .. t_l) scaled dt/4
    double dt;          // Euler substep
    double s;           // trace factor (1 -/+ dt tr A)^l (R5)
    double Mtau[16];    // e^{A tau}, row stride 4
    double Q[16];
};

// Device table, one entry per substep n < l (n <= l for Crank-Nicolson; host computed,
// uploaded per predict):
//   E_n = e^{-A n dt} Q e^{-A^T n dt}   (so D_n = B^-1 E_n B^-T, R3)
//   P_n = e^{A n dt}                    (B_n = P_n B, for AXIS_LITERAL)
struct SubstepEntry {
    double E[16];
    double P[16];
};

// Likelihood parameters (kernel param).
struct LikParams {
    int kind, nz, nx, pad;
    double H[16];       // nz x nx, row stride 4
    double Rinv[16];    // nz x nz, row stride 4
    double lognorm;     // -0.5 log((2 pi)^nz det R)  or  -log(sigma sqrt(2 pi))
    double inv_sigma;
    // TERRAIN_GM (kind 2): h = bilinear(terrain) at (x[ix], x[iy]); GM noise
    int ncomp, ix, iy, trow, tcol, pad2;
    double gm_logc[4];  // log w_g - 0.5 log(2 pi var_g)
    double gm_mu[4];
    double gm_ivar[4];  // 1 / var_g
    double tx0, ty0, tidx, tidy;   // table origin and inverse spacings
    const double* terrain;         // device table [trow][tcol]
};

struct Dims {
    int nx;
    int n[4];               // sizes of the block this context/shard holds (axis 0 first)
    int H0;                 // N_0/2 + 1 (half spectrum along axis 0)
    long long ntot;         // real points per filter in the block
    long long nspec;        // complex half-spectrum points per filter in the block
    int batch;
    int ng[4];              // global grid sizes (== n unless sharded along the last axis)
    int lo[4];              // global index of the block's first point per axis
    int src_lo, src_n;      // regrid source window along the last axis (global start, planes)
    int grid;               // grid design from a covariance: 0 axis-aligned (R12), 1 eigen-aligned (R28)
};

// R28 (the covariance-aligned grids of the refs of P:346): grid matrix
// whose columns are the eigenvectors of cov (stride 4, symmetric) scaled to +-ks standard
// deviations: cov = V diag(lam) V^T by cyclic Jacobi rotations; eigenvector j, in order of
// decreasing lam (lower index first on ties), takes the still free axis a of its largest
// |V[a][j]| (lowest axis on ties), signed so that V[a][j] > 0; B[:, a] = v_j 2 ks sqrt(lam_j) / n[a].
// A diagonal cov gives the axis-aligned grid of R12. Returns false unless every lam > 0.
__host__ __device__ inline bool eigen_grid(int nx, const int* n, const double* cov, double ks, double* B) {
    double a[16], v[16];
    for (int i = 0; i < 16; ++i) {
        a[i] = cov[i];
        v[i] = (i % 5 == 0) ? 1.0 : 0.0;
        B[i] = 0.0;
    }
    for (int sweep = 0; sweep < 32; ++sweep) {
        double off = 0.0, dia = 0.0;
        for (int p = 0; p < nx; ++p) {
            dia += a[p * 4 + p] * a[p * 4 + p];
            for (int q = p + 1; q < nx; ++q) off += a[p * 4 + q] * a[p * 4 + q];
        }
        if (!(off > 1e-36 * dia)) break;
        for (int p = 0; p < nx; ++p)
            for (int q = p + 1; q < nx; ++q) {
                const double apq = a[p * 4 + q];
                if (apq == 0.0) continue;
                const double th = (a[q * 4 + q] - a[p * 4 + p]) / (2.0 * apq);
                const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(fma(th, th, 1.0)));
                const double c = 1.0 / sqrt(fma(t, t, 1.0)), s = t * c;
                for (int k = 0; k < nx; ++k) {         // A <- A J, V <- V J
                    const double akp = a[k * 4 + p], akq = a[k * 4 + q];
                    a[k * 4 + p] = c * akp - s * akq;
                    a[k * 4 + q] = s * akp + c * akq;
                    const double vkp = v[k * 4 + p], vkq = v[k * 4 + q];
                    v[k * 4 + p] = c * vkp - s * vkq;
                    v[k * 4 + q] = s * vkp + c * vkq;
                }
                for (int k = 0; k < nx; ++k) {         // A <- J^T A
                    const double apk = a[p * 4 + k], aqk = a[q * 4 + k];
                    a[p * 4 + k] = c * apk - s * aqk;
                    a[q * 4 + k] = s * apk + c * aqk;
                }
            }
    }
    bool done[4] = {false, false, false, false}, used[4] = {false, false, false, false};
    for (int r = 0; r < nx; ++r) {
        int j = -1;
        for (int jj = 0; jj < nx; ++jj)
            if (!done[jj] && (j < 0 || a[jj * 4 + jj] > a[j * 4 + j])) j = jj;
        done[j] = true;
        const double lam = a[j * 4 + j];
        if (!(lam > 0.0 && lam < 1e300)) return false;
        int ax = -1;
        for (int k = 0; k < nx; ++k)
            if (!used[k] && (ax < 0 || fabs(v[k * 4 + j]) > fabs(v[ax * 4 + j]))) ax = k;
        used[ax] = true;
        const double sc = (v[ax * 4 + j] < 0.0 ? -2.0 : 2.0) * ks * sqrt(lam) / n[ax];
        for (int k = 0; k < nx; ++k) B[k * 4 + ax] = sc * v[k * 4 + j];
    }
    return true;
}

// Number of doubles per filter in the pencil path's epoch-coefficient buffer.
// pencil path: 4 + 10 l + 16 (scale, Euler factors, likelihood quadratic form);
// resident path: 24 + 3 l rounded up to even (kernels_resident.cu)
// plane path: 64 + 10 l (kernels_plane.cu)
inline int coef_stride(int l) { return 80 + 10 * l; }   // (Crank-Nicolson: l + 1 coefficient sets)

// ---------------------------------------------------------------------------
// launchers (implemented in the .cu files); all return a cudaError_t and
// increment *launches by the number of kernels launched.
// ---------------------------------------------------------------------------
struct Twiddles {        // per distinct axis length: forward table e^{-2 pi i m / N}
    const void* tw[4];   // device pointers per axis (complex of dtype)
};

struct PencilBufs {
    void* W;             // real weights [batch][ntot]
    void* W2;            // second real buffer (regrid target)
    void* S;             // complex half spectrum [batch][nspec]
    void* S2 = nullptr;  // second spectrum buffer (plane path, nx = 4: out-of-place strided pass)
    FilterState* st;
    double* partials;    // reduction scratch
    double* coef;        // [batch][coef_stride(l)]
    const SubstepEntry* sub;
    const double* z;     // [batch][nz]
    const double* gauss; // [batch][nx + 16 + 1] mean, inverse cov, log norm (set_gaussian)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;   // if set: recorded around the dominant kernel
};

cudaError_t launch_init_gaussian(const Dims& d, int dtype, PencilBufs& b, cudaStream_t s, int64_t* launches);
cudaError_t launch_normalise_state(const Dims& d, int dtype, PencilBufs& b, cudaStream_t s, int64_t* launches);
cudaError_t launch_update(const Dims& d, int dtype, PencilBufs& b, const LikParams& lp,
                          cudaStream_t s, int64_t* launches);
cudaError_t launch_regrid(const Dims& d, int dtype, PencilBufs& b, double k_sigma,
                          cudaStream_t s, int64_t* launches);   // swaps b.W / b.W2
bool cluster_epoch_supported(const Dims& d, int dtype, const ModelParams& mp);
cudaError_t launch_cluster_epoch(const Dims& d, PencilBufs& b, const Twiddles& tw, const ModelParams& mp,
                                 const LikParams* lp, double ks, cudaStream_t s, int64_t* launches);
bool line_epoch_supported(const Dims& d, int nsets);
cudaError_t launch_line_epoch(const Dims& d, int dtype, PencilBufs& b, const Twiddles& tw, const ModelParams& mp,
                              const LikParams* lp, double ks, cudaStream_t s, int64_t* launches);
cudaError_t launch_predict_pencil(const Dims& d, int dtype, PencilBufs& b, const Twiddles& tw,
                                  const ModelParams& mp, const LikParams* lp /* null = no update */,
                                  cudaStream_t s, int64_t* launches);
cudaError_t launch_scale_out(const Dims& d, int dtype, const PencilBufs& b, void* dst,
                             cudaStream_t s, int64_t* launches);

cudaError_t launch_pack_moments(const Dims& d, const FilterState* st, double* out, cudaStream_t s,
                                int64_t* launches);

// sharded building blocks (slab decomposition along the last axis; pmf_sharded.cpp)
enum { SH_PH_FWD = 1, SH_PH_PSI = 2, SH_PH_INV = 4 };
cudaError_t sh_prep(const Dims& d, PencilBufs& b, const ModelParams& mp, const LikParams* lp, cudaStream_t s,
                    int64_t* launches);
cudaError_t sh_phase(const Dims& d, int dtype, PencilBufs& b, const Twiddles& tw, const ModelParams& mp,
                     const LikParams* lp, int phase, void* psibuf, long long psiI, long long ioff, double* tot,
                     cudaStream_t s, int64_t* launches);
cudaError_t sh_pack(int dtype, void* S, void* send, long long I, int planes, const long long* d_off, int world,
                    int unpack, cudaStream_t s, int64_t* launches);
cudaError_t sh_points(const Dims& d, int dtype, PencilBufs& b, int mode, const LikParams& lp, double* tot,
                      cudaStream_t s, int64_t* launches);
cudaError_t sh_regrid(const Dims& d, int dtype, const void* src, void* dst, PencilBufs& b, double ks, double* tot,
                      cudaStream_t s, int64_t* launches);
cudaError_t launch_finalize_tot(const Dims& d, FilterState* st, const double* tot, int mode, double ks,
                                cudaStream_t s, int64_t* launches);
cudaError_t launch_sum_ranks(const double* in, double* out, int world, int n, cudaStream_t s, int64_t* launches);

// plane path (nx >= 3, N_0 = N_1 in {32, 64, 96, 128}): fused regrid + predict + update
bool plane_supported(const Dims& d, int l);
size_t plane_partials_doubles(const Dims& d);
cudaError_t launch_plane(const Dims& d, int dtype, PencilBufs& b, const ModelParams& mp, const LikParams* lp,
                         double k_sigma /* < 0 = no regrid */, cudaStream_t s, int64_t* launches);

// nx = 4 fp64 three-pass route (kernels_quad.cu): after the forward plane pass (spectrum
// S[filter][j3][j2][k1][k0]), K2 writes S2 in the transposed layout [filter][k1][k0][j3][j2]
// and K3 reads it; called by launch_plane between its forward pass and finaliser
bool quad_supported(const Dims& d, int dtype);
int quad_debug_counters(double* out, int n, int reset);
// the sharded nx = 4 route (slab over j3; pmf_sharded.cpp): plane prep without regrid, forward
// plane pass writing per-destination k0 blocks, K2 / K3 on the exchanged blocks, per-shard totals
cudaError_t launch_plane_prep(const Dims& d, PencilBufs& b, const ModelParams& mp, const LikParams* lp, cudaStream_t s,
                              int64_t* launches);
cudaError_t launch_plane_fwd_chunks(const Dims& d, PencilBufs& b, const ModelParams& mp, int chunks,
                                    long long chunk_stride, double* dcpart, int pbeg, int pend, cudaStream_t s,
                                    int64_t* launches);
cudaError_t launch_plane_fin_tot(const Dims& d, PencilBufs& b, const ModelParams& mp, double* tot, int update,
                                 cudaStream_t s, int64_t* launches);
cudaError_t launch_quad_mid_shard(const Dims& d, PencilBufs& b, const ModelParams& mp, int rank, int world,
                                  const void* in, void* out, int kbeg, int kend, cudaStream_t s, int64_t* launches);
cudaError_t launch_quad_inv_shard(const Dims& d, PencilBufs& b, const ModelParams& mp, const LikParams* lp, int rank,
                                  int world, const void* in, double* part, cudaStream_t s, int64_t* launches,
                                  int* ginv);
cudaError_t launch_shard_sum(const double* dcpart, int nplanes, const double* part, int ginv, int update, double* tot,
                             cudaStream_t s, int64_t* launches);
int resident_debug_counters(double* out, int n, int reset);
cudaError_t launch_quad(const Dims& d, PencilBufs& b, const ModelParams& mp, int range, bool up, double* dcpart,
                        double* dc3, double* part, cudaStream_t s, int64_t* launches, int* ginv);

// FDM baseline predictor (eq:FST; kernels_fdm.cu): prep + DST-I passes on FP64 tensor
// cores; the caller normalises (explicit sum) and runs the update
bool fdm_supported(const Dims& d, int dtype, int l);
size_t fdm_coef_doubles(int batch);
cudaError_t launch_fdm_predict(const Dims& d, int dtype, PencilBufs& b, const ModelParams& mp, double trace_base,
                               cudaStream_t s, int64_t* launches);

// resident (one CTA per filter) fused epoch kernel
bool resident_supported(const Dims& d, int dtype);
cudaError_t launch_resident(const Dims& d, int dtype, PencilBufs& b, const Twiddles& tw,
                            const ModelParams* mp /* null = no predict */,
                            const LikParams* lp /* null = no update */,
                            double regrid_k_sigma /* < 0 = no regrid */,
                            cudaStream_t s, int64_t* launches);

}  // namespace pmf
