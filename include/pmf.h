/*
 * pmf.h -- C ABI of the B200-native spectral point-mass filter (PMF) hot path.
 *
 * Method: Matousek, Dunik, Brandner, "Efficient Spectral Differentiation in
 * Grid-Based Continuous State Estimation" (FUSION 2024, arXiv 2412.07240).
 * Citations "P:<n>" are lines of PAPER.md; readings "R<n>" are listed in
 * DESIGN.md §3.
 *
 * Model (eq:dynam / eq:meas):  dx = A x dt + dw,  E[dw dw^T] = Q dt
 * (Q is the FPE diffusion matrix of eq:fokker P:55, R1), z_k = h(x_k) + v_k.
 *
 * A filter's density is a point-mass density (PMD, eq:PDF_pm P:116) on an
 * N_0 x ... x N_{nx-1} equidistant grid that moves with the drift (eq:gridMov
 * P:142). Point j = (j_0..j_{nx-1}) sits at the physical location
 *        xi_j = c + B u_j,   u_j[m] = j_m - (N_m - 1)/2          (R10)
 * with c the grid centre and B the (possibly sheared) nx x nx placement matrix.
 *
 * MEMORY LAYOUT (R-layout, P:114/P:346 MATLAB reshape): weights of one filter
 * are N_0*...*N_{nx-1} values with axis 0 FASTEST; filters are stacked
 * batch-major (filter index slowest). Real type per pmf_config.dtype (double
 * or float). Matrices are row-major, nx x nx, packed (stride nx).
 *
 * OWNERSHIP: the caller owns every host array and device buffer it passes; they
 * are read (or written) during the call only. The context owns its device
 * buffers (weights, spectrum, per-filter state) and its work is enqueued on
 * pmf_config.stream. Host outputs (pmf_moments, pmf_get_weights to host,
 * pmf_get_grid) synchronise that stream; nothing else does.
 *
 * LAZINESS: pmf_predict and pmf_regrid validate their arguments and RECORD the
 * operation; it is executed (fused with what follows) by the next call that
 * needs the density: pmf_update, pmf_get_weights, pmf_get_grid, pmf_sync. Results are identical to eager execution.
 *
 * ERRORS: every int-returning call returns PMF_OK (0) or a negative PMF_E_*
 * code; pmf_last_error() gives a message. A failed call leaves the context
 * unchanged unless the code is PMF_E_CUDA or PMF_E_NCCL (the context is then
 * unusable).
 * There is no CPU fallback: the library requires a CUDA device (sm_100a).
 */
#ifndef PMF_H
#define PMF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PMF_MAX_NX 4
#define PMF_MAX_NZ 4

/* return codes */
#define PMF_OK               0
#define PMF_E_ARG           -1  /* bad argument (null pointer, bad enum, nx/nz range, non-diagonal Q in AXIS_LITERAL mode) */
#define PMF_E_ODD_N         -2  /* points per axis odd (the spectral interpolant needs even N)             */
#define PMF_E_RADIX         -3  /* N has a prime factor other than 2,3,5,7,11,13,17, or N outside [4, 1024]     */
#define PMF_E_Q_NOT_PSD     -4  /* Q not symmetric positive semi-definite                                         */
#define PMF_E_SINGULAR_GRID -5  /* grid matrix B not invertible                                                    */
#define PMF_E_NO_SUPPORT    -6  /* normaliser zero/non-finite: measurement incompatible with grid support,       */
                                /* or degenerate posterior covariance at regrid (R12)                            */
#define PMF_E_DT            -7  /* dt <= 0, steps < 1, or Euler trace factor base 1 -/+ dt tr(A) <= 0 (R5)       */
#define PMF_E_STATE         -8  /* call out of order (e.g. predict before a density was set)                     */
#define PMF_E_CUDA          -9  /* CUDA runtime failure or no usable device                                        */
#define PMF_E_NOMEM        -10  /* device allocation failed                                                        */
#define PMF_E_NCCL         -11  /* NCCL failure (sharded contexts): libnccl.so.2 missing, communicator init, a     */
                                /* collective's enqueue, or an asynchronous communicator error (polled with      */
                                /* ncclCommGetAsyncError after every exchange); the context is then unusable      */

/* enums */
#define PMF_F64 0
#define PMF_F32 1

#define PMF_DIFF_FULL          0  /* R3: index-space diffusion D_n = B_n^-1 Q B_n^-T, cross terms kept (default) */
#define PMF_DIFF_AXIS_LITERAL  1  /* Alg. 2-3 literally: per-axis L^(m) = N ||B_n[:,m]||, no cross    */
#define PMF_DIFF_FDM           2  /* the paper's FDM baseline (eq:FDM P:146-150, zero Dirichlet boundary) in its
                                     eigen / sine-transform form (eq:FST P:199-202): diagonal Q, fp64,
                                     N_m in {32, 64, 96, 128}, <= 64 substeps; not sharded. DST-I on FP64
                                     tensor cores; regrid and update as for the other modes             */

#define PMF_TRACE_PHYSICAL (-1)   /* R5: s = (1 - dt tr A)^l   (eq:easyFPE P:92)                                   */
#define PMF_TRACE_PRINTED    1    /* Alg. 4 as printed: s = (1 + dt tr A)^l; normalised output identical   */

#define PMF_PATH_AUTO     0  /* resident kernel when it fits, else the plane path when it fits, else pencil      */
#define PMF_PATH_PENCIL   1  /* multi-pass per-axis pencil kernels (any nx <= 4)                                */
#define PMF_PATH_RESIDENT 2  /* one CTA per filter, whole half-spectrum in shared memory (nx = 2, N0 = N1 = 128)   */
#define PMF_PATH_PLANE    3  /* (i0,i1)-plane kernels + strided passes with the regrid fused into the forward pass:
                                nx = 3, 4; N0 = N1 in {32, 64, 96, 128}; N_m in {16, 32, 64, 96, 128} for m >= 2;
                                substeps <= 64 per predict (longer intervals run on the pencil kernels)       */

#define PMF_STEP_EULER 0
#define PMF_STEP_CN    1

#define PMF_GRID_AXIS  0   /* R12: regrid target axis-aligned, B' = diag(2 k_sigma sqrt(cov_mm) / N_m)            */
#define PMF_GRID_EIGEN 1   /* R28: aligned with the covariance eigenvectors (the refs of P:346): B' columns =
                              eigenvectors v_j * 2 k_sigma sqrt(lambda_j) / N_m, eigenvector j (decreasing lambda)
                              on the free axis of its largest |component|, that component > 0. Also used for the
                              initial grid of pmf_set_gaussian. PMF_DIFF_FULL only; not sharded                  */

#define PMF_LIK_LINEAR_GAUSS 0   /* z = H x + v, v ~ N(0, R), nz <= 4 (eq:meas P:36)                               */
#define PMF_LIK_RANGE_GAUSS  1   /* z = ||x|| + v, v ~ N(0, sigma^2), nz = 1 (C3)                                   */
#define PMF_LIK_TERRAIN_GM   2   /* the paper's §VI model: z = h(x[ix], x[iy]) + v, h the terrain table
                                    of pmf_set_terrain (bilinear, clamped to the table), v ~ sum_g w_g N(mu_g, var_g),
                                    ncomp <= 4 components; nz = 1                                                 */

typedef struct pmf_ctx pmf_ctx;

typedef struct {
    int   nx;          /* state dimension, 1..4                                                    */
    int   n[4];        /* points per axis N_m (even, factors 2,3,5,7,11,13,17 only, 4 <= N_m <= 1024;
                          n[m] for m>=nx ignored)                                                   */
    int   batch;       /* number of independent filters sharing A, Q and the likelihood kind       */
    int   dtype;       /* PMF_F64 or PMF_F32 (storage + transform precision; reductions are fp64)   */
    int   diff_mode;   /* PMF_DIFF_FULL (default 0), PMF_DIFF_AXIS_LITERAL or PMF_DIFF_FDM         */
    int   trace_sign;  /* PMF_TRACE_PHYSICAL (0 is read as PHYSICAL) or PMF_TRACE_PRINTED          */
    int   path;        /* PMF_PATH_AUTO / PENCIL / RESIDENT / PLANE                                 */
    int   device;      /* CUDA device ordinal the context lives on                                 */
    void* stream;      /* cudaStream_t to enqueue on; NULL = the legacy default stream             */
    int   step;        /* PMF_STEP_EULER (0, the paper's semi-implicit Euler substeps)
                          or PMF_STEP_CN (Crank-Nicolson, second order in dt; R27, "higher order
                          time stepping" = the paper's future work). CN runs on every path
                          (resident, plane, pencil) and is not combined with PMF_DIFF_FDM       */
    int   grid;        /* PMF_GRID_AXIS (0) or PMF_GRID_EIGEN: how pmf_set_gaussian and pmf_regrid
                          design a grid from a covariance                                           */
} pmf_config;

typedef struct {
    int    kind;       /* PMF_LIK_*                                                                 */
    int    nz;         /* measurement dimension (LINEAR_GAUSS: 1..4; RANGE_GAUSS: 1)                */
    double H[16];      /* LINEAR_GAUSS: nz x nx row-major, packed                                  */
    double R[16];      /* LINEAR_GAUSS: nz x nz noise covariance, symmetric positive definite       */
    double sigma;      /* RANGE_GAUSS: noise standard deviation > 0                                 */
    int    ncomp;      /* TERRAIN_GM: mixture components 1..4                                      */
    double gm_w[4];    /* TERRAIN_GM: weights >= 0 (normalised by the library)                     */
    double gm_mu[4];   /* TERRAIN_GM: component means                                              */
    double gm_var[4];  /* TERRAIN_GM: component variances > 0                                     */
} pmf_likelihood;

/* Create a context: validates sizes (PMF_E_ODD_N, PMF_E_RADIX), A (nx x nx) and
 * Q (nx x nx, symmetric PSD -> else PMF_E_Q_NOT_PSD), allocates the device
 * buffers on cfg->device. No density is set yet (PMF_E_STATE until
 * pmf_set_gaussian / pmf_set_state). *out receives the handle. */
int pmf_create(const pmf_config* cfg, const double* A, const double* Q, pmf_ctx** out);

/* Release every device buffer (synchronises the stream). NULL is a no-op. */
void pmf_destroy(pmf_ctx* ctx);

/* Message of the last error on this context (or of the last failed
 * pmf_create in this thread when ctx is NULL). Never NULL. */
const char* pmf_last_error(const pmf_ctx* ctx);

/* Initial density p(x_0) (P:48 footnote): for each filter b, the grid
 * c = mean_b, B = diag(2 k_sigma sqrt(cov_b[m][m]) / N_m) (R10; with PMF_GRID_EIGEN
 * the eigenvector-aligned B of R28), weights
 * N(xi; mean_b, cov_b) normalised so vol * sum w = 1 (vol = |det B|, R9).
 * mean: host batch x nx; cov: host batch x nx x nx (SPD). */
int pmf_set_gaussian(pmf_ctx* ctx, const double* mean, const double* cov, double k_sigma);

/* Terrain table for PMF_LIK_TERRAIN_GM ("a table function that assigns
 * altitude to each combination of ... it covers"): heights[r * ncol + c] is the
 * altitude at (x0 + c dx, y0 + r dy); state components ix, iy are the horizontal
 * position. Between nodes h is bilinear; outside the table the nearest edge value is
 * used (reading R26). The host array is copied to the device (the caller keeps
 * ownership). Errors: PMF_E_ARG for nrow/ncol < 2, dx/dy <= 0, ix/iy outside the state. */
int pmf_set_terrain(pmf_ctx* ctx, const double* heights, int nrow, int ncol, double x0, double y0, double dx,
                    double dy, int ix, int iy);

/* Set an arbitrary state: grid (center: host batch x nx, B: host batch x nx x nx)
 * and weights (batch x N_total in dtype, host or device per weights_on_device;
 * a device pointer must be on cfg->device). The weights are normalised on
 * entry (vol * sum w = 1). PMF_E_SINGULAR_GRID if some B is singular. */
int pmf_set_state(pmf_ctx* ctx, const double* center, const double* B,
                  const void* weights, int weights_on_device);

/* Time update over one prediction interval tau = dt * steps with `steps` Euler
 * substeps of length dt: Alg. 1-6 of §V.B --
 * forward DFT per axis (1/N each, eq:fourtrsf P:221), multiply by
 * s * prod_{n<steps} psi_n with psi_n the semi-implicit Euler factor of Alg. 3
 * (R2-R4, R7) on the grid at the start of substep n, inverse DFT,
 * normalise (Alg. 6; closed form, R9). The grid moves: c <- e^{A tau} c,
 * B <- e^{A tau} B (eq:gridMov P:142-148). Lazy (see LAZINESS).
 * cfg.step = PMF_STEP_CN: psi_n = (1 - dt/4 q_n) / (1 + dt/4 q_{n+1}) (R27).
 * cfg.diff_mode = PMF_DIFF_FDM: the explicit FDM instead (eq:FST), normalised by
 * summation (it does not conserve mass).
 * PMF_E_DT if dt <= 0, steps < 1 or 1 -/+ dt tr(A) <= 0 (FDM / plane: also steps > 64
 * where those kernels are required). */
int pmf_predict(pmf_ctx* ctx, double dt, int steps);

/* Measurement update (Bayes, eq:filt P:46): w_i <- w_i p(z - h(xi_i)) at the
 * (moved) grid points (R13), normaliser C = vol sum w_i p(z|xi_i),
 * w <- w / C; the moments of the posterior (R14) are computed on
 * the device in the same pass (fused into the inverse transform for the Gaussian
 * kinds; PMF_LIK_TERRAIN_GM runs as its own point pass after the predict).
 * z: batch x nz doubles, host or device. PMF_E_STATE for TERRAIN_GM without a
 * terrain table.
 * Per-filter failure (C == 0 or non-finite) is reported by pmf_moments
 * (PMF_E_NO_SUPPORT). */
int pmf_update(pmf_ctx* ctx, const double* z, int z_on_device, const pmf_likelihood* lik);

/* Copy the posterior moments of the last update to host arrays (any may be
 * NULL): mean batch x nx, cov batch x nx x nx, log_norm batch (log of the
 * P:49 normaliser). Packs (nx + nx^2 + 2) doubles per filter on the device and copies
 * them to pinned memory; synchronises. PMF_E_STATE before the first update,
 * PMF_E_NO_SUPPORT if any filter's last update failed. */
int pmf_moments(pmf_ctx* ctx, double* mean, double* cov, double* log_norm);

/* Bytes pmf_moments copies device -> host per call ((nx + nx^2 + 2) doubles per filter). */
int64_t pmf_moments_bytes(const pmf_ctx* ctx);

/* Asynchronous form of pmf_moments for pipelined callers: enqueues the packing and the
 * device -> host copy of the last update's moments into `dst` (pmf_moments_bytes bytes,
 * host memory the caller owns -- pinned for a truly asynchronous copy) on the context's
 * stream and returns at once. Record of filter b at dst + b (nx + nx^2 + 2) doubles:
 * mean[nx], cov[nx*nx] (row-major), log normaliser, failure flag (nonzero: that filter's
 * last update failed, the PMF_E_NO_SUPPORT of pmf_moments). Valid after pmf_sync (or any
 * synchronising call). PMF_E_STATE before the first update. */
int pmf_moments_async(pmf_ctx* ctx, double* dst);

/* Re-centre every filter's grid on its last posterior (R12; the paper is silent,
 * north_star "re-centre the grid"): c' = mean, B' = diag(2 k_sigma sqrt(cov_mm)/N_m)
 * (PMF_GRID_EIGEN: the eigenvector-aligned B' of R28, see pmf_config.grid),
 * multilinear interpolation of the old weights at the new points with zero
 * ghost nodes, renormalised. Lazy. PMF_E_STATE before the first update.
 * The mean and covariance are those of the last pmf_update (predictions do not
 * recompute them): call it right after an update, as pmf_step does. After
 * predictions with no update in between it re-centres on the stale posterior
 * and can cut off mass that has drifted away (the next update may then fail
 * with PMF_E_NO_SUPPORT). */
int pmf_regrid(pmf_ctx* ctx, double k_sigma);

/* One filter epoch = pmf_predict(dt, steps); pmf_update(z, lik); pmf_regrid(k_sigma)
 * (the regrid stays pending and is fused into the next epoch's load). */
int pmf_step(pmf_ctx* ctx, double dt, int steps, const double* z, int z_on_device,
             const pmf_likelihood* lik, double k_sigma);

/* ---------------------------------------------------------------------------
 * Sharded contexts: ONE filter (batch = 1, nx >= 2) whose grid
 * is split into `world` slabs along its LAST axis (N_{nx-1} divisible by world).
 * A predict does two all-to-all transposes (the last-axis transform needs whole
 * pencils), an update one all-reduce of the moment sums, a regrid a grouped
 * send/recv of the old planes each rank's new slab reads (R12). Everything else
 * is local. The filter state (grid, moments) is replicated on every rank.
 *
 * pmf_nccl_unique_id: rank 0 creates the NCCL id (128 bytes) that every rank
 * passes to pmf_create_sharded (broadcast it, e.g. with torch.distributed).
 * libnccl.so.2 is loaded on first use (dlopen); PMF_E_NCCL if unavailable.
 *
 * pmf_create_sharded: cfg->n are the GLOBAL sizes. unique_id != NULL: this
 * process is `rank` of `world` (one GPU each, NCCL over NVLink). unique_id ==
 * NULL: "virtual ranks" -- all `world` slabs live in this one context on one
 * device and the collectives become device copies; results equal the real
 * sharded path up to the order of the all-reduce sum.
 * Weights passed to pmf_set_state / returned by pmf_get_weights are the slabs
 * the context holds, in slab order (virtual: the whole grid; real: the local
 * slab, N_0 x ... x N_{nx-2} x (N_{nx-1}/world) values). */
int pmf_nccl_unique_id(void* out128);
int pmf_create_sharded(const pmf_config* cfg, const double* A, const double* Q, int rank, int world,
                       const void* unique_id, pmf_ctx** out);
/* Number of slabs the grid is split into (1 for an ordinary context). */
int pmf_world(const pmf_ctx* ctx);

/* Normalised density values (vol * sum = 1) of all filters on their current
 * grids, batch x N_total in dtype; dst on host or on cfg->device. Flushes
 * pending work. */
int pmf_get_weights(pmf_ctx* ctx, void* dst, int dst_on_device);

/* Current grids: center batch x nx, B batch x nx x nx (host; either may be NULL).
 * Flushes pending work and synchronises. */
int pmf_get_grid(pmf_ctx* ctx, double* center, double* B);

/* Flush pending work and wait for the stream. */
int pmf_sync(pmf_ctx* ctx);

/* Number of kernels this context has launched so far. */
int64_t pmf_launch_count(const pmf_ctx* ctx);

/* Kernel timing: while enabled, CUDA events are recorded on the context's stream
 * around the dominant kernel of every executed prediction (the resident epoch
 * kernel, the plane path's last-axis Psi pass, the FDM's last-axis DST kernel, or
 * the whole pencil predict); pmf_profile_read waits for them and
 * returns the summed milliseconds and the number of timed launches, then resets.
 * pmf_profile(ctx, 1) also resets. */
int pmf_profile(pmf_ctx* ctx, int enable);
int pmf_profile_read(pmf_ctx* ctx, double* total_ms, int64_t* count);

/* CUDA-graph replay of the launch sequence of a flush (default on; env PMF_NO_GRAPHS=1
   turns it off at creation). When the pending work, the likelihood and the buffers
   equal those of an earlier flush, the captured graph is replayed instead of
   re-launching every kernel (an epoch of pmf_step repeats the same sequence). Needs a
   non-legacy stream (cfg.stream != NULL); capture failures fall back to direct
   launches. Results are bitwise identical either way. */
int pmf_use_graphs(pmf_ctx* ctx, int enable);

/* Bytes of device memory owned by the context. */
int64_t pmf_device_bytes(const pmf_ctx* ctx);

/* Kernel path the context uses (PMF_PATH_PENCIL, PMF_PATH_RESIDENT or PMF_PATH_PLANE). */
int pmf_path(const pmf_ctx* ctx);

/* Kernel family that ran the predict of the most recent flush (a CUDA-graph replay repeats
   the captured one): PMF_EPOCH_NONE before any predict, else one of
     PMF_EPOCH_PENCIL   multi-kernel pencil predict (prep, per-axis transforms, finalize)
     PMF_EPOCH_LINE     nx = 1: regrid + predict + update + moments in one launch
     PMF_EPOCH_CLUSTER  nx = 2 at 256^2: the whole epoch in one 16- (or 8-) CTA cluster launch
     PMF_EPOCH_RESIDENT nx = 2 at 128^2: one CTA per filter, the whole epoch in one launch
     PMF_EPOCH_PLANE    nx = 3, 4: plane kernels + strided passes
     PMF_EPOCH_FDM      the FDM / DST-I baseline predictor (diff_mode = PMF_DIFF_FDM)
     PMF_EPOCH_SHARDED  slab-sharded context (pmf_create_sharded)
   Returns -1 for a null context. Diagnostic only: results do not depend on it. */
#define PMF_EPOCH_NONE     0
#define PMF_EPOCH_PENCIL   1
#define PMF_EPOCH_LINE     2
#define PMF_EPOCH_CLUSTER  3
#define PMF_EPOCH_RESIDENT 4
#define PMF_EPOCH_PLANE    5
#define PMF_EPOCH_FDM      6
#define PMF_EPOCH_SHARDED  7
int pmf_epoch_kernel(const pmf_ctx* ctx);

/* Library version string. */
const char* pmf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PMF_H */
