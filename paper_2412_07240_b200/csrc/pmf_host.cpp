// pmf_host.cpp -- C ABI runtime of the spectral PMF (include/pmf.h).
//
// Owns the device buffers of a context, validates arguments, computes the
// per-prediction model constants on the host in fp64 (matrix exponentials of
// the drift, eq:gridMov P:142-148; trace factor, Alg. 4), and drives the
// kernels. predict/regrid are recorded and executed lazily (fused with the
// update that follows), see include/pmf.h "LAZINESS".
#include "../../include/pmf.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "pmf_internal.h"
#include "pmf_ctx_impl.h"

using namespace pmf;

namespace {
thread_local std::string g_create_error = "";
}  // namespace

// ============================================================================ helpers
static int fail(pmf_ctx* c, int code, const std::string& msg) {
    if (c) c->err = msg;
    else g_create_error = msg;
    return code;
}

static int cuda_fail(pmf_ctx* c, cudaError_t e, const char* where) {
    return fail(c, PMF_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(ctx, x, where)                                      \
    do {                                                       \
        cudaError_t e_ = (x);                                  \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, where); \
    } while (0)

static void mat_mul(int n, const double* A, const double* B, double* C) {  // stride 4
    double T[16] = {0};
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int k = 0; k < n; ++k) s += A[i * 4 + k] * B[k * 4 + j];
            T[i * 4 + j] = s;
        }
    std::memcpy(C, T, sizeof(T));
}

// e^{M}: scaling and squaring with a degree-20 Taylor polynomial (||M/2^k|| <= 1/2
// makes the truncation error < 1e-25 relative).
static void expm4(int n, const double* M, double* out) {
    double norm = 0.0;
    for (int i = 0; i < n; ++i) {
        double r = 0.0;
        for (int j = 0; j < n; ++j) r += std::fabs(M[i * 4 + j]);
        norm = std::max(norm, r);
    }
    int k = 0;
    while (norm > 0.5) { norm *= 0.5; ++k; }
    double X[16] = {0}, S[16] = {0}, T[16] = {0};
    const double sc = std::ldexp(1.0, -k);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) X[i * 4 + j] = M[i * 4 + j] * sc;
    for (int i = 0; i < n; ++i) { S[i * 4 + i] = 1.0; T[i * 4 + i] = 1.0; }
    for (int t = 1; t <= 20; ++t) {
        mat_mul(n, T, X, T);
        for (int i = 0; i < 16; ++i) T[i] /= t;
        for (int i = 0; i < 16; ++i) S[i] += T[i];
    }
    for (int s = 0; s < k; ++s) mat_mul(n, S, S, S);
    std::memcpy(out, S, sizeof(S));
}

// eigenvalues of a symmetric n x n (stride 4) matrix by cyclic Jacobi
static void sym_eig(int n, const double* Ain, double* ev) {
    double A[16];
    std::memcpy(A, Ain, sizeof(A));
    for (int sweep = 0; sweep < 60; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += A[p * 4 + q] * A[p * 4 + q];
        if (off < 1e-300) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                double apq = A[p * 4 + q];
                if (std::fabs(apq) < 1e-300) continue;
                double th = 0.5 * (A[q * 4 + q] - A[p * 4 + p]) / apq;
                double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
                double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < n; ++k) {
                    double akp = A[k * 4 + p], akq = A[k * 4 + q];
                    A[k * 4 + p] = c * akp - s * akq;
                    A[k * 4 + q] = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {
                    double apk = A[p * 4 + k], aqk = A[q * 4 + k];
                    A[p * 4 + k] = c * apk - s * aqk;
                    A[q * 4 + k] = s * apk + c * aqk;
                }
            }
    }
    for (int i = 0; i < n; ++i) ev[i] = A[i * 4 + i];
}

static double det_inv(int n, const double* Ain, double* Ai) {  // host Gauss-Jordan, stride 4
    double M[16], I[16] = {0};
    std::memcpy(M, Ain, sizeof(M));
    for (int i = 0; i < n; ++i) I[i * 4 + i] = 1.0;
    double det = 1.0;
    for (int col = 0; col < n; ++col) {
        int piv = col;
        for (int r = col + 1; r < n; ++r)
            if (std::fabs(M[r * 4 + col]) > std::fabs(M[piv * 4 + col])) piv = r;
        if (M[piv * 4 + col] == 0.0) return 0.0;
        if (piv != col) {
            for (int k = 0; k < 4; ++k) {
                std::swap(M[col * 4 + k], M[piv * 4 + k]);
                std::swap(I[col * 4 + k], I[piv * 4 + k]);
            }
            det = -det;
        }
        double p = M[col * 4 + col];
        det *= p;
        for (int k = 0; k < 4; ++k) { M[col * 4 + k] /= p; I[col * 4 + k] /= p; }
        for (int r = 0; r < n; ++r) {
            if (r == col) continue;
            double f = M[r * 4 + col];
            for (int k = 0; k < 4; ++k) { M[r * 4 + k] -= f * M[col * 4 + k]; I[r * 4 + k] -= f * I[col * 4 + k]; }
        }
    }
    if (Ai) std::memcpy(Ai, I, sizeof(I));
    return det;
}

static void unpack(int n, const double* src, double* dst) {  // packed n x n -> stride 4
    for (int i = 0; i < 16; ++i) dst[i] = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) dst[i * 4 + j] = src[i * n + j];
}

static bool radix_ok(int N) {
    if (N < 4 || N > 1024) return false;
    int m = N;
    for (int q : {2, 3, 5, 7, 11, 13, 17})
        while (m % q == 0) m /= q;
    return m == 1;
}

static int dalloc(pmf_ctx* c, void** p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) { cudaGetLastError(); return fail(c, PMF_E_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e)); }
    c->bytes += (int64_t)bytes;
    return PMF_OK;
}

static PencilBufs bufs(pmf_ctx* c) {
    PencilBufs b;
    b.W = c->W; b.W2 = c->W2; b.S = c->S; b.S2 = c->S2; b.st = c->st; b.partials = c->partials; b.coef = c->coef;
    b.sub = c->sub; b.z = c->z; b.gauss = c->gauss;
    return b;
}

// events around the dominant kernel of this predict (pmf_profile)
static void attach_events(pmf_ctx* c, PencilBufs& b) {
    if (c->prof) {
        if ((int)c->evs.size() < 2 * (c->nev + 1)) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            c->evs.push_back(e0);
            c->evs.push_back(e1);
        }
        b.ev0 = c->evs[2 * c->nev];
        b.ev1 = c->evs[2 * c->nev + 1];
        ++c->nev;
    }
}

static Twiddles twid(pmf_ctx* c) {
    Twiddles t;
    for (int i = 0; i < 4; ++i) t.tw[i] = c->tw[i];
    return t;
}

// Model constants of a prediction interval tau = dt*steps: e^{A tau}, the trace
// factor s (R5), and per-substep E_n = e^{-A n dt} Q e^{-A^T n dt}, P_n = e^{A n dt}.
static int prepare_model(pmf_ctx* c, double dt, int steps) {
    if (c->cached_dt == dt && c->cached_steps == steps) return PMF_OK;
    const int nx = c->d.nx;
    ModelParams mp{};
    mp.nx = nx;
    mp.l = steps;
    mp.diff_mode = c->cfg.diff_mode;
    mp.step = c->cfg.step;
    const int nsets = steps + (mp.step ? 1 : 0);      // Crank-Nicolson: grids t_0 .. t_l
    mp.dt = dt;
    double trA = 0.0;
    for (int a = 0; a < nx; ++a) trA += c->A[a * 4 + a];
    const int sgn = (c->cfg.trace_sign == PMF_TRACE_PRINTED) ? 1 : -1;
    mp.s = std::pow(1.0 + sgn * dt * trA, steps);
    double M[16];
    for (int i = 0; i < 16; ++i) M[i] = c->A[i] * (dt * steps);
    expm4(nx, M, mp.Mtau);
    std::memcpy(mp.Q, c->Q, sizeof(mp.Q));
    std::vector<SubstepEntry> tab(nsets);
    for (int s = 0; s < nsets; ++s) {
        double Mn[16], En[16], EnT[16], T1[16];
        for (int i = 0; i < 16; ++i) Mn[i] = -c->A[i] * (dt * s);
        expm4(nx, Mn, En);                            // e^{-A n dt}
        for (int i = 0; i < 4; ++i)
            for (int j = 0; j < 4; ++j) EnT[i * 4 + j] = En[j * 4 + i];
        mat_mul(nx, En, c->Q, T1);
        mat_mul(nx, T1, EnT, tab[s].E);
        for (int i = 0; i < 16; ++i) Mn[i] = c->A[i] * (dt * s);
        expm4(nx, Mn, tab[s].P);
    }
    size_t need = sizeof(SubstepEntry) * nsets;
    if (need > c->sub_bytes) {
        if (c->sub) { cudaFree(c->sub); c->bytes -= (int64_t)c->sub_bytes; c->sub = nullptr; }
        int r = dalloc(c, (void**)&c->sub, need);
        if (r) return r;
        c->sub_bytes = need;
    }
    size_t cneed = sizeof(double) * coef_stride(steps) * (size_t)c->d.batch;
    cneed = std::max(cneed, sizeof(double) * fdm_coef_doubles(c->d.batch));
    if (cneed > c->coef_bytes) {
        if (c->coef) { cudaFree(c->coef); c->bytes -= (int64_t)c->coef_bytes; c->coef = nullptr; }
        int r = dalloc(c, (void**)&c->coef, cneed);
        if (r) return r;
        c->coef_bytes = cneed;
    }
    CK(c, cudaMemcpyAsync(c->sub, tab.data(), need, cudaMemcpyHostToDevice, c->stream), "upload substep table");
    // the host vector dies at return: make the copy complete before that
    CK(c, cudaStreamSynchronize(c->stream), "sync model upload");
    c->mp = mp;
    c->cached_dt = dt;
    c->cached_steps = steps;
    return PMF_OK;
}

static int make_lik(pmf_ctx* c, const pmf_likelihood* lik, LikParams& lp) {
    if (!lik) return fail(c, PMF_E_ARG, "likelihood is NULL");
    const int nx = c->d.nx;
    lp = LikParams{};
    lp.kind = lik->kind;
    lp.nx = nx;
    if (lik->kind == PMF_LIK_RANGE_GAUSS) {
        if (!(lik->sigma > 0.0)) return fail(c, PMF_E_ARG, "range likelihood needs sigma > 0");
        lp.nz = 1;
        lp.inv_sigma = 1.0 / lik->sigma;
        lp.lognorm = -std::log(lik->sigma * std::sqrt(2.0 * M_PI));
        return PMF_OK;
    }
    if (lik->kind == PMF_LIK_TERRAIN_GM) {
        if (!c->terrain) return fail(c, PMF_E_STATE, "TERRAIN_GM likelihood needs pmf_set_terrain first");
        if (lik->ncomp < 1 || lik->ncomp > 4) return fail(c, PMF_E_ARG, "TERRAIN_GM: ncomp must be 1..4");
        double wsum = 0.0;
        for (int g = 0; g < lik->ncomp; ++g) {
            if (!(lik->gm_w[g] >= 0.0) || !(lik->gm_var[g] > 0.0) || !std::isfinite(lik->gm_mu[g]))
                return fail(c, PMF_E_ARG, "TERRAIN_GM: weights >= 0, variances > 0, finite means");
            wsum += lik->gm_w[g];
        }
        if (!(wsum > 0.0)) return fail(c, PMF_E_ARG, "TERRAIN_GM: weights sum to zero");
        lp.nz = 1;
        lp.ncomp = lik->ncomp;
        for (int g = 0; g < lik->ncomp; ++g) {
            lp.gm_logc[g] = std::log(lik->gm_w[g] / wsum) - 0.5 * std::log(2.0 * M_PI * lik->gm_var[g]);
            lp.gm_mu[g] = lik->gm_mu[g];
            lp.gm_ivar[g] = 1.0 / lik->gm_var[g];
        }
        lp.ix = c->t_ix;
        lp.iy = c->t_iy;
        lp.trow = c->t_rows;
        lp.tcol = c->t_cols;
        lp.tx0 = c->t_x0;
        lp.ty0 = c->t_y0;
        lp.tidx = 1.0 / c->t_dx;
        lp.tidy = 1.0 / c->t_dy;
        lp.terrain = c->terrain;
        return PMF_OK;
    }
    if (lik->kind != PMF_LIK_LINEAR_GAUSS) return fail(c, PMF_E_ARG, "unknown likelihood kind");
    const int nz = lik->nz;
    if (nz < 1 || nz > PMF_MAX_NZ) return fail(c, PMF_E_ARG, "nz must be 1..4");
    lp.nz = nz;
    for (int i = 0; i < nz; ++i)
        for (int a = 0; a < nx; ++a) lp.H[i * 4 + a] = lik->H[i * nx + a];
    double R[16], Ri[16];
    unpack(nz, lik->R, R);
    double det = det_inv(nz, R, Ri);
    if (!(det > 0.0)) return fail(c, PMF_E_ARG, "R must be positive definite");
    std::memcpy(lp.Rinv, Ri, sizeof(Ri));
    lp.lognorm = -0.5 * (nz * std::log(2.0 * M_PI) + std::log(det));
    return PMF_OK;
}

// The caller's z is read during the call only (pmf.h OWNERSHIP): host arrays are copied
// into a context-owned pinned staging slot (double-buffered, each slot fenced by an event)
// and the asynchronous H2D copy reads that slot, never the caller's memory after return.
static int upload_z(pmf_ctx* c, const double* z, int on_device, int nz) {
    if (!z) return fail(c, PMF_E_ARG, "z is NULL");
    size_t bytes = sizeof(double) * nz * (size_t)c->d.batch;
    if (on_device) {
        CK(c, cudaMemcpyAsync(c->z, z, bytes, cudaMemcpyDeviceToDevice, c->stream), "upload z");
        return PMF_OK;
    }
    const int k = c->z_slot;
    if (!c->z_stage[k]) {
        CK(c, cudaMallocHost((void**)&c->z_stage[k], sizeof(double) * PMF_MAX_NZ * (size_t)c->d.batch),
           "cudaMallocHost (z staging)");
        CK(c, cudaEventCreateWithFlags(&c->z_ev[k], cudaEventDisableTiming), "z staging event");
    } else {
        CK(c, cudaEventSynchronize(c->z_ev[k]), "z staging slot reuse");   // its previous copy is done
    }
    std::memcpy(c->z_stage[k], z, bytes);
    CK(c, cudaMemcpyAsync(c->z, c->z_stage[k], bytes, cudaMemcpyHostToDevice, c->stream), "upload z");
    CK(c, cudaEventRecord(c->z_ev[k], c->stream), "z staging event");
    c->z_slot ^= 1;
    return PMF_OK;
}

// Execute pending regrid/predict, optionally fused with an update (launches directly).
static int flush_direct(pmf_ctx* c, const LikParams* lp) {
    if (c->sh) {
        if (c->pend.predict) c->epoch_kernel = PMF_EPOCH_SHARDED;
        return sh_flush(c, lp);
    }
    if (lp && lp->kind == PMF_LIK_TERRAIN_GM) {
        // the table likelihood is not fused into the transform kernels: predict (+ regrid)
        // first, then the standalone point update
        if (c->pend.predict || c->pend.regrid) {
            int r = flush_direct(c, nullptr);
            if (r) return r;
        }
        PencilBufs b = bufs(c);
        cudaError_t e = launch_update(c->d, c->dtype, b, *lp, c->stream, &c->launches);
        if (e != cudaSuccess) return cuda_fail(c, e, "update");
        return PMF_OK;
    }
    PencilBufs b = bufs(c);
    cudaError_t e = cudaSuccess;
    if (c->cfg.diff_mode == PMF_DIFF_FDM) {
        // FDM baseline: [regrid] -> DST-I predict (eq:FST) -> normalise by summation -> [update]
        if (c->pend.regrid) {
            e = launch_regrid(c->d, c->dtype, b, c->pend.k_sigma, c->stream, &c->launches);
            if (e != cudaSuccess) return cuda_fail(c, e, "regrid");
            std::swap(c->W, c->W2);
            b = bufs(c);
        }
        if (c->pend.predict) {
            if (!fdm_supported(c->d, c->dtype, c->pend.steps))
                return fail(c, PMF_E_DT, "FDM predictor: at most 64 substeps per predict");
            double trA = 0.0;
            for (int a = 0; a < c->d.nx; ++a) trA += c->A[a * 4 + a];
            const int sgn = (c->cfg.trace_sign == PMF_TRACE_PRINTED) ? 1 : -1;
            attach_events(c, b);
            c->epoch_kernel = PMF_EPOCH_FDM;
            e = launch_fdm_predict(c->d, c->dtype, b, c->mp, 1.0 + sgn * c->mp.dt * trA, c->stream, &c->launches);
            if (e != cudaSuccess) return cuda_fail(c, e, "FDM predict");
            b.ev0 = b.ev1 = nullptr;
            e = launch_normalise_state(c->d, c->dtype, b, c->stream, &c->launches);
            if (e != cudaSuccess) return cuda_fail(c, e, "FDM normalise");
        }
        if (lp) {
            e = launch_update(c->d, c->dtype, b, *lp, c->stream, &c->launches);
            if (e != cudaSuccess) return cuda_fail(c, e, "update");
        }
        c->pend = Pending{};
        return PMF_OK;
    }
    // nx = 1: regrid + predict + update + moments of every filter in ONE launch
    if (c->d.nx == 1 && c->pend.predict && line_epoch_supported(c->d, c->pend.steps + (c->mp.step ? 1 : 0)) &&
        std::getenv("PMF_NO_LINE_EPOCH") == nullptr) {
        attach_events(c, b);
        c->epoch_kernel = PMF_EPOCH_LINE;
        e = launch_line_epoch(c->d, c->dtype, b, twid(c), c->mp, lp, c->pend.regrid ? c->pend.k_sigma : -1.0,
                              c->stream, &c->launches);
        if (e != cudaSuccess) return cuda_fail(c, e, "line epoch kernel");
        c->pend = Pending{};
        return PMF_OK;
    }
    // nx = 2 at 256^2 (fp64, Euler): the whole epoch in ONE launch of an 8-CTA cluster that
    // keeps the half spectrum in distributed shared memory (kernels_cluster.cu)
    if (c->path == PMF_PATH_PENCIL && c->pend.predict && cluster_epoch_supported(c->d, c->dtype, c->mp) &&
        std::getenv("PMF_NO_CLUSTER") == nullptr) {
        attach_events(c, b);
        c->epoch_kernel = PMF_EPOCH_CLUSTER;
        e = launch_cluster_epoch(c->d, b, twid(c), c->mp, lp, c->pend.regrid ? c->pend.k_sigma : -1.0, c->stream,
                                 &c->launches);
        if (e != cudaSuccess) return cuda_fail(c, e, "cluster epoch kernel");
        c->pend = Pending{};
        return PMF_OK;
    }
    // the resident kernel keeps 3 coefficients per substep (l + 1 sets for Crank-Nicolson) in
    // two shared-memory buffers next to its 141 KB spectrum: up to 1024 substeps per call
    const bool resident = c->path == PMF_PATH_RESIDENT && c->pend.predict && c->pend.steps <= 1024;
    if (resident) {
        attach_events(c, b);
        c->epoch_kernel = PMF_EPOCH_RESIDENT;
        e = launch_resident(c->d, c->dtype, b, twid(c), &c->mp, lp, c->pend.regrid ? c->pend.k_sigma : -1.0,
                            c->stream, &c->launches);
        if (e != cudaSuccess) return cuda_fail(c, e, "resident epoch kernel");
        c->pend = Pending{};
        return PMF_OK;
    }
    // plane path: regrid (if pending) fused into the forward pass, predict, update
    if (c->path == PMF_PATH_PLANE && c->pend.predict && plane_supported(c->d, c->pend.steps)) {
        attach_events(c, b);
        c->epoch_kernel = PMF_EPOCH_PLANE;
        e = launch_plane(c->d, c->dtype, b, c->mp, lp, c->pend.regrid ? c->pend.k_sigma : -1.0, c->stream,
                         &c->launches);
        if (e != cudaSuccess) return cuda_fail(c, e, "plane path");
        c->pend = Pending{};
        return PMF_OK;
    }
    if (c->pend.regrid) {
        e = launch_regrid(c->d, c->dtype, b, c->pend.k_sigma, c->stream, &c->launches);
        if (e != cudaSuccess) return cuda_fail(c, e, "regrid");
        std::swap(c->W, c->W2);
    }
    if (c->pend.predict && !c->S && c->d.nx > 1) {   // resident context asked for a very long interval
        int r = dalloc(c, &c->S, 2 * c->esize * (size_t)c->d.nspec * c->d.batch);
        if (r) return r;
    }
    b = bufs(c);
    if (c->pend.predict) {
        attach_events(c, b);
        c->epoch_kernel = PMF_EPOCH_PENCIL;
        e = launch_predict_pencil(c->d, c->dtype, b, twid(c), c->mp, lp, c->stream, &c->launches);
        if (e != cudaSuccess) return cuda_fail(c, e, "predict");
    } else if (lp) {
        e = launch_update(c->d, c->dtype, b, *lp, c->stream, &c->launches);
        if (e != cudaSuccess) return cuda_fail(c, e, "update");
    }
    c->pend = Pending{};
    return PMF_OK;
}

// Replay the flush as a CUDA graph when the same work was captured before: an epoch of
// pmf_step launches the identical kernel sequence with identical arguments (the buffers
// are fixed; the pencil regrid alternates W / W2, which is part of the key). Capture
// needs a non-legacy stream; any capture failure falls back to direct launches.
static void graph_key(const pmf_ctx* c, const LikParams* lp, GraphKey& k) {
    std::memset(&k, 0, sizeof(k));
    k.path = c->path;
    k.predict = c->pend.predict;
    k.steps = c->pend.steps;
    k.regrid = c->pend.regrid;
    k.has_lp = lp != nullptr;
    k.prof = c->prof;
    k.diff_mode = c->cfg.diff_mode;
    k.dt = c->pend.dt;
    k.k_sigma = c->pend.k_sigma;
    if (lp) std::memcpy(&k.lp, lp, sizeof(LikParams));
    k.W = c->W;
    k.W2 = c->W2;
    k.S = c->S;
    k.S2 = c->S2;
    k.sub = c->sub;
    k.coef = c->coef;
    k.terrain = c->terrain;
    k.partials = c->partials;
    k.z = c->z;
}

static int flush(pmf_ctx* c, const LikParams* lp) {
    const bool work = c->pend.predict || c->pend.regrid || lp;
    if (c->sh || !c->graphs || c->stream == nullptr || !work) return flush_direct(c, lp);
    GraphKey key;
    graph_key(c, lp, key);
    GraphEntry* hit = nullptr;
    for (auto& g : c->gcache)
        if (std::memcmp(&g.key, &key, sizeof(key)) == 0) hit = &g;
    if (hit) {
        if (c->prof && hit->ev_node[0] && hit->ev_node[1]) {
            // a fresh event pair per replay (pmf_profile_read sums the pairs)
            PencilBufs b;
            attach_events(c, b);
            CK(c, cudaGraphExecEventRecordNodeSetEvent(hit->exec, hit->ev_node[0], b.ev0), "graph event");
            CK(c, cudaGraphExecEventRecordNodeSetEvent(hit->exec, hit->ev_node[1], b.ev1), "graph event");
        }
        CK(c, cudaGraphLaunch(hit->exec, c->stream), "graph launch");
        if (hit->swaps) std::swap(c->W, c->W2);
        c->launches += hit->launches;
        c->pend = Pending{};
        return PMF_OK;
    }
    if (c->gcache.size() >= 8) return flush_direct(c, lp);
    // capture this flush
    const Pending saved = c->pend;
    void* W0 = c->W;
    const int64_t l0 = c->launches;
    const int nev0 = c->nev;
    if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
        cudaGetLastError();
        c->graphs = false;
        return flush_direct(c, lp);
    }
    int r = flush_direct(c, lp);
    cudaGraph_t g = nullptr;
    cudaError_t ec = cudaStreamEndCapture(c->stream, &g);
    cudaGraphExec_t exec = nullptr;
    if (r == PMF_OK && ec == cudaSuccess && g && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess) {
        GraphEntry e;
        e.key = key;
        e.exec = exec;
        e.swaps = c->W != W0;
        e.launches = c->launches - l0;
        if (c->prof && c->nev > nev0) {
            // the event-record nodes of the pair this flush attached (retargeted per replay)
            cudaEvent_t want[2] = {c->evs[2 * nev0], c->evs[2 * nev0 + 1]};
            size_t n = 0;
            cudaGraphGetNodes(g, nullptr, &n);
            std::vector<cudaGraphNode_t> nodes(n);
            cudaGraphGetNodes(g, nodes.data(), &n);
            for (auto nd : nodes) {
                cudaGraphNodeType ty;
                cudaGraphNodeGetType(nd, &ty);
                if (ty != cudaGraphNodeTypeEventRecord) continue;
                cudaEvent_t ev;
                cudaGraphEventRecordNodeGetEvent(nd, &ev);
                for (int q = 0; q < 2; ++q)
                    if (ev == want[q]) e.ev_node[q] = nd;
            }
        }
        e.graph = g;
        c->gcache.push_back(e);
        CK(c, cudaGraphLaunch(exec, c->stream), "graph launch");
        return PMF_OK;
    }
    // capture failed: undo the host-side effects and launch directly
    cudaGetLastError();
    if (g) cudaGraphDestroy(g);
    if (exec) cudaGraphExecDestroy(exec);
    c->graphs = false;
    c->pend = saved;
    if (c->W != W0) std::swap(c->W, c->W2);
    c->launches = l0;
    c->nev = nev0;
    return flush_direct(c, lp);
}

template <typename T>
static void make_twiddles(int N, std::vector<T>& out) {
    out.resize(2 * N);
    const long double pi = 3.141592653589793238462643383279502884L;
    for (int m = 0; m < N; ++m) {
        long double ang = 2.0L * pi * (long double)m / (long double)N;
        out[2 * m] = (T)cosl(ang);
        out[2 * m + 1] = (T)(-sinl(ang));
    }
}

// argument validation shared by pmf_create and pmf_create_sharded (no device access)
int pmf_validate_model(const pmf_config* cfg, const double* A, const double* Q, double* Qs) {
    const int nx = cfg->nx;
    if (nx < 1 || nx > PMF_MAX_NX) return fail(nullptr, PMF_E_ARG, "nx must be 1..4");
    if (cfg->batch < 1) return fail(nullptr, PMF_E_ARG, "batch must be >= 1");
    if (cfg->dtype != PMF_F64 && cfg->dtype != PMF_F32) return fail(nullptr, PMF_E_ARG, "bad dtype");
    if (cfg->diff_mode != PMF_DIFF_FULL && cfg->diff_mode != PMF_DIFF_AXIS_LITERAL && cfg->diff_mode != PMF_DIFF_FDM)
        return fail(nullptr, PMF_E_ARG, "bad diff_mode");
    if (cfg->step != PMF_STEP_EULER && cfg->step != PMF_STEP_CN) return fail(nullptr, PMF_E_ARG, "bad step");
    if (cfg->grid != PMF_GRID_AXIS && cfg->grid != PMF_GRID_EIGEN) return fail(nullptr, PMF_E_ARG, "bad grid");
    if (cfg->grid == PMF_GRID_EIGEN && cfg->diff_mode != PMF_DIFF_FULL)
        return fail(nullptr, PMF_E_ARG, "eigen-aligned grids need PMF_DIFF_FULL (cross terms)");
    if (cfg->diff_mode == PMF_DIFF_FDM) {
        if (cfg->step != PMF_STEP_EULER) return fail(nullptr, PMF_E_ARG, "FDM predictor: explicit steps only");
        if (cfg->dtype != PMF_F64) return fail(nullptr, PMF_E_ARG, "FDM predictor: fp64 only");
        for (int m = 0; m < nx; ++m)
            if (cfg->n[m] != 32 && cfg->n[m] != 64 && cfg->n[m] != 96 && cfg->n[m] != 128)
                return fail(nullptr, PMF_E_RADIX, "FDM predictor: N per axis in {32, 64, 96, 128}");
    }
    for (int m = 0; m < nx; ++m) {
        if (cfg->n[m] % 2) return fail(nullptr, PMF_E_ODD_N, "points per axis must be even (P:219)");
        if (!radix_ok(cfg->n[m])) return fail(nullptr, PMF_E_RADIX, "N must be a product of 2, 3, 5, 7, 11, 13, 17 in [4, 1024]");
    }
    unpack(nx, Q, Qs);
    for (int i = 0; i < nx; ++i) {
        for (int j = 0; j < nx; ++j) {
            if (!std::isfinite(Qs[i * 4 + j]) || !std::isfinite(A[i * nx + j]))
                return fail(nullptr, PMF_E_ARG, "A and Q must be finite");
            double scale = std::max(std::fabs(Qs[i * 4 + j]), std::fabs(Qs[j * 4 + i]));
            if (std::fabs(Qs[i * 4 + j] - Qs[j * 4 + i]) > 1e-12 * std::max(scale, 1e-300) &&
                std::fabs(Qs[i * 4 + j] - Qs[j * 4 + i]) > 0)
                return fail(nullptr, PMF_E_Q_NOT_PSD, "Q must be symmetric");
        }
    }
    double ev[4];
    sym_eig(nx, Qs, ev);
    double qmax = 0.0;
    for (int i = 0; i < nx; ++i) qmax = std::max(qmax, std::fabs(ev[i]));
    for (int i = 0; i < nx; ++i)
        if (ev[i] < -1e-12 * std::max(qmax, 1e-300)) return fail(nullptr, PMF_E_Q_NOT_PSD, "Q must be PSD");
    if (cfg->diff_mode == PMF_DIFF_AXIS_LITERAL || cfg->diff_mode == PMF_DIFF_FDM)
        for (int i = 0; i < nx; ++i)
            for (int j = 0; j < nx; ++j)
                if (i != j && Qs[i * 4 + j] != 0.0)
                    return fail(nullptr, PMF_E_ARG,
                                "AXIS_LITERAL / FDM need a diagonal Q (Alg. 3 uses Q^(m,m); eq:FDM per axis)");

    return PMF_OK;
}

// ---------------------------------------------------------------- shared helpers (pmf_ctx_impl.h)
void pmf_profile_events(pmf_ctx* c, cudaEvent_t* e0, cudaEvent_t* e1) {
    PencilBufs b;
    attach_events(c, b);
    *e0 = b.ev0;
    *e1 = b.ev1;
}
int pmf_fail(pmf_ctx* c, int code, const std::string& msg) { return fail(c, code, msg); }
int pmf_cuda_fail(pmf_ctx* c, cudaError_t e, const char* where) { return cuda_fail(c, e, where); }
int pmf_dalloc(pmf_ctx* c, void** p, size_t bytes) { return dalloc(c, p, bytes); }
int pmf_prepare_model(pmf_ctx* c, double dt, int steps) { return prepare_model(c, dt, steps); }
int pmf_make_lik(pmf_ctx* c, const pmf_likelihood* lik, LikParams& lp) { return make_lik(c, lik, lp); }
double pmf_det_inv(int n, const double* A, double* Ai) { return det_inv(n, A, Ai); }
void pmf_unpack(int n, const double* src, double* dst) { unpack(n, src, dst); }
template <typename T>
void pmf_make_twiddles(int N, std::vector<T>& out) { make_twiddles<T>(N, out); }
template void pmf_make_twiddles<double>(int, std::vector<double>&);
template void pmf_make_twiddles<float>(int, std::vector<float>&);

// ============================================================================ ABI
extern "C" {

const char* pmf_version(void) { return "pmf-b200 0.1 (sm_100a)"; }

const char* pmf_last_error(const pmf_ctx* ctx) {
    if (!ctx) return g_create_error.c_str();
    return ctx->err.c_str();
}

int pmf_create(const pmf_config* cfg, const double* A, const double* Q, pmf_ctx** out) {
    if (!cfg || !A || !Q || !out) return fail(nullptr, PMF_E_ARG, "null argument");
    *out = nullptr;
    const int nx = cfg->nx;
    double Qs[16];
    {
        int rv = pmf_validate_model(cfg, A, Q, Qs);
        if (rv) return rv;
    }

    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(nullptr, PMF_E_CUDA, "no CUDA device available (the library has no CPU fallback)");
    }
    if (cfg->device < 0 || cfg->device >= ndev) return fail(nullptr, PMF_E_ARG, "bad device ordinal");
    e = cudaSetDevice(cfg->device);
    if (e != cudaSuccess) return fail(nullptr, PMF_E_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, cfg->device);
    if (prop.major != 10) return fail(nullptr, PMF_E_CUDA, "device is not sm_100 (Blackwell B200)");

    pmf_ctx* c = new pmf_ctx();
    c->cfg = *cfg;
    c->dtype = cfg->dtype;
    c->esize = cfg->dtype == PMF_F64 ? 8 : 4;
    c->stream = (cudaStream_t)cfg->stream;
    c->graphs = std::getenv("PMF_NO_GRAPHS") == nullptr;
    unpack(nx, A, c->A);
    std::memcpy(c->Q, Qs, sizeof(Qs));
    Dims& d = c->d;
    d.nx = nx;
    d.ntot = 1;
    for (int m = 0; m < 4; ++m) d.n[m] = m < nx ? cfg->n[m] : 1;
    for (int m = 0; m < nx; ++m) d.ntot *= d.n[m];
    d.H0 = d.n[0] / 2 + 1;
    d.nspec = d.ntot / d.n[0] * d.H0;
    d.batch = cfg->batch;
    for (int m = 0; m < 4; ++m) {
        d.ng[m] = d.n[m];
        d.lo[m] = 0;
    }
    d.src_lo = 0;
    d.src_n = d.n[nx - 1];
    d.grid = cfg->grid;

    bool res_ok = resident_supported(d, c->dtype);
    bool plane_ok = plane_supported(d, 1);
    if (cfg->path == PMF_PATH_RESIDENT && !res_ok) {
        delete c;
        return fail(nullptr, PMF_E_ARG, "resident path not supported for this grid/dtype");
    }
    if (cfg->path == PMF_PATH_PLANE && !plane_ok) {
        delete c;
        return fail(nullptr, PMF_E_ARG, "plane path not supported for this grid");
    }
    if (cfg->path == PMF_PATH_PENCIL) c->path = PMF_PATH_PENCIL;
    else if (cfg->path == PMF_PATH_RESIDENT || (cfg->path == PMF_PATH_AUTO && res_ok)) c->path = PMF_PATH_RESIDENT;
    else if (cfg->path == PMF_PATH_PLANE || (cfg->path == PMF_PATH_AUTO && plane_ok)) c->path = PMF_PATH_PLANE;
    else c->path = PMF_PATH_PENCIL;

    const size_t wbytes = c->esize * (size_t)d.ntot * d.batch;
    int r = PMF_OK;
    if (!r) r = dalloc(c, &c->W, wbytes);
    if (!r) r = dalloc(c, &c->W2, wbytes);
    if (!r && c->path != PMF_PATH_RESIDENT && nx > 1) r = dalloc(c, &c->S, 2 * c->esize * (size_t)d.nspec * d.batch);
    if (!r && c->path == PMF_PATH_PLANE && nx == 4) r = dalloc(c, &c->S2, 2 * c->esize * (size_t)d.nspec * d.batch);
    if (!r) r = dalloc(c, (void**)&c->st, sizeof(FilterState) * d.batch);
    // reduction scratch: the largest per-pass block count (pencil C2R rows / points kernels)
    size_t nblk = (size_t)d.batch * 1024;
    nblk = std::max(nblk, (size_t)(d.ntot / d.n[0]) * d.batch);
    c->partials_bytes = nblk * NMOM * sizeof(double);
    if (!r) r = dalloc(c, (void**)&c->partials, c->partials_bytes);
    if (!r) r = dalloc(c, (void**)&c->z, sizeof(double) * PMF_MAX_NZ * d.batch);
    if (!r) r = dalloc(c, (void**)&c->gauss, sizeof(double) * 21 * d.batch);
    if (!r) r = dalloc(c, (void**)&c->mom_dev, sizeof(double) * (nx + nx * nx + 2) * d.batch);
    if (!r && cudaMallocHost((void**)&c->mom_host, sizeof(double) * (nx + nx * nx + 2) * d.batch) != cudaSuccess)
        r = fail(c, PMF_E_NOMEM, "cudaMallocHost (moments)");
    for (int m = 0; m < nx && !r; ++m) {
        const int N = d.n[m];
        if (c->dtype == PMF_F64) {
            std::vector<double> t;
            make_twiddles(N, t);
            r = dalloc(c, &c->tw[m], t.size() * sizeof(double));
            if (!r && cudaMemcpy(c->tw[m], t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
                r = fail(c, PMF_E_CUDA, "twiddle upload");
        } else {
            std::vector<float> t;
            make_twiddles(N, t);
            r = dalloc(c, &c->tw[m], t.size() * sizeof(float));
            if (!r && cudaMemcpy(c->tw[m], t.data(), t.size() * sizeof(float), cudaMemcpyHostToDevice) != cudaSuccess)
                r = fail(c, PMF_E_CUDA, "twiddle upload");
        }
    }
    if (!r) {
        std::vector<FilterState> z(d.batch);
        std::memset(z.data(), 0, sizeof(FilterState) * d.batch);
        if (cudaMemcpy(c->st, z.data(), sizeof(FilterState) * d.batch, cudaMemcpyHostToDevice) != cudaSuccess)
            r = fail(c, PMF_E_CUDA, "state init");
    }
    if (r) {
        std::string m = c->err;
        pmf_destroy(c);
        if (!m.empty()) g_create_error = m;
        return r;
    }
    *out = c;
    return PMF_OK;
}

void pmf_destroy(pmf_ctx* c) {
    if (!c) return;
    if (c->sh) sh_destroy(c);
    cudaSetDevice(c->cfg.device);
    cudaStreamSynchronize(c->stream);
    for (auto& g : c->gcache) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
    }
    void* ptrs[] = {c->W, c->W2, c->S, c->S2, c->terrain, c->st, c->partials, c->coef, c->sub, c->z, c->gauss, c->mom_dev,
                    c->tw[0], c->tw[1], c->tw[2], c->tw[3]};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (c->mom_host) cudaFreeHost(c->mom_host);
    for (int k = 0; k < 2; ++k) {
        if (c->z_stage[k]) cudaFreeHost(c->z_stage[k]);
        if (c->z_ev[k]) cudaEventDestroy(c->z_ev[k]);
    }
    for (cudaEvent_t e : c->evs) cudaEventDestroy(e);
    delete c;
}

int pmf_set_gaussian(pmf_ctx* c, const double* mean, const double* cov, double k_sigma) {
    if (!c || !mean || !cov) return fail(c, PMF_E_ARG, "null argument");
    if (!(k_sigma > 0.0)) return fail(c, PMF_E_ARG, "k_sigma must be > 0");
    if (c->sh) return sh_set_gaussian(c, mean, cov, k_sigma);
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    const Dims& d = c->d;
    const int nx = d.nx;
    std::vector<FilterState> st(d.batch);
    std::vector<double> g(21 * (size_t)d.batch, 0.0);
    for (int b = 0; b < d.batch; ++b) {
        FilterState& f = st[b];
        std::memset(&f, 0, sizeof(f));
        double P[16], Pi[16];
        unpack(nx, cov + (size_t)b * nx * nx, P);
        double det = det_inv(nx, P, Pi);
        if (!(det > 0.0)) return fail(c, PMF_E_ARG, "cov must be positive definite");
        for (int a = 0; a < nx; ++a) {
            f.c[a] = mean[(size_t)b * nx + a];
            f.B[a * 4 + a] = 2.0 * k_sigma * std::sqrt(P[a * 4 + a]) / d.n[a];   // R10
            g[21 * (size_t)b + a] = mean[(size_t)b * nx + a];
        }
        if (d.grid == PMF_GRID_EIGEN && !eigen_grid(nx, d.n, P, k_sigma, f.B))   // R28
            return fail(c, PMF_E_ARG, "cov must be positive definite");
        for (int i = 0; i < 16; ++i) g[21 * (size_t)b + 4 + i] = Pi[i];
        g[21 * (size_t)b + 20] = -0.5 * (nx * std::log(2.0 * M_PI) + std::log(det));
        f.scale = 1.0;
    }
    c->pend = Pending{};
    CK(c, cudaMemcpyAsync(c->st, st.data(), sizeof(FilterState) * d.batch, cudaMemcpyHostToDevice, c->stream),
       "state upload");
    CK(c, cudaMemcpyAsync(c->gauss, g.data(), sizeof(double) * g.size(), cudaMemcpyHostToDevice, c->stream),
       "gauss upload");
    PencilBufs b = bufs(c);
    cudaError_t e = launch_init_gaussian(d, c->dtype, b, c->stream, &c->launches);
    if (e != cudaSuccess) return cuda_fail(c, e, "init_gaussian");
    CK(c, cudaStreamSynchronize(c->stream), "set_gaussian sync");
    c->have_density = true;
    c->have_update = false;
    return PMF_OK;
}

int pmf_set_state(pmf_ctx* c, const double* center, const double* B, const void* weights, int on_device) {
    if (!c || !center || !B || !weights) return fail(c, PMF_E_ARG, "null argument");
    if (c->sh) return sh_set_state(c, center, B, weights, on_device);
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    const Dims& d = c->d;
    const int nx = d.nx;
    std::vector<FilterState> st(d.batch);
    for (int b = 0; b < d.batch; ++b) {
        FilterState& f = st[b];
        std::memset(&f, 0, sizeof(f));
        unpack(nx, B + (size_t)b * nx * nx, f.B);
        if (det_inv(nx, f.B, nullptr) == 0.0) return fail(c, PMF_E_SINGULAR_GRID, "grid matrix B is singular");
        for (int a = 0; a < nx; ++a) f.c[a] = center[(size_t)b * nx + a];
        f.scale = 1.0;
    }
    c->pend = Pending{};
    CK(c, cudaMemcpyAsync(c->st, st.data(), sizeof(FilterState) * d.batch, cudaMemcpyHostToDevice, c->stream),
       "state upload");
    CK(c, cudaMemcpyAsync(c->W, weights, c->esize * (size_t)d.ntot * d.batch,
                          on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream),
       "weights upload");
    PencilBufs b = bufs(c);
    cudaError_t e = launch_normalise_state(d, c->dtype, b, c->stream, &c->launches);
    if (e != cudaSuccess) return cuda_fail(c, e, "normalise");
    CK(c, cudaStreamSynchronize(c->stream), "set_state sync");
    c->have_density = true;
    c->have_update = false;
    return PMF_OK;
}

int pmf_predict(pmf_ctx* c, double dt, int steps) {
    if (!c) return fail(c, PMF_E_ARG, "null context");
    if (!c->have_density) return fail(c, PMF_E_STATE, "no density set");
    if (!(dt > 0.0) || steps < 1 || !std::isfinite(dt)) return fail(c, PMF_E_DT, "dt must be > 0 and steps >= 1");
    double trA = 0.0;
    for (int a = 0; a < c->d.nx; ++a) trA += c->A[a * 4 + a];
    const int sgn = (c->cfg.trace_sign == PMF_TRACE_PRINTED) ? 1 : -1;
    if (!(1.0 + sgn * dt * trA > 0.0)) return fail(c, PMF_E_DT, "Euler trace factor base 1 -/+ dt tr(A) <= 0 (R5)");
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    if (c->pend.predict) {   // two predicts in a row: run the first one now
        int r = flush(c, nullptr);
        if (r) return r;
    }
    if (c->cfg.diff_mode == PMF_DIFF_FDM && !c->sh && !fdm_supported(c->d, c->dtype, steps))
        return fail(c, PMF_E_DT, "FDM predictor: at most 64 substeps per predict");
    int r = prepare_model(c, dt, steps);
    if (r) return r;
    c->pend.predict = true;
    c->pend.dt = dt;
    c->pend.steps = steps;
    return PMF_OK;
}

int pmf_update(pmf_ctx* c, const double* z, int z_on_device, const pmf_likelihood* lik) {
    if (!c) return fail(c, PMF_E_ARG, "null context");
    if (!c->have_density) return fail(c, PMF_E_STATE, "no density set");
    LikParams lp;
    int r = make_lik(c, lik, lp);
    if (r) return r;
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    r = upload_z(c, z, z_on_device, lp.nz);
    if (r) return r;
    r = flush(c, &lp);
    if (r) return r;
    c->have_update = true;
    return PMF_OK;
}

int pmf_regrid(pmf_ctx* c, double k_sigma) {
    if (!c) return fail(c, PMF_E_ARG, "null context");
    if (!c->have_update) return fail(c, PMF_E_STATE, "regrid needs the moments of an update");
    if (!(k_sigma > 0.0)) return fail(c, PMF_E_ARG, "k_sigma must be > 0");
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    if (c->pend.regrid || c->pend.predict) {
        int r = flush(c, nullptr);
        if (r) return r;
    }
    c->pend.regrid = true;
    c->pend.k_sigma = k_sigma;
    return PMF_OK;
}

int pmf_step(pmf_ctx* c, double dt, int steps, const double* z, int z_on_device, const pmf_likelihood* lik,
             double k_sigma) {
    int r = pmf_predict(c, dt, steps);
    if (r) return r;
    r = pmf_update(c, z, z_on_device, lik);
    if (r) return r;
    return pmf_regrid(c, k_sigma);
}

int pmf_moments(pmf_ctx* c, double* mean, double* cov, double* log_norm) {
    if (!c) return fail(c, PMF_E_ARG, "null context");
    if (!c->have_update) return fail(c, PMF_E_STATE, "no update has run");
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    const Dims& d = c->d;
    const int nx = d.nx, stride = nx + nx * nx + 2;
    const size_t bytes = sizeof(double) * stride * (size_t)d.batch;
    cudaError_t e = launch_pack_moments(d, c->st, c->mom_dev, c->stream, &c->launches);
    if (e != cudaSuccess) return cuda_fail(c, e, "pack moments");
    CK(c, cudaMemcpyAsync(c->mom_host, c->mom_dev, bytes, cudaMemcpyDeviceToHost, c->stream), "moments download");
    CK(c, cudaStreamSynchronize(c->stream), "moments sync");
    int bad = 0;
    for (int b = 0; b < d.batch; ++b) {
        const double* f = c->mom_host + (size_t)b * stride;
        if (f[stride - 1] != 0.0) bad = 1;
        if (mean)
            for (int a = 0; a < nx; ++a) mean[(size_t)b * nx + a] = f[a];
        if (cov)
            for (int q = 0; q < nx * nx; ++q) cov[(size_t)b * nx * nx + q] = f[nx + q];
        if (log_norm) log_norm[b] = f[nx + nx * nx];
    }
    if (bad) return fail(c, PMF_E_NO_SUPPORT, "measurement incompatible with grid support (some filter)");
    return PMF_OK;
}

int pmf_moments_async(pmf_ctx* c, double* dst) {
    if (!c || !dst) return fail(c, PMF_E_ARG, "null argument");
    if (c->sh) return fail(c, PMF_E_ARG, "pmf_moments_async: not for sharded contexts");
    if (!c->have_update) return fail(c, PMF_E_STATE, "no update has run");
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    // (a recorded regrid / predict stays pending, as with pmf_moments: the moments are the
    // last update's, and the pending work fuses into the next epoch's launch)
    cudaError_t e = launch_pack_moments(c->d, c->st, c->mom_dev, c->stream, &c->launches);
    if (e != cudaSuccess) return cuda_fail(c, e, "pack moments");
    CK(c, cudaMemcpyAsync(dst, c->mom_dev, (size_t)pmf_moments_bytes(c), cudaMemcpyDeviceToHost, c->stream),
       "moments download");
    return PMF_OK;
}

int64_t pmf_moments_bytes(const pmf_ctx* c) {
    return c ? (int64_t)sizeof(double) * (c->d.nx + c->d.nx * c->d.nx + 2) * c->d.batch : 0;
}

int pmf_get_weights(pmf_ctx* c, void* dst, int dst_on_device) {
    if (!c || !dst) return fail(c, PMF_E_ARG, "null argument");
    if (!c->have_density) return fail(c, PMF_E_STATE, "no density set");
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    int r = flush(c, nullptr);
    if (r) return r;
    if (c->sh) return sh_get_weights(c, dst, dst_on_device);
    const Dims& d = c->d;
    size_t bytes = c->esize * (size_t)d.ntot * d.batch;
    PencilBufs b = bufs(c);
    if (dst_on_device) {
        cudaError_t e = launch_scale_out(d, c->dtype, b, dst, c->stream, &c->launches);
        if (e != cudaSuccess) return cuda_fail(c, e, "scale_out");
        return PMF_OK;
    }
    void* tmp = c->W2;
    bool own = false;
    if (!tmp) {
        int rr = dalloc(c, &tmp, bytes);
        if (rr) return rr;
        own = true;
    }
    cudaError_t e = launch_scale_out(d, c->dtype, b, tmp, c->stream, &c->launches);
    if (e == cudaSuccess) e = cudaMemcpyAsync(dst, tmp, bytes, cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (own) { cudaFree(tmp); c->bytes -= (int64_t)bytes; }
    if (e != cudaSuccess) return cuda_fail(c, e, "get_weights");
    return PMF_OK;
}

int pmf_get_grid(pmf_ctx* c, double* center, double* B) {
    if (!c) return fail(c, PMF_E_ARG, "null context");
    if (!c->have_density) return fail(c, PMF_E_STATE, "no density set");
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    int r = flush(c, nullptr);
    if (r) return r;
    const Dims& d = c->d;
    std::vector<FilterState> st(d.batch);
    CK(c, cudaMemcpyAsync(st.data(), c->st, sizeof(FilterState) * d.batch, cudaMemcpyDeviceToHost, c->stream),
       "state download");
    CK(c, cudaStreamSynchronize(c->stream), "grid sync");
    const int nx = d.nx;
    for (int b = 0; b < d.batch; ++b)
        for (int a = 0; a < nx; ++a) {
            if (center) center[(size_t)b * nx + a] = st[b].c[a];
            if (B)
                for (int q = 0; q < nx; ++q) B[(size_t)b * nx * nx + a * nx + q] = st[b].B[a * 4 + q];
        }
    return PMF_OK;
}

int pmf_sync(pmf_ctx* c) {
    if (!c) return fail(c, PMF_E_ARG, "null context");
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    if (c->have_density) {
        int r = flush(c, nullptr);
        if (r) return r;
    }
    CK(c, cudaStreamSynchronize(c->stream), "sync");
    return PMF_OK;
}

int64_t pmf_launch_count(const pmf_ctx* c) { return c ? c->launches : 0; }

int pmf_set_terrain(pmf_ctx* c, const double* heights, int nrow, int ncol, double x0, double y0, double dx,
                    double dy, int ix, int iy) {
    if (!c || !heights) return fail(c, PMF_E_ARG, "null argument");
    if (c->sh) return fail(c, PMF_E_ARG, "terrain likelihood: not for sharded contexts");
    if (nrow < 2 || ncol < 2 || !(dx > 0.0) || !(dy > 0.0) || ix < 0 || iy < 0 || ix >= c->d.nx ||
        iy >= c->d.nx || ix == iy)
        return fail(c, PMF_E_ARG, "terrain: nrow, ncol >= 2; dx, dy > 0; ix != iy state components");
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    const size_t bytes = sizeof(double) * (size_t)nrow * ncol;
    if (c->terrain) {
        CK(c, cudaStreamSynchronize(c->stream), "sync");
        cudaFree(c->terrain);
        c->terrain = nullptr;
    }
    int r = dalloc(c, (void**)&c->terrain, bytes);
    if (r) return r;
    CK(c, cudaMemcpy(c->terrain, heights, bytes, cudaMemcpyHostToDevice), "terrain upload");
    c->t_rows = nrow;
    c->t_cols = ncol;
    c->t_x0 = x0;
    c->t_y0 = y0;
    c->t_dx = dx;
    c->t_dy = dy;
    c->t_ix = ix;
    c->t_iy = iy;
    return PMF_OK;
}

int pmf_use_graphs(pmf_ctx* c, int enable) {
    if (!c) return fail(c, PMF_E_ARG, "null context");
    c->graphs = enable != 0;
    return PMF_OK;
}

int pmf_profile(pmf_ctx* c, int enable) {
    if (!c) return fail(c, PMF_E_ARG, "null context");
    c->prof = enable != 0;
    c->nev = 0;
    return PMF_OK;
}

int pmf_profile_read(pmf_ctx* c, double* total_ms, int64_t* count) {
    if (!c || !total_ms || !count) return fail(c, PMF_E_ARG, "null argument");
    CK(c, cudaSetDevice(c->cfg.device), "cudaSetDevice");
    double tot = 0.0;
    for (int i = 0; i < c->nev; ++i) {
        CK(c, cudaEventSynchronize(c->evs[2 * i + 1]), "profile event");
        float ms = 0.0f;
        CK(c, cudaEventElapsedTime(&ms, c->evs[2 * i], c->evs[2 * i + 1]), "profile elapsed");
        tot += ms;
    }
    *total_ms = tot;
    *count = c->nev;
    c->nev = 0;
    return PMF_OK;
}
int64_t pmf_device_bytes(const pmf_ctx* c) { return c ? c->bytes : 0; }
int pmf_path(const pmf_ctx* c) { return c ? c->path : -1; }
int pmf_epoch_kernel(const pmf_ctx* c) { return c ? c->epoch_kernel : -1; }

}  // extern "C"

// Debug only (not in pmf.h): per-phase cycle counters of the nx = 4 three-pass kernels in
// builds compiled with -DPMF_QPROF (tools/qprof.py); zeros otherwise.
extern "C" int pmf_debug_counters(double* out, int n, int reset) {
    int r = quad_debug_counters(out, n < 16 ? n : 16, reset);
    if (r == 0 && n > 16) r = resident_debug_counters(out + 16, n - 16, reset);
    return r;
}
