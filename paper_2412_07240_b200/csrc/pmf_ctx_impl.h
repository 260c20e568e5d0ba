// pmf_ctx_impl.h -- the context object behind the C ABI and the host helpers
// shared by pmf_host.cpp (single-device contexts) and pmf_sharded.cpp (contexts
// whose grid is split into slabs along the last axis). Not part of the ABI.
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/pmf.h"
#include "pmf_internal.h"

namespace pmf {
struct ShardSet;   // pmf_sharded.cpp
}

struct Pending {
    bool predict = false;
    double dt = 0.0;
    int steps = 0;
    bool regrid = false;
    double k_sigma = 0.0;
};

// A captured flush (CUDA graph) and what replaying it must redo on the host.
struct GraphKey {
    int path, predict, steps, regrid, has_lp, prof, diff_mode, pad;
    double dt, k_sigma;
    pmf::LikParams lp;
    // every device pointer a captured kernel takes as an argument: a reallocation (e.g.
    // prepare_model growing sub / coef for more substeps) must miss the cache
    void* W;
    void* W2;
    void* S;
    void* S2;
    void* sub;
    void* coef;
    void* terrain;
    void* partials;
    void* z;
};
struct GraphEntry {
    GraphKey key;
    cudaGraph_t graph = nullptr;                        // kept: its node handles address the exec
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t ev_node[2] = {nullptr, nullptr};   // event-record nodes (profiling)
    bool swaps = false;                                 // the flush swapped W / W2
    int64_t launches = 0;                               // kernels per replay
};

struct pmf_ctx {
    pmf_config cfg{};
    pmf::Dims d{};
    int dtype = 0;
    int path = PMF_PATH_PENCIL;
    int epoch_kernel = PMF_EPOCH_NONE;   // kernel family of the last flush that ran a predict
    size_t esize = 8;
    double A[16]{}, Q[16]{};
    cudaStream_t stream = nullptr;
    // device buffers
    void* W = nullptr;
    void* W2 = nullptr;
    void* S = nullptr;
    void* S2 = nullptr;
    double* terrain = nullptr;       // TERRAIN_GM likelihood table (pmf_set_terrain)
    int t_rows = 0, t_cols = 0, t_ix = 0, t_iy = 0;
    double t_x0 = 0, t_y0 = 0, t_dx = 1, t_dy = 1;
    pmf::FilterState* st = nullptr;
    double* partials = nullptr;
    size_t partials_bytes = 0;
    double* coef = nullptr;
    size_t coef_bytes = 0;
    pmf::SubstepEntry* sub = nullptr;
    size_t sub_bytes = 0;
    double* z = nullptr;
    // pinned staging of host measurements (pmf_update/pmf_step with z in host memory): the
    // caller's array is copied on the host during the call, the H2D copy reads the staging
    // slot; a slot is reused only after its previous copy completed (event)
    double* z_stage[2] = {nullptr, nullptr};
    cudaEvent_t z_ev[2] = {nullptr, nullptr};
    int z_slot = 0;
    double* gauss = nullptr;
    double* mom_dev = nullptr;       // compact moments [batch][nx + nx^2 + 2]
    double* mom_host = nullptr;      // pinned host mirror
    void* tw[4] = {nullptr, nullptr, nullptr, nullptr};
    int64_t bytes = 0;
    // host-side model cache (per (dt, steps))
    double cached_dt = -1.0;
    int cached_steps = -1;
    pmf::ModelParams mp{};
    // state machine
    bool have_density = false;
    bool have_update = false;
    Pending pend;
    int64_t launches = 0;
    // kernel timing (pmf_profile): event pairs around the dominant kernel of each flush
    bool prof = false;
    std::vector<cudaEvent_t> evs;
    int nev = 0;
    std::string err;
    // CUDA-graph replay of flushes (pmf_step loops launch the same sequence every epoch)
    bool graphs = true;
    std::vector<GraphEntry> gcache;
    // sharded context (slab decomposition along the last axis), else null
    pmf::ShardSet* sh = nullptr;
};

// helpers implemented in pmf_host.cpp
int pmf_fail(pmf_ctx* c, int code, const std::string& msg);
int pmf_cuda_fail(pmf_ctx* c, cudaError_t e, const char* where);
int pmf_dalloc(pmf_ctx* c, void** p, size_t bytes);
int pmf_prepare_model(pmf_ctx* c, double dt, int steps);
int pmf_make_lik(pmf_ctx* c, const pmf_likelihood* lik, pmf::LikParams& lp);
double pmf_det_inv(int n, const double* A, double* Ai);
void pmf_unpack(int n, const double* src, double* dst);
void pmf_profile_events(pmf_ctx* c, cudaEvent_t* e0, cudaEvent_t* e1);   // null when not profiling
int pmf_validate_model(const pmf_config* cfg, const double* A, const double* Q, double* Qs);
template <typename T>
void pmf_make_twiddles(int N, std::vector<T>& out);

// sharded contexts (pmf_sharded.cpp)
int sh_set_gaussian(pmf_ctx* c, const double* mean, const double* cov, double k_sigma);
int sh_set_state(pmf_ctx* c, const double* center, const double* B, const void* weights, int on_device);
int sh_flush(pmf_ctx* c, const pmf::LikParams* lp);
int sh_get_weights(pmf_ctx* c, void* dst, int on_device);
void sh_destroy(pmf_ctx* c);
