// pmf_sharded.cpp -- one large filter split into slabs along its LAST axis over
// several ranks (slab decomposition with two all-to-all
// transposes per predict and an all-reduce of the moment sums per update).
//
//   rank r holds planes [r n_loc, (r+1) n_loc) of axis L = nx-1 (real weights)
//   predict: prep -> R2C + forward C2C axes 1..L-1 (local) -> pack -> ALL-TO-ALL
//            -> last axis forward * s Psi * inverse on rank r's share of the
//               other wavenumbers (full pencils along L) -> ALL-TO-ALL back
//            -> unpack -> inverse C2C L-1..1 + C2R (+ likelihood) (local)
//   update:  per-rank moment sums -> ALL-REDUCE -> normaliser and moments
//   regrid:  host computes, from the (replicated) filter state, which old planes
//            every rank's new slab reads (R12's multilinear map); the planes move
//            by grouped send/recv into a window buffer; local resampling; sums
//            all-reduced for the renormalisation.
//
// Communication goes through an Exchanger: NCCL (libnccl loaded with dlopen;
// grouped ncclSend/ncclRecv and ncclAllReduce on the context's stream) for one
// rank per process, or in-process device copies for "virtual ranks" -- all
// shards in one context on one GPU, which runs the identical sharded code path
// and is what the single-GPU parity tests exercise.
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pmf_ctx_impl.h"

using namespace pmf;

namespace pmf {

// ---------------------------------------------------------------- NCCL (dynamically loaded)
struct NcclApi {
    using Res = int;
    using Comm = void*;
    struct UniqueId { char internal[128]; };
    Res (*GetUniqueId)(UniqueId*) = nullptr;
    Res (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
    Res (*CommDestroy)(Comm) = nullptr;
    Res (*Send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
    Res (*Recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
    Res (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
    Res (*GroupStart)() = nullptr;
    Res (*GroupEnd)() = nullptr;
    Res (*CommGetAsyncError)(Comm, Res*) = nullptr;
    const char* (*GetErrorString)(Res) = nullptr;
    bool ok = false;
    std::string why;
    static NcclApi& get() {
        static NcclApi a = load();
        return a;
    }
    static NcclApi load() {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.why = std::string("dlopen libnccl.so.2: ") + dlerror();
            return a;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        a.GetUniqueId = (Res(*)(UniqueId*))sym("ncclGetUniqueId");
        a.CommInitRank = (Res(*)(Comm*, int, UniqueId, int))sym("ncclCommInitRank");
        a.CommDestroy = (Res(*)(Comm))sym("ncclCommDestroy");
        a.Send = (Res(*)(const void*, size_t, int, int, Comm, cudaStream_t))sym("ncclSend");
        a.Recv = (Res(*)(void*, size_t, int, int, Comm, cudaStream_t))sym("ncclRecv");
        a.AllReduce = (Res(*)(const void*, void*, size_t, int, int, Comm, cudaStream_t))sym("ncclAllReduce");
        a.GroupStart = (Res(*)())sym("ncclGroupStart");
        a.GroupEnd = (Res(*)())sym("ncclGroupEnd");
        a.GetErrorString = (const char* (*)(Res))sym("ncclGetErrorString");
        a.CommGetAsyncError = (Res(*)(Comm, Res*))sym("ncclCommGetAsyncError");
        a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.AllReduce && a.GroupStart &&
               a.GroupEnd && a.CommGetAsyncError;
        if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
        return a;
    }
};
constexpr int NCCL_INT8 = 0, NCCL_FLOAT64 = 8, NCCL_SUM = 0, NCCL_IN_PROGRESS = 7;

// an NCCL call's failure (r != 0), with the library's message
static int nccl_fail(pmf_ctx* c, int r, const char* what) {
    NcclApi& api = NcclApi::get();
    std::string m = std::string(what) + " failed";
    if (api.GetErrorString) m += std::string(": ") + api.GetErrorString(r);
    return pmf_fail(c, PMF_E_NCCL, m);
}

struct Shard {
    int rank = 0;
    Dims d{};                 // local slab dims (n[L] = n_loc, lo[L] = rank * n_loc)
    void* W = nullptr;        // local real weights
    void* Wwin = nullptr;     // regrid source window (old planes)
    size_t win_planes = 0;
    void* S = nullptr;        // local half spectrum [n_loc][I]
    void* send = nullptr;     // packed blocks / back-exchange receive
    void* recv = nullptr;     // transposed block T [N_L][I_r]
    FilterState* st = nullptr;
    double* partials = nullptr;
    double* coef = nullptr;
    size_t coef_bytes = 0;
    double* tot = nullptr;    // [NMOM] per-rank sums (all-reduced in place)
    double* gauss = nullptr;
};

// one copy of `bytes` from shard-rank src (buffer offset so) to shard-rank dst (offset do)
struct Xfer {
    int src, dst;
    size_t so, dof, bytes;
};

struct ShardSet {
    int world = 1;
    int rank = 0;                       // real mode: this process's rank; virtual: -1
    bool virt = false;
    int L = 0, n_loc = 0;
    long long I = 0;                    // inner size H0 * N_1 * ... * N_{L-1}
    std::vector<long long> off;         // inner ranges per rank (world + 1)
    long long* d_off = nullptr;
    size_t plane_real = 0;              // elements per real plane (N_0 * ... * N_{L-1})
    std::vector<Shard> sh;              // virtual: world shards; real: 1
    NcclApi::Comm comm = nullptr;
    double* sum_scratch = nullptr;      // virtual all-reduce staging [world][NMOM]
    // pipelined all-to-alls of the three-pass route: the exchanges run on `xs` (a second
    // stream), ordered against the compute stream by events (created on first use)
    cudaStream_t xs = nullptr;
    std::vector<cudaEvent_t> ev;
};

}  // namespace pmf

// ============================================================================ exchanger
// asynchronous communicator errors (a peer died, a network/NVLink fault): polled after
// every enqueued exchange -- non-blocking; ncclInProgress is not an error
static int nccl_poll(pmf_ctx* c) {
    NcclApi& api = NcclApi::get();
    int ae = 0;
    if (int r = api.CommGetAsyncError(c->sh->comm, &ae)) return nccl_fail(c, r, "ncclCommGetAsyncError");
    if (ae != 0 && ae != NCCL_IN_PROGRESS) return nccl_fail(c, ae, "NCCL communicator (asynchronous error)");
    return PMF_OK;
}

static int exchange(pmf_ctx* c, const std::vector<Xfer>& xs, void* (*sbuf)(Shard&), void* (*rbuf)(Shard&),
                    cudaStream_t st = nullptr) {
    ShardSet& S = *c->sh;
    if (!st) st = c->stream;
    if (S.virt) {
        for (const Xfer& x : xs) {
            char* src = (char*)sbuf(S.sh[x.src]) + x.so;
            char* dst = (char*)rbuf(S.sh[x.dst]) + x.dof;
            if (x.bytes) {
                cudaError_t e = cudaMemcpyAsync(dst, src, x.bytes, cudaMemcpyDeviceToDevice, st);
                if (e != cudaSuccess) return pmf_cuda_fail(c, e, "virtual exchange");
            }
        }
        return PMF_OK;
    }
    NcclApi& api = NcclApi::get();
    Shard& me = S.sh[0];
    api.GroupStart();
    for (const Xfer& x : xs) {
        if (!x.bytes) continue;
        if (x.src == S.rank && x.dst == S.rank) {
            cudaError_t e = cudaMemcpyAsync((char*)rbuf(me) + x.dof, (char*)sbuf(me) + x.so, x.bytes,
                                            cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) { api.GroupEnd(); return pmf_cuda_fail(c, e, "local exchange"); }
        } else if (x.src == S.rank) {
            int r = api.Send((char*)sbuf(me) + x.so, x.bytes, NCCL_INT8, x.dst, S.comm, st);
            if (r) { api.GroupEnd(); return nccl_fail(c, r, "ncclSend"); }
        } else if (x.dst == S.rank) {
            int r = api.Recv((char*)rbuf(me) + x.dof, x.bytes, NCCL_INT8, x.src, S.comm, st);
            if (r) { api.GroupEnd(); return nccl_fail(c, r, "ncclRecv"); }
        }
    }
    if (int r = api.GroupEnd()) return nccl_fail(c, r, "ncclGroupEnd");
    return nccl_poll(c);
}

// sum of the shards' tot[0..n) over ranks (n <= NTOT), written back to every shard
constexpr int NTOT = NMOM + 1;          // 15 moment sums + the DC of the three-pass route
static int allreduce_tot(pmf_ctx* c, int n = NMOM) {
    ShardSet& S = *c->sh;
    if (!S.virt) {
        NcclApi& api = NcclApi::get();
        if (int r = api.AllReduce(S.sh[0].tot, S.sh[0].tot, n, NCCL_FLOAT64, NCCL_SUM, S.comm, c->stream))
            return nccl_fail(c, r, "ncclAllReduce");
        return nccl_poll(c);
    }
    // virtual: host-free reduction in rank order -- gather, sum on device, scatter
    for (int r = 0; r < S.world; ++r) {
        cudaError_t e = cudaMemcpyAsync(S.sum_scratch + r * n, S.sh[r].tot, n * sizeof(double),
                                        cudaMemcpyDeviceToDevice, c->stream);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "virtual allreduce gather");
    }
    cudaError_t e = launch_sum_ranks(S.sum_scratch, S.sh[0].tot, S.world, n, c->stream, &c->launches);
    if (e != cudaSuccess) return pmf_cuda_fail(c, e, "virtual allreduce sum");
    for (int r = 1; r < S.world; ++r) {
        e = cudaMemcpyAsync(S.sh[r].tot, S.sh[0].tot, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "virtual allreduce scatter");
    }
    return PMF_OK;
}

static PencilBufs shard_bufs(pmf_ctx* c, Shard& s) {
    PencilBufs b;
    b.W = s.W;
    b.W2 = nullptr;
    b.S = s.S;
    b.st = s.st;
    b.partials = s.partials;
    b.coef = s.coef;
    b.sub = c->sub;
    b.z = c->z;
    b.gauss = s.gauss;
    return b;
}

static Twiddles twid(pmf_ctx* c) {
    Twiddles t;
    for (int i = 0; i < 4; ++i) t.tw[i] = c->tw[i];
    return t;
}

static int finalize_all(pmf_ctx* c, int mode, double ks) {
    ShardSet& S = *c->sh;
    int r = allreduce_tot(c);
    if (r) return r;
    for (Shard& s : S.sh) {
        cudaError_t e = launch_finalize_tot(s.d, s.st, s.tot, mode, ks, c->stream, &c->launches);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "finalize");
    }
    return PMF_OK;
}

// ============================================================================ create / destroy
extern "C" int pmf_nccl_unique_id(void* out128) {
    if (!out128) return pmf_fail(nullptr, PMF_E_ARG, "null argument");
    NcclApi& api = NcclApi::get();
    if (!api.ok) return pmf_fail(nullptr, PMF_E_NCCL, api.why);
    NcclApi::UniqueId id;
    if (int r = api.GetUniqueId(&id)) return nccl_fail(nullptr, r, "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
    return PMF_OK;
}

extern "C" int pmf_create_sharded(const pmf_config* cfg, const double* A, const double* Q, int rank, int world,
                                  const void* unique_id, pmf_ctx** out) {
    if (!cfg || !A || !Q || !out) return pmf_fail(nullptr, PMF_E_ARG, "null argument");
    *out = nullptr;
    double Qs[16];
    int rv = pmf_validate_model(cfg, A, Q, Qs);
    if (!rv && cfg->diff_mode == PMF_DIFF_FDM) rv = pmf_fail(nullptr, PMF_E_ARG, "FDM predictor: not sharded");
    if (!rv && cfg->grid != PMF_GRID_AXIS) rv = pmf_fail(nullptr, PMF_E_ARG, "eigen-aligned grids: not sharded");
    if (rv) return rv;
    const int nx = cfg->nx, L = nx - 1;
    if (nx < 2) return pmf_fail(nullptr, PMF_E_ARG, "sharding needs nx >= 2 (slabs along the last axis)");
    if (cfg->batch != 1) return pmf_fail(nullptr, PMF_E_ARG, "a sharded context holds one filter (batch = 1)");
    if (world < 1 || cfg->n[L] % world) return pmf_fail(nullptr, PMF_E_ARG, "N of the last axis must divide by world");
    const bool virt = unique_id == nullptr;
    if (!virt && (rank < 0 || rank >= world)) return pmf_fail(nullptr, PMF_E_ARG, "bad rank");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return pmf_fail(nullptr, PMF_E_CUDA, "no CUDA device available (the library has no CPU fallback)");
    }
    if (cfg->device < 0 || cfg->device >= ndev) return pmf_fail(nullptr, PMF_E_ARG, "bad device ordinal");
    cudaSetDevice(cfg->device);
    pmf_ctx* c = new pmf_ctx();
    c->cfg = *cfg;
    c->dtype = cfg->dtype;
    c->esize = cfg->dtype == PMF_F64 ? 8 : 4;
    c->stream = (cudaStream_t)cfg->stream;
    c->path = PMF_PATH_PENCIL;
    pmf_unpack(nx, A, c->A);
    std::memcpy(c->Q, Qs, sizeof(Qs));
    // global dims (used by pmf_moments / pmf_get_grid through c->d and c->st)
    Dims& g = c->d;
    g.nx = nx;
    g.ntot = 1;
    for (int m = 0; m < 4; ++m) g.n[m] = m < nx ? cfg->n[m] : 1;
    for (int m = 0; m < nx; ++m) g.ntot *= g.n[m];
    g.H0 = g.n[0] / 2 + 1;
    g.nspec = g.ntot / g.n[0] * g.H0;
    g.batch = 1;
    for (int m = 0; m < 4; ++m) { g.ng[m] = g.n[m]; g.lo[m] = 0; }
    g.src_lo = 0;
    g.src_n = g.n[L];
    ShardSet* S = new ShardSet();
    c->sh = S;
    S->world = world;
    S->virt = virt;
    S->rank = virt ? -1 : rank;
    S->L = L;
    S->n_loc = g.n[L] / world;
    S->I = g.nspec / g.n[L];
    S->plane_real = (size_t)(g.ntot / g.n[L]);
    S->off.resize(world + 1);
    for (int r = 0; r <= world; ++r) S->off[r] = S->I * r / world;
    int err = PMF_OK;
    auto fail = [&](int code, const std::string& m) {
        if (!err) err = pmf_fail(c, code, m);
        return err;
    };
    if (!virt) {
        NcclApi& api = NcclApi::get();
        if (!api.ok) fail(PMF_E_NCCL, api.why);
        else {
            NcclApi::UniqueId id;
            std::memcpy(&id, unique_id, sizeof(id));
            if (int r = api.CommInitRank(&S->comm, world, id, rank)) {
                const std::string m = std::string("ncclCommInitRank failed") +
                                      (api.GetErrorString ? std::string(": ") + api.GetErrorString(r) : "");
                fail(PMF_E_NCCL, m);
            }
        }
    }
    const int nshards = virt ? world : 1;
    const size_t cs = c->esize * 2;                 // complex element
    long long Imax = 0;
    for (int r = 0; r < world; ++r) Imax = std::max(Imax, S->off[r + 1] - S->off[r]);
    for (int k = 0; k < nshards && !err; ++k) {
        Shard sd;
        sd.rank = virt ? k : rank;
        sd.d = g;
        sd.d.n[L] = S->n_loc;
        sd.d.lo[L] = sd.rank * S->n_loc;
        sd.d.ntot = g.ntot / world;
        sd.d.nspec = g.nspec / world;
        sd.d.src_lo = sd.d.lo[L];
        sd.d.src_n = S->n_loc;
        sd.win_planes = (size_t)std::min(g.n[L], S->n_loc + 8);
        const size_t spec = (size_t)std::max<long long>(S->n_loc * S->I, (long long)g.n[L] * Imax);
        if (!err && pmf_dalloc(c, &sd.W, c->esize * (size_t)sd.d.ntot)) err = PMF_E_NOMEM;
        if (!err && pmf_dalloc(c, &sd.Wwin, c->esize * S->plane_real * sd.win_planes)) err = PMF_E_NOMEM;
        if (!err && pmf_dalloc(c, &sd.S, cs * (size_t)S->n_loc * S->I)) err = PMF_E_NOMEM;
        if (!err && pmf_dalloc(c, &sd.send, cs * spec)) err = PMF_E_NOMEM;
        if (!err && pmf_dalloc(c, &sd.recv, cs * spec)) err = PMF_E_NOMEM;
        if (!err && pmf_dalloc(c, (void**)&sd.st, sizeof(FilterState))) err = PMF_E_NOMEM;
        if (!err && pmf_dalloc(c, (void**)&sd.partials, sizeof(double) * NMOM * 2048)) err = PMF_E_NOMEM;
        if (!err && pmf_dalloc(c, (void**)&sd.tot, sizeof(double) * NTOT)) err = PMF_E_NOMEM;
        if (!err && pmf_dalloc(c, (void**)&sd.gauss, sizeof(double) * 21)) err = PMF_E_NOMEM;
        S->sh.push_back(sd);
    }
    if (!err && pmf_dalloc(c, (void**)&S->d_off, sizeof(long long) * (world + 1))) err = PMF_E_NOMEM;
    if (!err && cudaMemcpy(S->d_off, S->off.data(), sizeof(long long) * (world + 1), cudaMemcpyHostToDevice))
        fail(PMF_E_CUDA, "upload offsets");
    if (!err && pmf_dalloc(c, (void**)&S->sum_scratch, sizeof(double) * NTOT * world)) err = PMF_E_NOMEM;
    // context-level buffers shared by the shards (same device): z, model table, moments, twiddles
    if (!err && pmf_dalloc(c, (void**)&c->z, sizeof(double) * PMF_MAX_NZ)) err = PMF_E_NOMEM;
    if (!err && pmf_dalloc(c, (void**)&c->mom_dev, sizeof(double) * (nx + nx * nx + 2))) err = PMF_E_NOMEM;
    if (!err && cudaMallocHost((void**)&c->mom_host, sizeof(double) * (nx + nx * nx + 2)) != cudaSuccess)
        fail(PMF_E_NOMEM, "cudaMallocHost");
    for (int m = 0; m < nx && !err; ++m) {
        const int N = g.n[m];
        if (c->dtype == PMF_F64) {
            std::vector<double> t;
            pmf_make_twiddles(N, t);
            if (pmf_dalloc(c, &c->tw[m], t.size() * sizeof(double))) err = PMF_E_NOMEM;
            else cudaMemcpy(c->tw[m], t.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice);
        } else {
            std::vector<float> t;
            pmf_make_twiddles(N, t);
            if (pmf_dalloc(c, &c->tw[m], t.size() * sizeof(float))) err = PMF_E_NOMEM;
            else cudaMemcpy(c->tw[m], t.data(), t.size() * sizeof(float), cudaMemcpyHostToDevice);
        }
    }
    if (!err) {
        FilterState z{};
        std::memset(&z, 0, sizeof(z));
        for (Shard& sd : S->sh) cudaMemcpy(sd.st, &z, sizeof(z), cudaMemcpyHostToDevice);
        c->st = S->sh[0].st;            // pmf_moments / pmf_get_grid read shard 0 (states are replicated)
    }
    if (err) {
        std::string m = c->err;
        pmf_destroy(c);
        pmf_fail(nullptr, err, m);
        return err;
    }
    *out = c;
    return PMF_OK;
}

void sh_destroy(pmf_ctx* c) {
    ShardSet* S = c->sh;
    cudaStreamSynchronize(c->stream);
    for (Shard& sd : S->sh) {
        void* ps[] = {sd.W, sd.Wwin, sd.S, sd.send, sd.recv, sd.st, sd.partials, sd.coef, sd.tot, sd.gauss};
        for (void* p : ps)
            if (p) cudaFree(p);
    }
    if (S->d_off) cudaFree(S->d_off);
    if (S->sum_scratch) cudaFree(S->sum_scratch);
    if (S->xs) cudaStreamSynchronize(S->xs);
    for (cudaEvent_t e : S->ev) cudaEventDestroy(e);
    if (S->xs) cudaStreamDestroy(S->xs);
    if (S->comm) NcclApi::get().CommDestroy(S->comm);
    c->st = nullptr;                    // aliased shard 0's state
    delete S;
    c->sh = nullptr;
}

// ============================================================================ density setters
int sh_set_gaussian(pmf_ctx* c, const double* mean, const double* cov, double k_sigma) {
    ShardSet& S = *c->sh;
    const int nx = c->d.nx;
    FilterState f{};
    std::memset(&f, 0, sizeof(f));
    double P[16], Pi[16];
    pmf_unpack(nx, cov, P);
    const double det = pmf_det_inv(nx, P, Pi);
    if (!(det > 0.0)) return pmf_fail(c, PMF_E_ARG, "cov must be positive definite");
    std::vector<double> gp(21, 0.0);
    for (int a = 0; a < nx; ++a) {
        f.c[a] = mean[a];
        f.B[a * 4 + a] = 2.0 * k_sigma * std::sqrt(P[a * 4 + a]) / c->d.n[a];   // R10 (global N)
        gp[a] = mean[a];
    }
    for (int i = 0; i < 16; ++i) gp[4 + i] = Pi[i];
    gp[20] = -0.5 * (nx * std::log(2.0 * M_PI) + std::log(det));
    f.scale = 1.0;
    c->pend = Pending{};
    for (Shard& sd : S.sh) {
        cudaMemcpyAsync(sd.st, &f, sizeof(f), cudaMemcpyHostToDevice, c->stream);
        cudaMemcpyAsync(sd.gauss, gp.data(), sizeof(double) * 21, cudaMemcpyHostToDevice, c->stream);
        PencilBufs b = shard_bufs(c, sd);
        cudaError_t e = sh_points(sd.d, c->dtype, b, 1, LikParams{}, sd.tot, c->stream, &c->launches);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "init gaussian");
    }
    int r = finalize_all(c, 1, 0.0);
    if (r) return r;
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return pmf_fail(c, PMF_E_CUDA, "set_gaussian sync");
    c->have_density = true;
    c->have_update = false;
    return PMF_OK;
}

int sh_set_state(pmf_ctx* c, const double* center, const double* B, const void* weights, int on_device) {
    ShardSet& S = *c->sh;
    const int nx = c->d.nx;
    FilterState f{};
    std::memset(&f, 0, sizeof(f));
    pmf_unpack(nx, B, f.B);
    if (pmf_det_inv(nx, f.B, nullptr) == 0.0) return pmf_fail(c, PMF_E_SINGULAR_GRID, "grid matrix B is singular");
    for (int a = 0; a < nx; ++a) f.c[a] = center[a];
    f.scale = 1.0;
    c->pend = Pending{};
    const size_t slab = c->esize * (size_t)S.sh[0].d.ntot;
    for (size_t k = 0; k < S.sh.size(); ++k) {
        Shard& sd = S.sh[k];
        cudaMemcpyAsync(sd.st, &f, sizeof(f), cudaMemcpyHostToDevice, c->stream);
        // weights: the slabs this context holds, in order (virtual: the whole grid)
        cudaMemcpyAsync(sd.W, (const char*)weights + k * slab, slab,
                        on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream);
        PencilBufs b = shard_bufs(c, sd);
        cudaError_t e = sh_points(sd.d, c->dtype, b, 2, LikParams{}, sd.tot, c->stream, &c->launches);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "normalise");
    }
    int r = finalize_all(c, 1, 0.0);
    if (r) return r;
    if (cudaStreamSynchronize(c->stream) != cudaSuccess) return pmf_fail(c, PMF_E_CUDA, "set_state sync");
    c->have_density = true;
    c->have_update = false;
    return PMF_OK;
}

// ============================================================================ regrid with plane exchange
static int sh_regrid_all(pmf_ctx* c, double ks) {
    ShardSet& S = *c->sh;
    const int nx = c->d.nx, L = S.L, NL = c->d.n[L];
    // replicated filter state -> host (the plane ranges are host-side NCCL counts)
    FilterState f;
    cudaError_t e = cudaMemcpyAsync(&f, S.sh[0].st, sizeof(f), cudaMemcpyDeviceToHost, c->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) return pmf_cuda_fail(c, e, "regrid state download");
    if (f.status) return pmf_fail(c, PMF_E_NO_SUPPORT, "regrid after a failed update");
    // the same map as the device (R12): v = B^-1 (c' + B' u' - c) + (N-1)/2
    double Bn[16] = {0}, cn[4], Bi[16];
    for (int a = 0; a < nx; ++a) {
        const double v = f.cov[a * 4 + a];
        if (!(v > 0.0) || !std::isfinite(v)) return pmf_fail(c, PMF_E_NO_SUPPORT, "degenerate covariance at regrid");
        cn[a] = f.mean[a];
        Bn[a * 4 + a] = 2.0 * ks * std::sqrt(v) / c->d.n[a];
    }
    pmf_det_inv(nx, f.B, Bi);
    double M[4] = {0, 0, 0, 0}, oL = 0.5 * (NL - 1);
    for (int b = 0; b < nx; ++b) {
        double s = 0.0;
        for (int k = 0; k < nx; ++k) s += Bi[L * 4 + k] * Bn[k * 4 + b];
        M[b] = s;
        oL += Bi[L * 4 + b] * (cn[b] - f.c[b]);
    }
    const size_t pb = c->esize * S.plane_real;          // bytes per real plane
    std::vector<Xfer> xs;
    std::vector<int> wlo(S.world), wn(S.world);
    for (int d = 0; d < S.world; ++d) {
        // range of the old last-axis coordinate over the corners of rank d's new slab
        double vmin = oL, vmax = oL;
        for (int b = 0; b < nx; ++b) {
            double ulo = -0.5 * (c->d.n[b] - 1), uhi = 0.5 * (c->d.n[b] - 1);
            if (b == L) {
                ulo = d * S.n_loc - 0.5 * (NL - 1);
                uhi = (d + 1) * S.n_loc - 1 - 0.5 * (NL - 1);
            }
            vmin += std::min(M[b] * ulo, M[b] * uhi);
            vmax += std::max(M[b] * ulo, M[b] * uhi);
        }
        int lo = (int)std::floor(std::max(vmin, -4.0)) - 1, hi = (int)std::floor(std::min(vmax, (double)NL + 4)) + 2;
        lo = std::max(lo, 0);
        hi = std::min(hi, NL - 1);
        wlo[d] = lo;
        wn[d] = std::max(0, hi - lo + 1);
    }
    // window capacity
    for (Shard& sd : S.sh) {
        const int d = sd.rank;
        if ((size_t)wn[d] > sd.win_planes) {
            cudaStreamSynchronize(c->stream);
            cudaFree(sd.Wwin);
            sd.Wwin = nullptr;
            if (pmf_dalloc(c, &sd.Wwin, pb * (size_t)wn[d])) return PMF_E_NOMEM;
            sd.win_planes = wn[d];
        }
    }
    if (!S.virt) {   // every rank must agree on the capacity needs of the others only for its own window
    }
    for (int d = 0; d < S.world; ++d)
        for (int s = 0; s < S.world; ++s) {
            const int a = std::max(wlo[d], s * S.n_loc), b2 = std::min(wlo[d] + wn[d], (s + 1) * S.n_loc);
            if (b2 > a) xs.push_back({s, d, (size_t)(a - s * S.n_loc) * pb, (size_t)(a - wlo[d]) * pb, (size_t)(b2 - a) * pb});
        }
    int r = exchange(c, xs, [](Shard& s) -> void* { return s.W; }, [](Shard& s) -> void* { return s.Wwin; });
    if (r) return r;
    for (Shard& sd : S.sh) {
        Dims dd = sd.d;
        dd.src_lo = wlo[sd.rank];
        dd.src_n = wn[sd.rank];
        PencilBufs b = shard_bufs(c, sd);
        e = sh_regrid(dd, c->dtype, sd.Wwin, sd.W, b, ks, sd.tot, c->stream, &c->launches);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "sharded regrid");
    }
    return finalize_all(c, 2, ks);
}

// ============================================================================ predict / update
// ============================================================================ three-pass route
// nx = 4, fp64, N_0 = N_1 in {32, 64, 96}, n2 = n3 in {16, .., 96}, N_0 divisible by world
// (kernels_quad.cu): rank r owns the j3 slab [r slab, (r+1) slab):
//   K1  forward plane pass over its planes; each spectrum row leaves in world k0 blocks,
//       block q = [j3 % slab][j2][k1][k0 in q's range] (contiguous per destination)
//   ALL-TO-ALL  block q of rank r -> rank q, stacked in rank order: [j3][j2][k1][k0 - q N0/G]
//   K2  rank q: the (j3, j2)-planes of its (k1, k0) items (whole planes: the axis-2/3 DFTs,
//       s Psi, inverses); output row j3 to block j3 / slab = [k0][k1][j3 % slab][j2]
//   ALL-TO-ALL back  block r of rank q -> rank r, stacked in rank order: [k0][k1][j3 % slab][j2]
//   K3  rank r: inverse DFT along axes 0, 1 of its planes, likelihood, weights, moment sums
//   ALL-REDUCE of {15 moment sums, DC} -> normaliser, closed-form scale, moments
// Both exchanges move every spectrum element once: 2 (G-1)/G x 16 B x H N^3 per rank and predict.
// the two all-to-all plans of the three-pass route: blocks of `blk` elements of `cb` bytes;
// x1: K1's block q on rank r -> rank q, slot r; x2: K2's block r on rank q -> rank r, slot q
static void quad_xfers(int G, size_t blk, size_t cb, std::vector<Xfer>& x1, std::vector<Xfer>& x2) {
    for (int r = 0; r < G; ++r)
        for (int q = 0; q < G; ++q) {
            x1.push_back({r, q, cb * q * blk, cb * r * blk, cb * blk});
            x2.push_back({q, r, cb * r * blk, cb * q * blk, cb * blk});
        }
}

static bool sh_quad_ok(pmf_ctx* c) {
    const Dims& g = c->d;
    const ShardSet& S = *c->sh;
    if (c->dtype != PMF_F64 || g.nx != 4 || g.n[0] != g.n[1] || g.n[2] != g.n[3]) return false;
    const int N = g.n[0], NQ = g.n[2];
    if ((N != 32 && N != 64 && N != 96) || (NQ != 16 && NQ != 32 && NQ != 64 && NQ != 96)) return false;
    if (N % S.world || (N / S.world) < 1 || c->mp.l + 1 > 64 || c->cfg.diff_mode != PMF_DIFF_FULL) return false;
    const char* e = std::getenv("PMF_NO_QUAD");
    return !(e && e[0] == '1');
}

// Chunks of the pipelined exchanges (PMF_XCHUNKS, default 4; 1 = one exchange after each pass)
static int xchunks() {
    const char* e = std::getenv("PMF_XCHUNKS");
    const int v = e ? std::atoi(e) : 4;
    return v < 1 ? 1 : (v > 16 ? 16 : v);
}

// the pieces of chunk [lo, hi) of every block in a plan: each (source, destination) block of
// `blk` elements is split along its outermost index (j3 % slab for K1's blocks, k0 for K2's),
// `inner` elements per index value
static void chunk_xfers(const std::vector<Xfer>& full, size_t cb, size_t inner, int lo, int hi,
                        std::vector<Xfer>& out) {
    out.clear();
    for (const Xfer& x : full)
        out.push_back({x.src, x.dst, x.so + cb * inner * lo, x.dof + cb * inner * lo, cb * inner * (hi - lo)});
}

static int sh_predict_quad(pmf_ctx* c, const LikParams* lp) {
    ShardSet& S = *c->sh;
    const Dims& g = c->d;
    const int G = S.world, N = g.n[0], H = N / 2 + 1, NQ = g.n[2], slab = S.n_loc, N0c = N / G;
    const size_t blk = (size_t)slab * NQ * H * N0c;            // complex elements per (source, destination)
    const size_t cb = c->esize * 2;
    const int nplanes = slab * NQ;
    cudaError_t e;
    // the two all-to-alls overlap the passes next to them. K1 runs in C1 chunks
    // of its slab (j3 ranges; each chunk's rows are contiguous in every destination block) and
    // chunk i's pieces leave while K1 works on chunk i + 1; K2 runs in C2 chunks of its k0
    // range and chunk i returns while K2 works on chunk i + 1. Exchanges on the stream S.xs,
    // ordered by events; K2 (K3) starts when the last piece of the first (second) exchange is in.
    // A single rank (G = 1: a 1-rank communicator or one virtual slab) keeps K2's output in the
    // unsharded route's k1-major order [k1][k0][j3][j2] (what K3 then reads), in which a k0
    // sub-range is neither contiguous nor addressed per chunk: K2 runs whole, one piece back.
    const int C1 = std::min(xchunks(), slab), C2 = G == 1 ? 1 : std::min(xchunks(), N0c);
    if (!S.xs && cudaStreamCreateWithFlags(&S.xs, cudaStreamNonBlocking) != cudaSuccess)
        return pmf_cuda_fail(c, cudaGetLastError(), "exchange stream");
    while ((int)S.ev.size() < 2 * 16 + 2) {
        cudaEvent_t ev;
        if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
            return pmf_cuda_fail(c, cudaGetLastError(), "exchange event");
        S.ev.push_back(ev);
    }
    cudaEvent_t* ev = S.ev.data();                              // [0, 16) K1 chunks, [16, 32) K2 chunks
    cudaEvent_t ev_x1 = S.ev[32], ev_x2 = S.ev[33];             // exchange 1 / 2 complete
    std::vector<Xfer> x1, x2, part;
    quad_xfers(G, blk, cb, x1, x2);
    for (Shard& sd : S.sh) {
        PencilBufs b = shard_bufs(c, sd);
        e = launch_plane_prep(sd.d, b, c->mp, lp, c->stream, &c->launches);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "sharded prep");
    }
    // the exchange stream may still be reading last predict's buffers: order it after this
    // predict's start (and everything before it on the compute stream)
    for (int i = 0; i < C1; ++i) {
        const int jb = (int)((long long)slab * i / C1), je = (int)((long long)slab * (i + 1) / C1);
        for (Shard& sd : S.sh) {
            PencilBufs b = shard_bufs(c, sd);
            e = launch_plane_fwd_chunks(sd.d, b, c->mp, G, (long long)blk, sd.partials, jb * NQ, je * NQ, c->stream,
                                        &c->launches);
            if (e != cudaSuccess) return pmf_cuda_fail(c, e, "sharded forward plane pass");
        }
        if ((e = cudaEventRecord(ev[i], c->stream)) != cudaSuccess || (e = cudaStreamWaitEvent(S.xs, ev[i], 0)))
            return pmf_cuda_fail(c, e, "exchange order");
        chunk_xfers(x1, cb, (size_t)NQ * H * N0c, jb, je, part);
        int rc = exchange(c, part, [](Shard& s) -> void* { return s.S; }, [](Shard& s) -> void* { return s.recv; },
                          S.xs);
        if (rc) return rc;
    }
    if ((e = cudaEventRecord(ev_x1, S.xs)) != cudaSuccess || (e = cudaStreamWaitEvent(c->stream, ev_x1, 0)))
        return pmf_cuda_fail(c, e, "exchange order");
    for (int i = 0; i < C2; ++i) {
        const int kb = (int)((long long)N0c * i / C2), ke = (int)((long long)N0c * (i + 1) / C2);
        for (Shard& sd : S.sh) {
            PencilBufs b = shard_bufs(c, sd);
            e = launch_quad_mid_shard(sd.d, b, c->mp, sd.rank, G, sd.recv, sd.send, kb, ke, c->stream, &c->launches);
            if (e != cudaSuccess) return pmf_cuda_fail(c, e, "sharded axis-2/3 pass");
        }
        if ((e = cudaEventRecord(ev[16 + i], c->stream)) != cudaSuccess ||
            (e = cudaStreamWaitEvent(S.xs, ev[16 + i], 0)))
            return pmf_cuda_fail(c, e, "exchange order");
        chunk_xfers(x2, cb, (size_t)H * slab * NQ, kb, ke, part);
        int rc = exchange(c, part, [](Shard& s) -> void* { return s.send; }, [](Shard& s) -> void* { return s.S; },
                          S.xs);
        if (rc) return rc;
    }
    if ((e = cudaEventRecord(ev_x2, S.xs)) != cudaSuccess || (e = cudaStreamWaitEvent(c->stream, ev_x2, 0)))
        return pmf_cuda_fail(c, e, "exchange order");
    int rc;
    for (Shard& sd : S.sh) {
        PencilBufs b = shard_bufs(c, sd);
        int ginv = 1;
        double* part_ = sd.partials + nplanes;
        e = launch_quad_inv_shard(sd.d, b, c->mp, lp, sd.rank, G, sd.S, part_, c->stream, &c->launches, &ginv);
        if (e == cudaSuccess)
            e = launch_shard_sum(sd.partials, nplanes, part_, ginv, lp ? 1 : 0, sd.tot, c->stream, &c->launches);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "sharded inverse plane pass");
    }
    rc = allreduce_tot(c, NTOT);
    if (rc) return rc;
    for (Shard& sd : S.sh) {
        PencilBufs b = shard_bufs(c, sd);
        e = launch_plane_fin_tot(sd.d, b, c->mp, sd.tot, lp ? 1 : 0, c->stream, &c->launches);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "sharded finalise");
    }
    return PMF_OK;
}

static int sh_predict_all(pmf_ctx* c, const LikParams* lp) {
    ShardSet& S = *c->sh;
    const size_t cs = c->esize * 2;
    const int cstride = coef_stride(c->mp.l);
    for (Shard& sd : S.sh) {
        const size_t need = sizeof(double) * cstride;
        if (need > sd.coef_bytes) {
            if (sd.coef) { cudaStreamSynchronize(c->stream); cudaFree(sd.coef); sd.coef = nullptr; }
            if (pmf_dalloc(c, (void**)&sd.coef, need)) return PMF_E_NOMEM;
            sd.coef_bytes = need;
        }
    }
    if (sh_quad_ok(c)) return sh_predict_quad(c, lp);
    cudaError_t e;
    for (Shard& sd : S.sh) {
        PencilBufs b = shard_bufs(c, sd);
        e = sh_prep(sd.d, b, c->mp, lp, c->stream, &c->launches);
        if (e == cudaSuccess)
            e = sh_phase(sd.d, c->dtype, b, twid(c), c->mp, lp, SH_PH_FWD, nullptr, -1, 0, nullptr, c->stream,
                         &c->launches);
        if (e == cudaSuccess) e = sh_pack(c->dtype, sd.S, sd.send, S.I, S.n_loc, S.d_off, S.world, 0, c->stream,
                                          &c->launches);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "sharded forward");
    }
    // transpose 1: block (s -> d) = n_loc x I_d, from send (packed by d) to recv [s][plane][I_d]
    std::vector<Xfer> x1, x2;
    for (int s = 0; s < S.world; ++s)
        for (int d = 0; d < S.world; ++d) {
            const long long Id = S.off[d + 1] - S.off[d];
            const size_t bytes = cs * (size_t)(S.n_loc * Id);
            x1.push_back({s, d, cs * (size_t)(S.n_loc * S.off[d]), cs * (size_t)(s * S.n_loc * Id), bytes});
            // back: d returns rows of slab s of its T to s, into s's packed layout
            x2.push_back({d, s, cs * (size_t)(s * S.n_loc * Id), cs * (size_t)(S.n_loc * S.off[d]), bytes});
        }
    int r = exchange(c, x1, [](Shard& s) -> void* { return s.send; }, [](Shard& s) -> void* { return s.recv; });
    if (r) return r;
    for (Shard& sd : S.sh) {
        PencilBufs b = shard_bufs(c, sd);
        const long long Id = S.off[sd.rank + 1] - S.off[sd.rank];
        e = sh_phase(sd.d, c->dtype, b, twid(c), c->mp, lp, SH_PH_PSI, sd.recv, Id, S.off[sd.rank], nullptr,
                     c->stream, &c->launches);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "sharded Psi");
    }
    r = exchange(c, x2, [](Shard& s) -> void* { return s.recv; }, [](Shard& s) -> void* { return s.send; });
    if (r) return r;
    for (Shard& sd : S.sh) {
        PencilBufs b = shard_bufs(c, sd);
        e = sh_pack(c->dtype, sd.S, sd.send, S.I, S.n_loc, S.d_off, S.world, 1, c->stream, &c->launches);
        if (e == cudaSuccess)
            e = sh_phase(sd.d, c->dtype, b, twid(c), c->mp, lp, SH_PH_INV, nullptr, -1, 0, lp ? sd.tot : nullptr,
                         c->stream, &c->launches);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "sharded inverse");
    }
    if (lp) return finalize_all(c, 0, 0.0);
    return PMF_OK;
}

int sh_flush(pmf_ctx* c, const LikParams* lp) {
    ShardSet& S = *c->sh;
    if (c->pend.regrid) {
        int r = sh_regrid_all(c, c->pend.k_sigma);
        if (r) return r;
    }
    if (c->pend.predict) {
        cudaEvent_t e0 = nullptr, e1 = nullptr;
        pmf_profile_events(c, &e0, &e1);          // time the whole sharded predict (+update)
        if (e0) cudaEventRecord(e0, c->stream);
        int r = sh_predict_all(c, lp);
        if (r) return r;
        if (e1) cudaEventRecord(e1, c->stream);
    } else if (lp) {
        for (Shard& sd : S.sh) {
            PencilBufs b = shard_bufs(c, sd);
            cudaError_t e = sh_points(sd.d, c->dtype, b, 0, *lp, sd.tot, c->stream, &c->launches);
            if (e != cudaSuccess) return pmf_cuda_fail(c, e, "sharded update");
        }
        int r = finalize_all(c, 0, 0.0);
        if (r) return r;
    }
    c->pend = Pending{};
    return PMF_OK;
}

int sh_get_weights(pmf_ctx* c, void* dst, int on_device) {
    ShardSet& S = *c->sh;
    const size_t slab = c->esize * (size_t)S.sh[0].d.ntot;
    for (size_t k = 0; k < S.sh.size(); ++k) {
        Shard& sd = S.sh[k];
        PencilBufs b = shard_bufs(c, sd);
        // scale_out into the shard's send buffer (>= slab), then copy out
        cudaError_t e = launch_scale_out(sd.d, c->dtype, b, sd.send, c->stream, &c->launches);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync((char*)dst + k * slab, sd.send, slab,
                                on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream);
        if (e != cudaSuccess) return pmf_cuda_fail(c, e, "sharded get_weights");
    }
    if (!on_device && cudaStreamSynchronize(c->stream) != cudaSuccess) return pmf_fail(c, PMF_E_CUDA, "sync");
    return PMF_OK;
}

extern "C" int pmf_world(const pmf_ctx* c) { return (c && c->sh) ? c->sh->world : 1; }

// Test hook (not in pmf.h; host only, no device): the three-pass route's exchange plans for
// `world` ranks and blocks of `blk` complex fp64 elements: 2 world^2 rows of (source rank,
// destination rank, source byte offset, destination byte offset, bytes), x1 then x2.
// chunk [lo, hi) of plan `which` (0: K1 -> K2, 1: K2 -> K3) with `inner` elements per value of
// the blocks' outermost index: the pieces sh_predict_quad's pipelined exchange issues
extern "C" int pmf_debug_quad_chunk(int world, long long blk, int which, long long inner, int lo, int hi,
                                    long long* out) {
    if (world < 1 || blk < 1 || inner < 1 || lo < 0 || hi < lo || !out || (which != 0 && which != 1)) return PMF_E_ARG;
    std::vector<Xfer> x1, x2, part;
    quad_xfers(world, (size_t)blk, 16, x1, x2);
    chunk_xfers(which ? x2 : x1, 16, (size_t)inner, lo, hi, part);
    long long* o = out;
    for (const Xfer& x : part) {
        *o++ = x.src;
        *o++ = x.dst;
        *o++ = (long long)x.so;
        *o++ = (long long)x.dof;
        *o++ = (long long)x.bytes;
    }
    return PMF_OK;
}

extern "C" int pmf_debug_quad_plan(int world, long long blk, long long* out) {
    if (world < 1 || blk < 1 || !out) return PMF_E_ARG;
    std::vector<Xfer> x1, x2;
    quad_xfers(world, (size_t)blk, 16, x1, x2);
    long long* o = out;
    for (const auto* v : {&x1, &x2})
        for (const Xfer& x : *v) {
            *o++ = x.src;
            *o++ = x.dst;
            *o++ = (long long)x.so;
            *o++ = (long long)x.dof;
            *o++ = (long long)x.bytes;
        }
    return PMF_OK;
}
