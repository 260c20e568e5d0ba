// bench_layout.cu -- memory-side microbenchmark for the C4 (96^4, fp64) spectrum
// layout: how fast can a plane pass write (and read) the "transposed" spectrum
// Y[k1][k0][j3][j2] (one (j2, j3) plane = 4704 complex, each to its own 147 KB-strided
// slot), compared with a contiguous copy and with the contiguous (j3, j2)-plane rows the
// fused (2,3) pass reads? No compute: every kernel only moves the bytes a pass moves.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_layout bench_layout.cu
//   ./bench_layout > layout.json
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <algorithm>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int NQ = 96, N0 = 96, H = 49;
constexpr int PLANES = NQ * NQ;            // (j2, j3)
constexpr int E = H * N0;                  // elements per plane (k1, k0)
constexpr size_t TOT = (size_t)PLANES * E; // complex elements

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(b)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned ph) {
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void tma_store5(const CUtensorMap* m, const void* src, int c0, int c1, int c2, int c3, int c4) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
                 ::"l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(su32(src)) : "memory");
}
__device__ __forceinline__ void tma_load5(const CUtensorMap* m, void* dst, unsigned long long* bar, int c0, int c1, int c2, int c3, int c4) {
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"(su32(dst)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(su32(bar)) : "memory");
}

// ---------------------------------------------------------------- contiguous copy (baseline)
__global__ void k_copy(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

// ---------------------------------------------------------------- per-thread scatter / gather
// MODE 0: 16 B per element, planes p = blockIdx + k grid (neighbour planes on neighbour CTAs)
// MODE 1: 16 B per element, CTA walks consecutive planes (neighbour planes one after the other)
// MODE 2: 32 B (plane pairs)
template <int MODE, bool WRITE>
__global__ void __launch_bounds__(384, 1) k_scatter(double2* Y) {
    extern __shared__ double2 sm[];
    for (int i = threadIdx.x; i < 2 * E; i += blockDim.x) sm[i] = double2{(double)i, 1.0};
    __syncthreads();
    const int units = MODE == 2 ? PLANES / 2 : PLANES;
    const int per = (units + gridDim.x - 1) / gridDim.x;
    for (int k = 0; k < per; ++k) {
        const int u = MODE == 0 || MODE == 2 ? blockIdx.x + k * gridDim.x : blockIdx.x * per + k;
        if (u >= units) break;
        if (MODE == 2) {
            const int p = 2 * u;
            for (int e = threadIdx.x; e < E; e += blockDim.x) {
                double* g = reinterpret_cast<double*>(Y + (size_t)e * PLANES + p);
                if (WRITE) {
                    const double2 a = sm[e], b = sm[E + e];
                    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(g), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y) : "memory");
                } else {
                    double4 r;
                    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(g));
                    sm[e] = double2{r.x, r.y};
                    sm[E + e] = double2{r.z, r.w};
                }
            }
        } else {
            for (int e = threadIdx.x; e < E; e += blockDim.x) {
                double2* g = Y + (size_t)e * PLANES + u;
                if (WRITE) __stcg(g, sm[e]);
                else sm[e] = __ldcg(g);
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- TMA tensor store / load
// map dims (innermost first): re/im 2, j2 96, j3 96, k0 96, k1 49 (doubles); box (2, PAIR, 1, 96, 1)
template <int PAIR, bool WRITE>
__global__ void __launch_bounds__(128, 1) k_tma(const __grid_constant__ CUtensorMap m) {
    extern __shared__ __align__(128) double2 sm[];          // [k1][k0][PAIR]
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + PAIR * E);
    if (threadIdx.x == 0) mbar_init(bar);
    for (int i = threadIdx.x; i < PAIR * E; i += blockDim.x) sm[i] = double2{(double)i, 1.0};
    __syncthreads();
    const int units = PLANES / PAIR;
    int k = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x, ++k) {
        const int p = u * PAIR, j2 = p % NQ, j3 = p / NQ;
        if (WRITE) {
            if (threadIdx.x < H) {
                fence_async();
                tma_store5(&m, sm + threadIdx.x * N0 * PAIR, 0, j2, j3, 0, threadIdx.x);
                bulk_commit();
                bulk_wait_read();
            }
        } else {
            if (threadIdx.x == 0) mbar_tx(bar, (unsigned)(PAIR * E * 16));
            __syncwarp();
            if (threadIdx.x < H) tma_load5(&m, sm + threadIdx.x * N0 * PAIR, bar, 0, j2, j3, 0, threadIdx.x);
            mbar_wait(bar, k & 1);
        }
        __syncthreads();
    }
    if (WRITE && threadIdx.x < H) bulk_wait_all();
}

// ---------------------------------------------------------------- contiguous (j3, j2) planes (fused pass reads/writes)
__global__ void __launch_bounds__(128, 1) k_rows(double2* Y, double2* Z) {
    extern __shared__ __align__(128) double2 sm[];          // [96][97]
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + NQ * (NQ + 1));
    if (threadIdx.x == 0) mbar_init(bar);
    __syncthreads();
    int k = 0;
    for (int e = blockIdx.x; e < E; e += gridDim.x, ++k) {
        const double2* src = Y + (size_t)e * PLANES;
        if (threadIdx.x == 0) mbar_tx(bar, NQ * NQ * 16);
        __syncwarp();
        if (threadIdx.x < NQ) {
            fence_async();
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su32(sm + threadIdx.x * (NQ + 1))), "l"(src + threadIdx.x * NQ), "r"(NQ * 16), "r"(su32(bar)) : "memory");
        }
        mbar_wait(bar, k & 1);
        if (threadIdx.x < NQ) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(Z + (size_t)e * PLANES + threadIdx.x * NQ),
                         "r"(su32(sm + threadIdx.x * (NQ + 1))), "r"(NQ * 16) : "memory");
            bulk_commit();
            bulk_wait_read();
        }
        __syncthreads();
    }
    if (threadIdx.x < NQ) bulk_wait_all();
}

static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;

static CUtensorMap make_map(double2* Y, int pair) {
    CUtensorMap m;
    cuuint64_t dims[5] = {2, NQ, NQ, N0, H};
    cuuint64_t str[4] = {16, 16ull * NQ, 16ull * PLANES, 16ull * PLANES * N0};
    cuuint32_t box[5] = {2, (cuuint32_t)pair, 1, N0, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, Y, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        fprintf(stderr, "cuTensorMapEncodeTiled failed %d\n", (int)r);
        exit(1);
    }
    return m;
}

template <typename F>
static void timeit(const char* name, double bytes, F f, bool last = false) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    f();
    CK(cudaDeviceSynchronize());
    std::vector<float> ts;
    for (int r = 0; r < 7; ++r) {
        CK(cudaEventRecord(e0));
        f();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    const float med = ts[ts.size() / 2];
    printf("  \"%s\": {\"ms\": %.4f, \"GBps\": %.1f}%s\n", name, med, bytes / (med * 1e-3) / 1e9, last ? "" : ",");
    fflush(stdout);
}

#include <algorithm>
int main() {
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q));
    int nsm = 148;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    double2 *Y, *Z;
    CK(cudaMalloc(&Y, TOT * 16));
    CK(cudaMalloc(&Z, TOT * 16));
    CK(cudaMemset(Y, 0, TOT * 16));
    CK(cudaMemset(Z, 0, TOT * 16));
    const double bytes = (double)TOT * 16;
    printf("{\n  \"what\": \"C4 spectrum (49 x 96 x 96 x 96 complex fp64 = %.0f MB) moved by layout; GBps = useful bytes / time\",\n", bytes / 1e6);
    timeit("copy_contiguous_rw", 2 * bytes, [&] { k_copy<<<nsm * 8, 512>>>((const double4*)Y, (double4*)Z, TOT / 2); });
    const size_t sm2 = 2 * E * 16;
    CK(cudaFuncSetAttribute(k_scatter<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2));
    CK(cudaFuncSetAttribute(k_scatter<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2));
    CK(cudaFuncSetAttribute(k_scatter<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2));
    CK(cudaFuncSetAttribute(k_scatter<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2));
    CK(cudaFuncSetAttribute(k_scatter<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2));
    CK(cudaFuncSetAttribute(k_scatter<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2));
    timeit("write16_neighbour_ctas", bytes, [&] { k_scatter<0, true><<<nsm, 384, sm2>>>(Y); });
    timeit("write16_same_cta_seq", bytes, [&] { k_scatter<1, true><<<nsm, 384, sm2>>>(Y); });
    timeit("write32_pairs", bytes, [&] { k_scatter<2, true><<<nsm, 384, sm2>>>(Y); });
    timeit("read16_neighbour_ctas", bytes, [&] { k_scatter<0, false><<<nsm, 384, sm2>>>(Y); });
    timeit("read16_same_cta_seq", bytes, [&] { k_scatter<1, false><<<nsm, 384, sm2>>>(Y); });
    timeit("read32_pairs", bytes, [&] { k_scatter<2, false><<<nsm, 384, sm2>>>(Y); });
    CUtensorMap m1 = make_map(Y, 1), m2 = make_map(Y, 2);
    const size_t st1 = E * 16 + 64, st2 = 2 * E * 16 + 64;
    CK(cudaFuncSetAttribute(k_tma<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, st1));
    CK(cudaFuncSetAttribute(k_tma<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, st2));
    CK(cudaFuncSetAttribute(k_tma<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, st1));
    CK(cudaFuncSetAttribute(k_tma<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, st2));
    timeit("tma_store16", bytes, [&] { k_tma<1, true><<<nsm, 128, st1>>>(m1); });
    timeit("tma_store32_pairs", bytes, [&] { k_tma<2, true><<<nsm, 128, st2>>>(m2); });
    timeit("tma_store16_2cta", bytes, [&] { k_tma<1, true><<<2 * nsm, 128, st1>>>(m1); });
    timeit("tma_load16", bytes, [&] { k_tma<1, false><<<nsm, 128, st1>>>(m1); });
    timeit("tma_load32_pairs", bytes, [&] { k_tma<2, false><<<nsm, 128, st2>>>(m2); });
    timeit("tma_load16_2cta", bytes, [&] { k_tma<1, false><<<2 * nsm, 128, st1>>>(m1); });
    const size_t sr = NQ * (NQ + 1) * 16 + 64;
    CK(cudaFuncSetAttribute(k_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, sr));
    timeit("rows_contiguous_rw", 2 * bytes, [&] { k_rows<<<nsm, 128, sr>>>(Y, Z); }, true);
    printf("}\n");
    return 0;
}
