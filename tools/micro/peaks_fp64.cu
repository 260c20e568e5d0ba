// peaks_fp64.cu -- measured FP64 peaks of this B200 ("before claiming ALU
// fractions, measure the FP64 peak"): DFMA issue rate (CUDA cores), DMMA
// (mma.sync m8n8k4 f64, the FP64 tensor path) and, for the fp32 instances, FFMA.
// Every kernel runs many independent FMA chains per thread over a full-chip grid;
// the SM clock during the run is derived from clock64() deltas over the event time.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks_fp64 peaks_fp64.cu
//   ./peaks_fp64 > peaks.json
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

template <typename T, int CH>
__global__ void k_fma(double* outd, int iters, long long* clk) {
    T* out = reinterpret_cast<T*>(outd);
    T a[CH];
    const T m = (T)0.999999, c = (T)1e-7;
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = (T)(threadIdx.x + i);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < CH; ++i) a[i] = fma(a[i], m, c);
    }
    long long t1 = clock64();
    T s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += a[i];
    if (s == (T)-1) out[threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

// D(8x8) += A(8x4) B(4x8), f64; NA independent accumulators per warp
template <int NA>
__global__ void k_dmma(double* out, int iters, long long* clk) {
    double a = 1.0 + threadIdx.x * 1e-3, b = 0.5 - threadIdx.x * 1e-4;
    double d[NA][2];
#pragma unroll
    for (int i = 0; i < NA; ++i) { d[i][0] = 0.0; d[i][1] = 0.0; }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < NA; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
    }
    long long t1 = clock64();
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < NA; ++i) s += d[i][0] + d[i][1];
    if (s == -1.0) out[threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}


// half the warps of every CTA issue DFMA chains, the other half DMMA: does the FP64
// tensor path run beside the DFMA pipe (sum > either alone) or share it?
__global__ void k_mixed(double* out, int iters, long long* clk) {
    const int w = threadIdx.x >> 5;
    long long t0 = clock64();
    double s = 0.0;
    if (w & 1) {
        double a = 1.0 + threadIdx.x * 1e-3, b = 0.5 - threadIdx.x * 1e-4;
        double d[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) { d[i][0] = 0.0; d[i][1] = 0.0; }
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(d[i][0]), "+d"(d[i][1]) : "d"(a), "d"(b));
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
    } else {
        double a[8];
        const double m = 0.999999, c = 1e-7;
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = (double)(threadIdx.x + i);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int r = 0; r < 8; ++r)
#pragma unroll
                for (int i = 0; i < 8; ++i) a[i] = fma(a[i], m, c);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s += a[i];
    }
    long long t1 = clock64();
    if (s == -1.0) out[threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <typename K>
static int run(const char* name, K kern, int blocks, int threads, int iters, double flop_per_iter_thread,
               double* out, long long* dclk, bool last) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    kern<<<blocks, threads>>>(out, iters / 8, dclk);   // warm-up
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    long long clk = 0;
    for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(e0));
        kern<<<blocks, threads>>>(out, iters, dclk);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) {
            best = ms;
            CK(cudaMemcpy(&clk, dclk, sizeof(clk), cudaMemcpyDeviceToHost));
        }
    }
    const double flops = flop_per_iter_thread * iters * (double)blocks * threads;
    const double tf = flops / (best * 1e-3) / 1e12;
    (void)clk;
    printf("  \"%s\": {\"tflops\": %.3f, \"ms\": %.3f}%s\n", name, tf, best, last ? "" : ",");
    return 0;
}

int main() {
    int dev = 0, nsm = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, dev));
    double* out;
    long long* clk;
    CK(cudaMalloc(&out, 1 << 20));
    CK(cudaMalloc(&clk, 8));
    printf("{\n  \"gpu\": \"%s\", \"sms\": %d,\n", p.name, nsm);
    // DFMA: 8 chains x 16 unrolled per iteration, 2 flop per FMA
    run("fp64_fma", k_fma<double, 8>, nsm * 8, 256, 4000, 2.0 * 16 * 8, out, clk, false);
    run("fp32_fma", k_fma<float, 8>, nsm * 8, 256, 8000, 2.0 * 16 * 8, out, clk, false);
    // DMMA m8n8k4: 2*8*8*4 = 512 flop per warp-MMA = 16 per thread
    run("fp64_dmma", k_dmma<8>, nsm * 8, 256, 4000, 16.0 * 8, out, clk, false);
    run("fp64_dfma_plus_dmma_half_warps_each", k_mixed, nsm * 8, 256, 4000, 128.0, out, clk, true);
    printf("}\n");
    return 0;
}
