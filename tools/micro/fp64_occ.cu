// fp64_occ.cu -- DFMA throughput vs. warps per SM and independent chains per thread
// (how much FP64 ILP/TLP does B200 need?). One CTA per SM.
#include <cstdio>
#include <vector>
#include <algorithm>

template <int CH>
__global__ void k(double* out, int iters) {
    double a[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-6;
    const double m = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
            for (int i = 0; i < CH; ++i) a[i] = fma(a[i], m, c);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += a[i];
    if (s == -1.0) out[threadIdx.x] = s;
}

template <int CH>
void run(int threads) {
    double* out;
    cudaMalloc(&out, 1 << 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    k<CH><<<148, threads>>>(out, 100);
    cudaDeviceSynchronize();
    std::vector<float> ts;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        k<CH><<<148, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    const double fl = 2.0 * 4 * CH * (double)iters * 148 * threads;
    printf("  \"warps%d_chains%d\": %.2f,\n", threads / 32, CH, fl / (ts[1] * 1e-3) / 1e12);
}

int main() {
    printf("{\n \"what\": \"DFMA TFLOP/s, one CTA per SM, independent FMA chains per thread\",\n");
    for (int th : {128, 256, 384, 512}) {
        run<1>(th); run<2>(th); run<4>(th); run<8>(th); run<12>(th);
    }
    printf(" \"end\": 0\n}\n");
}
