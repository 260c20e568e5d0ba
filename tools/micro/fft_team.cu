// fft_team.cu -- the K2 (k_q_mid) FFT work in isolation: a 96 x 96 complex fp64 plane
// resident in shared memory, per item F2 (96 row FFTs), F3 (96 column FFTs forward x
// const x inverse), I2 (96 row inverse FFTs), no global traffic. Measures how close the
// team-of-8 register FFT (plane_common.cuh) comes to the FP64 pipe, per variant:
//   V0  twiddles W^{ts} loaded from the shared table (the production code)
//   V1  twiddles from one load per thread + a product tree in registers
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//        -I ../../paper_2412_07240_b200/csrc -o fft_team fft_team.cu
#include <cstdio>
#include <vector>
#include <algorithm>

#include "plane_common.cuh"

using namespace pmf;
using namespace pmf::pln;
using V = double2;

constexpr int NQ = 96, R = 12, P = NQ + 1;

// twiddle product tree: w[s] = W^{t s}, s = 1..R-1, from w1 = W^t (depth 4)
template <bool INV>
__device__ __forceinline__ void tw_tree(V w1, V* w) {
    if (INV) w1.y = -w1.y;
    auto sq = [](V a) { return V{fma(a.x, a.x, -a.y * a.y), 2.0 * a.x * a.y}; };
    w[1] = w1;
    w[2] = sq(w1);
    w[3] = cmul(w[2], w1);
    w[4] = sq(w[2]);
    w[5] = cmul(w[4], w1);
    w[6] = sq(w[3]);
    w[7] = cmul(w[4], w[3]);
    w[8] = sq(w[4]);
    w[9] = cmul(w[8], w1);
    w[10] = sq(w[5]);
    w[11] = cmul(w[8], w[3]);
}

template <int VAR, bool INV, typename SLOT>
__device__ __forceinline__ void tdft(V* x, V* pa, V* pb, V* ex, const V* tw, int t, SLOT slot) {
    if constexpr (VAR == 0 || VAR == 2) {
        team_dft<R, INV>(x, pa, pb, ex, tw, t, slot);
    } else {
        reg::dft12<INV>(x);
        V w[R];
        tw_tree<INV>(tw[8 + t], w);
#pragma unroll
        for (int s = 1; s < R; ++s) x[s] = cmul(x[s], w[s]);
        __syncwarp();
#pragma unroll
        for (int s = 0; s < R; ++s) ex[slot(s, t)] = x[s];
        __syncwarp();
        if (s_on<R>(t)) {
            const int sa = s_a<R>(t), sb = s_b<R>(t);
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) {
                pa[tt] = ex[slot(sa, tt)];
                pb[tt] = ex[slot(sb, tt)];
            }
            reg::dft8<INV>(pa);
            reg::dft8<INV>(pb);
        }
        __syncwarp();
    }
}

template <int VAR, bool INV, typename SLOT>
__device__ __forceinline__ void tdft_dif(V* pa, V* pb, V* x, V* ex, const V* tw, int t, SLOT slot) {
    if constexpr (VAR == 0 || VAR == 2) {
        team_dft_dif<R, INV>(pa, pb, x, ex, tw, t, slot);
    } else {
        __syncwarp();
        if (s_on<R>(t)) {
            const int sa = s_a<R>(t), sb = s_b<R>(t);
            reg::dft8<INV>(pa);
            reg::dft8<INV>(pb);
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) {
                ex[slot(sa, tt)] = pa[tt];
                ex[slot(sb, tt)] = pb[tt];
            }
        }
        __syncwarp();
#pragma unroll
        for (int s = 0; s < R; ++s) x[s] = ex[slot(s, t)];
        V w[R];
        tw_tree<INV>(tw[8 + t], w);
#pragma unroll
        for (int s = 1; s < R; ++s) x[s] = cmul(x[s], w[s]);
        reg::dft12<INV>(x);
        __syncwarp();
    }
}

template <int VAR, int TEAMS>
__global__ void __launch_bounds__(8 * TEAMS, 1) k_fft(double* out, int items) {
    constexpr int NT = 8 * TEAMS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* X = reinterpret_cast<V*>(smem_raw);
    V* tw = X + NQ * P;
    const int tid = threadIdx.x, q = tid >> 3;
    int t = tid & 7;
    init_tw<NQ>(tw);
    for (int i = tid; i < NQ * P; i += NT) X[i] = V{1e-3 * (i % 97), 1e-3 * (i % 89)};
    __syncthreads();
    auto rs = [](int s2, int tt) { return rslot(s2, tt); };
    auto cs = [](int s2, int tt) { return rslot(s2, tt) * P; };
    for (int it = 0; it < items; ++it) {
#pragma unroll 1
        for (int j3 = q; j3 < NQ; j3 += TEAMS) {           // F2
            if (VAR == 2) asm volatile("" : "+r"(t));     // opaque: no hoisted per-thread addresses
            V* row = X + j3 * P;
            V x[R], pa[8], pb[8];
#pragma unroll
            for (int r = 0; r < R; ++r) x[r] = row[t + 8 * r];
            tdft<VAR, false>(x, pa, pb, row, tw, t, rs);
            if (s_on<R>(t)) {
                const int sa = s_a<R>(t), sb = s_b<R>(t);
#pragma unroll
                for (int qq = 0; qq < 8; ++qq) {
                    row[sa + R * qq] = pa[qq];
                    row[sb + R * qq] = pb[qq];
                }
            }
        }
        __syncthreads();
#pragma unroll 1
        for (int k2 = q; k2 < NQ; k2 += TEAMS) {           // F3
            if (VAR == 2) asm volatile("" : "+r"(t));     // opaque: no hoisted per-thread addresses
            V* col = X + k2;
            V x[R], pa[8], pb[8];
#pragma unroll
            for (int r = 0; r < R; ++r) x[r] = col[(t + 8 * r) * P];
            tdft<VAR, false>(x, pa, pb, col, tw, t, cs);
#pragma unroll
            for (int qq = 0; qq < 8; ++qq) {
                pa[qq] = V{pa[qq].x * (1.0 / 96), pa[qq].y * (1.0 / 96)};
                pb[qq] = V{pb[qq].x * (1.0 / 96), pb[qq].y * (1.0 / 96)};
            }
            tdft_dif<VAR, true>(pa, pb, x, col, tw, t, cs);
#pragma unroll
            for (int r = 0; r < R; ++r) col[(t + 8 * r) * P] = x[r];
        }
        __syncthreads();
#pragma unroll 1
        for (int j3 = q; j3 < NQ; j3 += TEAMS) {           // I2
            if (VAR == 2) asm volatile("" : "+r"(t));     // opaque: no hoisted per-thread addresses
            V* row = X + j3 * P;
            V x[R], pa[8], pb[8];
            if (s_on<R>(t)) {
                const int sa = s_a<R>(t), sb = s_b<R>(t);
#pragma unroll
                for (int qq = 0; qq < 8; ++qq) {
                    pa[qq] = row[sa + R * qq];
                    pb[qq] = row[sb + R * qq];
                }
            }
            tdft_dif<VAR, true>(pa, pb, x, row, tw, t, rs);
#pragma unroll
            for (int r = 0; r < R; ++r) row[t + 8 * r] = V{x[r].x * (1.0 / 96), x[r].y * (1.0 / 96)};
        }
        __syncthreads();
    }
    if (tid == 0) out[blockIdx.x] = X[5].x + X[P + 7].y;
}

template <int VAR, int TEAMS>
static void run(const char* name, int items, bool last = false) {
    constexpr int NT = 8 * TEAMS;
    const size_t smem = sizeof(V) * (NQ * P + NQ);
    cudaFuncSetAttribute(k_fft<VAR, TEAMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    double* out;
    cudaMalloc(&out, 148 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fft<VAR, TEAMS><<<148, NT, smem>>>(out, 2);
    cudaDeviceSynchronize();
    std::vector<float> ts;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_fft<VAR, TEAMS><<<148, NT, smem>>>(out, items);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    const double us_item = 1e3 * ts[2] / items;
    // the production C4 K2 runs 4704 / 148 = 31.8 items per SM
    printf("  \"%s\": {\"us_per_item_per_sm\": %.3f, \"c4_k2_fft_only_us\": %.1f, \"err\": \"%s\"}%s\n", name, us_item,
           us_item * 4704.0 / 148.0, cudaGetErrorString(cudaGetLastError()), last ? "" : ",");
}


// V3: stage 2 one s-value at a time (8 complex live), the spectral row kept in exchange-slot
// order between the passes (X(s + R q) at slot(s, q)): every thread writes back only the
// slots it read, so no second warp sync and no pa/pb pair in registers
template <bool INV, typename SLOT>
__device__ __forceinline__ void st1(V* x, V* ex, const V* tw, int t, SLOT slot) {
    // DIT stage 1: x[r] (element t + 8r) -> ex[slot(s, t)] = Y_t(s) W^{ts}
    reg::dft12<INV>(x);
#pragma unroll
    for (int s = 1; s < R; ++s) x[s] = twid<INV>(x[s], tw[s * 8 + t]);
#pragma unroll
    for (int s = 0; s < R; ++s) ex[slot(s, t)] = x[s];
}
template <bool INV, typename SLOT>
__device__ __forceinline__ void st1_dif(V* x, V* ex, const V* tw, int t, SLOT slot) {
    // DIF stage 1 (inverse of st1's layout): ex[slot(s, t)] -> x[r] = element t + 8r
#pragma unroll
    for (int s = 0; s < R; ++s) x[s] = ex[slot(s, t)];
#pragma unroll
    for (int s = 1; s < R; ++s) x[s] = twid<INV>(x[s], tw[s * 8 + t]);
    reg::dft12<INV>(x);
}
// stage 2 on this thread's own s values: f(s, p) transforms the 8 values in place
template <typename SLOT, typename F>
__device__ __forceinline__ void st2(V* ex, int t, SLOT slot, F f) {
    if (s_on<R>(t)) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int s = h ? s_b<R>(t) : s_a<R>(t);
            V p[8];
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) p[tt] = ex[slot(s, tt)];
            f(s, p);
#pragma unroll
            for (int tt = 0; tt < 8; ++tt) ex[slot(s, tt)] = p[tt];
        }
    }
}

template <int TEAMS>
__global__ void __launch_bounds__(8 * TEAMS, 1) k_fft3(double* out, int items) {
    constexpr int NT = 8 * TEAMS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* X = reinterpret_cast<V*>(smem_raw);
    V* tw = X + NQ * P;
    const int tid = threadIdx.x, q = tid >> 3, t = tid & 7;
    init_tw<NQ>(tw);
    for (int i = tid; i < NQ * P; i += NT) X[i] = V{1e-3 * (i % 97), 1e-3 * (i % 89)};
    __syncthreads();
    auto rs = [](int s2, int tt) { return rslot(s2, tt); };
    auto cs = [](int s2, int tt) { return rslot(s2, tt) * P; };
    for (int it = 0; it < items; ++it) {
#pragma unroll 1
        for (int j3 = q; j3 < NQ; j3 += TEAMS) {           // F2 -> row in slot order
            V* row = X + j3 * P;
            V x[R];
#pragma unroll
            for (int r = 0; r < R; ++r) x[r] = row[t + 8 * r];
            __syncwarp();
            st1<false>(x, row, tw, t, rs);
            __syncwarp();
            st2(row, t, rs, [](int, V* p) { reg::dft8<false>(p); });
            __syncwarp();
        }
        __syncthreads();
#pragma unroll 1
        for (int k2 = q; k2 < NQ; k2 += TEAMS) {           // F3 on column pos(k2)
            V* col = X + rslot(k2 % R, k2 / R);
            V x[R];
#pragma unroll
            for (int r = 0; r < R; ++r) x[r] = col[(t + 8 * r) * P];
            __syncwarp();
            st1<false>(x, col, tw, t, cs);
            __syncwarp();
            st2(col, t, cs, [](int, V* p) {
                reg::dft8<false>(p);
#pragma unroll
                for (int qq = 0; qq < 8; ++qq) p[qq] = V{p[qq].x * (1.0 / 96), p[qq].y * (1.0 / 96)};
                reg::dft8<true>(p);
            });
            __syncwarp();
            st1_dif<true>(x, col, tw, t, cs);
            __syncwarp();
#pragma unroll
            for (int r = 0; r < R; ++r) col[(t + 8 * r) * P] = x[r];
        }
        __syncthreads();
#pragma unroll 1
        for (int j3 = q; j3 < NQ; j3 += TEAMS) {           // I2 from slot order
            V* row = X + j3 * P;
            st2(row, t, rs, [](int, V* p) { reg::dft8<true>(p); });
            __syncwarp();
            V x[R];
            st1_dif<true>(x, row, tw, t, rs);
            __syncwarp();
#pragma unroll
            for (int r = 0; r < R; ++r) row[t + 8 * r] = V{x[r].x * (1.0 / 96), x[r].y * (1.0 / 96)};
        }
        __syncthreads();
    }
    if (tid == 0) out[blockIdx.x] = X[5].x + X[P + 7].y;
}

template <int TEAMS>
static void run3(const char* name, int items, bool last = false) {
    constexpr int NT = 8 * TEAMS;
    const size_t smem = sizeof(V) * (NQ * P + NQ);
    cudaFuncSetAttribute(k_fft3<TEAMS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    double* out;
    cudaMalloc(&out, 148 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fft3<TEAMS><<<148, NT, smem>>>(out, 2);
    cudaDeviceSynchronize();
    std::vector<float> ts;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        k_fft3<TEAMS><<<148, NT, smem>>>(out, items);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        ts.push_back(ms);
    }
    std::sort(ts.begin(), ts.end());
    const double us_item = 1e3 * ts[2] / items;
    printf("  \"%s\": {\"us_per_item_per_sm\": %.3f, \"c4_k2_fft_only_us\": %.1f, \"err\": \"%s\"}%s\n", name, us_item,
           us_item * 4704.0 / 148.0, cudaGetErrorString(cudaGetLastError()), last ? "" : ",");
}

int main() {
    printf("{\n");
    run<0, 32>("v0_table_twiddles_8w", 64);
    run<1, 32>("v1_tree_twiddles_8w", 64);
    run<0, 48>("v0_table_twiddles_12w", 64);
    run<1, 48>("v1_tree_twiddles_12w", 64);
    run<2, 32>("v2_opaque_t_8w", 64);
    run<2, 48>("v2_opaque_t_12w", 64);
    run3<32>("v3_half_stage2_slot_order_8w", 64);
    run3<48>("v3_half_stage2_slot_order_12w", 64, true);
    printf("}\n");
    return 0;
}
