// kernels_fdm.cu -- the paper's FDM baseline predictor in its
// efficient eigen form: explicit central differences with zero Dirichlet boundary
// (eq:FDM P:146-150, eq:fdiff P:158-164) have the DST-I eigenvectors R for every
// substep of the moving grid, so l steps are
//
//     P' = R^{-1} ( Lambda (.) R P ),  Lambda = prod_{n<l} lambda_n,  R^{-1} = 2/(N+1) R
//
// (eq:FST P:199-202), applied axis by axis in nx dimensions with
// lambda_n(j) = b_n + sum_m 2 a_{m,n} cos((j_m+1) pi/(N_m+1)),
// a_{m,n} = Q_mm dt / (2 delta_{m,n}^2), b_n = 1 - dt tr A - sum_m 2 a_{m,n}
// (readings R23-R25).
//
// DST-I sizes 2(N+1) (194 for N = 96) do not suit an FFT, so each axis transform is
// a dense batched GEMM on the FP64 tensor cores (mma.sync m8n8k4 .f64, DMMA):
// out[k][t] = sum_j S[k][j] in[j][t] over tiles of 32 pencils, S[k][j] =
// sin((k+1)(j+1) pi/(N+1)) read from its 2(N+1)-entry sine table. The last axis fuses forward
// transform, Lambda and inverse transform in one pass. fp64 only.
#include <algorithm>
#include <cmath>

#include "device_common.cuh"

namespace pmf {
namespace fdm {

constexpr int TP = 32;      // pencils per tile
constexpr int NTH = 128;    // 4 warps; warp w owns output rows [w NA/4, (w+1) NA/4)
constexpr int LMAX = 64;    // substeps held per filter in shared memory
constexpr int GLP = LMAX + 1;   // per-pencil table pitch (odd: lanes of different pencils in distinct banks)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// per-filter coefficient block: [n * 4 + m] = a_{m,n}, [4 LMAX + n] = b_n
__host__ __device__ constexpr int cstride() { return 5 * LMAX; }

// ============================================================================ prep (1 thread per filter)
template <int NX>
__global__ void k_fdm_prep(FilterState* st, double* coef, ModelParams mp, const SubstepEntry* __restrict__ sub,
                           double trace_base, int batch) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= batch) return;
    FilterState& f = st[b];
    double* P = coef + (long long)b * cstride();
    if (f.status != 0) return;
    for (int n = 0; n < mp.l; ++n) {
        double Bn[16];
        for (int i = 0; i < 16; ++i) Bn[i] = 0.0;
        mat_mul4(NX, sub[n].P, f.B, Bn);                     // grid at the start of substep n
        double asum = 0.0;
#pragma unroll
        for (int m = 0; m < NX; ++m) {
            double len2 = 0.0;
#pragma unroll
            for (int r = 0; r < NX; ++r) len2 = fma(Bn[r * 4 + m], Bn[r * 4 + m], len2);
            const double am = mp.Q[m * 4 + m] * mp.dt / (2.0 * len2);
            P[n * 4 + m] = am;
            asum += am;
        }
        P[4 * LMAX + n] = trace_base - 2.0 * asum;
    }
    double Bl[16], cl[4];
    for (int i = 0; i < 16; ++i) Bl[i] = 0.0;
    mat_mul4(NX, mp.Mtau, f.B, Bl);
    for (int a = 0; a < NX; ++a) {
        double s = 0.0;
        for (int k = 0; k < NX; ++k) s = fma(mp.Mtau[a * 4 + k], f.c[k], s);
        cl[a] = s;
    }
    for (int a = 0; a < NX; ++a) f.c[a] = cl[a];
    for (int i = 0; i < 16; ++i) f.B[i] = Bl[i];
}

// ============================================================================ DST-I pass along one axis
// MODE 0: forward (R), 1: inverse (2/(N+1) R), 2: last axis, forward x Lambda x inverse.
// AX0: the axis is contiguous (pencils are rows); else pencils along stride I.
struct DstArgs {
    double* W;
    const double* coef;
    long long I, O;         // strided: inner count and outer count; AX0: I = rows per filter, O = batch
    int ocpf;               // o values per filter
    int nx, l;
    int n[4];               // sizes per axis
    int axis;
};

// S[k][j] = sin((k+1)(j+1) pi/(N+1)) takes only 2(N+1) distinct values: the A fragments
// are read from the table T[m] = sin(m pi/(N+1)), m = (k+1)(j+1) mod 2(N+1), advanced by
// an integer step per k-slice, instead of a resident N x N matrix (135 KB at N = 128):
// the CTA needs ~45 KB of shared memory and two fit on an SM.
template <int NA, bool AX0, int MODE>
__global__ void __launch_bounds__(NTH, 3) k_dst(DstArgs a) {
    constexpr int M2 = 2 * (NA + 1);           // period of the sine table
    constexpr int IP = TP + 8;                 // tile pitch: B-fragment rows 8 doubles apart
    constexpr int MT = NA / 32;                // m8 tiles per warp (NA / 4 rows / 8)
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* X = reinterpret_cast<double*>(smem_raw);          // [NA][IP] tile (j or k rows, t columns)
    double* gl = X + NA * IP;                                 // [TP][GLP] per-pencil Lambda terms
    double* Ts = gl + TP * GLP;                               // [M2] sine table
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int m = tid; m < M2; m += NTH) Ts[m] = sinpi((double)m / (double)(NA + 1));
    __syncthreads();
    const long long tiles = (a.I + TP - 1) / TP, ntile = a.O * tiles;
    const int r0 = warp * (NA / 4);            // this warp's output rows
    // table index of this lane's A-fragment element (row r0 + 8 mi + lane/4, column kk + lane%4)
    // at kk = 0, and its advance per k-slice of 4 columns
    int idx0[MT], step[MT];
#pragma unroll
    for (int mi = 0; mi < MT; ++mi) {
        const int r1 = r0 + 8 * mi + (lane >> 2) + 1;
        idx0[mi] = (r1 * ((lane & 3) + 1)) % M2;
        step[mi] = (4 * r1) % M2;
    }
    auto gemm = [&](double acc[MT][4][2]) {
        int idx[MT];
#pragma unroll
        for (int mi = 0; mi < MT; ++mi) {
            idx[mi] = idx0[mi];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        }
#pragma unroll 4
        for (int kk = 0; kk < NA; kk += 4) {
            double bf[4];
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) bf[ni] = X[(kk + (lane & 3)) * IP + 8 * ni + (lane >> 2)];
#pragma unroll
            for (int mi = 0; mi < MT; ++mi) {
                const double af = Ts[idx[mi]];
                idx[mi] += step[mi];
                idx[mi] -= (idx[mi] >= M2) ? M2 : 0;
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af, bf[ni]);
            }
        }
    };
    // accumulators -> tile rows (k) in shared memory, scaled
    auto put = [&](double acc[MT][4][2], double sc) {
#pragma unroll
        for (int mi = 0; mi < MT; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) {
                const int k = r0 + 8 * mi + (lane >> 2), t = 8 * ni + 2 * (lane & 3);
                X[k * IP + t] = acc[mi][ni][0] * sc;
                X[k * IP + t + 1] = acc[mi][ni][1] * sc;
            }
    };
    for (long long blk = blockIdx.x; blk < ntile; blk += gridDim.x) {
        const long long o = blk / tiles, i0 = (blk - o * tiles) * TP;
        const int cnt = (int)(a.I - i0 < TP ? a.I - i0 : TP);
        // ---------------------------------------------------------------- load the tile: X[j][t]
        if (AX0) {
            const double* src = a.W + (o * a.I + i0) * NA;    // rows i0.. of filter o, NA each
            for (int e = tid; e < TP * NA; e += NTH) {
                const int t = e / NA, j = e - t * NA;
                X[j * IP + t] = t < cnt ? src[(long long)t * NA + j] : 0.0;
            }
        } else {
            const double* src = a.W + o * NA * a.I + i0;
            for (int e = tid; e < TP * NA; e += NTH) {
                const int j = e / TP, t = e - j * TP;
                X[j * IP + t] = t < cnt ? src[(long long)j * a.I + t] : 0.0;
            }
        }
        if (MODE == 2) {
            // per pencil: g_n = b_n + sum_{m != axis} 2 a_{m,n} cos((j_m+1) pi/(N_m+1))
            const long long filt = o / a.ocpf;
            const double* cf = a.coef + filt * cstride();
            for (int e = tid; e < TP * a.l; e += NTH) {
                const int t = e / a.l, n = e - t * a.l;
                // multi-index of the pencil: axes 0 .. axis-1 in the inner index, axes > axis in o
                long long in = i0 + t, oo = o - filt * a.ocpf;
                double g = cf[4 * LMAX + n];
                for (int m = 0; m < a.nx; ++m) {
                    if (m == a.axis) continue;
                    int jm;
                    if (m < a.axis) {
                        jm = (int)(in % a.n[m]);
                        in /= a.n[m];
                    } else {
                        jm = (int)(oo % a.n[m]);
                        oo /= a.n[m];
                    }
                    g = fma(2.0 * cf[n * 4 + m], cospi((double)(jm + 1) / (double)(a.n[m] + 1)), g);
                }
                gl[t * GLP + n] = g;
            }
        }
        __syncthreads();
        double acc[MT][4][2];
        gemm(acc);
        __syncthreads();                       // every warp has read the tile
        if (MODE == 2) {
            const long long filt = o / a.ocpf;
            const double* cf = a.coef + filt * cstride();
#pragma unroll
            for (int mi = 0; mi < MT; ++mi) {
                const int k = r0 + 8 * mi + (lane >> 2);
                const double ck = 2.0 * cospi((double)(k + 1) / (double)(NA + 1));
#pragma unroll
                for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int t = 8 * ni + 2 * (lane & 3) + e;
                        double lam = 1.0;
                        for (int n = 0; n < a.l; ++n) lam *= fma(cf[n * 4 + a.axis], ck, gl[t * GLP + n]);
                        acc[mi][ni][e] *= lam;
                    }
            }
            put(acc, 1.0);
            __syncthreads();
            gemm(acc);
            __syncthreads();
        }
        put(acc, MODE == 0 ? 1.0 : 2.0 / (NA + 1));
        __syncthreads();
        // ---------------------------------------------------------------- store: X[k][t]
        if (AX0) {
            double* dst = a.W + (o * a.I + i0) * NA;
            for (int e = tid; e < TP * NA; e += NTH) {
                const int t = e / NA, k = e - t * NA;
                if (t < cnt) dst[(long long)t * NA + k] = X[k * IP + t];
            }
        } else {
            double* dst = a.W + o * NA * a.I + i0;
            for (int e = tid; e < TP * NA; e += NTH) {
                const int k = e / TP, t = e - k * TP;
                if (t < cnt) dst[(long long)k * a.I + t] = X[k * IP + t];
            }
        }
        __syncthreads();
    }
}

}  // namespace fdm

using namespace fdm;

bool fdm_supported(const Dims& d, int dtype, int l) {
    if (dtype != 0 || l > LMAX) return false;
    for (int m = 0; m < d.nx; ++m)
        if (d.n[m] != 32 && d.n[m] != 64 && d.n[m] != 96 && d.n[m] != 128) return false;
    return true;
}

size_t fdm_coef_doubles(int batch) { return (size_t)cstride() * batch; }

template <int NA>
static cudaError_t dst_pass(DstArgs a, bool ax0, int mode, cudaStream_t s) {
    const size_t smem = sizeof(double) * ((size_t)NA * (TP + 8) + (size_t)TP * GLP + 2 * (NA + 1));
    auto launch = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        int dev = 0, nsm = 148, occ = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NTH, smem);
        if (e != cudaSuccess) return e;
        const long long work = a.O * ((a.I + TP - 1) / TP);
        const int grid = (int)std::max(1LL, std::min(work, (long long)nsm * std::max(occ, 1)));
        kern<<<grid, NTH, smem, s>>>(a);
        return cudaGetLastError();
    };
    if (ax0) {
        if (mode == 0) return launch(k_dst<NA, true, 0>);
        if (mode == 1) return launch(k_dst<NA, true, 1>);
        return launch(k_dst<NA, true, 2>);
    }
    if (mode == 0) return launch(k_dst<NA, false, 0>);
    if (mode == 1) return launch(k_dst<NA, false, 1>);
    return launch(k_dst<NA, false, 2>);
}

static cudaError_t dst_axis(const Dims& d, PencilBufs& b, int m, int mode, int l, cudaStream_t s) {
    DstArgs a{};
    a.W = (double*)b.W;
    a.coef = b.coef;
    a.nx = d.nx;
    a.l = l;
    a.axis = m;
    for (int q = 0; q < 4; ++q) a.n[q] = d.n[q];
    const bool ax0 = m == 0;
    if (ax0) {
        a.I = d.ntot / d.n[0];          // rows per filter
        a.O = d.batch;
        a.ocpf = 1;
    } else {
        long long I = 1, O = d.batch, ocpf = 1;
        for (int q = 0; q < m; ++q) I *= d.n[q];
        for (int q = m + 1; q < d.nx; ++q) {
            O *= d.n[q];
            ocpf *= d.n[q];
        }
        a.I = I;
        a.O = O;
        a.ocpf = (int)ocpf;
    }
    // MODE 2 on axis 0 (nx = 1): the pencil's other indices are none; the strided decode
    // treats rows as the inner index, which for nx = 1 is a single row per filter
    switch (d.n[m]) {
        case 32: return dst_pass<32>(a, ax0, mode, s);
        case 64: return dst_pass<64>(a, ax0, mode, s);
        case 96: return dst_pass<96>(a, ax0, mode, s);
        case 128: return dst_pass<128>(a, ax0, mode, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_fdm_predict(const Dims& d, int dtype, PencilBufs& b, const ModelParams& mp, double trace_base,
                               cudaStream_t s, int64_t* launches) {
    if (!fdm_supported(d, dtype, mp.l)) return cudaErrorInvalidValue;
    switch (d.nx) {
        case 1: k_fdm_prep<1><<<(d.batch + 127) / 128, 128, 0, s>>>(b.st, b.coef, mp, b.sub, trace_base, d.batch); break;
        case 2: k_fdm_prep<2><<<(d.batch + 127) / 128, 128, 0, s>>>(b.st, b.coef, mp, b.sub, trace_base, d.batch); break;
        case 3: k_fdm_prep<3><<<(d.batch + 127) / 128, 128, 0, s>>>(b.st, b.coef, mp, b.sub, trace_base, d.batch); break;
        default: k_fdm_prep<4><<<(d.batch + 127) / 128, 128, 0, s>>>(b.st, b.coef, mp, b.sub, trace_base, d.batch); break;
    }
    ++*launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const int L = d.nx - 1;
    for (int m = 0; m < L; ++m) {
        if ((e = dst_axis(d, b, m, 0, mp.l, s)) != cudaSuccess) return e;
        ++*launches;
    }
    if (b.ev0) cudaEventRecordWithFlags(b.ev0, s, cudaEventRecordExternal);
    if ((e = dst_axis(d, b, L, 2, mp.l, s)) != cudaSuccess) return e;
    if (b.ev1) cudaEventRecordWithFlags(b.ev1, s, cudaEventRecordExternal);
    ++*launches;
    for (int m = L - 1; m >= 0; --m) {
        if ((e = dst_axis(d, b, m, 1, mp.l, s)) != cudaSuccess) return e;
        ++*launches;
    }
    return cudaSuccess;
}

}  // namespace pmf
