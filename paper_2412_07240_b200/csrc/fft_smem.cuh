// fft_smem.cuh -- mixed-radix (2, 3, 4) Stockham autosort FFT on a tile of P
// pencils held in shared memory (pencil p at offset p*PS, PS >= N).
// Forward uses e^{-2 pi i js/N} (eq:fourtrsf P:221) WITHOUT the 1/N (the
// scales of all axes are folded into the spectral multiplier); the inverse uses
// e^{+2 pi i js/N}. Twiddles come from a per-N table tw[m] = e^{-2 pi i m/N}
// computed once on the host in extended precision.
#pragma once
#include "device_common.cuh"

namespace pmf {

struct FFTPlan {
    int N;
    int nst;
    int r[16];
};

template <int R, bool INV, typename V> struct SmallDFT;

template <bool INV, typename V> struct SmallDFT<2, INV, V> {
    static __device__ __forceinline__ void run(V* v) {
        V a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    }
};

template <bool INV, typename V> struct SmallDFT<4, INV, V> {
    static __device__ __forceinline__ void run(V* v) {
        V a = cadd(v[0], v[2]), b = csub(v[0], v[2]);
        V c = cadd(v[1], v[3]), d = mul_mi<INV>(csub(v[1], v[3]));
        v[0] = cadd(a, c);
        v[2] = csub(a, c);
        v[1] = cadd(b, d);
        v[3] = csub(b, d);
    }
};

template <bool INV, typename V> struct SmallDFT<3, INV, V> {
    static __device__ __forceinline__ void run(V* v) {
        using T = decltype(v[0].x);
        const T h = T(0.8660254037844386467637231707529361834714);   // sin(2 pi / 3)
        V t1 = cadd(v[1], v[2]);
        V t2 = {v[0].x - T(0.5) * t1.x, v[0].y - T(0.5) * t1.y};
        V d = csub(v[1], v[2]);
        V t3 = mul_mi<INV>(V{h * d.x, h * d.y});                    // -i h (v1 - v2) forward
        v[0] = cadd(v[0], t1);
        v[1] = cadd(t2, t3);
        v[2] = csub(t2, t3);
    }
};

template <int R, bool INV, typename V>
__device__ __forceinline__ void stockham_stage(const V* __restrict__ src, V* __restrict__ dst, int N,
                                               int Ns, int P, int PS, const V* __restrict__ tw) {
    const int NR = N / R;
    const int total = P * NR;
    const int twstep = N / (Ns * R);
    // exact float-reciprocal division: the fractional part of (x + 0.5)/d is >= 0.5/d >> float error
    const float invNR = 1.0f / (float)NR, invNs = 1.0f / (float)Ns;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int p = (int)(((float)t + 0.5f) * invNR);
        const int j = t - p * NR;
        const int jq = (int)(((float)j + 0.5f) * invNs);
        const int k = j - jq * Ns;
        const V* s = src + p * PS;
        V v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = s[j + r * NR];
        if (Ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                V w = tw[r * k * twstep];
                if (INV) w.y = -w.y;
                v[r] = cmul(v[r], w);
            }
        }
        SmallDFT<R, INV, V>::run(v);
        const int idxD = jq * Ns * R + k;
        V* d = dst + p * PS;
#pragma unroll
        for (int r = 0; r < R; ++r) d[idxD + r * Ns] = v[r];
    }
}

// Transform the P pencils in `a` (uses `b` as ping-pong scratch). The caller
// must __syncthreads() before the call; returns the buffer holding the result
// (synchronised).
template <bool INV, typename V>
__device__ V* smem_fft(V* a, V* b, int P, int PS, const FFTPlan& pl, const V* __restrict__ tw) {
    int Ns = 1;
    for (int s = 0; s < pl.nst; ++s) {
        const int R = pl.r[s];
        if (R == 4) stockham_stage<4, INV>(a, b, pl.N, Ns, P, PS, tw);
        else if (R == 2) stockham_stage<2, INV>(a, b, pl.N, Ns, P, PS, tw);
        else stockham_stage<3, INV>(a, b, pl.N, Ns, P, PS, tw);
        __syncthreads();
        V* t = a; a = b; b = t;
        Ns *= R;
    }
    return a;
}

}  // namespace pmf
