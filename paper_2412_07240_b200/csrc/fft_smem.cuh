// fft_smem.cuh -- mixed-radix (2, 3, 4 + direct 5, 7, 11, 13, 17) Stockham autosort FFT on a tile of P
// pencils held in shared memory (pencil p at offset p*PS, PS >= N).
// Forward uses e^{-2 pi i js/N} (eq:fourtrsf P:221) WITHOUT the 1/N (the
// scales of all axes are folded into the spectral multiplier); the inverse uses
// e^{+2 pi i js/N}. Twiddles come from a per-N table tw[m] = e^{-2 pi i m/N}
// computed once on the host in extended precision.
#pragma once
#include "device_common.cuh"
#include "fft_reg.cuh"

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

// Radix 17 (the paper's N_pa = 34 = 2 x 17 grids) with constant coefficients and
// the symmetric pairing of j and 17 - j: X[k] = A_k -/+ i B_k, X[17-k] = A_k +/- i B_k with
// A_k = v0 + sum_j (v_j + v_{17-j}) cos(2 pi jk/17), B_k = sum_j (v_j - v_{17-j}) sin(2 pi jk/17)
// -- 256 FMA for 17 outputs instead of 272 complex multiplies.
// cos / sin (2 pi m / 17), m = 0..8 (folded to immediates once the loops are unrolled)
__host__ __device__ __forceinline__ constexpr double r17c(int m) {
    return m == 0 ? 1.0 : m == 1 ? 0.93247222940435581 : m == 2 ? 0.73900891722065909 : m == 3 ? 0.44573835577653831
         : m == 4 ? 0.092268359463302016 : m == 5 ? -0.27366299007208289 : m == 6 ? -0.60263463637925629
         : m == 7 ? -0.85021713572961399 : -0.98297309968390179;
}
__host__ __device__ __forceinline__ constexpr double r17s(int m) {
    return m == 0 ? 0.0 : m == 1 ? 0.36124166618715292 : m == 2 ? 0.67369564364655721 : m == 3 ? 0.89516329135506234
         : m == 4 ? 0.99573417629503447 : m == 5 ? 0.96182564317281904 : m == 6 ? 0.7980172272802396
         : m == 7 ? 0.52643216287735606 : 0.18374951781657037;
}
template <bool INV, typename V> struct SmallDFT<17, INV, V> {
    static __device__ __forceinline__ void run(V* v) {
        using T = decltype(v[0].x);
        V a[9], b[9];
        V x0 = v[0];
#pragma unroll
        for (int j = 1; j <= 8; ++j) {
            a[j] = cadd(v[j], v[17 - j]);
            b[j] = csub(v[j], v[17 - j]);
            x0 = cadd(x0, a[j]);
        }
#pragma unroll
        for (int k = 1; k <= 8; ++k) {
            V A = v[0], B = V{T(0), T(0)};
#pragma unroll
            for (int j = 1; j <= 8; ++j) {
                const int m = (j * k) % 17;                         // compile-time after unrolling
                const T cs = (T)(m <= 8 ? r17c(m) : r17c(17 - m));
                const T sn = (T)(m <= 8 ? r17s(m) : -r17s(17 - m));
                A = V{fma(a[j].x, cs, A.x), fma(a[j].y, cs, A.y)};
                B = V{fma(b[j].x, sn, B.x), fma(b[j].y, sn, B.y)};
            }
            // forward: X_k = A - i B, X_{17-k} = A + i B; inverse: the conjugate pairing
            const V mB = V{B.y, -B.x};                              // -i B
            v[k] = INV ? csub(A, mB) : cadd(A, mB);
            v[17 - k] = INV ? cadd(A, mB) : csub(A, mB);
        }
        v[0] = x0;
    }
};

// Direct DFT of a small odd prime size R (5, 7, 11, 13, 17): X[k] = sum_j v[j] W_R^{jk},
// W_R^{m} = tw[(N/R) m] from the length-N table (the paper's grids N_pa = 34, 80, 200
// are not 2^a 3^b: P:413).
template <int R, bool INV, typename V>
__device__ __forceinline__ void prime_dft(V* v, const V* __restrict__ tw, int N) {
    V out[R];
    const int st = N / R;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        V acc = v[0];
#pragma unroll
        for (int j = 1; j < R; ++j) {
            V w = tw[st * ((j * k) % R)];
            if (INV) w.y = -w.y;
            const V t = cmul(v[j], w);
            acc = cadd(acc, t);
        }
        out[k] = acc;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) v[k] = out[k];
}

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
        if constexpr (R == 2 || R == 3 || R == 4) SmallDFT<R, INV, V>::run(v);
        else prime_dft<R, INV>(v, tw, N);
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
        else if (R == 3) stockham_stage<3, INV>(a, b, pl.N, Ns, P, PS, tw);
        else if (R == 5) stockham_stage<5, INV>(a, b, pl.N, Ns, P, PS, tw);
        else if (R == 7) stockham_stage<7, INV>(a, b, pl.N, Ns, P, PS, tw);
        else if (R == 11) stockham_stage<11, INV>(a, b, pl.N, Ns, P, PS, tw);
        else if (R == 13) stockham_stage<13, INV>(a, b, pl.N, Ns, P, PS, tw);
        else stockham_stage<17, INV>(a, b, pl.N, Ns, P, PS, tw);
        __syncthreads();
        V* t = a; a = b; b = t;
        Ns *= R;
    }
    return a;
}

// ---------------------------------------------------------------------------
// Compile-time Stockham FFT for the common pencil lengths: radix sequence,
// strides and divisors are constants, radix-8 stages run reg::dft8.
template <int N>
__host__ __device__ constexpr int ct_nstages() {
    return (N == 64 || N == 32 || N == 24 || N == 16 || N == 12 || N == 34) ? 2
         : (N == 96 || N == 128 || N == 256 || N == 48 || N == 192 || N == 384 || N == 512) ? 3 : 0;
}
template <int N>
__host__ __device__ constexpr int ct_radix(int st) {
    // first stage (Ns = 1) takes the largest radix: no twiddles there
    return N == 34 ? (st == 0 ? 17 : 2) : N == 64 ? 8 : N == 32 ? (st == 0 ? 8 : 4) : N == 24 ? (st == 0 ? 8 : 3) : N == 16 ? 4 : N == 12 ? (st == 0 ? 4 : 3)
         : N == 96 ? (st == 0 ? 8 : st == 1 ? 4 : 3) : N == 128 ? (st == 0 ? 8 : 4) : N == 256 ? (st < 2 ? 8 : 4)
         : N == 48 ? (st < 2 ? 4 : 3) : N == 192 ? (st < 2 ? 8 : 3) : N == 384 ? (st < 2 ? 8 : 6) : N == 512 ? 8 : 0;
}
template <int N>
inline constexpr bool ct_supported = ct_nstages<N>() > 0;

// Shared-memory layout of the compile-time path: one pad slot every 8 complex
// (sx), so the stride-R writes of a Stockham stage hit distinct bank groups.
template <int NC>
__host__ __device__ __forceinline__ int sx(int j) { return NC > 0 ? j + (j >> 3) : j; }
template <int NC>
__host__ __device__ __forceinline__ int pencil_stride(int N) { return NC > 0 ? NC + NC / 8 + 1 : N + 1; }

template <int R, bool INV, typename V>
__device__ __forceinline__ void reg_dft(V* v) {
    if constexpr (R == 8) reg::dft8<INV>(v);
    else if constexpr (R == 4) reg::r4<INV>(v[0], v[1], v[2], v[3]);
    else if constexpr (R == 6) {
        // 6 = 2 x 3: radix-3 over (0,2,4) and (1,3,5), twiddle W6, radix-2
        V a[3] = {v[0], v[2], v[4]}, b[3] = {v[1], v[3], v[5]};
        SmallDFT<3, INV, V>::run(a);
        SmallDFT<3, INV, V>::run(b);
        using T = decltype(v[0].x);
        const T h = T(0.8660254037844386467637231707529361834714);
        // W6^1 = (1/2, -h) forward, W6^2 = (-1/2, -h)
        const T sg = INV ? h : -h;
        b[1] = V{fma(b[1].x, T(0.5), -b[1].y * sg), fma(b[1].x, sg, b[1].y * T(0.5))};
        b[2] = V{fma(b[2].x, T(-0.5), -b[2].y * sg), fma(b[2].x, sg, b[2].y * T(-0.5))};
        for (int k = 0; k < 3; ++k) {
            v[k] = cadd(a[k], b[k]);
            v[k + 3] = csub(a[k], b[k]);
        }
    } else SmallDFT<R, INV, V>::run(v);
}

template <int N, int R, int NS, bool INV, typename V>
__device__ __forceinline__ void ct_stage(const V* __restrict__ src, V* __restrict__ dst, int P,
                                         const V* __restrict__ tw) {
    constexpr int NR = N / R, PS = N + N / 8 + 1, TWS = N / (NS * R);
    const int total = P * NR;
    for (int t = threadIdx.x; t < total; t += blockDim.x) {
        const int p = t / NR, j = t - p * NR;
        const int jq = j / NS, k = j - jq * NS;
        const V* s = src + p * PS;
        V v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = s[sx<N>(j + r * NR)];
        if constexpr (NS > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) {
                V w = tw[r * k * TWS];
                if (INV) w.y = -w.y;
                v[r] = cmul(v[r], w);
            }
        }
        reg_dft<R, INV>(v);
        V* d = dst + p * PS;
        const int o = jq * NS * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) d[sx<N>(o + r * NS)] = v[r];
    }
}

template <int N, int ST, int NS, bool INV, typename V>
__device__ __forceinline__ V* ct_fft_rec(V* a, V* b, int P, const V* __restrict__ tw) {
    if constexpr (ST >= ct_nstages<N>()) {
        return a;
    } else {
        constexpr int R = ct_radix<N>(ST);
        ct_stage<N, R, NS, INV>(a, b, P, tw);
        __syncthreads();
        return ct_fft_rec<N, ST + 1, NS * R, INV>(b, a, P, tw);
    }
}

// NC > 0: compile-time transform of length NC; NC == 0: the runtime plan.
template <int NC, bool INV, typename V>
__device__ __forceinline__ V* fft_any(V* a, V* b, int P, int PS, const FFTPlan& pl, const V* __restrict__ tw) {
    if constexpr (NC > 0) return ct_fft_rec<NC, 0, 1, INV>(a, b, P, tw);
    else return smem_fft<INV>(a, b, P, PS, pl, tw);
}

}  // namespace pmf
