// fft_reg.cuh -- small DFTs held in registers (natural order in and out):
// radix 4, 8, 16 (4x4) with the constant twiddles of W16. Used by the resident
// epoch kernel (16 x 8 decomposition of the 128-point transforms) and by the
// compile-time Stockham stages of the pencil path.
#pragma once
#include "device_common.cuh"

namespace pmf {
namespace reg {

template <typename T> struct K {
    static constexpr T C1 = T(0.92387953251128675613);   // cos(pi/8)
    static constexpr T S1 = T(0.38268343236508977173);   // sin(pi/8)
    static constexpr T R2 = T(0.70710678118654752440);   // 1/sqrt(2)
};

// multiply by W16^e (forward: e^{-2 pi i e/16}; inverse: conjugate)
template <int E, bool INV, typename V>
__device__ __forceinline__ V w16(V a) {
    using T = decltype(a.x);
    constexpr int e = E & 15;
    if constexpr (e == 0) return a;
    else if constexpr (e == 4) return mul_mi<INV>(a);
    else if constexpr (e == 8) return V{-a.x, -a.y};
    else if constexpr (e == 12) return mul_mi<!INV>(a);
    else if constexpr (e == 2 || e == 6 || e == 10 || e == 14) {
        // (1 - i)/sqrt2 rotated by multiples of -i
        V b = a;
        if constexpr (e == 6) b = mul_mi<INV>(a);
        else if constexpr (e == 10) b = V{-a.x, -a.y};
        else if constexpr (e == 14) b = mul_mi<!INV>(a);
        const T r = K<T>::R2;
        if (INV) return V{(b.x - b.y) * r, (b.x + b.y) * r};
        return V{(b.x + b.y) * r, (b.y - b.x) * r};
    } else {
        const double ang = 2.0 * 3.14159265358979323846 * e / 16.0;
        // compile-time constants for e = 1,3,5,7,9,11,13,15
        T c, s;
        if constexpr (e == 1 || e == 15) { c = K<T>::C1; s = K<T>::S1; }
        else if constexpr (e == 3 || e == 13) { c = K<T>::S1; s = K<T>::C1; }
        else if constexpr (e == 5 || e == 11) { c = -K<T>::S1; s = K<T>::C1; }
        else { c = -K<T>::C1; s = K<T>::S1; }
        (void)ang;
        if constexpr (e > 8) s = -s;     // sin(2 pi e/16) < 0 for e > 8
        // forward multiplier (c, -s); inverse (c, s)
        const T si = INV ? s : -s;
        return V{fma(a.x, c, -a.y * si), fma(a.x, si, a.y * c)};
    }
}

template <bool INV, typename V>
__device__ __forceinline__ void r4(V& a0, V& a1, V& a2, V& a3) {
    V s02 = cadd(a0, a2), d02 = csub(a0, a2);
    V s13 = cadd(a1, a3), d13 = mul_mi<INV>(csub(a1, a3));
    a0 = cadd(s02, s13);
    a2 = csub(s02, s13);
    a1 = cadd(d02, d13);
    a3 = csub(d02, d13);
}

// in-place 16-point DFT, natural order in and out
template <bool INV, typename V>
__device__ __forceinline__ void dft16(V* x) {
    // radix-4 over r2 for each r1: x[r1 + 4 r2] -> Y(r1, s2) at x[r1 + 4 s2]
#pragma unroll
    for (int r1 = 0; r1 < 4; ++r1) r4<INV>(x[r1], x[r1 + 4], x[r1 + 8], x[r1 + 12]);
    x[5] = w16<1, INV>(x[5]);
    x[9] = w16<2, INV>(x[9]);
    x[13] = w16<3, INV>(x[13]);
    x[6] = w16<2, INV>(x[6]);
    x[10] = w16<4, INV>(x[10]);
    x[14] = w16<6, INV>(x[14]);
    x[7] = w16<3, INV>(x[7]);
    x[11] = w16<6, INV>(x[11]);
    x[15] = w16<9, INV>(x[15]);
    // radix-4 over r1 for each s2: (x[4 s2 + r1]) -> X(s2 + 4 s1)
    V y[16];
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) {
        V a0 = x[4 * s2], a1 = x[4 * s2 + 1], a2 = x[4 * s2 + 2], a3 = x[4 * s2 + 3];
        r4<INV>(a0, a1, a2, a3);
        y[s2] = a0;
        y[s2 + 4] = a1;
        y[s2 + 8] = a2;
        y[s2 + 12] = a3;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = y[i];
}

// in-place 8-point DFT, natural order in and out
template <bool INV, typename V>
__device__ __forceinline__ void dft8(V* x) {
    using T = decltype(x[0].x);
    // radix-4 over r2 for r1 = 0, 1: x[r1 + 2 r2]
    V a0 = x[0], a1 = x[2], a2 = x[4], a3 = x[6];
    V b0 = x[1], b1 = x[3], b2 = x[5], b3 = x[7];
    r4<INV>(a0, a1, a2, a3);
    r4<INV>(b0, b1, b2, b3);
    const T r = K<T>::R2;
    // twiddle W8^{s2} on the r1 = 1 branch
    if (INV) {
        b1 = V{(b1.x - b1.y) * r, (b1.x + b1.y) * r};
        b2 = mul_mi<true>(b2);
        b3 = V{-(b3.x + b3.y) * r, (b3.x - b3.y) * r};
    } else {
        b1 = V{(b1.x + b1.y) * r, (b1.y - b1.x) * r};
        b2 = mul_mi<false>(b2);
        b3 = V{(b3.y - b3.x) * r, -(b3.x + b3.y) * r};
    }
    x[0] = cadd(a0, b0);
    x[4] = csub(a0, b0);
    x[1] = cadd(a1, b1);
    x[5] = csub(a1, b1);
    x[2] = cadd(a2, b2);
    x[6] = csub(a2, b2);
    x[3] = cadd(a3, b3);
    x[7] = csub(a3, b3);
}

// radix 3 (forward: W3 = e^{-2 pi i/3}), natural order
template <bool INV, typename V>
__device__ __forceinline__ void r3(V& a0, V& a1, V& a2) {
    using T = decltype(a0.x);
    const T h = T(0.86602540378443864676);     // sin(2 pi/3)
    const V t1 = cadd(a1, a2);
    const V t2 = V{fma(T(-0.5), t1.x, a0.x), fma(T(-0.5), t1.y, a0.y)};
    const V d = csub(a1, a2);
    const V t3 = mul_mi<INV>(V{h * d.x, h * d.y});
    a0 = cadd(a0, t1);
    a1 = cadd(t2, t3);
    a2 = csub(t2, t3);
}

// multiply by W12^E (forward e^{-2 pi i E/12}; inverse: conjugate), E in {1,2,3,4,6}
template <int E, bool INV, typename V>
__device__ __forceinline__ V w12(V a) {
    using T = decltype(a.x);
    if constexpr (E == 3) return mul_mi<INV>(a);
    else if constexpr (E == 6) return V{-a.x, -a.y};
    else {
        constexpr T h = T(0.86602540378443864676);
        constexpr T c = E == 1 ? h : (E == 2 ? T(0.5) : T(-0.5));
        constexpr T s = E == 1 ? T(0.5) : h;
        const T si = INV ? s : -s;
        return V{fma(a.x, c, -a.y * si), fma(a.x, si, a.y * c)};
    }
}

// in-place 12-point DFT (4 x 3 Cooley-Tukey), natural order in and out:
// r = r1 + 4 r2 -> radix 3 over r2, twiddle W12^{r1 s2}, radix 4 over r1 -> k = s2 + 3 s1
template <bool INV, typename V>
__device__ __forceinline__ void dft12(V* x) {
#pragma unroll
    for (int r1 = 0; r1 < 4; ++r1) r3<INV>(x[r1], x[r1 + 4], x[r1 + 8]);
    x[5] = w12<1, INV>(x[5]);
    x[9] = w12<2, INV>(x[9]);
    x[6] = w12<2, INV>(x[6]);
    x[10] = w12<4, INV>(x[10]);
    x[7] = w12<3, INV>(x[7]);
    x[11] = w12<6, INV>(x[11]);
    V y[12];
#pragma unroll
    for (int s2 = 0; s2 < 3; ++s2) {
        V a0 = x[4 * s2], a1 = x[4 * s2 + 1], a2 = x[4 * s2 + 2], a3 = x[4 * s2 + 3];
        r4<INV>(a0, a1, a2, a3);
        y[s2] = a0;
        y[s2 + 3] = a1;
        y[s2 + 6] = a2;
        y[s2 + 9] = a3;
    }
#pragma unroll
    for (int i = 0; i < 12; ++i) x[i] = y[i];
}

}  // namespace reg
}  // namespace pmf
