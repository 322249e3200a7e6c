// fm_dft.cuh — register-resident small DFTs (radix 2/3/4/5/8/16) for the
// spatial tile FFT and the per-pixel tonal inverse FFT.
//
// Forward DFT: X[k] = sum_n x[n] W_R^{nk}, W_R = exp(-2*pi*i/R).
// Inverse (INV=true) uses conj(W) and is unnormalised; the 1/N factors of
// the whole pipeline are folded into the cached SE spectrum.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fm {

// work-list entry flag (int2.y of the per-ladder unit lists): the unit is
// "full" — its plane 0 is a known constant, not computed or stored
constexpr int kJobFull = 1 << 30;

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// a * b
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ float2 cmulc(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, a.y * b.y), fmaf(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }  // a * (-i)
__device__ __forceinline__ float2 mul_pi(float2 a) { return make_float2(-a.y, a.x); }  // a * (+i)
__device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// cos(2*pi*j/16); j is a compile-time constant after unrolling so the switch folds.
__device__ __forceinline__ float cos16(int j) {
  switch (j & 15) {
    case 0: return 1.0f;
    case 1: return 0.923879532511286756f;
    case 2: return 0.707106781186547524f;
    case 3: return 0.382683432365089772f;
    case 4: return 0.0f;
    case 5: return -0.382683432365089772f;
    case 6: return -0.707106781186547524f;
    case 7: return -0.923879532511286756f;
    case 8: return -1.0f;
    case 9: return -0.923879532511286756f;
    case 10: return -0.707106781186547524f;
    case 11: return -0.382683432365089772f;
    case 12: return 0.0f;
    case 13: return 0.382683432365089772f;
    case 14: return 0.707106781186547524f;
    default: return 0.923879532511286756f;
  }
}
__device__ __forceinline__ float sin16(int j) { return cos16(j - 4); }

// v * W_R^e (forward) or v * conj(W_R^e) (inverse), for R | 16, e compile-time.
template <int R, bool INV>
__device__ __forceinline__ float2 twc(float2 v, int e) {
  const int j = (e * (16 / R)) & 15;
  if (j == 0) return v;
  if (j == 4) return INV ? mul_pi(v) : mul_mi(v);
  if (j == 8) return make_float2(-v.x, -v.y);
  if (j == 12) return INV ? mul_mi(v) : mul_pi(v);
  const float c = cos16(j);
  const float s = INV ? sin16(j) : -sin16(j);
  return cmul(v, make_float2(c, s));
}

template <int R, bool INV>
__device__ __forceinline__ void dft(float2 (&x)[R]);

template <bool INV>
__device__ __forceinline__ void dft2_(float2 (&x)[2]) {
  const float2 a = x[0], b = x[1];
  x[0] = cadd(a, b);
  x[1] = csub(a, b);
}

template <bool INV>
__device__ __forceinline__ void dft4_(float2 (&x)[4]) {
  const float2 t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]);
  const float2 t2 = cadd(x[1], x[3]), t3 = csub(x[1], x[3]);
  const float2 r = INV ? mul_pi(t3) : mul_mi(t3);
  x[0] = cadd(t0, t2);
  x[2] = csub(t0, t2);
  x[1] = cadd(t1, r);
  x[3] = csub(t1, r);
}

// R = A*B four-step in registers, natural input and output order:
// X[k1 + A*k2] = sum_{n2<B} W_B^{n2 k2} W_R^{n2 k1} sum_{n1<A} x[n2 + B*n1] W_A^{n1 k1}
template <int A, int B, bool INV>
__device__ __forceinline__ void dft_ab(float2 (&x)[A * B]) {
  constexpr int R = A * B;
  float2 t[R];
#pragma unroll
  for (int n2 = 0; n2 < B; ++n2) {
    float2 a[A];
#pragma unroll
    for (int n1 = 0; n1 < A; ++n1) a[n1] = x[n2 + B * n1];
    dft<A, INV>(a);
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) t[n2 * A + k1] = twc<R, INV>(a[k1], n2 * k1);
  }
#pragma unroll
  for (int k1 = 0; k1 < A; ++k1) {
    float2 b[B];
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) b[n2] = t[n2 * A + k1];
    dft<B, INV>(b);
#pragma unroll
    for (int k2 = 0; k2 < B; ++k2) x[k1 + A * k2] = b[k2];
  }
}

template <bool INV>
__device__ __forceinline__ void dft3_(float2 (&x)[3]) {
  const float s3 = 0.866025403784438647f;  // sin(2*pi/3)
  const float2 t1 = cadd(x[1], x[2]);
  const float2 t2 = make_float2(fmaf(-0.5f, t1.x, x[0].x), fmaf(-0.5f, t1.y, x[0].y));
  const float2 d = csub(x[1], x[2]);
  const float2 t3 = make_float2(s3 * d.x, s3 * d.y);
  const float2 r = INV ? mul_pi(t3) : mul_mi(t3);
  x[0] = cadd(x[0], t1);
  x[1] = cadd(t2, r);
  x[2] = csub(t2, r);
}

template <bool INV>
__device__ __forceinline__ void dft5_(float2 (&x)[5]) {
  const float c1 = 0.309016994374947424f;   // cos(2pi/5)
  const float c2 = -0.809016994374947424f;  // cos(4pi/5)
  const float s1 = 0.951056516295153572f;   // sin(2pi/5)
  const float s2 = 0.587785252292473129f;   // sin(4pi/5)
  const float2 t1 = cadd(x[1], x[4]), t2 = cadd(x[2], x[3]);
  const float2 t3 = csub(x[1], x[4]), t4 = csub(x[2], x[3]);
  const float2 x0 = x[0];
  const float2 a1 = make_float2(x0.x + c1 * t1.x + c2 * t2.x, x0.y + c1 * t1.y + c2 * t2.y);
  const float2 a2 = make_float2(x0.x + c2 * t1.x + c1 * t2.x, x0.y + c2 * t1.y + c1 * t2.y);
  const float2 b1 = make_float2(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y);
  const float2 b2 = make_float2(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y);
  const float2 r1 = INV ? mul_pi(b1) : mul_mi(b1);
  const float2 r2 = INV ? mul_pi(b2) : mul_mi(b2);
  x[0] = make_float2(x0.x + t1.x + t2.x, x0.y + t1.y + t2.y);
  x[1] = cadd(a1, r1);
  x[4] = csub(a1, r1);
  x[2] = cadd(a2, r2);
  x[3] = csub(a2, r2);
}

template <int R, bool INV>
__device__ __forceinline__ void dft(float2 (&x)[R]) {
  if constexpr (R == 1) {
  } else if constexpr (R == 2) {
    dft2_<INV>(x);
  } else if constexpr (R == 3) {
    dft3_<INV>(x);
  } else if constexpr (R == 4) {
    dft4_<INV>(x);
  } else if constexpr (R == 5) {
    dft5_<INV>(x);
  } else if constexpr (R == 8) {
    dft_ab<2, 4, INV>(x);
  } else if constexpr (R == 16) {
    dft_ab<4, 4, INV>(x);
  } else {
    static_assert(R == 1, "unsupported radix");
  }
}

}  // namespace fm
