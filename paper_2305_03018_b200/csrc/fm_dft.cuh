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

// Complex primitives.  On sm_100 every one of them is ONE packed f32x2
// instruction (FADD2 / FMUL2 / FFMA2: same lane throughput as two scalar ops,
// half the issue slots): a real scale rides as a broadcast operand and the
// "times +-i" swizzle + sign as operand modifiers, so a complex multiply is
// FMUL2 + FFMA2.  The host path (codelet tests) computes the same formulas.
#if defined(__CUDA_ARCH__) && __CUDA_ARCH__ >= 1000
__device__ __forceinline__ unsigned long long pk2(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long r) {
  float a, b;
  asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
  return make_float2(a, b);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return upk2(r);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.x, b.y)));
  return upk2(r);
}
// a + i b,  a - i b
__device__ __forceinline__ float2 cadd_i(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(-b.y, b.x)));
  return upk2(r);
}
__device__ __forceinline__ float2 csub_i(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(b.y, -b.x)));
  return upk2(r);
}
// s a
__device__ __forceinline__ float2 cscale(float2 a, float s) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(s, s)));
  return upk2(r);
}
// s a + c
__device__ __forceinline__ float2 cfma(float s, float2 a, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a.x, a.y)), "l"(pk2(s, s)), "l"(pk2(c.x, c.y)));
  return upk2(r);
}
// s (i a) + c,  s (-i a) + c
__device__ __forceinline__ float2 cfma_i(float s, float2 a, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(-a.y, a.x)), "l"(pk2(s, s)), "l"(pk2(c.x, c.y)));
  return upk2(r);
}
__device__ __forceinline__ float2 cfma_mi(float s, float2 a, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a.y, -a.x)), "l"(pk2(s, s)), "l"(pk2(c.x, c.y)));
  return upk2(r);
}
#else
__host__ __device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ float2 cadd_i(float2 a, float2 b) { return make_float2(a.x - b.y, a.y + b.x); }
__host__ __device__ __forceinline__ float2 csub_i(float2 a, float2 b) { return make_float2(a.x + b.y, a.y - b.x); }
__host__ __device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ float2 cfma(float s, float2 a, float2 c) {
  return make_float2(fmaf(s, a.x, c.x), fmaf(s, a.y, c.y));
}
__host__ __device__ __forceinline__ float2 cfma_i(float s, float2 a, float2 c) {
  return make_float2(fmaf(s, -a.y, c.x), fmaf(s, a.x, c.y));
}
__host__ __device__ __forceinline__ float2 cfma_mi(float s, float2 a, float2 c) {
  return make_float2(fmaf(s, a.y, c.x), fmaf(s, -a.x, c.y));
}
#endif
// a * b = b.x a + b.y (i a)
__host__ __device__ __forceinline__ float2 cmul(float2 a, float2 b) { return cfma_i(b.y, a, cscale(a, b.x)); }
// a * conj(b) = b.x a + b.y (-i a)
__host__ __device__ __forceinline__ float2 cmulc(float2 a, float2 b) { return cfma_mi(b.y, a, cscale(a, b.x)); }
__host__ __device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }  // a * (-i)
__host__ __device__ __forceinline__ float2 mul_pi(float2 a) { return make_float2(-a.y, a.x); }  // a * (+i)
__host__ __device__ __forceinline__ float2 conjf2(float2 a) { return make_float2(a.x, -a.y); }

// cos(2*pi*j/16); j is a compile-time constant after unrolling so the switch folds.
__host__ __device__ __forceinline__ float cos16(int j) {
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
__host__ __device__ __forceinline__ float sin16(int j) { return cos16(j - 4); }

// v * W_R^e (forward) or v * conj(W_R^e) (inverse), for R | 16, e compile-time.
template <int R, bool INV>
__host__ __device__ __forceinline__ float2 twc(float2 v, int e) {
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
__host__ __device__ __forceinline__ void dft(float2 (&x)[R]);

template <bool INV>
__host__ __device__ __forceinline__ void dft2_(float2 (&x)[2]) {
  const float2 a = x[0], b = x[1];
  x[0] = cadd(a, b);
  x[1] = csub(a, b);
}

template <bool INV>
__host__ __device__ __forceinline__ void dft4_(float2 (&x)[4]) {
  const float2 t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]);
  const float2 t2 = cadd(x[1], x[3]), t3 = csub(x[1], x[3]);
  x[0] = cadd(t0, t2);
  x[2] = csub(t0, t2);
  x[1] = INV ? cadd_i(t1, t3) : csub_i(t1, t3);
  x[3] = INV ? csub_i(t1, t3) : cadd_i(t1, t3);
}

// R = A*B four-step in registers, natural input and output order:
// X[k1 + A*k2] = sum_{n2<B} W_B^{n2 k2} W_R^{n2 k1} sum_{n1<A} x[n2 + B*n1] W_A^{n1 k1}
template <int A, int B, bool INV>
__host__ __device__ __forceinline__ void dft_ab(float2 (&x)[A * B]) {
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
__host__ __device__ __forceinline__ void dft3_(float2 (&x)[3]) {
  const float s3 = 0.866025403784438647f;  // sin(2*pi/3)
  const float2 t1 = cadd(x[1], x[2]);
  const float2 t2 = cfma(-0.5f, t1, x[0]);
  const float2 d = csub(x[1], x[2]);
  x[0] = cadd(x[0], t1);
  // t2 +- s3 (i d) (inverse), t2 -+ s3 (i d) (forward)
  x[1] = INV ? cfma_i(s3, d, t2) : cfma_mi(s3, d, t2);
  x[2] = INV ? cfma_mi(s3, d, t2) : cfma_i(s3, d, t2);
}

template <bool INV>
__host__ __device__ __forceinline__ void dft5_(float2 (&x)[5]) {
  const float c1 = 0.309016994374947424f;   // cos(2pi/5)
  const float c2 = -0.809016994374947424f;  // cos(4pi/5)
  const float s1 = 0.951056516295153572f;   // sin(2pi/5)
  const float s2 = 0.587785252292473129f;   // sin(4pi/5)
  const float2 t1 = cadd(x[1], x[4]), t2 = cadd(x[2], x[3]);
  const float2 t3 = csub(x[1], x[4]), t4 = csub(x[2], x[3]);
  const float2 x0 = x[0];
  const float2 a1 = cfma(c2, t2, cfma(c1, t1, x0));
  const float2 a2 = cfma(c1, t2, cfma(c2, t1, x0));
  const float2 b1 = cfma(s2, t4, cscale(t3, s1));
  const float2 b2 = cfma(-s1, t4, cscale(t3, s2));
  x[0] = cadd(x0, cadd(t1, t2));
  // a +- i b (inverse), a -+ i b (forward)
  x[1] = INV ? cadd_i(a1, b1) : csub_i(a1, b1);
  x[4] = INV ? csub_i(a1, b1) : cadd_i(a1, b1);
  x[2] = INV ? cadd_i(a2, b2) : csub_i(a2, b2);
  x[3] = INV ? csub_i(a2, b2) : cadd_i(a2, b2);
}

// ---------------------------------------------------------------------------
// FMA-shaped radix-8 / radix-16 codelets.  Four-step (A x 4) in registers like
// dft_ab, but the second-stage twiddles are folded into the radix-4
// butterflies: a W8-type twiddle h(1 -/+ i) becomes two adds whose scale h
// rides in the butterfly FMAs, and a general twiddle c(1 -/+ i tan) becomes two
// FMAs with the cosine again carried by the butterfly FMAs
// (DFT16: 144 instead of 160 FP instructions, DFT8: 52 instead of 56).
// sigma = -1 forward (W = exp(-2 pi i/16)), +1 inverse.

// Radix-4 stage over b_n = W^{n e} a_n for the W8-type row (e = 2 in units of
// W16): outputs X_{k2} = sum_n W4^{n k2} b_n, k2 = 0..3.
template <bool INV>
__host__ __device__ __forceinline__ void bfly4_w8(float2 a0, float2 a1, float2 a2, float2 a3, float2& X0, float2& X1,
                                                  float2& X2, float2& X3) {
  constexpr float h = 0.707106781186547524f;
  constexpr float sg = INV ? 1.0f : -1.0f;
  // b2 = sigma*i*a2: S = a0 + b2, D = a0 - b2
  const float2 S = INV ? cadd_i(a0, a2) : csub_i(a0, a2);
  const float2 D = INV ? csub_i(a0, a2) : cadd_i(a0, a2);
  // b1 + b3 = h P', b1 - b3 = h Q'  (b1 = W^2 a1, b3 = W^6 a3)
  const float2 d = csub(a1, a3), e = cadd(a1, a3);
  const float2 P = INV ? cadd_i(d, e) : csub_i(d, e);
  const float2 Q = INV ? cadd_i(e, d) : csub_i(e, d);
  X0 = cfma(h, P, S);
  X2 = cfma(-h, P, S);
  X1 = cfma_i(sg * h, Q, D);
  X3 = cfma_i(-sg * h, Q, D);
}

template <bool INV>
__host__ __device__ __forceinline__ void dft8_(float2 (&x)[8]) {
  float2 a[4][2];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    a[n2][0] = cadd(x[n2], x[n2 + 4]);
    a[n2][1] = csub(x[n2], x[n2 + 4]);
  }
  float2 b[4] = {a[0][0], a[1][0], a[2][0], a[3][0]};
  dft4_<INV>(b);
  x[0] = b[0];
  x[2] = b[1];
  x[4] = b[2];
  x[6] = b[3];
  bfly4_w8<INV>(a[0][1], a[1][1], a[2][1], a[3][1], x[1], x[3], x[5], x[7]);
}

template <bool INV>
__host__ __device__ __forceinline__ void dft16_(float2 (&x)[16]) {
  constexpr float h = 0.707106781186547524f;
  constexpr float c1 = 0.923879532511286756f;  // cos(pi/8)
  constexpr float t1 = 0.414213562373095049f;  // tan(pi/8)
  constexpr float sg = INV ? 1.0f : -1.0f;
  float2 a[4][4];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    float2 v[4] = {x[n2], x[n2 + 4], x[n2 + 8], x[n2 + 12]};
    dft4_<INV>(v);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) a[n2][k1] = v[k1];
  }
  // k1 = 0: plain radix-4
  {
    float2 b[4] = {a[0][0], a[1][0], a[2][0], a[3][0]};
    dft4_<INV>(b);
    x[0] = b[0];
    x[4] = b[1];
    x[8] = b[2];
    x[12] = b[3];
  }
  // k1 = 2: twiddles W^0, W^2, W^4, W^6
  bfly4_w8<INV>(a[0][2], a[1][2], a[2][2], a[3][2], x[2], x[6], x[10], x[14]);
  // k1 = 1: twiddles W^0, W^1, W^2, W^3
  {
    const float2 a0 = a[0][1], a1 = a[1][1], a2 = a[2][1], a3 = a[3][1];
    // b2 = W^2 a2 = h (a2.x - s a2.y, a2.y + s a2.x)
    const float2 A2 = INV ? cadd_i(a2, a2) : csub_i(a2, a2);
    const float2 S = cfma(h, A2, a0);
    const float2 D = cfma(-h, A2, a0);
    // b1 = W^1 a1 = c1 u, b3 = W^3 a3 = c1 v
    const float2 u = cfma_i(sg * t1, a1, a1);
    const float2 v = cfma_i(sg, a3, cscale(a3, t1));
    const float2 p = cadd(u, v), q = csub(u, v);
    x[1] = cfma(c1, p, S);
    x[9] = cfma(-c1, p, S);
    x[5] = cfma_i(sg * c1, q, D);
    x[13] = cfma_i(-sg * c1, q, D);
  }
  // k1 = 3: twiddles W^0, W^3, W^6, W^9 (= -W^1)
  {
    const float2 a0 = a[0][3], a1 = a[1][3], a2 = a[2][3], a3 = a[3][3];
    // b2 = W^6 a2 = -h (a2 - s i a2) = -h B2
    const float2 B2 = INV ? csub_i(a2, a2) : cadd_i(a2, a2);
    const float2 S = cfma(-h, B2, a0);
    const float2 D = cfma(h, B2, a0);
    // b1 = W^3 a1 = c1 v1, b3 = W^9 a3 = -c1 u3
    const float2 v1 = cfma_i(sg, a1, cscale(a1, t1));
    const float2 u3 = cfma_i(sg * t1, a3, a3);
    const float2 p = csub(v1, u3), q = cadd(v1, u3);
    x[3] = cfma(c1, p, S);
    x[11] = cfma(-c1, p, S);
    x[7] = cfma_i(sg * c1, q, D);
    x[15] = cfma_i(-sg * c1, q, D);
  }
}

// v * W_32^j (forward) or v * conj(W_32^j), j in [0, 16) compile-time
template <bool INV>
__host__ __device__ __forceinline__ float2 tw32(float2 v, int j) {
  if (j == 0) return v;
  if (j == 8) return INV ? mul_pi(v) : mul_mi(v);
  if ((j & 1) == 0) return twc<16, INV>(v, j / 2);
  // cos(2 pi j / 32) for odd j
  constexpr float c1 = 0.980785280403230449f, c3 = 0.831469612302545237f;
  constexpr float c5 = 0.555570233019602225f, c7 = 0.195090322016128268f;
  const int jj = j < 8 ? j : 16 - j;   // cos(2 pi (16 - j)/32) = -cos(2 pi j/32), sin equal
  const float c0 = jj == 1 ? c1 : jj == 3 ? c3 : jj == 5 ? c5 : c7;
  const float s0 = jj == 1 ? c7 : jj == 3 ? c5 : jj == 5 ? c3 : c1;   // sin(2 pi jj/32) = cos(2 pi (8-jj)/32)
  const float c = j < 8 ? c0 : -c0;
  return cmul(v, make_float2(c, INV ? s0 : -s0));
}

// cos / sin (2 pi j / 128) for a compile-time j in [0, 128): quarter-wave table
__host__ __device__ constexpr float cos128q(int i) {
  constexpr float q[33] = {1.000000000000000000f, 0.998795456205172405f, 0.995184726672196929f, 0.989176509964781014f, 0.980785280403230431f, 0.970031253194543974f, 0.956940335732208824f, 0.941544065183020806f, 0.923879532511286738f, 0.903989293123443338f, 0.881921264348355050f, 0.857728610000272118f, 0.831469612302545236f, 0.803207531480644943f, 0.773010453362736993f, 0.740951125354959106f, 0.707106781186547573f, 0.671558954847018330f, 0.634393284163645488f, 0.595699304492433468f, 0.555570233019602289f, 0.514102744193221661f, 0.471396736825997809f, 0.427555093430282196f, 0.382683432365089837f, 0.336889853392220051f, 0.290284677254462331f, 0.242980179903263982f, 0.195090322016128331f, 0.146730474455361748f, 0.098017140329560770f, 0.049067674327418126f, 0.000000000000000061f};
  return q[i];
}
__host__ __device__ constexpr float cos128(int j) {
  return (j >> 5) == 0 ? cos128q(j & 31) : (j >> 5) == 1 ? -cos128q(32 - (j & 31))
         : (j >> 5) == 2 ? -cos128q(j & 31) : cos128q(32 - (j & 31));
}
__host__ __device__ constexpr float sin128(int j) { return cos128((j + 96) & 127); }   // sin x = cos(x - pi/2)
// v * W_128^j (forward) or v * conj(W_128^j), j compile-time
template <bool INV>
__host__ __device__ __forceinline__ float2 tw128(float2 v, int j) {
  j &= 127;
  if (j == 0) return v;
  if (j == 32) return INV ? mul_pi(v) : mul_mi(v);
  if (j == 64) return make_float2(-v.x, -v.y);
  if (j == 96) return INV ? mul_mi(v) : mul_pi(v);
  return cmul(v, make_float2(cos128(j), INV ? sin128(j) : -sin128(j)));
}

// 32-point DFT in registers, permuted frequency order (radix-2 DIF step, then two
// DFT16s): forward takes x[n] natural and leaves X[2r] in x[r], X[2r+1] in
// x[16+r]; the inverse variant takes that order and returns natural order.
template <bool INV>
__host__ __device__ __forceinline__ void dft32p_fwd(float2 (&x)[32]) {
  float2 lo[16], hi[16];
#pragma unroll
  for (int n = 0; n < 16; ++n) {
    lo[n] = cadd(x[n], x[n + 16]);
    hi[n] = tw32<INV>(csub(x[n], x[n + 16]), n);
  }
  dft16_<INV>(lo);
  dft16_<INV>(hi);
#pragma unroll
  for (int n = 0; n < 16; ++n) {
    x[n] = lo[n];
    x[n + 16] = hi[n];
  }
}
template <bool INV>
__host__ __device__ __forceinline__ void dft32p_inv(float2 (&x)[32]) {
  float2 lo[16], hi[16];
#pragma unroll
  for (int n = 0; n < 16; ++n) {
    lo[n] = x[n];
    hi[n] = x[n + 16];
  }
  dft16_<INV>(lo);
  dft16_<INV>(hi);
#pragma unroll
  for (int n = 0; n < 16; ++n) {
    const float2 t = tw32<INV>(hi[n], n);
    x[n] = cadd(lo[n], t);
    x[n + 16] = csub(lo[n], t);
  }
}
// frequency held by register r after dft32p_fwd
__host__ __device__ constexpr int dft32p_freq(int r) { return r < 16 ? 2 * r : 2 * (r - 16) + 1; }

template <int R, bool INV>
__host__ __device__ __forceinline__ void dft(float2 (&x)[R]) {
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
    dft8_<INV>(x);
  } else if constexpr (R == 16) {
    dft16_<INV>(x);
  } else {
    static_assert(R == 1, "unsupported radix");
  }
}

}  // namespace fm
