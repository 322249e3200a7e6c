// fm_tonal_coop.cuh — inverse tonal transform for long tonal axes (40 < N <= 160),
// several threads per pixel.
//
// Same job as tonal_kernel_t (fm_tonal.cuh: irfftn's tonal axis + rint + deviation,
// fft_conv.py:139-149, and project_with_validity, umbra.py:189-205), but a
// one-thread-per-pixel FFT of this length needs 2N complex registers (spills) or a
// 16N-byte shared-memory array per thread (one 64-thread CTA per SM).  Here a CTA
// owns 32 neighbouring pixels and G threads share each pixel: the length-N inverse
// DFT runs as two register passes over ONE in-place shared-memory array
// S[k][pixel] (8 N bytes per pixel):
//
//   pack   S[k], S[N-k] = c2r packing of X[k], X[N-k] loaded from global memory
//          (coalesced per plane, 16-bit planes unpacked), one pair per thread and step
//   pass 1 for b < N2:  Y_b[c] = sum_a S[N2 a + b] W_N1^{a c};  S[N2 c + b] = W_N^{b c} Y_b[c]
//   pass 2 for c < N1:  z[c + N1 d] = sum_b S[N2 c + b] W_N2^{b d}    (registers)
//   threshold / top degree / deviation from the registers, combined over the G threads
//
// with k = N2 a + b, n = c + N1 d (W_N^{k n} = W_N1^{a c} W_N^{b c} W_N2^{b d}).
// Thread (g, pixel) = (tid / 32, tid % 32) takes b = g, g + G, ... and c = g, g + G, ...:
// every warp holds one g, so its 32 lanes touch 32 consecutive pixels of the same
// element (conflict-free 256-byte accesses) and all table indices are warp-uniform
// (constant-bank broadcasts).  The sub-transforms are the compile-time register
// FFTs of fm_tonal.cuh (N1, N2 <= 25).
#pragma once
#include "fm_tonal.cuh"

namespace fm {

// N = N1 * N2 with G | N1 and G | N2 (every thread gets whole sub-transforms)
struct CoopSplit { int n1, n2, g; };
__host__ __device__ constexpr CoopSplit coop_split(int n) {
  switch (n) {
    case 45: return {3, 15, 3};
    case 48: return {4, 12, 4};
    case 50: return {5, 10, 5};
    case 54: return {6, 9, 3};
    case 60: return {6, 10, 2};
    case 64: return {8, 8, 4};
    case 72: return {6, 12, 3};
    case 75: return {5, 15, 5};
    case 80: return {8, 10, 2};
    case 81: return {9, 9, 3};
    case 90: return {6, 15, 3};
    case 96: return {8, 12, 4};
    case 100: return {10, 10, 5};
    case 108: return {9, 12, 3};
    case 120: return {10, 12, 2};
    case 125: return {5, 25, 5};
    case 128: return {8, 16, 4};
    case 135: return {9, 15, 3};
    case 144: return {12, 12, 4};
    case 150: return {10, 15, 5};
    case 160: return {10, 16, 2};
    default: return {0, 0, 0};
  }
}
constexpr int kCoopPix = 32;
__host__ __device__ constexpr bool coop_ok(int n) { return coop_split(n).g != 0; }
__host__ __device__ constexpr int coop_threads(int n) { return coop_ok(n) ? coop_split(n).g * kCoopPix : 32; }
__host__ __device__ constexpr int coop_smem(int n) { return n * kCoopPix * 8; }

// the array holding stock_run's result (ping-pong parity of the stage count)
template <int M>
__device__ __forceinline__ float2 (&stock_result(float2 (&v)[M], float2 (&w)[M]))[M] {
  if constexpr (num_radices(M) % 2 == 0) return v;
  else return w;
}

constexpr int kCoopGMax = 5;

// One CTA's work: 32 pixels (block `blk`) of the unit `job`; threads with g >= G (none in the
// per-entry launches) would only join the barriers.
template <int N>
__device__ __forceinline__ void coop_body(const TonalArgs& a, float x0_full, int2 job, int blk, float2* csm, int (*s_top)[kCoopPix]) {
  constexpr CoopSplit sp = coop_split(N);
  constexpr int N1 = sp.n1, N2 = sp.n2, G = sp.g, PIX = kCoopPix;
  static_assert(N1 * N2 == N && N1 % G == 0 && N2 % G == 0 && G <= kCoopGMax, "split");
  constexpr int off = tonal_off(N);
  const int pix = threadIdx.x & (PIX - 1), g = threadIdx.x / PIX;
  const bool act = g < G;
  const TonalPix pp = tonal_pixel_job(a, job, blk * PIX + pix);
  float2* S = csm + pix;
  const float invq = a.chat_invq_T / (float)(2 * N);

  // ---- load + c2r packing: thread g takes the pairs (k, N - k), k = g, g + G, ... <= N/2,
  // straight from global memory (coalesced per plane, 16-bit planes unpacked):
  // Z[k] = s + i m, Z[N-k] = s^* + i m^* with s = X[k] + X[N-k]^*, m = w_k (X[k] - X[N-k]^*),
  // w_k = exp(2 pi i k / 2N)  (tonal_kernel_pipe's packing; k = 0 and k = N/2 are the same
  // formula, their second value is absent / identical)
  if (act) {
    const size_t plane = a.wpx;
    const unsigned int* src4 = reinterpret_cast<const unsigned int*>(a.chat) + pp.src;
    const float2* src8 = a.chat + pp.src;
    constexpr int NP = N / 2 + 1, UB = 8;
#pragma unroll 1
    for (int j0 = g; j0 < NP; j0 += G * UB) {
      float2 xk[UB], xm[UB];
      if (!pp.live) {
#pragma unroll
        for (int u = 0; u < UB; ++u) xk[u] = xm[u] = make_float2(0.f, 0.f);
      } else if (a.chat16) {   // (the element format is uniform per launch)
        unsigned int rk[UB], rm[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int k = min(j0 + G * u, NP - 1);
          rk[u] = __ldcs(src4 + (size_t)k * plane);
          rm[u] = __ldcs(src4 + (size_t)(N - k) * plane);
        }
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          xk[u] = unpack16(rk[u], invq);
          xm[u] = unpack16(rm[u], invq);
        }
      } else {
#pragma unroll
        for (int u = 0; u < UB; ++u) {
          const int k = min(j0 + G * u, NP - 1);
          xk[u] = __ldcs(src8 + (size_t)k * plane);
          xm[u] = __ldcs(src8 + (size_t)(N - k) * plane);
        }
      }
      if (j0 == 0 && pp.full && pp.live) xk[0] = make_float2(x0_full, 0.f);
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int k = j0 + G * u;
        if (k < NP) {
          const float2 xc = conjf2(xm[u]);
          const float2 sk = cadd(xk[u], xc), m = cmul(c_ttw[off + k], csub(xk[u], xc));
          S[k * PIX] = cadd_i(sk, m);
          if (k > 0) S[(N - k) * PIX] = cadd_i(conjf2(sk), conjf2(m));
        }
      }
    }
  }
  __syncthreads();
  // ---- pass 1: length-N1 transforms over a (stride N2), twiddle W_N^{b c}, in place
#pragma unroll 1
  for (int b = act ? g : N2; b < N2; b += G) {
    float2 v[N1], w[N1];
#pragma unroll
    for (int i = 0; i < N1; ++i) v[i] = S[(N2 * i + b) * PIX];
    stock_run<N1, 0, 1>(v, w);
    float2(&r)[N1] = stock_result<N1>(v, w);
    S[b * PIX] = r[0];
#pragma unroll
    for (int c = 1; c < N1; ++c) S[(N2 * c + b) * PIX] = cmul(r[c], c_ttw[off + 2 * b * c]);
  }
  __syncthreads();
  // ---- pass 2: length-N2 transforms over b (contiguous), outputs n = c + N1 d
  float dev = 0.f;
  int top = -1;
#pragma unroll 1
  for (int c = act ? g : N1; c < N1; c += G) {
    float2 v[N2], w[N2];
#pragma unroll
    for (int i = 0; i < N2; ++i) v[i] = S[(N2 * c + i) * PIX];
    stock_run<N2, 0, 1>(v, w);
    float2(&r)[N2] = stock_result<N2>(v, w);
#pragma unroll
    for (int d = 0; d < N2; ++d) {
      const float2 z = r[d];
      const float2 m = cadd(z, make_float2(12582912.0f, 12582912.0f));
      const float2 e = csub(z, csub(m, make_float2(12582912.0f, 12582912.0f)));
      dev = fmaxf(dev, fmaxf(fabsf(e.x), fabsf(e.y)));
      const int n = c + N1 * d;
      const int t = z.y > 0.5f ? 2 * n + 1 : (z.x > 0.5f ? 2 * n : -1);
      top = max(top, t);
    }
  }
  if (act) s_top[g][pix] = top;
  __syncthreads();
  if (g == 0 && pp.live) {
#pragma unroll
    for (int j = 1; j < G; ++j) top = max(top, s_top[j][pix]);
    store_out(a, pp.dst, top >= 0 ? a.out_sign * (top + a.se_min) + pp.anchor : a.fill);
    if (a.valid) a.valid[pp.dst] = top >= 0 ? 1 : 0;
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) dev = fmaxf(dev, __shfl_xor_sync(0xffffffffu, dev, o2));
  if ((threadIdx.x & 31) == 0 && dev > 0.f) atomicMax(reinterpret_cast<int*>(a.dev_max), __float_as_int(dev));
}

// one launch per ladder entry: grid (units of the entry, 32-pixel blocks)
template <int N>
__global__ void __launch_bounds__(coop_threads(N)) tonal_kernel_coop(const TonalArgs a) {
  extern __shared__ __align__(16) float2 csm[];   // S[N][PIX]
  __shared__ int s_top[kCoopGMax][kCoopPix];
  coop_body<N>(a, a.x0_full, a.list[blockIdx.x], (int)blockIdx.y, csm, s_top);
}

}  // namespace fm
