// fm_naive.cuh — exact direct max-plus dilation / min-plus erosion.
//
// GPU restatement of the reference's naive operators (dilate_naive,
// morphology.py:65-85; erode_naive, morphology.py:88-113): for every output
// pixel, max (min) over the defined SE entries of f(x - y) + b(y)
// (f(x + y) - b(y)); pixels with no pair get `fill` and validity 0.  It is the
// large-configuration verification path and the method="naive" operator; the
// FFT pipeline never calls it.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace fm {

struct NaiveArgs {
  const void* img;
  const uint8_t* img_def;
  int img_dtype;
  int H, W;           // image extent (1-D: H = 1)
  int OH, OW;         // output extent
  int CY, CX;         // input index = out index + C -/+ j
  int erode;          // 0: max f(a+C-j)+b ; 1: min f(a+C+j)-b
  const int4* ent;    // SE entries (jy, jx, value, 0)
  int nent;
  int fill;
  int32_t* out;
  uint8_t* valid;
};

__device__ __forceinline__ int naive_load(const void* img, int dtype, int64_t i) {
  if (dtype == 0) return (int)__ldg(reinterpret_cast<const uint8_t*>(img) + i);
  if (dtype == 1) return (int)__ldg(reinterpret_cast<const uint16_t*>(img) + i);
  return __ldg(reinterpret_cast<const int32_t*>(img) + i);
}

__global__ void __launch_bounds__(256) naive_kernel(const NaiveArgs a) {
  constexpr int kChunk = 1024;
  __shared__ int4 se[kChunk];
  const int ox = blockIdx.x * 32 + (threadIdx.x & 31);
  const int oy = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int img = blockIdx.z;
  const bool live = ox < a.OW && oy < a.OH;
  const int64_t base = (int64_t)img * a.H * a.W;
  const int sgn = a.erode ? 1 : -1;
  int acc = a.erode ? INT32_MAX : INT32_MIN;
  bool any = false;
  for (int c0 = 0; c0 < a.nent; c0 += kChunk) {
    const int n = min(kChunk, a.nent - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) se[i] = a.ent[c0 + i];
    __syncthreads();
    if (!live) continue;
    for (int e = 0; e < n; ++e) {
      const int4 s = se[e];
      const int iy = oy + a.CY + sgn * s.x;
      const int ix = ox + a.CX + sgn * s.y;
      if (iy < 0 || iy >= a.H || ix < 0 || ix >= a.W) continue;
      const int64_t gi = base + (int64_t)iy * a.W + ix;
      if (a.img_def && !a.img_def[gi]) continue;
      const int f = naive_load(a.img, a.img_dtype, gi);
      if (a.erode) acc = min(acc, f - s.z);
      else acc = max(acc, f + s.z);
      any = true;
    }
  }
  if (live) {
    const int64_t o = ((int64_t)img * a.OH + oy) * a.OW + ox;
    a.out[o] = any ? acc : a.fill;
    if (a.valid) a.valid[o] = any ? 1 : 0;
  }
}

}  // namespace fm
