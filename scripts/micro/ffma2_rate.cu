// Microbenchmark: throughput of packed FFMA2/FADD2 (f32x2) vs scalar FFMA on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) { u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r; }
__device__ __forceinline__ u64 fadd2(u64 a, u64 b) { u64 r; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b)); return r; }
template <int MODE>
__global__ void k(float* out, int iters, float s) {
  float acc[16]; u64 p[8];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int i = 0; i < 8; ++i) { float2 f = make_float2(acc[2*i], acc[2*i+1]); p[i] = *reinterpret_cast<u64*>(&f); }
  float2 ss = make_float2(s, s); u64 sp = *reinterpret_cast<u64*>(&ss);
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], s, 0.5f);
    } else if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = ffma2(p[i], sp, sp);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = fadd2(p[i], sp);
    }
  }
  float t = 0;
  for (int i = 0; i < 16; ++i) t += acc[i];
  for (int i = 0; i < 8; ++i) { float2 f = *reinterpret_cast<float2*>(&p[i]); t += f.x + f.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 20000;
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (mode == 0) k<0><<<148 * 8, 512>>>(o, iters, 0.999f);
      if (mode == 1) k<1><<<148 * 8, 512>>>(o, iters, 0.999f);
      if (mode == 2) k<2><<<148 * 8, 512>>>(o, iters, 0.999f);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double lane_ops = 148.0 * 8 * 512 * iters * 16;   // fp32 lane-ops (2 per f32x2 instr)
      double instr = (mode == 0 ? 16.0 : 8.0) * 148.0 * 8 * 512 * iters / 32;
      if (rep) printf("mode %d (%s): %.3f ms, %.1f Tlane-op/s, %.2f warp-instr/clk/SM at 1.965 GHz\n", mode,
                      mode == 0 ? "FFMA" : mode == 1 ? "FFMA2" : "FADD2", ms, lane_ops / ms / 1e9,
                      instr / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
  return 0;
}
