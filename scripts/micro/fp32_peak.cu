// Microbenchmark: FP32 FMA peak of the B200 per SM clock (the conv kernel's roofline
// denominator).  Every thread runs independent FFMA2 (fma.rn.f32x2) chains; the
// elapsed SM cycles come from clock64 inside each CTA, so the result is flop per
// SM clock, independent of the clock the box happens to run at.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp32_peak fp32_peak.cu && ./fp32_peak
// prints one JSON line: {"flops_per_clock": <whole GPU>, "sms": ..., ...}
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;

__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

template <bool PACKED>
__global__ void k(float* out, u64* cycles, int iters, float s) {
  float acc[16];
  u64 p[8];
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3f + i;
  for (int i = 0; i < 8; ++i) {
    float2 f = make_float2(acc[2 * i], acc[2 * i + 1]);
    p[i] = *reinterpret_cast<u64*>(&f);
  }
  float2 ss = make_float2(s, s);
  const u64 sp = *reinterpret_cast<u64*>(&ss);
  __syncthreads();
  const u64 t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (PACKED) {
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = ffma2(p[i], sp, sp);
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = fmaf(acc[i], s, 0.5f);
    }
  }
  __syncthreads();
  const u64 t1 = clock64();
  float t = 0;
  for (int i = 0; i < 16; ++i) t += acc[i];
  for (int i = 0; i < 8; ++i) {
    float2 f = *reinterpret_cast<float2*>(&p[i]);
    t += f.x + f.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int ctas = sms, nt = 1024, iters = 20000;   // one 1024-thread CTA per SM
  float* o;
  u64* cyc;
  cudaMalloc(&o, (size_t)ctas * nt * 4);
  cudaMalloc(&cyc, ctas * sizeof(u64));
  double best[2] = {0, 0};
  for (int mode = 0; mode < 2; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      if (mode) k<true><<<ctas, nt>>>(o, cyc, iters, 0.999f);
      else k<false><<<ctas, nt>>>(o, cyc, iters, 0.999f);
      cudaDeviceSynchronize();
      u64 h[1024];
      cudaMemcpy(h, cyc, ctas * sizeof(u64), cudaMemcpyDeviceToHost);
      u64 mx = 0;
      for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
      // flops per SM per clock: 2 per FMA lane-op, 16 lane-ops per thread per iteration
      const double f = 2.0 * 16.0 * nt * (double)iters / (double)mx;
      if (f > best[mode]) best[mode] = f;
    }
  printf("{\"flops_per_clock\": %.1f, \"sms\": %d, \"per_sm_per_clock_ffma\": %.2f, "
         "\"per_sm_per_clock_ffma2\": %.2f, \"how\": \"scripts/micro/fp32_peak.cu: independent FMA chains, "
         "one 1024-thread CTA per SM, clock64 cycles, best of 3; flops_per_clock = SMs x best per-SM rate\"}\n",
         sms * (best[0] > best[1] ? best[0] : best[1]), sms, best[0], best[1]);
  return 0;
}
