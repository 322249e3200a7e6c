// Microbenchmark: HBM read bandwidth reachable by S SMs while a blocker kernel
// holds the other SMs (one 1024-thread CTA per SM using the whole register file,
// spinning on clock64 only), i.e. the premise of co-scheduling the HBM-bound
// tonal pass on a small SM partition beside the compute-bound conv pass.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(1024, 1) blocker(long long cycles, int* sink) {
  extern __shared__ char s[];
  const long long t0 = clock64();
  float x = threadIdx.x;
  while (clock64() - t0 < cycles) x = x * 0.999f + 1.0f;
  if (x == 12345.f) sink[0] = 1;   // keep the loop
  s[threadIdx.x] = (char)x;
}
__global__ void stream(const float4* __restrict__ a, size_t n, float* out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const float4 x0 = __ldcs(a + i), x1 = __ldcs(a + i + stride), x2 = __ldcs(a + i + 2 * stride), x3 = __ldcs(a + i + 3 * stride);
    acc += x0.x + x1.y + x2.z + x3.w;
  }
  if (acc == 12345.f) out[0] = acc;
}
int main() {
  const size_t bytes = (size_t)2 << 30, n = bytes / 16;
  float4* a; float* o; int* sink;
  cudaMalloc(&a, bytes); cudaMalloc(&o, 4); cudaMalloc(&sink, 4); cudaMemset(a, 0, bytes);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(blocker, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t sb, ss; cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int Ss[] = {16, 32, 48, 64, 96, 148};
  for (int S : Ss) {
    for (int occ : {4, 8, 16}) {
      const int nb = nsm - S;
      if (nb > 0) blocker<<<nb, 1024, 200 * 1024, sb>>>(2000000000LL / 40, sink);   // ~25 ms at 2 GHz
      volatile long long spin = 0; for (long long q = 0; q < 3000000; ++q) spin += q;   // let the blockers land
      cudaEventRecord(e0, ss);
      stream<<<S * occ, 256, 0, ss>>>(a, n, o);
      cudaEventRecord(e1, ss);
      cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("S=%3d SMs occ=%2d: %.3f ms  %.0f GB/s  (%.1f GB/s per SM)\n", S, occ, ms, bytes / ms / 1e6, bytes / ms / 1e6 / S);
    }
  }
  return 0;
}
