// fm_direct.cuh — exact full-mode integer convolution (direct summation).
//
// Replaces direct_full / conv_full_direct (fft_conv.py:94-111) on the device
// for the generic N-D (ndim <= 3) count-convolution API: one thread per output
// element, int64 accumulation over the overlapping entries of b.  Used for
// operands that are not tonal one-hot volumes (those go through the FFT tile
// path in count mode); exact, so its deviation is 0.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace fm {

struct DirectArgs {
  int64_t as[3], bs[3], os[3];   // padded to 3 axes (leading 1s)
  const int64_t* a;
  const int64_t* b;
  int64_t* out;
  int64_t nout;
};

__global__ void __launch_bounds__(256) conv_direct_kernel(const DirectArgs d) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= d.nout) return;
  const int64_t o2 = idx % d.os[2], r = idx / d.os[2];
  const int64_t o1 = r % d.os[1], o0 = r / d.os[1];
  int64_t acc = 0;
  const int64_t j0a = max((int64_t)0, o0 - (d.as[0] - 1)), j0b = min(d.bs[0] - 1, o0);
  const int64_t j1a = max((int64_t)0, o1 - (d.as[1] - 1)), j1b = min(d.bs[1] - 1, o1);
  const int64_t j2a = max((int64_t)0, o2 - (d.as[2] - 1)), j2b = min(d.bs[2] - 1, o2);
  for (int64_t j0 = j0a; j0 <= j0b; ++j0)
    for (int64_t j1 = j1a; j1 <= j1b; ++j1) {
      const int64_t* brow = d.b + (j0 * d.bs[1] + j1) * d.bs[2];
      const int64_t* arow = d.a + ((o0 - j0) * d.as[1] + (o1 - j1)) * d.as[2];
      for (int64_t j2 = j2a; j2 <= j2b; ++j2) acc += brow[j2] * arow[o2 - j2];
    }
  d.out[idx] = acc;
}

}  // namespace fm
