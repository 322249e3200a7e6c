// fm_fft64.cuh — generic N-D FP64 FFT convolution of integer volumes, and the
// tonal lift / projection of the count level.
//
// The hot path (fm_tile128.cuh + fm_tonal.cuh) convolves tonal one-hot volumes
// in FP32 by tiles.  The reference's count-level API also takes ARBITRARY
// non-negative integer operands of rank 1..3 (and umbra volumes of 3-D grids,
// rank 4): conv_full_fft_with_stats (fft_conv.py:128-150) — rfftn / product /
// irfftn in f64 at the padded shape of the next_fast_size ladder, slice, rint,
// deviation.  This file is that computation on the device, in FP64 like the
// reference, so its precision budget (2^52, fft_conv.py:114-125) applies
// unchanged:
//   * fft64_stage<R>: one Stockham radix-R pass along one axis of a
//     [outer][n][inner] complex volume (R in {2,3,4,5}: the ladder sizes
//     2^k and 45*2^k factor into them); twiddles by sincospi in FP64;
//   * pad / product / finish kernels: zero-padded embed of the int64 operands,
//     pointwise spectral product, and slice + rint + max|x - rint x| + int64 store.
// And the two count-level maps of umbra.py:
//   * umbra_kernel: build_umbra (umbra.py:177-186), bits[x, g(x)] = 1;
//   * project_kernel: project_with_validity's window reduction (umbra.py:189-205),
//     top = highest t with count >= 1, valid = any.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace fm {

constexpr int kFft64NT = 256;

__device__ __forceinline__ double2 z_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 z_mul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// exp(sign * 2 pi i * num / den)
__device__ __forceinline__ double2 z_root(int sign, int64_t num, int64_t den) {
  double s, c;
  sincospi(2.0 * (double)(num % den) / (double)den, &s, &c);
  return make_double2(c, sign * s);
}

// One Stockham pass of radix R along the middle axis of [outer][n][inner]:
// input index j + r*m (m = n/R), output (j/Ns)*Ns*R + j%Ns + r*Ns.
template <int R>
__global__ void __launch_bounds__(kFft64NT) fft64_stage(const double2* __restrict__ in, double2* __restrict__ out,
                                                         int64_t outer, int64_t n, int64_t inner, int64_t Ns,
                                                         int sign) {
  const int64_t m = n / R;
  const int64_t total = outer * m * inner;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % inner;
    const int64_t oj = t / inner;
    const int64_t j = oj % m, o = oj / m;
    const int64_t jm = j % Ns;
    const double2* src = in + (o * n) * inner + i;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[(j + r * m) * inner];
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = z_mul(v[r], z_root(sign, jm * r, Ns * R));
    }
    // length-R DFT (R <= 5: direct sums over exact FP64 roots)
    double2 y[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      double2 acc = v[0];
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const int e = (r * k) % R;
        if (e == 0) acc = z_add(acc, v[r]);
        else if (R == 4 && e == 2) acc = make_double2(acc.x - v[r].x, acc.y - v[r].y);
        else if (R == 2) acc = make_double2(acc.x - v[r].x, acc.y - v[r].y);
        else if (R == 4) acc = z_add(acc, e == 1 ? make_double2(-sign * v[r].y, sign * v[r].x)
                                                 : make_double2(sign * v[r].y, -sign * v[r].x));
        else acc = z_add(acc, z_mul(v[r], z_root(sign, e, R)));
      }
      y[k] = acc;
    }
    double2* dst = out + (o * n + (j / Ns) * Ns * R + jm) * inner + i;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[(int64_t)r * Ns * inner] = y[r];
  }
}

struct Shape4 {
  int64_t d[4];
};

// zero-padded embed of an int64 operand of shape `s` into the complex volume of shape `p`
__global__ void fft64_pad(const int64_t* __restrict__ a, Shape4 s, Shape4 p, double2* __restrict__ out) {
  const int64_t total = p.d[0] * p.d[1] * p.d[2] * p.d[3];
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t, idx = 0;
    bool in = true;
    int64_t c[4];
    for (int k = 3; k >= 0; --k) {
      c[k] = r % p.d[k];
      r /= p.d[k];
      in = in && c[k] < s.d[k];
    }
    if (in) idx = ((c[0] * s.d[1] + c[1]) * s.d[2] + c[2]) * s.d[3] + c[3];
    out[t] = make_double2(in ? (double)a[idx] : 0.0, 0.0);
  }
}

__global__ void fft64_product(double2* __restrict__ a, const double2* __restrict__ b, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    a[t] = z_mul(a[t], b[t]);
}

// slice [0, o) of the padded inverse, scale, rint, deviation, int64 store
__global__ void fft64_finish(const double2* __restrict__ x, Shape4 p, Shape4 o, double scale,
                             int64_t* __restrict__ out, unsigned long long* dev_bits) {
  const int64_t total = o.d[0] * o.d[1] * o.d[2] * o.d[3];
  double dev = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = t, c[4];
    for (int k = 3; k >= 0; --k) {
      c[k] = r % o.d[k];
      r /= o.d[k];
    }
    const int64_t src = ((c[0] * p.d[1] + c[1]) * p.d[2] + c[2]) * p.d[3] + c[3];
    const double v = x[src].x * scale;
    const double rv = rint(v);
    dev = fmax(dev, fabs(v - rv));
    out[t] = (int64_t)rv;
  }
  for (int o2 = 16; o2 > 0; o2 >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o2));
  // non-negative doubles order like their bit patterns
  if ((threadIdx.x & 31) == 0 && dev > 0.0) atomicMax(dev_bits, (unsigned long long)__double_as_longlong(dev));
}

// build_umbra: bits [npx][l_r + 1] int64, zeroed by the caller; one 1 per defined pixel
__global__ void umbra_kernel(const int64_t* __restrict__ values, const uint8_t* __restrict__ defined, int64_t npx,
                             int64_t t, int64_t* __restrict__ bits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npx; i += (int64_t)gridDim.x * blockDim.x) {
    if (defined && !defined[i]) continue;
    const int64_t v = values[i];
    if (v >= 0 && v < t) bits[i * t + v] = 1;
  }
}

// project_with_validity over a contiguous window [npx][t]
__global__ void project_kernel(const int64_t* __restrict__ window, int64_t npx, int64_t t,
                               int64_t* __restrict__ values, uint8_t* __restrict__ valid) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npx; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t* col = window + i * t;
    int64_t top = -1;
    for (int64_t k = t - 1; k >= 0; --k)
      if (col[k] >= 1) {
        top = k;
        break;
      }
    values[i] = top >= 0 ? top : 0;
    valid[i] = top >= 0 ? 1 : 0;
  }
}

}  // namespace fm
