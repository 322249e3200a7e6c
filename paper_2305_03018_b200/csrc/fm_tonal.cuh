// fm_tonal.cuh — per-pixel inverse tonal transform fused with the threshold
// and the highest-nonzero-degree reduction (Step 3 of the paper).
//
// Replaces irfftn's tonal axis + slice + rint + deviation check
// (fft_conv.py:139-149) and project_with_validity (umbra.py:189-205) + the
// erosion duality store (morphology.py:175-180): for every output pixel the
// K = T/2+1 complex spectral values Chat[k] (already scaled by 1/T) are turned
// into the T real counts c(t) with a half-length complex inverse FFT
// (c2r packing), then
//     value = max{ t : c(t) > 0.5 }   (np.rint(c) >= 1, umbra.py:198)
//     valid = any t with c(t) > 0.5   (has_any, umbra.py:199)
// and out = valid ? out_sign*(value + se_min) + anchor : fill, where the anchor
// is the unit's min f (dilation) or max f (erosion).  One launch per tonal
// length of the plan's ladder covers the units that use it.  max|c - rint(c)| is
// reduced block-wide and atomically into the plan's deviation slot.
#pragma once
#include "fm_async.cuh"
#include "fm_dft.cuh"

namespace fm {

struct TonalArgs {
  const float2* chat;     // [imgs][units][K_max][wpx] window-local planes
  int K_max;              // planes per unit in chat
  int N, T;               // this launch's tonal length T = 2N (one ladder entry)
  int nstages;
  int radix[12];
  const float2* twN;      // generic kernel: [N] exp(+2 pi i j / N)
  const float2* wT;       // generic kernel: [N] exp(+2 pi i k / T)
  const int2* list;       // units of this ladder entry: (img, unit)
  const int4* unit_param; // [imgs][units]: x = anchor
  int units, wpx;         // wpx: plane stride (even), npx: pixels per unit
  int npx, njobs;         // njobs: units in list (pipelined kernel)
  uint32_t qx_magic, tx_magic;  // ceil(2^32 / QX), ceil(2^32 / tiles_x) (0 for a divisor of 1): exact quotients below 2^16
  int unit0, upl;         // first unit of this launch, chat slots per image
  int two_d, QY, QX, OH, OW, tiles_x, unit_step_x;
  void* out;              // [imgs][OH][OW] of out_dtype
  int out_dtype;          // 0 int32, 1 uint8, 2 uint16, 3 int16
  uint8_t* valid;         // nullable
  int out_sign, se_min, fill;
  int stride;             // generic kernel: per-pixel smem stride (float2), odd
  float* dev_max;         // max |c - rint c| (float bits, atomicMax as int)
  // count-volume mode (generic kernel): counts[pixel][d], d = t + (anchor - count_base)
  int32_t* counts;
  int count_len, count_base;
  // units flagged "full" (unit_param.w bit 1: window inside the image, no gaps)
  // have plane 0 = (defined SE entries) / T everywhere; the conv kernel skips it
  float x0_full;
  int use_tma;            // pipelined kernel: stages by 2-D tensor copies (maps passed beside the args)
  int tma_row0;           // first map row of this launch's spectral buffer set (double-buffered plans)
  // device-dispatched kernel (small launches): every ladder entry in one launch
  const int* bucket_count;   // [L] units per ladder entry
  const int* ladder;         // [L] N of each entry
  const int2* lists;         // [L][cap] work lists
  int L, cap, se_count;
  // 16-bit spectral planes (plan chat16): each complex value stored as two int16
  // fixed-point numbers; value = stored * chat_invq_T / T (see fm_abi.cu)
  int chat16;
  float chat_invq_T;
};

// One spectral value of pixel index `idx` (elements of the window-local planes):
// complex64, or a pair of int16 fixed-point numbers scaled by `invq` (16-bit planes).
__device__ __forceinline__ float2 unpack16(uint32_t w, float invq) {
#ifndef FM_UNPACK_MAGIC   // (the XU-free variant below measured 2.7% slower at c5: the tonal pass is FMA-pipe bound)
  float re, im;
  asm("cvt.rn.f32.s16 %0, %1;" : "=f"(re) : "h"((unsigned short)(w & 0xFFFFu)));
  asm("cvt.rn.f32.s16 %0, %1;" : "=f"(im) : "h"((unsigned short)(w >> 16)));
  return make_float2(re * invq, im * invq);
#else
  // int16 -> float without the XU pipe's cvt: s + 32768 spliced under the exponent of
  // 2^23 (one xor, two byte permutes), then an exact packed subtract and the scale
  const uint32_t b = w ^ 0x80008000u;
  const float2 f = make_float2(__uint_as_float(__byte_perm(b, 0x4B000000u, 0x7410)),
                               __uint_as_float(__byte_perm(b, 0x4B000000u, 0x7432)));
  return cscale(csub(f, make_float2(8421376.f, 8421376.f)), invq);
#endif
}
__device__ __forceinline__ float2 chat_ld(const TonalArgs& a, size_t idx, float invq) {
  if (a.chat16) return unpack16(__ldcs(reinterpret_cast<const unsigned int*>(a.chat) + idx), invq);
  return __ldcs(a.chat + idx);
}

__device__ __forceinline__ void store_out(const TonalArgs& a, size_t i, int v) {
  switch (a.out_dtype) {
    case 1: reinterpret_cast<uint8_t*>(a.out)[i] = (uint8_t)v; break;
    case 2: reinterpret_cast<uint16_t*>(a.out)[i] = (uint16_t)v; break;
    case 3: reinterpret_cast<int16_t*>(a.out)[i] = (int16_t)v; break;
    default: reinterpret_cast<int32_t*>(a.out)[i] = v; break;
  }
}

// Pixel p of the work unit list[blockIdx.y]: chat offset, output offset, anchor.
struct TonalPix {
  bool live, full;
  size_t src, dst;
  int anchor;
};
__device__ __forceinline__ TonalPix tonal_pixel_job(const TonalArgs& a, int2 job, int p) {
  const int img = job.x, unit = job.y & ~kJobFull;
  TonalPix r;
  int oy, ox;
  if (a.two_d) {
    // magic 0 encodes a divisor of 1 (2^32 does not fit)
    const int ty = a.tx_magic ? (int)__umulhi((uint32_t)unit, a.tx_magic) : unit, tx = unit - ty * a.tiles_x;
    const int wy = a.qx_magic ? (int)__umulhi((uint32_t)p, a.qx_magic) : p, wx = p - wy * a.QX;
    oy = ty * a.QY + wy;
    ox = tx * a.QX + wx;
  } else {
    oy = 0;
    ox = unit * a.unit_step_x + p;
  }
  r.live = p < a.npx && oy < a.OH && ox < a.OW;
  r.src = ((size_t)img * a.upl + (unit - a.unit0)) * a.K_max * (size_t)a.wpx + p;
  r.dst = ((size_t)img * a.OH + oy) * a.OW + ox;
  const int4 up = a.unit_param[(size_t)img * a.units + unit];
  r.anchor = r.live ? up.x : 0;
  r.full = (up.w & 2) != 0;
  return r;
}
__device__ __forceinline__ TonalPix tonal_pixel(const TonalArgs& a, int p) {
  return tonal_pixel_job(a, a.list[blockIdx.x], p);   // grid: x = work unit, y = pixel block
}

template <int R>
__device__ __forceinline__ void stockham_stage(const float2* in, float2* out, int N, int Ns,
                                               const float2* twN) {
  const int M = N / R;
  const int tstep = N / (Ns * R);
  for (int j = 0; j < M; ++j) {
    float2 v[R];
    const int jm = j % Ns;
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = in[j + r * M];
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], twN[(jm * r * tstep) % N]);
    }
    dft<R, true>(v);
    const int idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) out[idxD + r * Ns] = v[r];
  }
}

// ---------------------------------------------------------------------------
// Compile-time tonal FFTs.  For every 5-smooth N <= 160 the inverse length-N
// FFT is a fully unrolled Stockham recursion (radices 8,4,2,3,5) whose
// twiddles are compile-time offsets into one __constant__ table (constant-bank
// operands, no index arithmetic).  N <= 80: the pixel's spectrum lives in
// registers; 80 < N <= 160: in a thread-interleaved shared-memory array.
#define FM_TONAL_NS                                                                                         \
  1, 2, 3, 4, 5, 6, 8, 9, 10, 12, 15, 16, 18, 20, 24, 25, 27, 30, 32, 36, 40, 45, 48, 50, 54, 60, 64, 72, 75, 80, \
      81, 90, 96, 100, 108, 120, 125, 128, 135, 144, 150, 160
constexpr int kTonalNs[] = {FM_TONAL_NS};
constexpr int kTonalCount = sizeof(kTonalNs) / sizeof(int);
constexpr int kTonalRegMax = 80;

__host__ __device__ constexpr int tonal_off(int n) {
  constexpr int ns[] = {FM_TONAL_NS};
  int off = 0;
  for (int i = 0; i < (int)(sizeof(ns) / sizeof(int)); ++i) {
    if (ns[i] == n) return off;
    off += 2 * ns[i];
  }
  return -1;
}
__host__ __device__ constexpr int tonal_tab_total() {
  constexpr int ns[] = {FM_TONAL_NS};
  int off = 0;
  for (int i = 0; i < (int)(sizeof(ns) / sizeof(int)); ++i) off += 2 * ns[i];
  return off;
}
constexpr int kTonalTabTotal = tonal_tab_total();

// W_{2N}^j = exp(+2 pi i j / (2N)), j < 2N, for each supported N (inverse sign).
__constant__ float2 c_ttw[kTonalTabTotal];

__host__ __device__ constexpr int radix_at(int n, int i) {
  const int ps[5] = {8, 4, 2, 3, 5};
  int idx = 0;
  for (int q = 0; q < 5; ++q)
    while (n % ps[q] == 0) {
      if (idx == i) return ps[q];
      n /= ps[q];
      ++idx;
    }
  return 0;
}
__host__ __device__ constexpr int num_radices(int n) {
  int c = 0;
  while (radix_at(n, c) != 0) ++c;
  return c;
}

template <int NT>
struct SmemArr {
  float2* p;
  __device__ __forceinline__ float2& operator[](int i) const { return p[i * NT]; }
};

template <class A> struct IsSmemArr { static constexpr bool value = false; };
template <int NT> struct IsSmemArr<SmemArr<NT>> { static constexpr bool value = true; };

template <int N, int R, int Ns, class A, class B>
__device__ __forceinline__ void stock_stage(A& in, B& out) {
  constexpr int M = N / R;
  constexpr int tstep = N / (Ns * R);
  constexpr int off = tonal_off(N);
  // register arrays need full unrolling (compile-time indices); shared-memory
  // arrays are walked with a rolled loop to keep register pressure bounded
  constexpr int U = IsSmemArr<A>::value ? 1 : M;
#pragma unroll U
  for (int j = 0; j < M; ++j) {
    float2 v[R];
    const int jm = j % Ns;
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = in[j + r * M];
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) {
        // exp(+2 pi i e / N); e is a constant after unrolling, so the trivial
        // twiddles (1, -1, +-i) fold away
        const int e = (jm * r * tstep) % N;
        if (e == 0) continue;
        if (4 * e == 2 * N) v[r] = make_float2(-v[r].x, -v[r].y);
        else if (4 * e == N) v[r] = mul_pi(v[r]);
        else if (4 * e == 3 * N) v[r] = mul_mi(v[r]);
        else v[r] = cmul(v[r], c_ttw[off + 2 * e]);
      }
    }
    dft<R, true>(v);
    const int idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) out[idxD + r * Ns] = v[r];
  }
}

template <int N, int I, int Ns, class A>
__device__ __forceinline__ void stock_run(A& a, A& b) {
  constexpr int R = radix_at(N, I);
  if constexpr (R != 0) {
    stock_stage<N, R, Ns>(a, b);
    stock_run<N, I + 1, Ns * R>(b, a);
  }
}

template <int N, class A>
__device__ __forceinline__ int tonal_threshold(const A& res, float& dev) {
  int top = -1;
  constexpr bool SMA = IsSmemArr<A>::value;
  constexpr int U = SMA ? 4 : N;
#pragma unroll U
  for (int n = 0; n < N; ++n) {
    const float2 z = res[n];
    // rint via the 1.5*2^23 magic (round-to-nearest-even, |c| < 2^22): FMA pipe,
    // not XU; both counts of the pair at once (packed f32x2 adds)
    const float2 m = cadd(z, make_float2(12582912.0f, 12582912.0f));
    const float2 d = csub(z, csub(m, make_float2(12582912.0f, 12582912.0f)));
    dev = fmaxf(dev, fmaxf(fabsf(d.x), fabsf(d.y)));
    if constexpr (SMA) {
      top = z.x > 0.5f ? 2 * n : top;
      top = z.y > 0.5f ? 2 * n + 1 : top;
    }
  }
  if constexpr (!SMA) {
    // register spectrum: the highest count > 0.5, searched from the top down
    // (a warp's pixels are neighbours with close tops, so it exits early)
#pragma unroll
    for (int n = N - 1; n >= 0; --n) {
      if (res[n].y > 0.5f) { top = 2 * n + 1; break; }
      if (res[n].x > 0.5f) { top = 2 * n; break; }
    }
  }
  return top;
}

template <int N, bool SM, int NT>
__global__ void __launch_bounds__(NT) tonal_kernel_t(const TonalArgs a) {
  constexpr int off = tonal_off(N);
  const TonalPix pp = tonal_pixel(a, blockIdx.y * NT + threadIdx.x);
  const size_t plane = a.wpx;
  float dev = 0.f;
  if (pp.live) {
    const float invq = a.chat_invq_T / (float)(2 * N);
    int top;
    if constexpr (!SM) {
      float2 X[N + 1];
      if (a.chat16) {   // (two loops: the element format is uniform per launch)
        const unsigned int* src = reinterpret_cast<const unsigned int*>(a.chat) + pp.src;
#pragma unroll
        for (int k = 0; k <= N; ++k) X[k] = unpack16(__ldcs(src + (size_t)k * plane), invq);
      } else {
        const float2* src = a.chat + pp.src;
#pragma unroll
        for (int k = 0; k <= N; ++k) X[k] = __ldcs(src + (size_t)k * plane);
      }
      if (pp.full) X[0] = make_float2(a.x0_full, 0.f);
      float2 A[N], B[N];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        const float2 xk = X[k], xc = conjf2(X[N - k]);
        A[k] = cadd(cadd(xk, xc), mul_pi(cmul(c_ttw[off + k], csub(xk, xc))));
      }
      stock_run<N, 0, 1>(A, B);
      if constexpr (num_radices(N) % 2 == 0) top = tonal_threshold<N>(A, dev);
      else top = tonal_threshold<N>(B, dev);
    } else {
      extern __shared__ __align__(16) float2 tsm_t[];
      SmemArr<NT> A{tsm_t + threadIdx.x}, B{tsm_t + (size_t)N * NT + threadIdx.x};
      // X[0..N-1] -> B, X[N] stays in a register
      if (a.chat16) {
        const unsigned int* src = reinterpret_cast<const unsigned int*>(a.chat) + pp.src;
#pragma unroll 8
        for (int k = 0; k < N; ++k) B[k] = unpack16(__ldcs(src + (size_t)k * plane), invq);
      } else {
        const float2* src = a.chat + pp.src;
#pragma unroll 8
        for (int k = 0; k < N; ++k) B[k] = __ldcs(src + (size_t)k * plane);
      }
      if (pp.full) B[0] = make_float2(a.x0_full, 0.f);
      const float2 xN = chat_ld(a, pp.src + (size_t)N * plane, invq);
#pragma unroll 4
      for (int k = 0; k < N; ++k) {
        const float2 xk = B[k];
        const float2 xc = conjf2(k == 0 ? xN : B[N - k]);
        A[k] = cadd(cadd(xk, xc), mul_pi(cmul(c_ttw[off + k], csub(xk, xc))));
      }
      stock_run<N, 0, 1>(A, B);
      if constexpr (num_radices(N) % 2 == 0) top = tonal_threshold<N>(A, dev);
      else top = tonal_threshold<N>(B, dev);
    }
    store_out(a, pp.dst, top >= 0 ? a.out_sign * (top + a.se_min) + pp.anchor : a.fill);
    if (a.valid) a.valid[pp.dst] = top >= 0 ? 1 : 0;
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) dev = fmaxf(dev, __shfl_xor_sync(0xffffffffu, dev, o2));
  if ((threadIdx.x & 31) == 0 && dev > 0.f) atomicMax(reinterpret_cast<int*>(a.dev_max), __float_as_int(dev));
}

// ---------------------------------------------------------------------------
// Device-dispatched tonal pass for small launches (one small image: latency bound).
// One CTA per (unit, pixel block) of ANY ladder entry: the entry, the unit and the
// block are decoded from the device per-ladder counts (walked in ladder order), and
// the compile-time inverse FFT of that entry's N is picked by a switch -- so the
// whole call needs no host round trip for the counts (the host-sized launches of
// tonal_kernel_pipe / tonal_kernel_t need them).  Register variants (N <= 40).
constexpr int kDispatchNMax = 40;

__host__ __device__ constexpr int tonal_ns_at(int i) {
  constexpr int ns[] = {FM_TONAL_NS};
  return ns[i];
}

template <int N>
__device__ __forceinline__ void tonal_pixel_reg(const TonalArgs& a, const TonalPix& pp, float& dev) {
  constexpr int off = tonal_off(N);
  const float x0 = (float)((double)a.se_count / (2.0 * N));
  const float invq = a.chat_invq_T / (float)(2 * N);
  float2 X[N + 1];
#pragma unroll
  for (int k = 0; k <= N; ++k)
    X[k] = (k == 0 && pp.full) ? make_float2(x0, 0.f) : chat_ld(a, pp.src + (size_t)k * a.wpx, invq);
  float2 A[N], B[N];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const float2 xk = X[k], xc = conjf2(X[N - k]);
    A[k] = cadd(cadd(xk, xc), mul_pi(cmul(c_ttw[off + k], csub(xk, xc))));
  }
  stock_run<N, 0, 1>(A, B);
  float d = 0.f;
  int top;
  if constexpr (num_radices(N) % 2 == 0) top = tonal_threshold<N>(A, d);
  else top = tonal_threshold<N>(B, d);
  dev = fmaxf(dev, d);
  store_out(a, pp.dst, top >= 0 ? a.out_sign * (top + a.se_min) + pp.anchor : a.fill);
  if (a.valid) a.valid[pp.dst] = top >= 0 ? 1 : 0;
}

template <int NMAX, int I = 0>
__device__ __forceinline__ void tonal_pixel_dispatch(int n, const TonalArgs& a, const TonalPix& pp, float& dev) {
  if constexpr (I < kTonalCount) {
    constexpr int NI = tonal_ns_at(I);
    if constexpr (NI <= NMAX) {
      if (n == NI) {
        tonal_pixel_reg<NI>(a, pp, dev);
        return;
      }
      tonal_pixel_dispatch<NMAX, I + 1>(n, a, pp, dev);
    }
  }
}

// NMAX: the longest tonal axis the instance serves (the plan's, rounded up to 10 / 16 / 40): the
// register count is that of the longest compile-time FFT in the switch, so plans with short
// tonal axes (c1: N <= 10, c2: N <= 16) get twice the resident CTAs of the N <= 40 instance
template <int NT, int NMAX>
__global__ void __launch_bounds__(NT) tonal_kernel_dispatch(const TonalArgs a) {
  __shared__ int s_li, s_rem;
  const int bpj = (a.npx + NT - 1) / NT;
  if (threadIdx.x < 32) {
    // warp-parallel walk of the per-ladder item counts (one load per lane, prefix by shuffles)
    const int lane = threadIdx.x;
    int rem = (int)blockIdx.x, found = -1;
    for (int base = 0; base < a.L && found < 0; base += 32) {
      const int l = base + lane;
      const int c = l < a.L ? a.bucket_count[l] * bpj : 0;
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int nb = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += nb;
      }
      const unsigned m = __ballot_sync(0xffffffffu, l < a.L && rem < incl);
      if (m) {
        const int l0 = __ffs(m) - 1;
        rem -= __shfl_sync(0xffffffffu, incl - c, l0);
        found = base + l0;
      } else {
        rem -= __shfl_sync(0xffffffffu, incl, 31);
      }
    }
    if (lane == 0) {
      s_li = found;
      s_rem = rem;
    }
  }
  __syncthreads();
  const int li = s_li;
  if (li < 0) return;   // grid sized for every unit of the launch; past the jobs
  const int j = s_rem / bpj, blk = s_rem - (s_rem / bpj) * bpj;
  const TonalPix pp = tonal_pixel_job(a, a.lists[(size_t)li * a.cap + j], blk * NT + threadIdx.x);
  float dev = 0.f;
  if (pp.live) tonal_pixel_dispatch<NMAX>(a.ladder[li], a, pp, dev);
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) dev = fmaxf(dev, __shfl_xor_sync(0xffffffffu, dev, o2));
  if ((threadIdx.x & 31) == 0 && dev > 0.f) atomicMax(reinterpret_cast<int*>(a.dev_max), __float_as_int(dev));
}

// ---------------------------------------------------------------------------
// Very short tonal axes (N <= kRowsNMax: one to five planes per pixel, e.g. flat wide SEs after
// the clamp, c4).  An item of the pipelined kernel would be a few hundred bytes and its ring
// handshake and per-item parameter loads dominate; one thread per pixel (tonal_kernel_t) pays two
// dependent parameter loads per pixel.  Here a thread takes PPT pixels of one unit (the unit's
// parameters are loop invariant, the plane loads of the PPT pixels are independent).
constexpr int kRowsNMax = 4;
template <int NT, int PPT>
__global__ void __launch_bounds__(NT) tonal_kernel_rows(const TonalArgs a) {
  const int2 job = a.list[blockIdx.x];
  float dev = 0.f;
#pragma unroll
  for (int u = 0; u < PPT; ++u) {
    const TonalPix pp = tonal_pixel_job(a, job, ((int)blockIdx.y * PPT + u) * NT + (int)threadIdx.x);
    if (!pp.live) continue;
    switch (a.N) {
      case 1: tonal_pixel_reg<1>(a, pp, dev); break;
      case 2: tonal_pixel_reg<2>(a, pp, dev); break;
      case 3: tonal_pixel_reg<3>(a, pp, dev); break;
      default: tonal_pixel_reg<4>(a, pp, dev); break;
    }
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) dev = fmaxf(dev, __shfl_xor_sync(0xffffffffu, dev, o2));
  if ((threadIdx.x & 31) == 0 && dev > 0.f) atomicMax(reinterpret_cast<int*>(a.dev_max), __float_as_int(dev));
}

// ---------------------------------------------------------------------------
// Pipelined register-variant kernel (N <= kTonalRegMax).  Persistent CTAs walk
// the (unit, pixel block) items of one ladder entry; the K spectral values of
// the next ST items are streamed into shared memory by bulk async copies (one
// cp.async.bulk per plane, issued by one thread, completion on an mbarrier),
// so HBM reads overlap the FFT and threshold work of the current item.
template <int N>
constexpr int tonal_pipe_nt() {
#ifdef FM_PIPE_NT_SMALL
  if (N <= 2) return FM_PIPE_NT_SMALL;   // one or two planes per pixel: larger items amortise the ring handshake
#endif
  return (N + 1) * 128 * 8 * 2 > 96 * 1024 ? 64 : 128;
}
#ifndef FM_PIPE_ST
#define FM_PIPE_ST 2
#endif
template <int N>
constexpr int tonal_pipe_st() { return FM_PIPE_ST; }   // two stages: more CTAs per SM beat a deeper ring (measured)
template <int N>
constexpr int tonal_pipe_smem() { return (N + 1) * tonal_pipe_nt<N>() * 8 * tonal_pipe_st<N>(); }

// NT consumer threads (one pixel each per item) + one producer warp; full[st]
// completes when the stage's bulk copies land, empty[st] when every consumer
// warp has read it.
// With tensor maps (tm: box {NT pixels, K planes}; tm1: {NT, K-1} for units
// whose plane 0 is known) the producer moves a whole stage with ONE 2-D TMA
// copy instead of one bulk copy per plane (whose address set-up made the
// single producer thread the bottleneck); out-of-range pixels of a unit's last
// block are zero-filled by the TMA unit and never stored.
template <int N, int NT, int ST>
__global__ void __launch_bounds__(NT + 32) tonal_kernel_pipe(const TonalArgs a, const __grid_constant__ CUtensorMap tm,
                                                             const __grid_constant__ CUtensorMap tm1) {
  constexpr int K = N + 1;
  constexpr int off = tonal_off(N);
  constexpr int NCW = NT / 32;
  extern __shared__ __align__(128) float2 tstg[];   // [ST][K][NT] of complex64 (or int16 pairs: chat16)
  unsigned char* stg_b = reinterpret_cast<unsigned char*>(tstg);
  const size_t esz = a.chat16 ? 4 : 8;               // bytes per stored spectral value
  const float invq = a.chat_invq_T / (float)(2 * N);
  __shared__ __align__(8) uint64_t full[ST], empty[ST];
  __shared__ int stage_k0[ST];   // 1: the stage's unit has a known plane 0 (not copied)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int bpj = (a.npx + NT - 1) / NT;
  const int items = a.njobs * bpj;
  if (tid == 0) {
    for (int st = 0; st < ST; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NCW) {
    // ---- producer
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      int i = 0;
      // the next item's work-list entry is loaded one iteration ahead, so its
      // latency overlaps the wait for a free stage
      int2 job_next = blockIdx.x < items ? a.list[blockIdx.x / bpj] : make_int2(0, 0);
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++i) {
        const int st = i % ST;
        const int2 job = job_next;
        const int item_next = item + gridDim.x;
        if (item_next < items) job_next = a.list[item_next / bpj];
        if (i >= ST) {
          mbar_wait(&empty[st], (uint32_t)(((i / ST) - 1) & 1));
          // the consumers read the stage through the generic proxy (released by
          // their arrives); order those reads before the async-proxy refill —
          // without this fence a stage was occasionally overwritten while read
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        const int j = item / bpj, blk = item - j * bpj;
        const int k0 = (job.y & kJobFull) ? 1 : 0;   // plane 0 known (not copied)
        if (a.use_tma) {
          stage_k0[st] = k0;   // published to the consumers by the arrive below
          mbar_expect_tx(&full[st], (uint32_t)(NT * esz * (K - k0)));
          const int row = a.tma_row0 + ((job.x * a.upl + ((job.y & ~kJobFull) - a.unit0)) * a.K_max) + k0;
          tma_load_2d(stg_b + ((size_t)st * K * NT + k0 * NT) * esz, k0 ? &tm1 : &tm, blk * NT, row, &full[st], pol);
          continue;
        }
        const char* src = reinterpret_cast<const char*>(a.chat) +
                          (((size_t)job.x * a.upl + ((job.y & ~kJobFull) - a.unit0)) * a.K_max * (size_t)a.wpx +
                           (size_t)blk * NT) * esz;
        const uint32_t bytes = (uint32_t)min(NT, a.wpx - blk * NT) * (uint32_t)esz;
        stage_k0[st] = k0;   // published to the consumers by the arrive below
        mbar_expect_tx(&full[st], bytes * (K - k0));
        unsigned char* dst = stg_b + (size_t)st * K * NT * esz;
#pragma unroll 1
        for (int k = k0; k < K; ++k)
          bulk_g2s(dst + (size_t)k * NT * esz, src + (size_t)k * a.wpx * esz, bytes, &full[st], pol);
      }
    }
    return;
  }
  // ---- consumers
  float dev = 0.f;
  int i = 0;
  for (int item = blockIdx.x; item < items; item += gridDim.x, ++i) {
    const int st = i % ST;
    mbar_wait(&full[st], (uint32_t)((i / ST) & 1));
    const int j = item / bpj, blk = item - j * bpj;
    const TonalPix pp = tonal_pixel_job(a, a.list[j], blk * NT + tid);
    const float2* xs8 = tstg + (size_t)st * K * NT + tid;
    const uint32_t* xs4 = reinterpret_cast<const uint32_t*>(tstg) + (size_t)st * K * NT + tid;
    auto xs = [&](int i) -> float2 { return a.chat16 ? unpack16(xs4[i], invq) : xs8[i]; };
    float2 A[N], B[N];
    // c2r packing Z[k] = s_k + i w_k d_k, s_k = X[k] + X[N-k]^*, d_k = X[k] - X[N-k]^*,
    // w_k = exp(+2 pi i k / T); the partner N-k reuses s, d and m = w_k d_k:
    // Z[N-k] = s^* + i m^*  (w_{N-k} = -w_k^*, d_{N-k} = -d_k^*)
    {
      const float2 x0 = stage_k0[st] ? make_float2(a.x0_full, 0.f) : xs(0);
      const float2 xc = conjf2(xs(N * NT));
      A[0] = cadd(cadd(x0, xc), mul_pi(csub(x0, xc)));
    }
#pragma unroll
    for (int k = 1; 2 * k < N; ++k) {
      const float2 xk = xs(k * NT), xm = conjf2(xs((N - k) * NT));
      const float2 sk = cadd(xk, xm), dk = csub(xk, xm);
      const float2 m = cmul(c_ttw[off + k], dk);
      A[k] = cadd_i(sk, m);                       // s + i m
      A[N - k] = cadd_i(conjf2(sk), conjf2(m));   // s^* + i m^*
    }
    if constexpr (N % 2 == 0 && N > 0) {
      const float2 xh = xs((N / 2) * NT);
      A[N / 2] = make_float2(2.f * xh.x, -2.f * xh.y);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);   // stage read into registers
    if (pp.live) {
      stock_run<N, 0, 1>(A, B);
      float d = 0.f;
      int top;
      if constexpr (num_radices(N) % 2 == 0) top = tonal_threshold<N>(A, d);
      else top = tonal_threshold<N>(B, d);
      dev = fmaxf(dev, d);
      store_out(a, pp.dst, top >= 0 ? a.out_sign * (top + a.se_min) + pp.anchor : a.fill);
      if (a.valid) a.valid[pp.dst] = top >= 0 ? 1 : 0;
    }
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) dev = fmaxf(dev, __shfl_xor_sync(0xffffffffu, dev, o2));
  if (lane == 0 && dev > 0.f) atomicMax(reinterpret_cast<int*>(a.dev_max), __float_as_int(dev));
}

// generic runtime-N fallback (N > 160)
__global__ void __launch_bounds__(128) tonal_kernel(const TonalArgs a) {
  extern __shared__ __align__(16) float2 tsm[];
  const int N = a.N;
  float2* twN = tsm;
  float2* wT = tsm + N;
  float2* bufA = tsm + 2 * N;
  float2* bufB = bufA + (size_t)blockDim.x * a.stride;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    twN[i] = a.twN[i];
    wT[i] = a.wT[i];
  }
  __syncthreads();

  const TonalPix pp = tonal_pixel(a, blockIdx.y * blockDim.x + threadIdx.x);
  const size_t plane = a.wpx;
  float dev = 0.f;
  if (pp.live) {
    const float invq = a.chat_invq_T / (float)(2 * N);
    float2* A = bufA + (size_t)threadIdx.x * a.stride;
    float2* B = bufB + (size_t)threadIdx.x * a.stride;
    if (a.chat16) {
      const unsigned int* src = reinterpret_cast<const unsigned int*>(a.chat) + pp.src;
      for (int k = 0; k <= N; ++k) A[k] = unpack16(__ldcs(src + (size_t)k * plane), invq);
    } else {
      const float2* src = a.chat + pp.src;
      for (int k = 0; k <= N; ++k) A[k] = __ldcs(src + (size_t)k * plane);
    }
    if (pp.full) A[0] = make_float2(a.x0_full, 0.f);
    // c2r packing: Z[k] = (X[k] + X[N-k]^*) + i w_T^{-k}... so that the
    // unnormalised length-N inverse DFT of Z gives z[n] = c(2n) + i c(2n+1).
    for (int k = 0; k < N; ++k) {
      const float2 xk = A[k];
      const float2 xc = conjf2(A[N - k]);
      const float2 s = cadd(xk, xc);
      const float2 d = csub(xk, xc);
      B[k] = cadd(s, mul_pi(cmul(wT[k], d)));
    }
    float2* in = B;
    float2* outb = A;
    int Ns = 1;
    for (int st = 0; st < a.nstages; ++st) {
      const int R = a.radix[st];
      switch (R) {
        case 2: stockham_stage<2>(in, outb, N, Ns, twN); break;
        case 3: stockham_stage<3>(in, outb, N, Ns, twN); break;
        case 4: stockham_stage<4>(in, outb, N, Ns, twN); break;
        case 5: stockham_stage<5>(in, outb, N, Ns, twN); break;
        default: stockham_stage<8>(in, outb, N, Ns, twN); break;
      }
      Ns *= R;
      float2* t = in;
      in = outb;
      outb = t;
    }
    int top = -1;
    int32_t* crow = a.counts ? a.counts + pp.dst * (size_t)a.count_len : nullptr;
    const int shift = pp.anchor - a.count_base;
    for (int n = 0; n < N; ++n) {
      const float2 z = in[n];
      dev = fmaxf(dev, fabsf(z.x - rintf(z.x)));
      dev = fmaxf(dev, fabsf(z.y - rintf(z.y)));
      if (z.x > 0.5f) top = 2 * n;
      if (z.y > 0.5f) top = 2 * n + 1;
      if (crow) {
        const int d0 = 2 * n + shift;
        if (d0 >= 0 && d0 < a.count_len) crow[d0] = (int32_t)rintf(z.x);
        if (d0 + 1 >= 0 && d0 + 1 < a.count_len) crow[d0 + 1] = (int32_t)rintf(z.y);
      }
    }
    if (!crow) store_out(a, pp.dst, top >= 0 ? a.out_sign * (top + a.se_min) + pp.anchor : a.fill);
    if (a.valid) a.valid[pp.dst] = top >= 0 ? 1 : 0;
  }
  if (blockDim.x >= 32) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dev = fmaxf(dev, __shfl_xor_sync(0xffffffffu, dev, off));
    if ((threadIdx.x & 31) == 0 && dev > 0.f) atomicMax(reinterpret_cast<int*>(a.dev_max), __float_as_int(dev));
  } else if (dev > 0.f) {   // partial-warp CTAs (very long tonal axes): no full-warp shuffle
    atomicMax(reinterpret_cast<int*>(a.dev_max), __float_as_int(dev));
  }
}

}  // namespace fm
