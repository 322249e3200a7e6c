// fm_fused.cuh — the tonal step (north_star (d)) fused into the conv tile kernel.
//
// Without it, every unit's K_t spatially-convolved spectral planes go to an HBM
// scratch and a separate tonal kernel (fm_tonal.cuh) reads them back.  Here the
// CTA that finishes a unit's LAST plane chunk runs the unit's inverse tonal FFT
// itself, right after the planes were written, while they are still in L2
// (one unit's planes are ~1.3 MB at c5; the ~150 units in flight fit the 126 MB
// L2), then discards those L2 lines (discard.global.L2: invalidated without a
// write-back) so the spectral volume never makes the round trip to HBM.
//
// Completion protocol: every CTA of a unit (its plane chunks) makes its chat
// stores visible device-wide (__threadfence by every thread, CTA barrier) and
// bumps the unit's counter; the CTA that sees count = chunks - 1 is the last,
// fences again (acquire) and streams the planes through shared memory with bulk
// async copies (served by L2), then resets the counter for the next launch.
//
// Per pixel the math is the tonal kernel's (fm_tonal.cuh): c2r packing, the
// compile-time length-N inverse FFT in registers, threshold c(t) > 0.5 with the
// highest such t (umbra.py:198-203), deviation max|c - rint c| (fft_conv.py:
// 143-148), typed store of value + validity.  Ladder entries with N above
// kFuseNMax keep the separate tonal kernel (register budget of the 512-thread
// conv CTA: 128 per thread).
#pragma once
#include "fm_tile.cuh"
#include "fm_tonal.cuh"   // (unpack16: 16-bit planes)

namespace fm {

constexpr int kFuseNMax = 40;

__host__ __device__ constexpr int tonal_n_at(int i) {
  constexpr int ns[] = {FM_TONAL_NS};
  return ns[i];
}

__device__ __forceinline__ void fused_store(const TileArgs& a, size_t i, int v) {
  switch (a.out_dtype) {
    case 1: reinterpret_cast<uint8_t*>(a.out)[i] = (uint8_t)v; break;
    case 2: reinterpret_cast<uint16_t*>(a.out)[i] = (uint16_t)v; break;
    case 3: reinterpret_cast<int16_t*>(a.out)[i] = (int16_t)v; break;
    default: reinterpret_cast<int32_t*>(a.out)[i] = v; break;
  }
}

__device__ __forceinline__ float2 ldcg2(const float2* p) {
  float2 r;
  asm volatile("ld.global.cg.v2.f32 {%0, %1}, [%2];" : "=f"(r.x), "=f"(r.y) : "l"(p));
  return r;
}

// One unit's tonal step: pixels p = tid + NT b, b = 0, 1, ... of its QY x QX window.
// The K planes of each pixel block stream from L2 into shared memory by bulk async copies
// (one per plane, issued by thread 0, completion on an mbarrier) one or two blocks ahead
// of the block being computed -- the conv kernel's tile buffers are free by now.
template <int N, int NT>
__device__ __forceinline__ void fused_tonal_unit(const TileArgs& a, const float2* chat_unit, int img, int unit,
                                                 int anchor, bool full, float2* stg, int stg_slots,
                                                 uint64_t* bars) {
  constexpr int K = N + 1;
  constexpr int off = tonal_off(N);
  const int tid = threadIdx.x;
  const int ty = unit / a.tiles_x, tx = unit - (unit / a.tiles_x) * a.tiles_x;
  const int npx = a.QY * a.QX;
  const int nblk = (npx + NT - 1) / NT;
  const int k0 = full ? 1 : 0;
  const int ST = 2 * K * NT <= stg_slots ? 2 : 1;
  const float x0 = (float)((double)a.se_count / (2.0 * N));
  // element size of the stored planes: complex64, or int16 pairs (16-bit planes)
  const int esz = a.chat16 ? 4 : 8;
  const float invq = a.chat16 ? 1.0f / (a.chat_q_T * (float)(2 * N)) : 1.f;
  const char* cu = reinterpret_cast<const char*>(chat_unit);
  unsigned char* sb = reinterpret_cast<unsigned char*>(stg);
  auto issue = [&](int blk, int st) {   // thread 0: the block's planes k0..K-1 into stage st
    const int p0 = blk * NT;
    const uint32_t bytes = (uint32_t)min(NT, a.wpx - p0) * (uint32_t)esz;   // wpx a multiple of 4: 16-byte multiples
    mbar_expect_tx(&bars[st], bytes * (uint32_t)(K - k0));
    for (int k = k0; k < K; ++k)
      bulk_g2s_nohint(sb + (size_t)(st * K + k) * NT * esz, cu + ((size_t)k * a.wpx + p0) * esz, bytes, &bars[st]);
  };
  if (tid == 0) {
    // the conv passes last wrote these bytes through the generic proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    issue(0, 0);
    if (ST == 2 && nblk > 1) issue(1, 1);
  }
  float dev = 0.f;
#pragma unroll 1
  for (int blk = 0; blk < nblk; ++blk) {
    const int st = ST == 2 ? (blk & 1) : 0;
    const uint32_t par = (uint32_t)((ST == 2 ? (blk >> 1) : blk) & 1);
    mbar_wait(&bars[st], par);
    float2 X[K];
    const float2* xs = stg + (size_t)st * K * NT + tid;
    const uint32_t* xs4 = reinterpret_cast<const uint32_t*>(stg) + (size_t)st * K * NT + tid;
#pragma unroll
    for (int k = 0; k < K; ++k)
      X[k] = (k == 0 && full) ? make_float2(x0, 0.f) : (a.chat16 ? unpack16(xs4[(size_t)k * NT], invq) : xs[(size_t)k * NT]);
    __syncthreads();   // every thread has read the stage
    if (tid == 0 && blk + ST < nblk) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(blk + ST, st);
    }
    const int p = blk * NT + tid;
    const int wy = p / a.QX, wx = p - (p / a.QX) * a.QX;
    const int oy = ty * a.QY + wy, ox = tx * a.QX + wx;
    if (p >= npx || oy >= a.OH || ox >= a.OW) continue;
    float2 A[N], B[N];
    {
      const float2 xc = conjf2(X[N]);
      A[0] = cadd(cadd(X[0], xc), mul_pi(csub(X[0], xc)));
    }
#pragma unroll
    for (int k = 1; 2 * k < N; ++k) {
      const float2 xk = X[k], xm = conjf2(X[N - k]);
      const float2 sk = cadd(xk, xm), dk = csub(xk, xm);
      const float2 m = cmul(c_ttw[off + k], dk);
      A[k] = cadd_i(sk, m);
      A[N - k] = cadd_i(conjf2(sk), conjf2(m));
    }
    if constexpr (N % 2 == 0 && N > 0) {
      const float2 xh = X[N / 2];
      A[N / 2] = make_float2(2.f * xh.x, -2.f * xh.y);
    }
    stock_run<N, 0, 1>(A, B);
    float d = 0.f;
    int top;
    if constexpr (num_radices(N) % 2 == 0) top = tonal_threshold<N>(A, d);
    else top = tonal_threshold<N>(B, d);
    dev = fmaxf(dev, d);
    const size_t dst = ((size_t)img * a.OH + oy) * a.OW + ox;
    fused_store(a, dst, top >= 0 ? a.out_sign * (top + a.se_min) + anchor : a.fill);
    if (a.valid) a.valid[dst] = top >= 0 ? 1 : 0;
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) dev = fmaxf(dev, __shfl_xor_sync(0xffffffffu, dev, o2));
  if ((tid & 31) == 0 && dev > 0.f) atomicMax(reinterpret_cast<int*>(a.dev_max), __float_as_int(dev));
}

template <int NT, int I = 0>
__device__ __forceinline__ void fused_tonal_dispatch(int n, const TileArgs& a, const float2* chat_unit, int img,
                                                     int unit, int anchor, bool full, float2* stg, int stg_slots,
                                                     uint64_t* bars) {
  if constexpr (I < kTonalCount) {
    constexpr int NI = tonal_n_at(I);
    if constexpr (NI <= kFuseNMax) {
      if (n == NI) {
        fused_tonal_unit<NI, NT>(a, chat_unit, img, unit, anchor, full, stg, stg_slots, bars);
        return;
      }
      fused_tonal_dispatch<NT, I + 1>(n, a, chat_unit, img, unit, anchor, full, stg, stg_slots, bars);
    }
  }
}

// Called by every thread of a conv CTA after its plane loop.  Returns after the
// unit's tonal step if this CTA completed the unit (and the unit's N is fused).
template <int NT>
__device__ __forceinline__ void fused_tail(const TileArgs& a, float2* chat_unit, int img, int unit, int K, int T,
                                           int k_chunk, float2* stg, int stg_slots) {
  const int N = T / 2;
  if (a.fuse_nmax == 0 || N > a.fuse_nmax) return;
  __shared__ int s_last;
  __shared__ __align__(8) uint64_t s_tbar[2];
  const int nch = (K + k_chunk - 1) / k_chunk;
  int* cnt = a.unit_done + ((size_t)img * a.upl + (unit - a.unit0));
  __threadfence();        // this thread's plane stores, device-wide
  __syncthreads();
  if (threadIdx.x == 0) {
    const int prev = nch > 1 ? atomicAdd(cnt, 1) : nch - 1;
    s_last = prev == nch - 1;
    if (s_last && nch > 1) *cnt = 0;   // self-reset for the next launch (no other CTA touches it now)
    __threadfence();      // acquire: the other chunks' stores before our reads
  }
  __syncthreads();
  if (!s_last) return;
  const int4 up = a.unit_param[(size_t)img * a.units + unit];
  const bool full = (up.w & 2) != 0;
  if (threadIdx.x == 0) {
    mbar_init(&s_tbar[0], 1);
    mbar_init(&s_tbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  fused_tonal_dispatch<NT>(N, a, chat_unit, img, unit, up.x, full, stg, stg_slots, s_tbar);
  if (a.discard) {
    // the unit's planes are consumed: drop their L2 lines without a write-back
    __syncthreads();
    const size_t esz = a.chat16 ? 4 : 8;
    const char* b0 = reinterpret_cast<const char*>(chat_unit) + (size_t)(full ? 1 : 0) * a.wpx * esz;
    const char* b1 = reinterpret_cast<const char*>(chat_unit) + (size_t)K * a.wpx * esz;
    const uintptr_t first = ((uintptr_t)b0 + 127) & ~(uintptr_t)127, last = (uintptr_t)b1 & ~(uintptr_t)127;
    for (uintptr_t l = first + (uintptr_t)threadIdx.x * 128; l < last; l += (uintptr_t)NT * 128)
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(l) : "memory");
  }
}

}  // namespace fm
