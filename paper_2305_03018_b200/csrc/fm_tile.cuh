// fm_tile.cuh — overlap-save tile FFT convolution of the tonal spectrum planes.
//
// One CTA owns one spatial tile (PY x PX, 2-D) or PY independent 1-D tiles of
// length PX, and loops over a chunk of tonal frequencies k.  Per k it
//   (a) encodes the tile on the fly: the tonal DFT of a one-hot column e_{v(x)}
//       is the single twiddle w_T^{k v(x)} (0 at gaps / outside the image), so
//       the (spatial x tonal) one-hot volume of build_umbra (umbra.py:177-186)
//       never exists;
//   (b) runs the forward 2-D FFT (y axis, then x axis; radix-R1 x radix-R2
//       four-step per axis, butterflies in registers, exchanges through a
//       padded shared-memory tile);
//   (c) multiplies by the cached SE spectrum for k (fa *= fb, fft_conv.py:137),
//       fused into the last forward pass;
//   (d) runs the inverse FFT (x axis, then y axis) and writes only the
//       overlap-save valid window of the tile to the spectral scratch
//       Chat[img][k][out_y][out_x] (complex64) for the tonal kernel.
// With SPEC=true the same code computes the SE spectrum (rfftn(b),
// fft_conv.py:135-136) once per plan and stores it in thread-register order.
//
// Data movement:
//  * every thread works on PAIRS of horizontally adjacent tile points, so each
//    shared-memory access is one 128-bit LDS/STS; rows are padded to PX+2
//    complex values (16-byte aligned; 8 consecutive rows at one x hit 8
//    distinct 16-byte bank groups, so row passes whose lanes run down the rows
//    are conflict-free; column passes read contiguous row segments); all
//    per-element offsets are compile-time immediates;
//  * the tonal DFT twiddle of the encode is one MUFU sincos on an exactly
//    reduced integer angle (no table, no shared memory);
//  * the SE spectrum for plane k (L2-resident, read by every tile) is streamed
//    into shared memory with per-thread cp.async (LDGSTS) in thread order, two
//    chunks ahead, so its L2 latency overlaps the FFT passes instead of
//    stalling the spectral product.
#pragma once
#include <type_traits>
#include "fm_async.cuh"
#include "fm_dft.cuh"

namespace fm {

constexpr uint16_t kSent = 0xFFFFu;  // "no one-hot entry": gap or outside the grid

template <int P> struct Split;
template <> struct Split<8> { static constexpr int R1 = 4, R2 = 2; };     // (1-D CTAs of 8 rows: y unused)
template <> struct Split<16> { static constexpr int R1 = 4, R2 = 4; };
template <> struct Split<32> { static constexpr int R1 = 8, R2 = 4; };
template <> struct Split<64> { static constexpr int R1 = 8, R2 = 8; };
template <> struct Split<128> { static constexpr int R1 = 16, R2 = 8; };
template <> struct Split<256> { static constexpr int R1 = 16, R2 = 16; };

// Twiddle tables W_P^j = exp(-2 pi i j / P) for P = 16..256, concatenated.
template <int P> struct TwOff;
template <> struct TwOff<16> { static constexpr int v = 0; };
template <> struct TwOff<32> { static constexpr int v = 16; };
template <> struct TwOff<64> { static constexpr int v = 48; };
template <> struct TwOff<128> { static constexpr int v = 112; };
template <> struct TwOff<256> { static constexpr int v = 240; };
constexpr int kTwTotal = 496;

struct TileArgs {
  // image batch (CONV) or SE (SPEC)
  const void* img;            // [batch][H][W] of img_dtype
  const uint8_t* img_def;     // nullable
  const int32_t* se_vals;     // SPEC: [my][mx]
  const uint8_t* se_def;      // SPEC: nullable
  int img_dtype;
  int H, W;                   // image array extent (1-D: H = 1)
  int OH, OW;                 // output region extent
  int DY, DX;                 // input index = out index + D + tile position
  int QY, QX;                 // valid outputs per tile per axis
  int my, mx;                 // SE extent per axis
  int tiles_x, tiles_total;   // tile grid (1-D: tiles_total = number of 1-D tiles)
  int T, K;                   // tonal length and planes (T/2+1)
  uint32_t magicT;            // floor(2^32 / T)
  int k_chunk;                // planes per CTA; 0: chosen on the device (fills conv_target CTAs)
  int conv_target;
  int enc_sign, enc_bias;     // v = enc_sign * f + enc_bias (CONV) / v = b - se_min (SPEC)
  const float4* spec;         // [K][thread order] SE spectrum, pairs (CONV reads)
  float4* spec_out;           // SPEC writes
  float spec_scale;           // SPEC: 1 / (PY_eff * PX * T)
  float2* chat;               // CONV: [imgs][units][K_max][wpx] (window-local pixels)
  const float2* enc_tab;      // encode tables exp(-2 pi i j / T), j <= T (entry T = 0); SPEC: this T's
  const int* enc_off;         // CONV: [ladder] offset of the ladder entry's table
  int* err;                   // value-range error flag
  // per-unit tonal length (CONV): a unit is one 2-D tile or one group of PY 1-D tiles
  const int4* unit_param;     // [imgs][units]: x = anchor (clamp level: v = f - anchor, or anchor - f for erosion), y = N_t, z = ladder index
  const int64_t* spec_off;    // [ladder] offset of the SE spectrum for N = ladder[i] (float4 units)
  int units;                  // units per image
  int unit0, upl;             // first unit of this launch, chat slots per image (units per launch)
  int K_max;                  // chat planes per unit (N_global + 1)
  int wpx;                    // plane stride of chat (even)
  // CONV launch order: jobs = the range kernel's work lists, largest tonal length first
  // each unit's planes are split into chunks of k_chunk (one CTA each)
  const int* bucket_count;    // [L]
  const int2* bucket_list;    // [L][cap] (img, unit)
  const int* ladder;          // [L] N of each ladder entry
  int cap, L;
  // fused tonal step (fm_fused.cuh, three-pass 128x128 kernel): the CTA completing a unit's
  // last plane chunk runs its inverse tonal FFT + threshold + store
  int chat16;                 // spectral planes stored as int16 pairs, value * (chat_q_T * T) (fm_abi.cu)
  float chat_q_T;
  int fuse_nmax;              // 0: off; else units with N_t <= fuse_nmax are finished here
  int discard;                // drop the consumed spectral lines from L2 (no write-back)
  int* unit_done;             // [imgs][upl] plane-chunk completion counters (self-resetting)
  void* out;                  // [imgs][OH][OW] of out_dtype (this launch's first image)
  int out_dtype;              // 0 int32, 1 uint8, 2 uint16, 3 int16
  uint8_t* valid;             // nullable
  int out_sign, se_min, fill, se_count;
  float* dev_max;             // max |c - rint c| (float bits, atomicMax as int)
};

__constant__ float2 c_tw[kTwTotal];

template <int PY, int PX, int NT, bool TWO_D>
struct TileCfg {
  static constexpr int R1x = Split<PX>::R1, R2x = Split<PX>::R2;
  static constexpr int R1y = TWO_D ? Split<PY>::R1 : 1;
  static constexpr int R2y = TWO_D ? Split<PY>::R2 : 1;
  static constexpr int RS = PX + 2;              // padded row stride (complex values)
  static constexpr int NPTS = PY * PX;
  static constexpr int XP = PX / 2;              // column pairs
  static constexpr int G_yA = TWO_D ? XP * R2y / NT : 0;   // items (xp, n2): R1y pairs each
  static constexpr int G_yB = TWO_D ? XP * R1y / NT : 0;   // items (xp, k1): R2y pairs each
  static constexpr int G_xA = PY * (R2x / 2) / NT;         // items (y, n2 pair): 2 x R1x values
  static constexpr int G_xB = PY * R1x / NT;               // items (y, k1): R2x values
  static_assert(!TWO_D || (G_yA >= 1 && G_yA * NT == XP * R2y && G_yB >= 1 && G_yB * NT == XP * R1y),
                "y-axis item split");
  static_assert(G_xA >= 1 && G_xA * NT == PY * (R2x / 2) && G_xB >= 1 && G_xB * NT == PY * R1x,
                "x-axis item split");
  static_assert(PX >= 16, "min tile edge 16");
  // x-axis passes: warp w owns rows [w*RPW, (w+1)*RPW), so the x pass A <-> B
  // exchanges stay inside one warp (__syncwarp instead of a CTA barrier)
  static constexpr int NW = NT / 32;
  static constexpr int RPW = PY / NW;
  static_assert(RPW * NW == PY && RPW * (R2x / 2) == 32 && G_xA == 1, "x pass A: one item per lane");
  // y pass B by warp-owned k1 groups (see the kernel): needs one 8-row group per warp
  static constexpr bool kWarpY = TWO_D && R1y == NW && R2y == RPW && XP % 32 == 0 && G_yB * 32 == XP;
  static constexpr int kBufBytes = PY * RS * 8;
  static constexpr int kSpecPairs = NPTS / 2;           // float4 per tonal plane
  static constexpr int SQ = R2x / 2;                    // float4 per x-pass-B item
  static constexpr int kChunkF4 = SQ * NT;              // float4 per spectrum chunk (one item per thread)
  static constexpr int NBUF = G_xB >= 2 ? 2 : 1;
  static constexpr int kSpecBytes = NBUF * kChunkF4 * 16;
  // CONV: a plane's first two spectrum chunks arrive by bulk async copies
  // (1-D TMA) issued a whole plane ahead, by the last warp to release the
  // buffer; the later chunks by per-thread cp.async into the thread's own
  // slots right after it consumed them (no cross-warp coupling mid-plane)
  static constexpr bool kBulkSpec = NBUF == 2 && G_xB >= 2;
  static constexpr uint32_t kChunkBytes = kChunkF4 * 16;
  static constexpr int kTvBytes = ((NPTS * 2 + 15) / 16) * 16;
  // x pass A twiddle pairs (W^{n2 k1}, W^{(n2+1) k1}) for the R2x/2 pair columns:
  // 16-byte slots, stride R1x+1 (conflict-free for the 4..8 distinct n2 of a
  // warp).  In 2-D they live in the row padding (free), in 1-D after the tiles.
  static constexpr int kTwxSlots = (R2x / 2) * (R1x + 1);
  static constexpr bool kTwxInPad = kTwxSlots <= PY;
  static constexpr int kTwxBytes = kTwxInPad ? 0 : kTwxSlots * 16;
  static constexpr int kSmemFixed = kBufBytes + kSpecBytes + kTvBytes + kTwxBytes;
  // encode table w_T^{-j}, j <= T (entry T = 0 for "no pixel"), in what is left
  // of the 227 KB (P = 128: T <= 95; beyond, the table is read from L1/L2)
  static constexpr int kEncAvail = (227 * 1024 - kSmemFixed - 256) / 8;  // 256: static smem of the kernel
  static constexpr int kEncSlots = kEncAvail < 0 ? 0 : (kEncAvail < 161 ? kEncAvail : 161);
  static constexpr int kSmemTotal = kSmemFixed + kEncSlots * 8;
};

__device__ __forceinline__ int load_img(const void* img, int dtype, int64_t i) {
  if (dtype == 0) return (int)__ldg(reinterpret_cast<const uint8_t*>(img) + i);
  if (dtype == 1) return (int)__ldg(reinterpret_cast<const uint16_t*>(img) + i);
  return __ldg(reinterpret_cast<const int32_t*>(img) + i);
}

// complex value -> two int16 fixed-point numbers (round to nearest, saturating)
__device__ __forceinline__ uint32_t pack16(float2 v, float q) {
  unsigned short re, im;
  asm("cvt.rni.sat.s16.f32 %0, %1;" : "=h"(re) : "f"(v.x * q));
  asm("cvt.rni.sat.s16.f32 %0, %1;" : "=h"(im) : "f"(v.y * q));
  return (uint32_t)re | ((uint32_t)im << 16);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// 16-byte global -> shared async copy (LDGSTS), L2-only caching
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One CTA's job: SPEC launches are (unit 0, plane chunk blockIdx.y) of one
// ladder entry; CONV launches map blockIdx.x to (img, unit, plane chunk) through
// the range kernel's per-ladder work lists, walked from the longest tonal length
// down (the longest units start first, so a launch ends without a tail of long
// stragglers).  Every thread calls it (it contains a CTA barrier); false = no work.
struct UnitJob {
  int img, unit, kchunk;
  int k_chunk;                // planes per CTA (device-chosen when the launch is sized on the device)
  int T, K, enc_bias, unit_li;
  uint32_t magicT;
  bool skip0;                 // CONV unit whose plane 0 is a known constant (fm_range.cuh "full")
  const float4* spec_base;    // SE spectrum of the unit's ladder entry
};

template <bool SPEC>
__device__ __forceinline__ bool decode_job(const TileArgs& a, UnitJob& j) {
  j.img = 0;
  j.unit = a.unit0 + blockIdx.x;
  j.kchunk = blockIdx.y;
  j.k_chunk = a.k_chunk;
  j.T = a.T;
  j.K = a.K;
  j.enc_bias = a.enc_bias;
  j.magicT = a.magicT;
  j.unit_li = 0;
  j.skip0 = false;
  j.spec_base = a.spec;
  if constexpr (!SPEC) {
    const int lane = threadIdx.x & 31;
    __shared__ int s_job[4];
    if (threadIdx.x < 32) {
      // k_chunk = 0: the launch was sized on the device (no host round trip for the
      // per-ladder counts): planes per CTA so that the jobs fill a.conv_target CTAs
      int kc = a.k_chunk;
      if (kc <= 0) {
        int planes = 0;
        for (int li = lane; li < a.L; li += 32) planes += a.bucket_count[li] * (a.ladder[li] + 1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) planes += __shfl_xor_sync(0xffffffffu, planes, o);
        kc = max(1, (planes + a.conv_target - 1) / a.conv_target);
      }
      int rem = (int)blockIdx.x, found = -1, fch = 1;
      for (int top = a.L - 1; top >= 0 && found < 0; top -= 32) {
        const int li = top - lane;
        const int ch = li >= 0 ? (a.ladder[li] + kc) / kc : 1;   // ceil((N+1)/k_chunk)
        const int c = li >= 0 ? a.bucket_count[li] * ch : 0;
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int nb = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += nb;
        }
        const unsigned m = __ballot_sync(0xffffffffu, li >= 0 && rem < incl);
        if (m) {
          const int l0 = __ffs(m) - 1;
          rem -= __shfl_sync(0xffffffffu, incl - c, l0);
          fch = __shfl_sync(0xffffffffu, ch, l0);
          found = top - l0;
        } else {
          rem -= __shfl_sync(0xffffffffu, incl, 31);
        }
      }
      if (lane == 0) {
        if (found < 0) {
          s_job[0] = -1;   // grid sized before the counts were known: no job left
        } else {
          const int u = rem / fch;
          const int2 job = a.bucket_list[(size_t)found * a.cap + u];
          s_job[0] = job.x;
          s_job[1] = job.y & ~kJobFull;
          s_job[2] = rem - u * fch;   // plane chunk of the unit
        }
        s_job[3] = kc;
      }
    }
    __syncthreads();
    if (s_job[0] < 0) return false;
    j.img = s_job[0];
    j.unit = s_job[1];
    j.kchunk = s_job[2];
    j.k_chunk = s_job[3];
    const int4 up = a.unit_param[(size_t)j.img * a.units + j.unit];
    j.K = up.y + 1;
    if (j.kchunk * j.k_chunk >= j.K) return false;   // this k-chunk is beyond the unit's planes
    j.T = 2 * up.y;
    j.magicT = (uint32_t)(0x100000000ull / (uint64_t)j.T);
    j.unit_li = up.z;
    j.skip0 = (up.w & 2) != 0;
    j.enc_bias = a.enc_sign > 0 ? -up.x : up.x;
    j.spec_base = a.spec + a.spec_off[up.z];
  }
  return true;
}

template <int PY, int PX, int NT, bool TWO_D, bool SPEC>
__global__ void __launch_bounds__(NT, 1) tile_conv_kernel(const TileArgs a) {
  using C = TileCfg<PY, PX, NT, TWO_D>;
  constexpr int RS = C::RS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* buf = reinterpret_cast<float2*>(smem_raw);
  float4* sbuf = reinterpret_cast<float4*>(smem_raw + C::kBufBytes);
  uint16_t* tv = reinterpret_cast<uint16_t*>(smem_raw + C::kBufBytes + C::kSpecBytes);
  const uint32_t* tv32 = reinterpret_cast<const uint32_t*>(tv);

  auto ld2 = [&](int y, int x) -> float4 { return *reinterpret_cast<const float4*>(buf + y * RS + x); };
  auto st2 = [&](int y, int x, float2 p, float2 q) {
    *reinterpret_cast<float4*>(buf + y * RS + x) = make_float4(p.x, p.y, q.x, q.y);
  };

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  UnitJob job;
  if (!decode_job<SPEC>(a, job)) return;
  const int img = job.img, unit = job.unit, kchunk_idx = job.kchunk;
  const int T = job.T, K = job.K, enc_bias = job.enc_bias, unit_li = job.unit_li;
  const uint32_t magicT = job.magicT;
  const bool skip0 = job.skip0;
  const float4* spec_base = job.spec_base;
  // encode table of this unit's T: shared memory when it fits, else global (L1)
  const float2* enc_g = SPEC ? a.enc_tab : a.enc_tab + a.enc_off[unit_li];
  float2* enc_s = reinterpret_cast<float2*>(smem_raw + C::kSmemFixed);
  // 2-D with room for two tables: per-plane tables M_k[t] = w_T^{(k t) mod T}
  // (double-buffered, M_k[T] = 0 for "no pixel"), so the encode is one LDS;
  // else the base table w_T^j with the index (k t) mod T reduced per element
  const bool mtab = TWO_D && 2 * (T + 1) <= C::kEncSlots;
  const bool enc_in_smem = !mtab && T + 1 <= C::kEncSlots;
  if (enc_in_smem)
    for (int j = tid; j <= T; j += NT) enc_s[j] = enc_g[j];
  const float2* encT = enc_in_smem ? enc_s : enc_g;
  auto build_mtab = [&](int kk) {
    float2* M = enc_s + (kk & 1) * (T + 1);
    for (int j = tid; j <= T; j += NT) M[j] = j < T ? enc_g[(kk * j) % T] : make_float2(0.f, 0.f);
  };
  const uint16_t sent = mtab ? (uint16_t)T : kSent;

  // ---- stage the tile's tonal indices v(x) (kSent = no entry)
  {
    int ty = 0, tx = 0;
    if (TWO_D && !SPEC) {
      ty = unit / a.tiles_x;
      tx = unit - ty * a.tiles_x;
    }
    int bad = 0;
    if constexpr (SPEC) {
      for (int p = tid; p < C::NPTS; p += NT) {
        const int py = p / PX, px = p - (p / PX) * PX;
        uint16_t t = sent;
        const int sy = TWO_D ? py : 0;
        if (sy < a.my && px < a.mx) {
          const int si = sy * a.mx + px;
          // ladder entries shorter than the SE's own value range are never used by a
          // unit (a unit's T exceeds max b - min b); reduce so their (unused) spectra
          // stay finite and the per-plane table (T + 1 entries) is never overrun
          if (a.se_def == nullptr || a.se_def[si]) t = (uint16_t)((a.se_vals[si] + a.enc_bias) % T);
        }
        tv[p] = t;
      }
    } else {
      // batches of GB independent (predicated) loads per thread, then the
      // conversions: the image reads overlap instead of paying one global
      // latency per pixel
      constexpr int IT = C::NPTS / NT;
      static_assert(IT * NT == C::NPTS, "staging split");
      constexpr int GB = IT < 16 ? IT : 16;
#pragma unroll 1
      for (int g0 = 0; g0 < IT; g0 += GB) {
        int raw[GB];
        bool ok[GB];
#pragma unroll
        for (int u = 0; u < GB; ++u) {
          const int p = tid + (g0 + u) * NT;
          const int py = p / PX, px = p - (p / PX) * PX;
          int iy, ix;
          bool rowok;
          if (TWO_D) {
            iy = ty * a.QY + a.DY + py;
            ix = tx * a.QX + a.DX + px;
            rowok = true;
          } else {
            const int tile = unit * PY + py;
            iy = 0;
            ix = tile * a.QX + a.DX + px;
            rowok = tile < a.tiles_total;
          }
          ok[u] = rowok && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
          raw[u] = 0;
          if (ok[u]) {
            const int64_t gi = ((int64_t)img * a.H + iy) * a.W + ix;
            raw[u] = load_img(a.img, a.img_dtype, gi);
            if (a.img_def != nullptr) ok[u] = a.img_def[gi] != 0;
          }
        }
#pragma unroll
        for (int u = 0; u < GB; ++u) {
          uint16_t t = sent;
          if (ok[u]) {
            // values below the unit's clamp level encode as the clamp (fm_range.cuh)
            const int v = max(a.enc_sign * raw[u] + enc_bias, 0);
            if (v >= T) bad = 1;
            else t = (uint16_t)v;
          }
          tv[tid + (g0 + u) * NT] = t;
        }
      }
    }
    if (!SPEC && bad) atomicOr(a.err, 1);
  }
  // x pass A twiddle pairs
  auto twx_slot = [&](int j) -> float4* {
    if constexpr (C::kTwxInPad) return reinterpret_cast<float4*>(buf + j * RS + PX);
    else return reinterpret_cast<float4*>(smem_raw + C::kBufBytes + C::kSpecBytes + C::kTvBytes) + j;
  };
  for (int j = tid; j < C::kTwxSlots; j += NT) {
    const int n2p = j / (C::R1x + 1), k1 = j - n2p * (C::R1x + 1);
    const int n2 = 2 * n2p;
    const float2 w0 = c_tw[TwOff<PX>::v + (n2 * k1) % PX];
    const float2 w1 = c_tw[TwOff<PX>::v + ((n2 + 1) * k1) % PX];
    *twx_slot(j) = make_float4(w0.x, w0.y, w1.x, w1.y);
  }
  __shared__ __align__(8) uint64_t s_full[2];   // spectrum ring (C::kBulkSpec)
  __shared__ int s_rel[2];                       // warps that released the buffer's chunk
  {
    const int k_first = kchunk_idx * job.k_chunk + ((skip0 && kchunk_idx == 0) ? 1 : 0);
    if (mtab) build_mtab(k_first);
    if constexpr (!SPEC && C::kBulkSpec) {
      if (tid == 0) {
        mbar_init(&s_full[0], 1);
        mbar_init(&s_full[1], 1);
        s_rel[0] = 0;
        s_rel[1] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (k_first < min(K, kchunk_idx * job.k_chunk + job.k_chunk)) {
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            mbar_expect_tx(&s_full[g], C::kChunkBytes);
            bulk_g2s_nohint(sbuf + g * C::kChunkF4, spec_base + (size_t)k_first * C::kSpecPairs + (size_t)g * C::kChunkF4,
                            C::kChunkBytes, &s_full[g]);
          }
        }
      }
    }
  }
  __syncthreads();
  const int ty = (TWO_D && !SPEC) ? unit / a.tiles_x : 0;
  const int tx = (TWO_D && !SPEC) ? unit - ty * a.tiles_x : 0;
  const int k_begin = kchunk_idx * job.k_chunk;
  // the plane loop bound lives in shared memory: under the kernel's register
  // pressure a register copy gets spilled and reloaded from local memory
  __shared__ int s_kend;
  if (tid == 0) s_kend = min(K, k_begin + job.k_chunk);
  __syncthreads();
  const volatile int* kend_s = &s_kend;
  // window-local output planes of this unit (slot = launch-local unit index)
  float2* chat_unit = SPEC ? nullptr : a.chat + ((size_t)img * a.upl + (unit - a.unit0)) * a.K_max * (size_t)a.wpx;

  // per-thread spectrum chunk copy: item g of plane k -> buffer g % NBUF (own slots only)
  auto spec_fetch = [&](int k, int g) {
    const float4* src = spec_base + (size_t)k * C::kSpecPairs + (size_t)g * C::kChunkF4 + tid;
    float4* dst = sbuf + (g % C::NBUF) * C::kChunkF4 + tid;
#pragma unroll
    for (int q = 0; q < C::SQ; ++q) cp_async16(dst + q * NT, src + q * NT);
    cp_async_commit();
  };

  int pord = 0;   // planes done (ring phase when chunks per plane is not a multiple of 4)
  for (int k = k_begin; k < *kend_s; ++k) {
    if (k == 0 && skip0) continue;   // plane 0 of a full unit: the tonal pass knows it
    if constexpr (!SPEC && !C::kBulkSpec) {
#pragma unroll
      for (int g = 0; g < C::NBUF; ++g) spec_fetch(k, g);
    }
    // encode helper: w_T^{k v} = exp(-2 pi i ((k v) mod T) / T) from the table;
    // the index is reduced exactly in integers, the sentinel reads entry T = 0
    auto enc = [&](uint32_t t) -> float2 {
      const uint32_t n = (uint32_t)k * t;
      uint32_t r = n - __umulhi(n, magicT) * (uint32_t)T;
      r = (r >= (uint32_t)T) ? r - (uint32_t)T : r;
      r = (t == kSent) ? (uint32_t)T : r;
      return encT[r];
    };

    if constexpr (TWO_D) {
      // ---------------- forward y, pass A (with encode): item (xp, n2)
      const float2* Mk = enc_s + (k & 1) * (T + 1);
      auto y_pass_a = [&](auto use_m) {
#pragma unroll
        for (int g = 0; g < C::G_yA; ++g) {
          const int i = tid + NT * g;
          const int xp = i % C::XP, n2 = i / C::XP;
          float2 wa[C::R1y], wb[C::R1y];
#pragma unroll
          for (int n1 = 0; n1 < C::R1y; ++n1) {
            const uint32_t tt = tv32[((n2 + C::R2y * n1) * PX) / 2 + xp];
            if constexpr (decltype(use_m)::value) {
              wa[n1] = Mk[tt & 0xFFFFu];
              wb[n1] = Mk[tt >> 16];
            } else {
              wa[n1] = enc(tt & 0xFFFFu);
              wb[n1] = enc(tt >> 16);
            }
          }
          dft<C::R1y, false>(wa);
          dft<C::R1y, false>(wb);
#pragma unroll
          for (int k1 = 0; k1 < C::R1y; ++k1) {
            float2 za = wa[k1], zb = wb[k1];
            if (k1 != 0) {
              const float2 w = c_tw[TwOff<PY>::v + n2 * k1];
              za = cmul(za, w);
              zb = cmul(zb, w);
            }
            st2(n2 + C::R2y * k1, 2 * xp, za, zb);
          }
        }
      };
      if (mtab) y_pass_a(std::true_type{});
      else y_pass_a(std::false_type{});
      __syncthreads();
      // next plane's table into the other buffer (its last reader, plane k-1's
      // y pass A, finished before this plane's first barrier)
      if (mtab && k + 1 < *kend_s) build_mtab(k + 1);
      // ---------------- forward y, pass B: item (xp, k1)
      // With one warp per k1 group (R1y == warps, R2y == rows per warp) the
      // group is exactly the warp's x-pass rows: y pass B, the x passes and
      // inverse y pass B then run warp-locally between two CTA barriers.
#pragma unroll
      for (int g = 0; g < C::G_yB; ++g) {
        const int i = tid + NT * g;
        const int xp = C::kWarpY ? lane + 32 * g : i % C::XP;
        const int k1 = C::kWarpY ? warp : i / C::XP;
        float2 wa[C::R2y], wb[C::R2y];
#pragma unroll
        for (int n2 = 0; n2 < C::R2y; ++n2) {
          const float4 p = ld2(n2 + C::R2y * k1, 2 * xp);
          wa[n2] = make_float2(p.x, p.y);
          wb[n2] = make_float2(p.z, p.w);
        }
        dft<C::R2y, false>(wa);
        dft<C::R2y, false>(wb);
#pragma unroll
        for (int k2 = 0; k2 < C::R2y; ++k2) st2(k2 + C::R2y * k1, 2 * xp, wa[k2], wb[k2]);
      }
      if constexpr (C::kWarpY) __syncwarp();
      else __syncthreads();
    }

    // ---------------- forward x, pass A: item (y, n2 pair); 1-D: with encode
#pragma unroll
    for (int g = 0; g < C::G_xA; ++g) {
      const int i = lane + 32 * g;
      const int y = warp * C::RPW + i % C::RPW, n2 = 2 * (i / C::RPW);
      float2 wa[C::R1x], wb[C::R1x];
#pragma unroll
      for (int n1 = 0; n1 < C::R1x; ++n1) {
        if constexpr (TWO_D) {
          const float4 p = ld2(y, n2 + C::R2x * n1);
          wa[n1] = make_float2(p.x, p.y);
          wb[n1] = make_float2(p.z, p.w);
        } else {
          const uint32_t tt = tv32[(y * PX + n2 + C::R2x * n1) / 2];
          wa[n1] = enc(tt & 0xFFFFu);
          wb[n1] = enc(tt >> 16);
        }
      }
      dft<C::R1x, false>(wa);
      dft<C::R1x, false>(wb);
#pragma unroll
      for (int k1 = 0; k1 < C::R1x; ++k1) {
        float2 za = wa[k1], zb = wb[k1];
        if (k1 != 0) {
          const float4 w = *twx_slot((n2 / 2) * (C::R1x + 1) + k1);
          za = cmul(za, make_float2(w.x, w.y));
          zb = cmul(zb, make_float2(w.z, w.w));
        }
        st2(y, n2 + C::R2x * k1, za, zb);
      }
    }
    __syncwarp();   // x pass B reads only rows owned by this warp

    // ---------------- forward x, pass B (+ spectral product + inverse x pass B): item (y, k1)
    {
      float4* so = SPEC ? a.spec_out + (size_t)k * C::kSpecPairs : nullptr;
#pragma unroll
      for (int g = 0; g < C::G_xB; ++g) {
        const int i = lane + 32 * g;
        const int y = warp * C::RPW + i % C::RPW, k1 = i / C::RPW;
        float2 w[C::R2x];
#pragma unroll
        for (int q = 0; q < C::SQ; ++q) {
          const float4 p = ld2(y, 2 * q + C::R2x * k1);
          w[2 * q] = make_float2(p.x, p.y);
          w[2 * q + 1] = make_float2(p.z, p.w);
        }
        dft<C::R2x, false>(w);
        if constexpr (SPEC) {
          const float s = a.spec_scale;
#pragma unroll
          for (int q = 0; q < C::SQ; ++q)
            so[(g * C::SQ + q) * NT + tid] =
                make_float4(w[2 * q].x * s, w[2 * q].y * s, w[2 * q + 1].x * s, w[2 * q + 1].y * s);
        } else {
          if (C::kBulkSpec && g < 2) {
            mbar_wait(&s_full[g], (uint32_t)(pord & 1));
          } else if (C::kBulkSpec) {
            // per-thread chunks g >= 2 (committed after items g-2, g-1)
            if (g + 1 < C::G_xB) cp_async_wait<1>();
            else cp_async_wait<0>();
          } else {
            // chunk g landed? (the newest NBUF-1 groups may still be in flight)
            if (g + C::NBUF <= C::G_xB) cp_async_wait<C::NBUF - 1>();
            else cp_async_wait<0>();
          }
          const float4* sp = sbuf + (g % C::NBUF) * C::kChunkF4 + tid;
          float4 s4[C::SQ];
#pragma unroll
          for (int q = 0; q < C::SQ; ++q) s4[q] = sp[q * NT];
#pragma unroll
          for (int q = 0; q < C::SQ; ++q) {
            w[2 * q] = cmul(w[2 * q], make_float2(s4[q].x, s4[q].y));
            w[2 * q + 1] = cmul(w[2 * q + 1], make_float2(s4[q].z, s4[q].w));
          }
          if (C::kBulkSpec && g + 2 >= C::G_xB) {
            // last chunks of the plane: release the buffer; the last warp to do so
            // refills it with the next plane's chunk (a bulk copy a whole plane ahead)
            __syncwarp();
            if (lane == 0) {
              __threadfence_block();
              const int b = g & 1;
              if (atomicAdd(&s_rel[b], 1) == C::NW - 1) {
                s_rel[b] = 0;
                if (k + 1 < *kend_s) {
                  // every warp's generic-proxy reads of the buffer happen before this
                  // (the release counter); order them before the async-proxy refill
                  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                  mbar_expect_tx(&s_full[b], C::kChunkBytes);
                  bulk_g2s_nohint(sbuf + b * C::kChunkF4,
                                  spec_base + (size_t)(k + 1) * C::kSpecPairs + (size_t)b * C::kChunkF4,
                                  C::kChunkBytes, &s_full[b]);
                }
              }
            }
          } else if (g + C::NBUF < C::G_xB) {
            // refill this thread's own slots (their values are consumed above)
            spec_fetch(k, g + C::NBUF);
          }
          dft<C::R2x, true>(w);
#pragma unroll
          for (int q = 0; q < C::SQ; ++q) st2(y, 2 * q + C::R2x * k1, w[2 * q], w[2 * q + 1]);
        }
      }
    }
    if constexpr (SPEC) {
      __syncthreads();
      continue;
    }
    __syncwarp();   // inverse x pass A reads only rows owned by this warp

    // ---------------- inverse x, pass A: item (y, n2 pair); 1-D: output store
#pragma unroll
    for (int g = 0; g < C::G_xA; ++g) {
      const int i = lane + 32 * g;
      const int y = warp * C::RPW + i % C::RPW, n2 = 2 * (i / C::RPW);
      float2 wa[C::R1x], wb[C::R1x];
#pragma unroll
      for (int k1 = 0; k1 < C::R1x; ++k1) {
        const float4 p = ld2(y, n2 + C::R2x * k1);
        wa[k1] = make_float2(p.x, p.y);
        wb[k1] = make_float2(p.z, p.w);
        if (k1 != 0) {
          const float4 w = *twx_slot((n2 / 2) * (C::R1x + 1) + k1);
          wa[k1] = cmulc(wa[k1], make_float2(w.x, w.y));
          wb[k1] = cmulc(wb[k1], make_float2(w.z, w.w));
        }
      }
      dft<C::R1x, true>(wa);
      dft<C::R1x, true>(wb);
      if constexpr (TWO_D) {
#pragma unroll
        for (int n1 = 0; n1 < C::R1x; ++n1) st2(y, n2 + C::R2x * n1, wa[n1], wb[n1]);
      } else {
        // 1-D output: row y is tile (blockIdx.x*PY + y); positions x >= mx-1 are valid;
        // window pixel p = y*QX + (x - (mx-1))
        const int tile = unit * PY + y;
        if (tile < a.tiles_total) {
          float2* dst = chat_unit + ((ptrdiff_t)k * a.wpx + (ptrdiff_t)y * a.QX - (a.mx - 1));
#pragma unroll
          for (int n1 = 0; n1 < C::R1x; ++n1) {
            const int x = n2 + C::R2x * n1;
            const int ox = tile * a.QX + x - (a.mx - 1);
            if (x >= a.mx - 1 && ox < a.OW) dst[x] = wa[n1];
            if (x + 1 >= a.mx - 1 && ox + 1 < a.OW) dst[x + 1] = wb[n1];
          }
        }
      }
    }
    if constexpr (TWO_D) {
      if constexpr (C::kWarpY) __syncwarp();
      else __syncthreads();
      // column pairs entirely left of the valid window are not needed any more
      const int xp_min = (a.mx - 1) / 2;
      // ---------------- inverse y, pass B: item (xp, k1)
#pragma unroll
      for (int g = 0; g < C::G_yB; ++g) {
        const int i = tid + NT * g;
        const int xp = C::kWarpY ? lane + 32 * g : i % C::XP;
        const int k1 = C::kWarpY ? warp : i / C::XP;
        if (xp < xp_min) continue;
        float2 wa[C::R2y], wb[C::R2y];
#pragma unroll
        for (int k2 = 0; k2 < C::R2y; ++k2) {
          const float4 p = ld2(k2 + C::R2y * k1, 2 * xp);
          wa[k2] = make_float2(p.x, p.y);
          wb[k2] = make_float2(p.z, p.w);
        }
        dft<C::R2y, true>(wa);
        dft<C::R2y, true>(wb);
#pragma unroll
        for (int n2 = 0; n2 < C::R2y; ++n2) st2(n2 + C::R2y * k1, 2 * xp, wa[n2], wb[n2]);
      }
      __syncthreads();
      // ---------------- inverse y, pass A + store of the valid window: item (xp, n2)
      // window pixel p = (y - (my-1)) * QX + (x - (mx-1))
      float2* dst = chat_unit + ((ptrdiff_t)k * a.wpx - (ptrdiff_t)(a.my - 1) * a.QX - (a.mx - 1));
#pragma unroll
      for (int g = 0; g < C::G_yA; ++g) {
        const int i = tid + NT * g;
        const int xp = i % C::XP, n2 = i / C::XP;
        if (xp < xp_min) continue;
        float2 wa[C::R1y], wb[C::R1y];
#pragma unroll
        for (int k1 = 0; k1 < C::R1y; ++k1) {
          const float4 p = ld2(n2 + C::R2y * k1, 2 * xp);
          wa[k1] = make_float2(p.x, p.y);
          wb[k1] = make_float2(p.z, p.w);
          if (k1 != 0) {
            const float2 w = c_tw[TwOff<PY>::v + n2 * k1];
            wa[k1] = cmulc(wa[k1], w);
            wb[k1] = cmulc(wb[k1], w);
          }
        }
        dft<C::R1y, true>(wa);
        dft<C::R1y, true>(wb);
        const int x = 2 * xp;
        const int ox = tx * a.QX + x - (a.mx - 1);
        const bool va = x >= a.mx - 1 && ox < a.OW;
        const bool vb = x + 1 >= a.mx - 1 && ox + 1 < a.OW;
        // rows y = n2 + R2y*n1 in [my-1, y_end) are stored; hoisted out of the n1 loop
        const int y_end = min(PY, a.OH - ty * a.QY + (a.my - 1));
        float2* col = dst + (ptrdiff_t)n2 * a.QX + x;
        const ptrdiff_t step = (ptrdiff_t)C::R2y * a.QX;
        // 16-byte stores when both columns are valid and every row start is aligned
        const bool pair = va && vb && (a.QX % 2 == 0) && ((reinterpret_cast<uintptr_t>(col) & 15) == 0);
#pragma unroll
        for (int n1 = 0; n1 < C::R1y; ++n1) {
          const int y = n2 + C::R2y * n1;
          if (y >= a.my - 1 && y < y_end) {
            float2* row = col + n1 * step;
            if (pair) {
              *reinterpret_cast<float4*>(row) = make_float4(wa[n1].x, wa[n1].y, wb[n1].x, wb[n1].y);
            } else {
              if (va) row[0] = wa[n1];
              if (vb) row[1] = wb[n1];
            }
          }
        }
      }
      // no barrier: the next plane's y pass A writes exactly the positions this
      // thread just read (same item partition), and no other thread reads them
    }
    ++pord;
  }
}

}  // namespace fm
