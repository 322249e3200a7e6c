// fm_range.cuh — per-unit tonal range (the local l_R of each tile).
//
// The reference sizes the tonal axis from the global data maxima
// (required_lr, umbra.py:172-174).  Exactness only needs, for every output
// pixel, a tonal length larger than the spread of the degrees that can meet
// there.  Two reductions of that spread are exact:
//
//  * shift: dilation commutes with constant shifts of f, so a unit encodes
//    v = f - min f over its input window (erosion: max f - f);
//  * clamp: if D is a lower bound of the dilation over the unit's output
//    pixels, replacing f(z) by max(f(z), D - max b) changes no output —
//    every raised pair sums to at most D, which never exceeds the true
//    maximum, and no pair is removed.  So values below c = D - max b may be
//    clamped to c, and the unit needs T_t > (max f - max(min f, c)) + (max b - min b).
//
// D = min over the unit's output pixels x of max over a small set S of SE
// taps (the highest-valued entries) of f(x - y) + b(y) — a lower bound of
// the dilation at x.  It is found by branch and bound: each pixel stops
// scanning taps as soon as its partial maximum reaches the running minimum,
// so most pixels touch only a few taps.  The input window is staged once in
// shared memory as int16 (out-of-image / undefined = -32768, which keeps any
// sum with b below every real candidate).
//
// The kernel then picks the smallest T_t = 2 N_t of the plan's ladder,
// records the unit's anchor (the clamp value in the image's own units) and
// appends the unit to the work list of its ladder entry (the tonal kernel is
// specialised per N).  Values outside [img_min, img_max] raise the error flag.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>
#include <type_traits>
#include "fm_dft.cuh"

namespace fm {

constexpr int kRangeNT = 256;
constexpr int kMaxBoundTaps = 128;
constexpr int16_t kWinUndef = -32768;
constexpr int kTapPadB = -(1 << 20);  // padding taps: never win a max
constexpr int kRangeSmemMax = 160 * 1024;

struct RangeArgs {
  const void* img;
  const uint8_t* img_def;
  int H, W;
  int two_d;
  int DY, DX, QY, QX;
  int win_y, win_x;       // input window extent of one unit
  int my, mx;             // SE extent (rows / columns of a split's window beyond its outputs)
  int tiles_x;            // 2-D tile grid width
  int units;              // units per image
  int unit0;              // first unit of this launch
  int unit_step_x;        // 1-D: output pixels per unit (tiles_per_unit * QX)
  int OH, OW;             // output extent (valid outputs of the last units are clipped)
  int enc_sign, enc_bias; // v = enc_sign * f + enc_bias in [0, vmax] (plan-wide)
  int vmax;
  int lr_se;              // se_max - se_min
  int cy, cx;             // SE centre, for the seed pixels
  int splits;             // CTAs per unit (output rows, or columns in 1-D, split between them)
  int skip0;              // the conv path may skip plane 0 of "full" units
  int warp_sync;          // bound taps walked warp-synchronously (else per-lane pixel queues)
  int ntaps;              // 0: no clamp; else a multiple of 8 (padded with kTapPadB taps)
  int flat_taps;          // every bound tap has b - se_min = 0 (flat SE, tap count a multiple of 8)
  int aligned;            // uint8 image rows 16-byte aligned (2-D, no mask): chunk-aligned staging
  const int* ladder;      // ascending N values
  int L;
  int4* unit_param;       // [imgs][units]
  int* bucket_count;      // [L]
  int2* bucket_list;      // [L][cap]
  int cap;
  int* err;
  int* part;              // splits > 1: [imgs*units][8] partial results + arrival count (self-resetting)
  int2 taps[kMaxBoundTaps];  // (offset in the unit window, b - se_min), best first: read from the
                             // constant bank, so a tap costs one add, one LDS and one add-max
};

template <int DT>
__device__ __forceinline__ int range_ld(const void* img, int64_t i) {
  if (DT == 0) return (int)__ldg(reinterpret_cast<const uint8_t*>(img) + i);
  if (DT == 1) return (int)__ldg(reinterpret_cast<const uint16_t*>(img) + i);
  return __ldg(reinterpret_cast<const int32_t*>(img) + i);
}

__device__ __forceinline__ void unit_finish(const RangeArgs& a, const int* lad, int img, int unit, int lo, int hi, int bound) {
  const bool any = lo <= hi;
  int c = any ? lo : 0;
  // bound: INT32_MAX = not computed, INT32_MIN = unknown (no clamp)
  if (any && bound != INT32_MAX && bound != INT32_MIN && (int64_t)bound - a.lr_se > c)
    c = (int)min((int64_t)bound - a.lr_se, (int64_t)hi);
  const int lr = any ? (hi - c) + a.lr_se : a.lr_se;
  int li = a.L - 1;
  for (int i = 0; i < a.L; ++i)
    if (2 * lad[i] >= lr + 1) {
      li = i;
      break;
    }
  // anchor in image units: v = f - anchor (dilation) / anchor - f (erosion)
  const int anchor = a.enc_sign * (c - a.enc_bias);
  // "full": the whole input window lies in the image and has no gaps, so every
  // valid output pairs with every defined SE entry and plane 0 is a constant
  bool full = false;
  if (a.skip0 && a.img_def == nullptr) {
    if (a.two_d) {
      const int ty = unit / a.tiles_x, tx = unit - ty * a.tiles_x;
      const int y0 = ty * a.QY + a.DY, x0 = tx * a.QX + a.DX;
      full = y0 >= 0 && y0 + a.win_y <= a.H && x0 >= 0 && x0 + a.win_x <= a.W;
    } else {
      const int x0 = unit * a.unit_step_x + a.DX;
      full = x0 >= 0 && x0 + a.win_x <= a.W;
    }
  }
  a.unit_param[(size_t)img * a.units + unit] = make_int4(anchor, lad[li], li, (any ? 1 : 0) | (full ? 2 : 0));
  const int slot = atomicAdd(&a.bucket_count[li], 1);
  a.bucket_list[(size_t)li * a.cap + slot] = make_int2(img, unit | (full ? kJobFull : 0));
}

// grid (units_in_launch * splits, images); split s of a unit handles output
// rows [s*QY/S, (s+1)*QY/S) (1-D: columns of the unit) and stages only the
// input rows those outputs read.
// WT: element type of the staged window: int16, or int8 when every encoded value fits 7 bits
// (half the shared memory: more resident CTAs for the clamp-bound walk)
template <int DT, typename WT = int16_t>
__global__ void __launch_bounds__(kRangeNT) range_kernel(const RangeArgs a) {
  extern __shared__ __align__(16) unsigned char swin_raw[];
  WT* swin = reinterpret_cast<WT*>(swin_raw);
  constexpr int kUndef = sizeof(WT) == 1 ? -128 : -32768;   // out-of-image / undefined: below every real candidate
  constexpr int kWMax = sizeof(WT) == 1 ? 127 : 32767;
  constexpr uint32_t kUndefWord = sizeof(WT) == 1 ? 0x80808080u : 0x80008000u;
  __shared__ int red[4][kRangeNT / 32];
  __shared__ int s_lo, s_hi, s_key, s_bound, s_last;
  __shared__ __align__(16) int s_toff[kMaxBoundTaps], s_tb[kMaxBoundTaps];
  __shared__ int s_lad[64];
  constexpr int NW = kRangeNT / 32;
  const int S = a.splits;
  const int lu = blockIdx.x / S, sp = blockIdx.x - lu * S;
  const int unit = a.unit0 + lu, img = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool stage = a.ntaps > 0;
  // geometry: window origin, this split's outputs [j0, j1) and staged window part
  int y0, x0, ny, nx, j0, j1, wy0, wy, wx0, wx;
  if (a.two_d) {
    const int ty = unit / a.tiles_x, tx = unit - ty * a.tiles_x;
    y0 = ty * a.QY + a.DY;
    x0 = tx * a.QX + a.DX;
    ny = min(a.QY, a.OH - ty * a.QY);
    nx = min(a.QX, a.OW - tx * a.QX);
    j0 = (int)((int64_t)sp * a.QY / S);
    j1 = (int)((int64_t)(sp + 1) * a.QY / S);
    wy0 = j0;
    wy = (j1 - j0) + a.my - 1;
    wx0 = 0;
    wx = a.win_x;
  } else {
    y0 = 0;
    x0 = unit * a.unit_step_x + a.DX;
    ny = 1;
    nx = min(a.unit_step_x, a.OW - unit * a.unit_step_x);
    j0 = (int)((int64_t)sp * a.unit_step_x / S);
    j1 = (int)((int64_t)(sp + 1) * a.unit_step_x / S);
    wy0 = 0;
    wy = 1;
    wx0 = j0;
    wx = (j1 - j0) + a.mx - 1;
  }
  if (tid == 0) s_bound = INT32_MAX;

  // ---- stage the window part (int16), min / max of v and the position of the minimum
  int lo = INT32_MAX, hi = INT32_MIN, bad = 0, key = INT32_MAX;
  const int xb = x0 + wx0;  // image column of window column 0
  // chunk-aligned staging (uint8, rows 16-byte aligned, no mask): staged column 0 is the
  // 16-aligned image column xa <= xb, the row stride ws a multiple of 16 -- every aligned
  // 16-pixel chunk of the image lands as two aligned 16-byte shared-memory stores
  const bool fast = DT == 0 && a.aligned && a.img_def == nullptr;
  const int xa = fast ? (xb & ~15) : xb, sh = xb - xa;
  const int ws = fast ? ((wx + 15) & ~15) + 16 : wx;
  for (int i = tid; i < a.ntaps; i += kRangeNT) {
    // host offsets index a window of row stride win_x (= wx in 2-D)
    const int off = a.taps[i].x;
    s_toff[i] = fast ? (off / wx) * ws + (off - (off / wx) * wx) : off;
    s_tb[i] = a.taps[i].y;
  }
  for (int i = tid; i < a.L && i < 64; i += kRangeNT) s_lad[i] = a.ladder[i];
  if (fast) {
    const int cpr = ws >> 4, total = wy * cpr;
    const float inv_cpr = 1.0f / (float)cpr;
    const uint8_t* img8 = reinterpret_cast<const uint8_t*>(a.img) + (int64_t)img * a.H * a.W;
#pragma unroll 2
    for (int it = tid; it < total; it += kRangeNT) {
      const int r = (int)(((float)it + 0.5f) * inv_cpr);
      const int ch = it - r * cpr;
      const int iy = y0 + wy0 + r, xc = xa + 16 * ch;   // W % 16 == 0: a chunk is inside or outside as a whole
      uint32_t pk[8];
      if (iy < 0 || iy >= a.H || xc < 0 || xc >= a.W) {
#pragma unroll
        for (int i = 0; i < 8; ++i) pk[i] = kUndefWord;
      } else {
        const uint4 wv = __ldg(reinterpret_cast<const uint4*>(img8 + (int64_t)iy * a.W + xc));
        const uint32_t wd[4] = {wv.x, wv.y, wv.z, wv.w};
        int v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = a.enc_sign * (int)__byte_perm(wd[e >> 2], 0, 0x4440 + (e & 3)) + a.enc_bias;
        const int c0 = 16 * ch - sh;   // window column of the chunk's first pixel
        int m = INT32_MAX, M = INT32_MIN;
        if (c0 >= 0 && c0 + 16 <= wx) {
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            m = min(m, v[e]);
            M = max(M, v[e]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (c0 + e >= 0 && c0 + e < wx) {
              m = min(m, v[e]);
              M = max(M, v[e]);
            }
        }
        if (m <= M) {
          lo = min(lo, m);
          hi = max(hi, M);
          key = min(key, (min(max(m, 0), 32767) << 16) | ((r * wx + max(c0, 0)) & 0xFFFF));
        }
        if (sizeof(WT) == 1) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            pk[i] = __byte_perm(__byte_perm((uint32_t)v[4 * i], (uint32_t)v[4 * i + 1], 0x0040),
                                __byte_perm((uint32_t)v[4 * i + 2], (uint32_t)v[4 * i + 3], 0x0040), 0x5410);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) pk[i] = __byte_perm((uint32_t)v[2 * i], (uint32_t)v[2 * i + 1], 0x5410);
        }
      }
      if (stage) {
        if (sizeof(WT) == 1) {
          *reinterpret_cast<uint4*>(swin + r * ws + 16 * ch) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(swin + r * ws + 16 * ch);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
    }
    bad = lo <= hi && (lo < 0 || hi > a.vmax);
  } else if (a.img_def == nullptr) {
    // 16-byte vector loads of aligned chunks covering each staged row part;
    // the window is first filled with "undefined" so that only in-image
    // columns need writing
    using T = typename std::conditional<DT == 0, uint8_t, typename std::conditional<DT == 1, uint16_t, int32_t>::type>::type;
    constexpr int EPC = 16 / (int)sizeof(T);
    if (stage) {
      constexpr int EPW = 4 / (int)sizeof(WT);
      const int nw = (wy * wx) / EPW;
      uint32_t* w32 = reinterpret_cast<uint32_t*>(swin);
      for (int i = tid; i < nw; i += kRangeNT) w32[i] = kUndefWord;
      for (int i = nw * EPW + tid; i < wy * wx; i += kRangeNT) swin[i] = (WT)kUndef;
      __syncthreads();
    }
    const int xs = max(xb, 0), xe = min(xb + wx, a.W);
    if (xs < xe) {
      const T* imgT = reinterpret_cast<const T*>(a.img);
      const int cpr = (xe - xs + 2 * EPC - 2) / EPC;  // chunks per row covering [xs, xe) at any alignment
      const int total = wy * cpr;
      const float inv_cpr = 1.0f / (float)cpr;
#pragma unroll 2
      for (int it = tid; it < total; it += kRangeNT) {
        const int r = (int)(((float)it + 0.5f) * inv_cpr);
        const int ch = it - r * cpr;
        const int iy = y0 + wy0 + r;
        if (iy < 0 || iy >= a.H) continue;
        const T* rowp = imgT + ((int64_t)img * a.H + iy) * a.W;
        const uintptr_t first = reinterpret_cast<uintptr_t>(rowp + xs) & ~(uintptr_t)15;
        const uintptr_t cb = first + 16u * (uintptr_t)ch;
        if (cb >= reinterpret_cast<uintptr_t>(rowp + xe)) continue;
        const uint4 wv = __ldg(reinterpret_cast<const uint4*>(cb));
        const int xc0 = (int)((const T*)cb - rowp);  // image column of the chunk's first element
        const uint32_t wd[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int e = 0; e < EPC; ++e) {
          const int x = xc0 + e;
          if (x < xs || x >= xe) continue;
          int f;
          if (DT == 0) f = (int)((wd[e >> 2] >> (8 * (e & 3))) & 0xFFu);
          else if (DT == 1) f = (int)((wd[e >> 1] >> (16 * (e & 1))) & 0xFFFFu);
          else f = (int)wd[e];
          const int v = a.enc_sign * f + a.enc_bias;
          lo = min(lo, v);
          hi = max(hi, v);
          bad |= (v < 0) | (v > a.vmax);
          const int sv = min(max(v, 0), kWMax);
          const int pos = r * wx + (x - xb);
          key = min(key, (sv << 16) | (pos & 0xFFFF));
          if (stage) swin[pos] = (WT)sv;
        }
      }
    }
  } else {
    const int rstep = a.two_d ? NW : 1, cstep = a.two_d ? 32 : kRangeNT;
    for (int r = a.two_d ? warp : 0; r < wy; r += rstep) {
      const int iy = y0 + wy0 + r;
      const bool rok = iy >= 0 && iy < a.H;
      const int64_t rb = ((int64_t)img * a.H + (rok ? iy : 0)) * a.W;
      WT* srow = swin + r * wx;
#pragma unroll 4
      for (int c = a.two_d ? lane : tid; c < wx; c += cstep) {
        const int ix = xb + c;
        int sv = kUndef;
        if (rok && (unsigned)ix < (unsigned)a.W) {
          const int64_t gi = rb + ix;
          if (a.img_def[gi]) {
            const int v = a.enc_sign * range_ld<DT>(a.img, gi) + a.enc_bias;
            lo = min(lo, v);
            hi = max(hi, v);
            bad |= (v < 0) | (v > a.vmax);
            sv = min(max(v, 0), kWMax);
            key = min(key, (sv << 16) | ((r * wx + c) & 0xFFFF));
          }
        }
        if (stage) srow[c] = (WT)sv;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    key = min(key, __shfl_xor_sync(0xffffffffu, key, o));
  }
  if (lane == 0) {
    red[0][warp] = lo;
    red[1][warp] = hi;
    red[2][warp] = bad;
    red[3][warp] = key;
  }
  __syncthreads();
  if (tid == 0) {
    for (int i = 1; i < NW; ++i) {
      lo = min(lo, red[0][i]);
      hi = max(hi, red[1][i]);
      bad |= red[2][i];
      key = min(key, red[3][i]);
    }
    if (bad) atomicOr(a.err, 1);
    s_lo = lo;
    s_hi = hi;
    s_key = key;
  }
  __syncthreads();
  lo = s_lo;
  hi = s_hi;

  // ---- lower bound D of the dilation over this split's outputs (branch and bound)
  const int jy_end = a.two_d ? min(j1, ny) : 1;
  const int jx_beg = a.two_d ? 0 : j0, jx_end = a.two_d ? nx : min(j1, nx);
  const int oy0 = a.two_d ? j0 : 0;  // first output row of the split (window row 0 of swin)
  if (stage && lo <= hi && oy0 < jy_end && jx_beg < jx_end) {
    const int floor_d = lo + a.lr_se;  // D <= floor_d gives no clamp
    {
      // seed: every warp evaluates one pixel exactly (lanes over taps), placed
      // around the part's minimum, where the smallest g is likely
      const int pos = s_key & 0xFFFF;
      const int zr = pos / wx, zc = pos - zr * wx;
      const int sy = (warp & 1) ? 3 : -3, sx = (warp & 2) ? 3 : -3, sc = warp >> 2;
      const int jy = min(max(zr - a.cy + sy * sc, 0), jy_end - 1 - oy0);
      const int jx = min(max(zc - a.cx + sx * sc, 0), jx_end - 1 - (a.two_d ? 0 : wx0));
      const int base = jy * ws + jx + sh;
      int g = INT32_MIN;
      for (int t = lane; t < a.ntaps; t += 32) g = max(g, (int)swin[base + s_toff[t]] + s_tb[t]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) g = max(g, __shfl_xor_sync(0xffffffffu, g, o));
      if (lane == 0) atomicMin(&s_bound, g);
    }
    __syncthreads();
    volatile int* vb = &s_bound;
    // breakpoints: D >= hi + 2 lr_se - 2 N + 1 lets the unit use ladder length N
    auto level_of = [&](int d) -> int {
      for (int i = 0; i < a.L; ++i) {
        const int th = hi + 2 * a.lr_se - 2 * s_lad[i] + 1;
        if (th <= d) return th;
      }
      return INT32_MIN;
    };
    // every lane walks its own queue of pixels (q += kRangeNT), one 8-tap group
    // per iteration, so lanes that stop early do not wait for the slowest one
    const int rows = jy_end - oy0, cols = jx_end - jx_beg;
    const int npx = rows * cols;
    const int xoff = a.two_d ? 0 : jx_beg - wx0;
    // q -> (jy, jx) with a high multiply by ceil(2^32/cols): exact for q < 2^16
    const uint32_t cmagic = cols > 1 ? (uint32_t)((0x100000000ull + cols - 1) / (uint64_t)cols) : 0u;
    auto base_of = [&](int q) {
      const int jy = cmagic ? (int)__umulhi((uint32_t)q, cmagic) : q;
      return jy * ws + (q - jy * cols) + xoff + sh;
    };
    // A pixel may stop as soon as g reaches the breakpoint level below the
    // running minimum: only the interval between ladder breakpoints that D
    // falls into changes the unit's tonal length.
    if (a.warp_sync) {
      // warps take 32 consecutive pixels and walk the taps together (same tap,
      // neighbouring pixels: conflict-free shared-memory reads); finished lanes idle
      for (int qb = warp * 32; qb < npx; qb += kRangeNT) {
        const int q = qb + lane;
        const bool act = q < npx;
        const int base = act ? base_of(q) : 0;
        int g = INT32_MIN, t = 0, seen = INT32_MIN, lvl = INT32_MIN;
        bool done = !act, stop_all = false;
        while (true) {
          const int bnd = __shfl_sync(0xffffffffu, *vb, 0);
          if (bnd != seen) {
            seen = bnd;
            lvl = level_of(bnd);
          }
          if (lvl <= floor_d) {
            stop_all = true;
            break;
          }
          if (!done && g >= lvl) done = true;
          if (!done && t >= a.ntaps) {
            if (g < bnd) atomicMin(&s_bound, g);
            done = true;
          }
          if (__all_sync(0xffffffffu, done)) break;
          if (!done) {
            const int4 o0 = *reinterpret_cast<const int4*>(s_toff + t), o1 = *reinterpret_cast<const int4*>(s_toff + t + 4);
            const int4 b0 = *reinterpret_cast<const int4*>(s_tb + t), b1 = *reinterpret_cast<const int4*>(s_tb + t + 4);
            g = max(g, (int)swin[base + o0.x] + b0.x);
            g = max(g, (int)swin[base + o0.y] + b0.y);
            g = max(g, (int)swin[base + o0.z] + b0.z);
            g = max(g, (int)swin[base + o0.w] + b0.w);
            g = max(g, (int)swin[base + o1.x] + b1.x);
            g = max(g, (int)swin[base + o1.y] + b1.y);
            g = max(g, (int)swin[base + o1.z] + b1.z);
            g = max(g, (int)swin[base + o1.w] + b1.w);
          }
          t += 8;
        }
        if (stop_all) break;
      }
    } else {
      const bool flat_taps = a.flat_taps != 0;
      int q = tid;
      if (q < npx) {
        int base = base_of(q), t = 0, g = INT32_MIN, seen = INT32_MIN, lvl = INT32_MIN;
        while (true) {
          const int bnd = *vb;
          if (bnd != seen) {
            seen = bnd;
            lvl = level_of(bnd);
          }
          if (lvl <= floor_d) break;  // no clamp possible: stop
#ifdef FM_RANGE_BRANCHY
          if (t >= a.ntaps || g >= lvl) {
            if (t >= a.ntaps && g < bnd) atomicMin(&s_bound, g);
            q += kRangeNT;
            if (q >= npx) break;
            base = base_of(q);
            t = 0;
            g = INT32_MIN;
          }
#else
          {
            // advance to the lane's next pixel by selects (no divergent region per iteration);
            // only the rare new minimum branches
            const bool all_taps = t >= a.ntaps, adv = all_taps || g >= lvl;
            if (all_taps && g < bnd) atomicMin(&s_bound, g);
            const int qn = q + kRangeNT;
            if (adv && qn >= npx) break;
            const int basen = base_of(min(qn, npx - 1));
            q = adv ? qn : q;
            base = adv ? basen : base;
            t = adv ? 0 : t;
            g = adv ? INT32_MIN : g;
          }
#endif
          const int4 o0 = *reinterpret_cast<const int4*>(s_toff + t), o1 = *reinterpret_cast<const int4*>(s_toff + t + 4);
          if (flat_taps) {
            // flat SE, no padding taps: every tap's b - se_min is 0 (no table loads, no adds)
            g = max(g, max(max((int)swin[base + o0.x], (int)swin[base + o0.y]), max((int)swin[base + o0.z], (int)swin[base + o0.w])));
            g = max(g, max(max((int)swin[base + o1.x], (int)swin[base + o1.y]), max((int)swin[base + o1.z], (int)swin[base + o1.w])));
          } else {
            const int4 b0 = *reinterpret_cast<const int4*>(s_tb + t), b1 = *reinterpret_cast<const int4*>(s_tb + t + 4);
            g = max(g, (int)swin[base + o0.x] + b0.x);
            g = max(g, (int)swin[base + o0.y] + b0.y);
            g = max(g, (int)swin[base + o0.z] + b0.z);
            g = max(g, (int)swin[base + o0.w] + b0.w);
            g = max(g, (int)swin[base + o1.x] + b1.x);
            g = max(g, (int)swin[base + o1.y] + b1.y);
            g = max(g, (int)swin[base + o1.z] + b1.z);
            g = max(g, (int)swin[base + o1.w] + b1.w);
          }
          t += 8;
        }
      }
    }
    __syncthreads();
  }
  // the unit's lower bound: the breakpoint level of the minimum (INT32_MIN: no clamp)
  int bound = INT32_MAX;
  if (stage && lo <= hi && s_bound != INT32_MAX) {
    bound = INT32_MIN;
    for (int i = 0; i < a.L; ++i) {
      const int th = hi + 2 * a.lr_se - 2 * s_lad[i] + 1;
      if (th <= s_bound) {
        bound = th > lo + a.lr_se ? th : INT32_MIN;
        break;
      }
    }
  }

  if (S == 1) {
    if (tid == 0) unit_finish(a, a.L <= 64 ? s_lad : a.ladder, img, unit, lo, hi, bound);
    return;
  }
  // ---- combine the splits: the last CTA to arrive finishes the unit
  if (tid == 0) {
    int* pr = a.part + ((size_t)img * a.units + unit) * 8;
    atomicMin(pr + 0, lo);
    atomicMax(pr + 1, hi);
    atomicMin(pr + 2, bound);
    __threadfence();
    s_last = atomicAdd(pr + 3, 1) == S - 1;
  }
  __syncthreads();
  if (s_last && tid == 0) {
    __threadfence();
    int* pr = a.part + ((size_t)img * a.units + unit) * 8;
    const int glo = atomicExch(pr + 0, INT32_MAX);
    const int ghi = atomicExch(pr + 1, INT32_MIN);
    const int gb = atomicExch(pr + 2, INT32_MAX);
    atomicExch(pr + 3, 0);
    unit_finish(a, a.L <= 64 ? s_lad : a.ladder, img, unit, glo, ghi, gb);
  }
}

// per-ladder unit counts -> mapped host memory (read by the host after an event)
__global__ void publish_counts(const int* __restrict__ counts, int* host_counts, int L) {
  for (int i = threadIdx.x; i < L; i += blockDim.x) reinterpret_cast<volatile int*>(host_counts)[i] = counts[i];
  __threadfence_system();
}

}  // namespace fm
