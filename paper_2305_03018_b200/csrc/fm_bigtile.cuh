// fm_bigtile.cuh — 256x256 overlap-save tiles for wide structuring elements.
//
// A 256^2 complex64 tile (512 KB) does not fit one SM, so the spatial FFT
// convolution of a (tile, plane) is split into three kernels that stream the
// tile through an HBM scratch S[item][256][256] (item = image, tile, plane):
//   big_rows_fwd  : encode w_T^{k v} + forward x FFT (radix 16x16) of 32 rows
//   big_cols      : forward y FFT of 32 columns, product with the SE spectrum,
//                   inverse y FFT; rows of the valid window written back
//   big_rows_inv  : inverse x FFT of 32 valid rows, valid columns -> Chat
// With a 101-wide SE the valid window grows from 28^2 (128 tile) to 156^2, so
// the FFT work per output pixel drops ~5x for about 1.8 MB of HBM traffic per
// (tile, plane).  The SE spectrum is computed by the same kernels (SPEC mode)
// and stored in the column kernel's thread order.  Positions after the forward
// passes are the four-step digit-permuted frequencies, as in fm_tile.cuh.
#pragma once
#include "fm_tile.cuh"

namespace fm {

constexpr int kBig = 256;        // tile edge
constexpr int kBigR = 16;        // 256 = 16 x 16 per axis
constexpr int kBigRows = 32;     // rows per row-kernel CTA
constexpr int kBigCols = 16;     // columns per column-kernel CTA
constexpr int kBigNT = 256;      // row kernels
constexpr int kBigColsNT = 128;  // column kernel: one y item per thread

struct BigArgs {
  // image batch (CONV) or SE (SPEC)
  const void* img;
  const uint8_t* img_def;
  const int32_t* se_vals;
  const uint8_t* se_def;
  int img_dtype;
  int H, W, OH, OW, DY, DX, QY, QX, my, mx, tiles_x;
  int enc_sign, enc_bias;     // SPEC: v = b + enc_bias
  int T, K;                   // SPEC launch: the ladder entry
  const int4* unit_param;     // CONV: [imgs][units]
  int units;
  int unit0, upl, nu;         // first unit, slots per image, units in this launch
  int lu0, nub;               // this launch's unit batch: launch-local units [lu0, lu0 + nub), grid z = imgs * nub
  int K_max;
  float2* S;                  // [imgs][units][K_max][256][256] (CONV) or [K][256][256] (SPEC)
  const float4* spec;         // CONV: ladder base; SPEC: output
  const int64_t* spec_off;    // [ladder] float4 offsets
  float spec_scale;
  float2* chat;               // [imgs][units][K_max][wpx]
  int wpx;
  int* err;
  int pair;                   // Nyquist planes of neighbouring units share one complex transform
};

// Nyquist-plane pairing.  Plane k = N of a unit (T = 2N) is REAL: w_T^{N v} = (-1)^v, and so is
// the SE's plane N.  Two launch-local neighbours (lu even, lu + 1) with the same tonal length
// therefore share ONE complex transform: z = a_lu + i a_{lu+1}, and z (*) h = a_lu (*) h +
// i a_{lu+1} (*) h splits into real and imaginary part because h is real.  The even unit's
// CTAs carry the pair, the odd unit's exit.  (c4: nearly every unit has N = 1 and, being
// "full", only that plane -- the three kernels do half the work.)
// returns 0: not paired, 1: carries the pair (partner = lu + 1), 2: carried by lu - 1 (exit)
__device__ __forceinline__ int big_pair_role(const BigArgs& a, int img, int lu, int k, const int4& up, int4& upp) {
  if (!a.pair || k != up.y) return 0;
  const int lup = lu ^ 1;
  if (lup >= a.nu) return 0;
  upp = a.unit_param[(size_t)img * a.units + a.unit0 + lup];
  if (upp.y != up.y) return 0;
  return (lu & 1) ? 2 : 1;
}

// ------------------------------------------------------------------ rows (x axis)
// CTA = 32 rows x 256 columns of one (image, tile, plane); 8 warps, 4 rows each.
template <bool FWD, bool SPEC>
__global__ void __launch_bounds__(kBigNT, 2) big_rows_kernel(const BigArgs a) {
  constexpr int PX = kBig, RS = PX + 2, R1 = kBigR, R2 = kBigR;
  constexpr int RPW = 4;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* buf = reinterpret_cast<float2*>(smem_raw);
  uint16_t* tv = reinterpret_cast<uint16_t*>(smem_raw + kBigRows * RS * 8);
  const uint32_t* tv32 = reinterpret_cast<const uint32_t*>(tv);
  float4* twx = reinterpret_cast<float4*>(smem_raw + kBigRows * RS * 8 + kBigRows * PX * 2);
  uint16_t* tv2 = reinterpret_cast<uint16_t*>(smem_raw + kBigRows * RS * 8 + kBigRows * PX * 2 + (kBigR / 2) * (kBigR + 1) * 16);
  const uint32_t* tv2_32 = reinterpret_cast<const uint32_t*>(tv2);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k = blockIdx.y;
  const int lu = SPEC ? 0 : a.lu0 + (int)(blockIdx.z % a.nub);
  const int unit = SPEC ? 0 : a.unit0 + lu;
  const int img = SPEC ? 0 : (int)(blockIdx.z / a.nub);
  int T = a.T, K = a.K, enc_bias = a.enc_bias, enc_bias2 = 0;
  bool paired = false;
  if constexpr (!SPEC) {
    const int4 up = a.unit_param[(size_t)img * a.units + unit];
    K = up.y + 1;
    T = 2 * up.y;
    enc_bias = a.enc_sign > 0 ? -up.x : up.x;
    if (k == 0 && (up.w & 2)) return;   // plane 0 of a full unit: the tonal pass knows it
    if (k < K) {
      int4 upp;
      const int role = big_pair_role(a, img, lu, k, up, upp);
      if (role == 2) return;
      paired = role == 1;
      enc_bias2 = a.enc_sign > 0 ? -upp.x : upp.x;
    }
  }
  if (k >= K) return;
  const int row0 = FWD ? blockIdx.x * kBigRows : (a.my - 1) + blockIdx.x * kBigRows;
  if (row0 >= kBig) return;
  const int ty = unit / max(a.tiles_x, 1), tx = unit - ty * max(a.tiles_x, 1);
  float2* Sitem = a.S + (((size_t)img * a.upl + lu) * a.K_max + k) * (size_t)(kBig * kBig);
  if constexpr (SPEC) Sitem = a.S + (size_t)k * (kBig * kBig);

  auto ld2 = [&](int y, int x) -> float4 { return *reinterpret_cast<const float4*>(buf + y * RS + x); };
  auto st2 = [&](int y, int x, float2 p, float2 q) {
    *reinterpret_cast<float4*>(buf + y * RS + x) = make_float4(p.x, p.y, q.x, q.y);
  };
  // twiddle pairs (W^{n2 k1}, W^{(n2+1) k1}), stride R1+1
  for (int j = tid; j < (R2 / 2) * (R1 + 1); j += kBigNT) {
    const int n2p = j / (R1 + 1), k1 = j - n2p * (R1 + 1), n2 = 2 * n2p;
    const float2 w0 = c_tw[TwOff<PX>::v + (n2 * k1) % PX];
    const float2 w1 = c_tw[TwOff<PX>::v + ((n2 + 1) * k1) % PX];
    twx[j] = make_float4(w0.x, w0.y, w1.x, w1.y);
  }

  if constexpr (FWD) {
    // ---- stage tonal indices of rows [row0, row0+32) of the tile's input window
    int bad = 0;
    if constexpr (SPEC) {
      for (int p = tid; p < kBigRows * PX; p += kBigNT) {
        const int py = row0 + p / PX, px = p % PX;
        uint16_t t = kSent;
        if (py < a.my && px < a.mx) {
          const int si = py * a.mx + px;
          if (a.se_def == nullptr || a.se_def[si]) t = (uint16_t)(a.se_vals[si] + a.enc_bias);
        }
        tv[p] = t;
      }
    } else {
      // batches of GB independent (predicated) loads per thread, then the
      // conversions: the image reads overlap instead of paying one latency each
      constexpr int IT = kBigRows * PX / kBigNT, GB = 16;
      static_assert(IT % GB == 0, "staging split");
      auto stage_unit = [&](int uty, int utx, int bias, uint16_t* tvd) {
        if (a.img_dtype == 0 && a.img_def == nullptr) {
          // uint8 images without a mask: 16-byte loads of the aligned chunks that cover each
          // row part inside the image (one load per 16 pixels instead of one per pixel)
          const int ixb = utx * a.QX + a.DX;              // image column of tile column 0
          const int xs = max(ixb, 0), xe = min(ixb + PX, a.W);
          for (int i = tid; i < kBigRows * PX / 2; i += kBigNT)
            reinterpret_cast<uint32_t*>(tvd)[i] = (uint32_t)kSent | ((uint32_t)kSent << 16);
          __syncthreads();
          if (xs < xe) {
            const uint8_t* base = reinterpret_cast<const uint8_t*>(a.img);
            constexpr int CPR = PX / 16 + 1;               // chunks covering 256 columns at any alignment
#pragma unroll 1
            for (int it = tid; it < kBigRows * CPR; it += kBigNT) {
              const int r = it / CPR, ch = it - r * CPR;
              const int iy = uty * a.QY + a.DY + row0 + r;
              if (iy < 0 || iy >= a.H) continue;
              const uint8_t* rowp = base + ((int64_t)img * a.H + iy) * a.W;
              const uintptr_t first = reinterpret_cast<uintptr_t>(rowp + xs) & ~(uintptr_t)15;
              const uintptr_t cb = first + 16u * (uintptr_t)ch;
              if (cb >= reinterpret_cast<uintptr_t>(rowp + xe)) continue;
              const uint4 wv = __ldg(reinterpret_cast<const uint4*>(cb));
              const int xc0 = (int)(reinterpret_cast<const uint8_t*>(cb) - rowp);
              const uint32_t wd[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                const int x = xc0 + e;
                if (x < xs || x >= xe) continue;
                const int f = (int)((wd[e >> 2] >> (8 * (e & 3))) & 0xFFu);
                const int v = max(a.enc_sign * f + bias, 0);
                if (v >= T) bad = 1;
                else tvd[r * PX + (x - ixb)] = (uint16_t)v;
              }
            }
          }
          return;
        }
#pragma unroll 1
        for (int g0 = 0; g0 < IT; g0 += GB) {
          int raw[GB];
          bool ok[GB];
#pragma unroll
          for (int u = 0; u < GB; ++u) {
            const int p = tid + (g0 + u) * kBigNT;
            const int py = row0 + p / PX, px = p % PX;
            const int iy = uty * a.QY + a.DY + py, ix = utx * a.QX + a.DX + px;
            ok[u] = iy >= 0 && iy < a.H && ix >= 0 && ix < a.W;
            raw[u] = 0;
            if (ok[u]) {
              const int64_t gi = ((int64_t)img * a.H + iy) * a.W + ix;
              raw[u] = load_img(a.img, a.img_dtype, gi);
              if (a.img_def != nullptr) ok[u] = a.img_def[gi] != 0;
            }
          }
#pragma unroll
          for (int u = 0; u < GB; ++u) {
            uint16_t t = kSent;
            if (ok[u]) {
              // values below the unit's clamp level encode as the clamp (fm_range.cuh)
              const int v = max(a.enc_sign * raw[u] + bias, 0);
              if (v >= T) bad = 1;
              else t = (uint16_t)v;
            }
            tvd[tid + (g0 + u) * kBigNT] = t;
          }
        }
      };
      stage_unit(ty, tx, enc_bias, tv);
      if (paired) {
        const int u2 = unit + 1, ty2 = u2 / max(a.tiles_x, 1);
        stage_unit(ty2, u2 - ty2 * max(a.tiles_x, 1), enc_bias2, tv2);
      }
    }
    if (!SPEC && bad) atomicOr(a.err, 1);
    __syncthreads();
    const uint32_t magicT = (uint32_t)(0x100000000ull / (uint64_t)T);
    const float two_pi_over_T = 6.28318530717958647692f / (float)T;
    auto enc = [&](uint32_t t) -> float2 {
      const uint32_t n = (uint32_t)k * t;
      uint32_t r = n - __umulhi(n, magicT) * (uint32_t)T;
      r = (r >= (uint32_t)T) ? r - (uint32_t)T : r;
      const int rr = (2 * r > (uint32_t)T) ? (int)r - T : (int)r;
      float sn, cs;
      __sincosf((float)rr * two_pi_over_T, &sn, &cs);
      const bool live = t != kSent;
      return make_float2(live ? cs : 0.f, live ? -sn : 0.f);
    };
    // ---- x pass A (encode): item (row, n2 pair), one per lane
    {
      const int y = warp * RPW + lane % RPW, n2 = 2 * (lane / RPW);
      float2 wa[R1], wb[R1];
      if (!SPEC && paired) {
        // Nyquist plane of two units: (-1)^v of this unit + i (-1)^v of its neighbour
        auto nyq = [](uint32_t t) -> float { return t == kSent ? 0.f : ((t & 1u) ? -1.f : 1.f); };
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) {
          const uint32_t tt = tv32[(y * PX + n2 + R2 * n1) / 2], t2 = tv2_32[(y * PX + n2 + R2 * n1) / 2];
          wa[n1] = make_float2(nyq(tt & 0xFFFFu), nyq(t2 & 0xFFFFu));
          wb[n1] = make_float2(nyq(tt >> 16), nyq(t2 >> 16));
        }
      } else {
#pragma unroll
        for (int n1 = 0; n1 < R1; ++n1) {
          const uint32_t tt = tv32[(y * PX + n2 + R2 * n1) / 2];
          wa[n1] = enc(tt & 0xFFFFu);
          wb[n1] = enc(tt >> 16);
        }
      }
      dft<R1, false>(wa);
      dft<R1, false>(wb);
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) {
        float2 za = wa[k1], zb = wb[k1];
        if (k1 != 0) {
          const float4 w = twx[(n2 / 2) * (R1 + 1) + k1];
          za = cmul(za, make_float2(w.x, w.y));
          zb = cmul(zb, make_float2(w.z, w.w));
        }
        st2(y, n2 + R2 * k1, za, zb);
      }
    }
    __syncwarp();
    // ---- x pass B: items (row, k1), two per lane; result rows -> S
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const int i = lane + 32 * g;
      const int y = warp * RPW + i % RPW, k1 = i / RPW;
      float2 w[R2];
#pragma unroll
      for (int q = 0; q < R2 / 2; ++q) {
        const float4 p = ld2(y, 2 * q + R2 * k1);
        w[2 * q] = make_float2(p.x, p.y);
        w[2 * q + 1] = make_float2(p.z, p.w);
      }
      dft<R2, false>(w);
#pragma unroll
      for (int q = 0; q < R2 / 2; ++q) st2(y, 2 * q + R2 * k1, w[2 * q], w[2 * q + 1]);
    }
    __syncthreads();
    // coalesced row stores (positions = permuted frequencies)
    for (int i = tid; i < kBigRows * (PX / 2); i += kBigNT) {
      const int y = i / (PX / 2), xp = i % (PX / 2);
      reinterpret_cast<float4*>(Sitem + (size_t)(row0 + y) * kBig)[xp] = ld2(y, 2 * xp);
    }
  } else {
    // ---- inverse: load valid rows, x pass B^-1, x pass A^-1, store valid columns
    const int nrows = min(kBigRows, kBig - row0);
#pragma unroll 4
    for (int i = tid; i < kBigRows * (PX / 2); i += kBigNT) {
      const int y = i / (PX / 2), xp = i % (PX / 2);
      if (y < nrows) cp_async16(buf + y * RS + 2 * xp, reinterpret_cast<const float4*>(Sitem + (size_t)(row0 + y) * kBig) + xp);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      const int i = lane + 32 * g;
      const int y = warp * RPW + i % RPW, k1 = i / RPW;
      float2 w[R2];
#pragma unroll
      for (int q = 0; q < R2 / 2; ++q) {
        const float4 p = ld2(y, 2 * q + R2 * k1);
        w[2 * q] = make_float2(p.x, p.y);
        w[2 * q + 1] = make_float2(p.z, p.w);
      }
      dft<R2, true>(w);
#pragma unroll
      for (int q = 0; q < R2 / 2; ++q) st2(y, 2 * q + R2 * k1, w[2 * q], w[2 * q + 1]);
    }
    __syncwarp();
    {
      const int y = warp * RPW + lane % RPW, n2 = 2 * (lane / RPW);
      float2 wa[R1], wb[R1];
#pragma unroll
      for (int k1 = 0; k1 < R1; ++k1) {
        const float4 p = ld2(y, n2 + R2 * k1);
        wa[k1] = make_float2(p.x, p.y);
        wb[k1] = make_float2(p.z, p.w);
        if (k1 != 0) {
          const float4 w = twx[(n2 / 2) * (R1 + 1) + k1];
          wa[k1] = cmulc(wa[k1], make_float2(w.x, w.y));
          wb[k1] = cmulc(wb[k1], make_float2(w.z, w.w));
        }
      }
      dft<R1, true>(wa);
      dft<R1, true>(wb);
#pragma unroll
      for (int n1 = 0; n1 < R1; ++n1) st2(y, n2 + R2 * n1, wa[n1], wb[n1]);
    }
    __syncthreads();
    // valid window store: tile row ty_row = row0 + y (>= my-1), columns x >= mx-1
    float2* dst = a.chat + (((size_t)img * a.upl + lu) * a.K_max + k) * (size_t)a.wpx;
    const int vx = kBig - (a.mx - 1);   // valid columns per row
    for (int i = tid; i < kBigRows * vx; i += kBigNT) {
      const int y = i / vx, c = i - (i / vx) * vx;
      const int row = row0 + y;
      if (y >= nrows) continue;
      const int oy = ty * a.QY + row - (a.my - 1), ox = tx * a.QX + c;
      const float2 v = buf[y * RS + (a.mx - 1) + c];
      if (oy < a.OH && ox < a.OW) dst[(size_t)(row - (a.my - 1)) * a.QX + c] = paired ? make_float2(v.x, 0.f) : v;
      if (paired) {
        // the neighbour's plane is the imaginary part; its own tile position bounds the store
        const int u2 = unit + 1, ty2 = u2 / max(a.tiles_x, 1), tx2 = u2 - ty2 * max(a.tiles_x, 1);
        const int oy2 = ty2 * a.QY + row - (a.my - 1), ox2 = tx2 * a.QX + c;
        if (oy2 < a.OH && ox2 < a.OW)
          (dst + (size_t)a.K_max * (size_t)a.wpx)[(size_t)(row - (a.my - 1)) * a.QX + c] = make_float2(v.y, 0.f);
      }
    }
  }
}

// ------------------------------------------------------------------ columns (y axis)
// CTA = 256 rows x 16 columns (8 column pairs) of one (image, tile, plane), 128 threads.
// y pass A items (xp, n2), y pass B items (xp, k1): one per thread each.
template <bool SPEC>
__global__ void __launch_bounds__(kBigColsNT, 3) big_cols_kernel(const BigArgs a) {
  constexpr int PY = kBig, PXC = kBigCols, RS = PXC + 2, R1 = kBigR, R2 = kBigR, XP = PXC / 2;
  constexpr int SQ = R2;  // float4 (pairs) per thread in y pass B
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* buf = reinterpret_cast<float2*>(smem_raw);
  float4* sbuf = reinterpret_cast<float4*>(smem_raw + PY * RS * 8);

  const int tid = threadIdx.x;
  const int cb = blockIdx.x, k = blockIdx.y;
  const int lu = SPEC ? 0 : a.lu0 + (int)(blockIdx.z % a.nub);
  const int unit = SPEC ? 0 : a.unit0 + lu;
  const int img = SPEC ? 0 : (int)(blockIdx.z / a.nub);
  int K = a.K;
  const float4* spec_plane = nullptr;
  if constexpr (!SPEC) {
    const int4 up = a.unit_param[(size_t)img * a.units + unit];
    K = up.y + 1;
    if (k >= K || (k == 0 && (up.w & 2))) return;   // past the unit's planes / known plane 0
    {
      int4 upp;
      if (big_pair_role(a, img, lu, k, up, upp) == 2) return;   // carried by the neighbour's CTAs
    }
    spec_plane = a.spec + a.spec_off[up.z] + ((size_t)k * (kBig / kBigCols) + cb) * (SQ * kBigColsNT);
    // the product's spectrum chunk streams in while the forward passes run
#pragma unroll
    for (int q = 0; q < SQ; ++q) cp_async16(sbuf + q * kBigColsNT + tid, spec_plane + q * kBigColsNT + tid);
    cp_async_commit();
  }
  float2* Sitem = SPEC ? a.S + (size_t)k * (kBig * kBig)
                       : a.S + (((size_t)img * a.upl + lu) * a.K_max + k) * (size_t)(kBig * kBig);
  auto ld2 = [&](int y, int x) -> float4 { return *reinterpret_cast<const float4*>(buf + y * RS + x); };
  auto st2 = [&](int y, int x, float2 p, float2 q) {
    *reinterpret_cast<float4*>(buf + y * RS + x) = make_float4(p.x, p.y, q.x, q.y);
  };
  // load 256 rows x 16 columns: all async copies in flight at once
#pragma unroll 4
  for (int i = tid; i < PY * XP; i += kBigColsNT) {
    const int y = i / XP, xp = i % XP;
    cp_async16(buf + y * RS + 2 * xp, reinterpret_cast<const float4*>(Sitem + (size_t)y * kBig + cb * PXC) + xp);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  // ---- forward y pass A: item (xp, n2)
  {
    const int xp = tid % XP, n2 = tid / XP;
    float2 wa[R1], wb[R1];
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) {
      const float4 p = ld2(n2 + R2 * n1, 2 * xp);
      wa[n1] = make_float2(p.x, p.y);
      wb[n1] = make_float2(p.z, p.w);
    }
    dft<R1, false>(wa);
    dft<R1, false>(wb);
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      float2 za = wa[k1], zb = wb[k1];
      if (k1 != 0) {
        const float2 w = c_tw[TwOff<PY>::v + n2 * k1];
        za = cmul(za, w);
        zb = cmul(zb, w);
      }
      st2(n2 + R2 * k1, 2 * xp, za, zb);
    }
  }
  __syncthreads();
  // ---- forward y pass B (+ product + inverse y pass B): item (xp, k1)
  {
    const int xp = tid % XP, k1 = tid / XP;
    float2 wa[R2], wb[R2];
#pragma unroll
    for (int n2 = 0; n2 < R2; ++n2) {
      const float4 p = ld2(n2 + R2 * k1, 2 * xp);
      wa[n2] = make_float2(p.x, p.y);
      wb[n2] = make_float2(p.z, p.w);
    }
    dft<R2, false>(wa);
    dft<R2, false>(wb);
    if constexpr (SPEC) {
      float4* so = const_cast<float4*>(a.spec) + ((size_t)k * (kBig / kBigCols) + cb) * (SQ * kBigColsNT);
      const float s = a.spec_scale;
#pragma unroll
      for (int q = 0; q < SQ; ++q) so[q * kBigColsNT + tid] = make_float4(wa[q].x * s, wa[q].y * s, wb[q].x * s, wb[q].y * s);
    } else {
      cp_async_wait<0>();
#pragma unroll
      for (int q = 0; q < SQ; ++q) {
        const float4 s = sbuf[q * kBigColsNT + tid];
        wa[q] = cmul(wa[q], make_float2(s.x, s.y));
        wb[q] = cmul(wb[q], make_float2(s.z, s.w));
      }
      dft<R2, true>(wa);
      dft<R2, true>(wb);
#pragma unroll
      for (int n2 = 0; n2 < R2; ++n2) st2(n2 + R2 * k1, 2 * xp, wa[n2], wb[n2]);
    }
  }
  if constexpr (SPEC) return;
  __syncthreads();
  // ---- inverse y pass A: item (xp, n2)
  {
    const int xp = tid % XP, n2 = tid / XP;
    float2 wa[R1], wb[R1];
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) {
      const float4 p = ld2(n2 + R2 * k1, 2 * xp);
      wa[k1] = make_float2(p.x, p.y);
      wb[k1] = make_float2(p.z, p.w);
      if (k1 != 0) {
        const float2 w = c_tw[TwOff<PY>::v + n2 * k1];
        wa[k1] = cmulc(wa[k1], w);
        wb[k1] = cmulc(wb[k1], w);
      }
    }
    dft<R1, true>(wa);
    dft<R1, true>(wb);
#pragma unroll
    for (int n1 = 0; n1 < R1; ++n1) st2(n2 + R2 * n1, 2 * xp, wa[n1], wb[n1]);
  }
  __syncthreads();
  // store the valid rows back (row-inverse kernel reads rows >= my-1)
  for (int i = tid; i < PY * XP; i += kBigColsNT) {
    const int y = i / XP, xp = i % XP;
    if (y < a.my - 1) continue;
    reinterpret_cast<float4*>(Sitem + (size_t)y * kBig + cb * PXC)[xp] = ld2(y, 2 * xp);
  }
}

constexpr int kBigRowsSmem = kBigRows * (kBig + 2) * 8 + 2 * kBigRows * kBig * 2 + (kBigR / 2) * (kBigR + 1) * 16;
constexpr int kBigColsSmem = kBig * (kBigCols + 2) * 8 + kBigR * kBigColsNT * 16;

}  // namespace fm
