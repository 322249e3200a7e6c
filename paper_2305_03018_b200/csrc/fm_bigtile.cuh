// fm_bigtile.cuh — 256x256 overlap-save tiles for wide structuring elements.
//
// A 256^2 complex64 tile (512 KB) does not fit one SM, so the spatial FFT
// convolution of a (tile, plane) is split into three kernels that stream the
// tile through an HBM scratch S[item][256][256] (item = image, tile, plane):
//   big_rows_fwd  : encode w_T^{k v} + forward x FFT (radix 16x16) of 32 rows
//   big_cols      : forward y FFT of 16 columns, product with the SE spectrum,
//                   inverse y FFT; rows of the valid window written back
//   big_rows_inv  : inverse x FFT of 32 valid rows, valid columns -> Chat
// Every thread owns ONE 16-point transform per pass (512 / 256 threads per CTA, <= 64 / 80
// registers): twice the resident warps of the earlier two-items-per-thread kernels, which
// ran at IPC ~1.4 per SM.  Row kernels keep a row as [k1][17] (17-stride: both passes'
// 64-bit accesses are conflict-free).
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
constexpr int kBigNT = 512;      // row kernels: one 16-point item per thread and pass
constexpr int kBigColsNT = 256;  // column kernel: one 16-point item per thread and pass
constexpr int kBigRS = kBigR * (kBigR + 1);   // row kernels: row stride of the [k1][17] layout (float2)
constexpr int kBigTvLd = kBig + 16;           // row stride of the staged tonal indices (chunk-aligned staging)

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
  // compact job list (big_jobs_kernel): grid (blocks, y, z) -> job y + z * gridDim.y = (image,
  // launch-local unit | plane << 16); nullptr: grid y = plane, z = unit x image
  const int2* jobs;
  const int* njobs;
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

// The live (image, unit, plane) items of a launch, compacted.  In the plain (plane, unit x image)
// grid a CTA whose item does not exist (planes past the unit's tonal length, plane 0 of a "full"
// unit, the Nyquist plane of a unit carried by its neighbour) holds a CTA slot with 70-100 KB of
// shared memory until its unit_param load returns: at c4 five of six CTAs were such exits, 12-20 %
// of the three kernels' warp samples.
__global__ void big_jobs_kernel(const BigArgs a, int n_imgs, int2* jobs, int* njobs, int cap) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_imgs * a.nu) return;
  const int img = i / a.nu, lu = i - img * a.nu;
  const int4 up = a.unit_param[(size_t)img * a.units + a.unit0 + lu];
  const int N = up.y, k0 = (up.w & 2) ? 1 : 0;
  int4 upp;
  const bool carried = big_pair_role(a, img, lu, N, up, upp) == 2;
  const int nj = (N - k0 + 1) - (carried ? 1 : 0);
  if (nj <= 0) return;
  int base = atomicAdd(njobs, nj);
  for (int k = k0; k <= N; ++k) {
    if (carried && k == N) continue;
    if (base < cap) jobs[base] = make_int2(img, lu | (k << 16));
    ++base;
  }
}

// (image, launch-local unit, plane) of a CTA; false: no such item
__device__ __forceinline__ bool big_decode(const BigArgs& a, int& img, int& lu, int& k) {
  if (a.jobs != nullptr) {
    const int j = (int)blockIdx.y + (int)blockIdx.z * (int)gridDim.y;
    if (j >= *a.njobs) return false;
    const int2 job = a.jobs[j];
    img = job.x;
    lu = job.y & 0xFFFF;
    k = job.y >> 16;
    return true;
  }
  k = blockIdx.y;
  lu = a.lu0 + (int)(blockIdx.z % a.nub);
  img = (int)(blockIdx.z / a.nub);
  return true;
}

// ------------------------------------------------------------------ rows (x axis)
// CTA = 32 rows x 256 columns of one (image, tile, plane); 16 warps, 2 rows each (both x
// passes stay inside the warp).  x = n2 + 16 n1 -> pass A: DFT16 over n1 (thread (row, n2)),
// twiddle W_256^{n2 k1}; pass B: DFT16 over n2 (thread (row, k1)); position k1*16 + k2 holds
// frequency k1 + 16 k2.  Shared row layout: slot k1*17 + j (j = n2, then k2; inverse: n1*17 + n2).
template <bool FWD, bool SPEC>
__global__ void __launch_bounds__(kBigNT, 2) big_rows_kernel(const BigArgs a) {
  constexpr int PX = kBig, RS = kBigRS, R = kBigR;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* buf = reinterpret_cast<float2*>(smem_raw);
  uint16_t* tv = reinterpret_cast<uint16_t*>(smem_raw + kBigRows * RS * 8);
  uint16_t* tv2 = tv + kBigRows * kBigTvLd;
  float2* tws = reinterpret_cast<float2*>(smem_raw + kBigRows * RS * 8 + 2 * kBigRows * kBigTvLd * 2);   // [n2][k1], stride 17

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int k = blockIdx.y, lu = 0, img = 0;
  if constexpr (!SPEC) {
    if (!big_decode(a, img, lu, k)) return;
  }
  const int unit = SPEC ? 0 : a.unit0 + lu;
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

  // x twiddles W_256^{n2 k1}
  if (tid < R * R) tws[(tid >> 4) * (R + 1) + (tid & 15)] = c_tw[TwOff<PX>::v + ((tid >> 4) * (tid & 15)) % PX];
  // this thread's items: row y of the warp's two, index j = n2 (pass A) / k1 (pass B)
  const int y = warp * 2 + (lane >> 4), j = lane & 15;
  float2* rowb = buf + y * RS;
  // position x' = 16 a + b of a row <-> slot a*17 + b
  auto slot = [](int x) { return (x >> 4) * (kBigR + 1) + (x & 15); };

  if constexpr (FWD) {
    // ---- stage tonal indices of rows [row0, row0+32) of the tile's input window
    int bad = 0, sh1 = 0, sh2 = 0;
    if constexpr (SPEC) {
      for (int p = tid; p < kBigRows * PX; p += kBigNT) {
        const int py = row0 + p / PX, px = p % PX;
        uint16_t t = kSent;
        if (py < a.my && px < a.mx) {
          const int si = py * a.mx + px;
          if (a.se_def == nullptr || a.se_def[si]) t = (uint16_t)(a.se_vals[si] + a.enc_bias);
        }
        tv[(p / PX) * kBigTvLd + px] = t;
      }
    } else {
      // returns the column shift sh: tile column c of row r is staged at tvd[r * kBigTvLd + sh + c]
      auto stage_unit = [&](int uty, int utx, int bias, uint16_t* tvd) -> int {
        const int ixb = utx * a.QX + a.DX;              // image column of tile column 0
        if (a.img_dtype == 0 && a.img_def == nullptr && (a.W & 15) == 0 &&
            (reinterpret_cast<uintptr_t>(a.img) & 15) == 0) {
          // uint8 rows 16-byte aligned, no mask: the staged row starts at the 16-aligned image
          // column xa <= ixb, so every aligned 16-pixel chunk of the image (inside or outside
          // the image as a whole) becomes two aligned 16-byte shared-memory stores
          const int xa = ixb & ~15, sh = ixb - xa;
          const uint8_t* base = reinterpret_cast<const uint8_t*>(a.img) + (int64_t)img * a.H * a.W;
          constexpr int CPR = kBigTvLd / 16;
#pragma unroll 1
          for (int it = tid; it < kBigRows * CPR; it += kBigNT) {
            const int r = it / CPR, ch = it - r * CPR;
            const int iy = uty * a.QY + a.DY + row0 + r, xc = xa + 16 * ch;
            uint32_t pk[8];
            if (iy < 0 || iy >= a.H || xc < 0 || xc >= a.W) {
#pragma unroll
              for (int i = 0; i < 8; ++i) pk[i] = (uint32_t)kSent | ((uint32_t)kSent << 16);
            } else {
              const uint4 wv = __ldg(reinterpret_cast<const uint4*>(base + (int64_t)iy * a.W + xc));
              const uint32_t wd[4] = {wv.x, wv.y, wv.z, wv.w};
              const int c0 = 16 * ch - sh;   // tile column of the chunk's first pixel
              uint32_t t16[16];
#pragma unroll
              for (int e = 0; e < 16; ++e) {
                const int v = max(a.enc_sign * (int)__byte_perm(wd[e >> 2], 0, 0x4440 + (e & 3)) + bias, 0);
                const bool in_tile = (unsigned)(c0 + e) < (unsigned)PX;
                if (in_tile && v >= T) bad = 1;
                t16[e] = (in_tile && v < T) ? (uint32_t)v : (uint32_t)kSent;
              }
#pragma unroll
              for (int i = 0; i < 8; ++i) pk[i] = t16[2 * i] | (t16[2 * i + 1] << 16);
            }
            uint4* dst = reinterpret_cast<uint4*>(tvd + r * kBigTvLd + 16 * ch);
            dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
            dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
          }
          return sh;
        }
        if (a.img_dtype == 0 && a.img_def == nullptr) {
          // uint8 images without a mask: 16-byte loads of the aligned chunks that cover each
          // row part inside the image (one load per 16 pixels instead of one per pixel)
          const int xs = max(ixb, 0), xe = min(ixb + PX, a.W);
          for (int i = tid; i < kBigRows * kBigTvLd / 2; i += kBigNT)
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
                else tvd[r * kBigTvLd + (x - ixb)] = (uint16_t)v;
              }
            }
          }
          return 0;
        }
        // generic path: batches of independent (predicated) loads per thread
        constexpr int IT = kBigRows * PX / kBigNT, GB = 16;
        static_assert(IT % GB == 0, "staging split");
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
            const int pp = tid + (g0 + u) * kBigNT;
            tvd[(pp / PX) * kBigTvLd + pp % PX] = t;
          }
        }
        return 0;
      };
      sh1 = stage_unit(ty, tx, enc_bias, tv);
      if (paired) {
        const int u2 = unit + 1, ty2 = u2 / max(a.tiles_x, 1);
        sh2 = stage_unit(ty2, u2 - ty2 * max(a.tiles_x, 1), enc_bias2, tv2);
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
    // ---- x pass A (encode): thread (y, n2 = j)
    {
      float2 w[R];
      const uint16_t* trow = tv + y * kBigTvLd + sh1 + j;
      if (!SPEC && paired) {
        // Nyquist plane of two units: (-1)^v of this unit + i (-1)^v of its neighbour
        auto nyq = [](uint32_t t) -> float { return t == kSent ? 0.f : ((t & 1u) ? -1.f : 1.f); };
        const uint16_t* trow2 = tv2 + y * kBigTvLd + sh2 + j;
#pragma unroll
        for (int n1 = 0; n1 < R; ++n1) w[n1] = make_float2(nyq(trow[R * n1]), nyq(trow2[R * n1]));
      } else {
#pragma unroll
        for (int n1 = 0; n1 < R; ++n1) w[n1] = enc(trow[R * n1]);
      }
      dft<R, false>(w);
      rowb[j] = w[0];
#pragma unroll
      for (int k1 = 1; k1 < R; ++k1) rowb[k1 * (R + 1) + j] = cmul(w[k1], tws[j * (R + 1) + k1]);
    }
    __syncwarp();
    // ---- x pass B: thread (y, k1 = j); the row then holds position k1*16 + k2 at slot k1*17 + k2
    {
      float2 w[R];
#pragma unroll
      for (int n2 = 0; n2 < R; ++n2) w[n2] = rowb[j * (R + 1) + n2];
      dft<R, false>(w);
#pragma unroll
      for (int k2 = 0; k2 < R; ++k2) rowb[j * (R + 1) + k2] = w[k2];
    }
    __syncthreads();
    // coalesced row stores (positions = permuted frequencies)
    for (int i = tid; i < kBigRows * (PX / 2); i += kBigNT) {
      const int yy = i / (PX / 2), xp = i % (PX / 2);
      const float2 p0 = buf[yy * RS + slot(2 * xp)], p1 = buf[yy * RS + slot(2 * xp + 1)];
      reinterpret_cast<float4*>(Sitem + (size_t)(row0 + yy) * kBig)[xp] = make_float4(p0.x, p0.y, p1.x, p1.y);
    }
  } else {
    // ---- inverse: load valid rows, x pass B^-1, x pass A^-1, store valid columns
    const int nrows = min(kBigRows, kBig - row0);
    {
      constexpr int IT = kBigRows * (PX / 2) / kBigNT;   // 8 float4 per thread, all loads in flight
      float4 v[IT];
#pragma unroll
      for (int u = 0; u < IT; ++u) {
        const int i = tid + u * kBigNT, yy = i / (PX / 2), xp = i % (PX / 2);
        v[u] = yy < nrows ? __ldcs(reinterpret_cast<const float4*>(Sitem + (size_t)(row0 + yy) * kBig) + xp)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < IT; ++u) {
        const int i = tid + u * kBigNT, yy = i / (PX / 2), xp = i % (PX / 2);
        buf[yy * RS + slot(2 * xp)] = make_float2(v[u].x, v[u].y);
        buf[yy * RS + slot(2 * xp + 1)] = make_float2(v[u].z, v[u].w);
      }
    }
    __syncthreads();
    {
      float2 w[R];
#pragma unroll
      for (int k2 = 0; k2 < R; ++k2) w[k2] = rowb[j * (R + 1) + k2];
      dft<R, true>(w);
#pragma unroll
      for (int n2 = 0; n2 < R; ++n2) rowb[j * (R + 1) + n2] = w[n2];
    }
    __syncwarp();
    {
      float2 w[R];
      w[0] = rowb[j];
#pragma unroll
      for (int k1 = 1; k1 < R; ++k1) w[k1] = cmulc(rowb[k1 * (R + 1) + j], tws[j * (R + 1) + k1]);
      dft<R, true>(w);
      // x = n2 + 16 n1 -> slot n1*17 + n2
#pragma unroll
      for (int n1 = 0; n1 < R; ++n1) rowb[n1 * (R + 1) + j] = w[n1];
    }
    __syncthreads();
    // valid window store: tile row ty_row = row0 + y (>= my-1), columns x >= mx-1
    float2* dst = a.chat + (((size_t)img * a.upl + lu) * a.K_max + k) * (size_t)a.wpx;
    const int vx = kBig - (a.mx - 1);   // valid columns per row
    for (int i = tid; i < kBigRows * vx; i += kBigNT) {
      const int yy = i / vx, c = i - (i / vx) * vx;
      const int row = row0 + yy;
      if (yy >= nrows) continue;
      const int oy = ty * a.QY + row - (a.my - 1), ox = tx * a.QX + c;
      const float2 v = buf[yy * RS + slot((a.mx - 1) + c)];
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
// CTA = 256 rows x 16 columns of one (image, tile, plane), 256 threads: thread (x, j) owns one
// 16-point transform per pass (y = n2 + 16 n1: pass A over n1 with j = n2, pass B over n2 with
// j = k1).  A warp's 64-bit accesses cover two rows of 16 consecutive columns.
template <bool SPEC>
__global__ void __launch_bounds__(kBigColsNT, 3) big_cols_kernel(const BigArgs a) {
  constexpr int PY = kBig, PXC = kBigCols, RS = PXC + 2, R = kBigR;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* buf = reinterpret_cast<float2*>(smem_raw);
  float2* sbuf = reinterpret_cast<float2*>(smem_raw + PY * RS * 8);   // [q][thread]

  const int tid = threadIdx.x;
  const int cb = blockIdx.x;
  int k = blockIdx.y, lu = 0, img = 0;
  if constexpr (!SPEC) {
    if (!big_decode(a, img, lu, k)) return;
  }
  const int unit = SPEC ? 0 : a.unit0 + lu;
  int K = a.K;
  if constexpr (!SPEC) {
    const int4 up = a.unit_param[(size_t)img * a.units + unit];
    K = up.y + 1;
    if (k >= K || (k == 0 && (up.w & 2))) return;   // past the unit's planes / known plane 0
    {
      int4 upp;
      if (big_pair_role(a, img, lu, k, up, upp) == 2) return;   // carried by the neighbour's CTAs
    }
  }
  float2* Sitem = SPEC ? a.S + (size_t)k * (kBig * kBig)
                       : a.S + (((size_t)img * a.upl + lu) * a.K_max + k) * (size_t)(kBig * kBig);
  // load 256 rows x 16 columns: all async copies in flight at once
  constexpr int XP = PXC / 2;
#pragma unroll 4
  for (int i = tid; i < PY * XP; i += kBigColsNT) {
    const int yy = i / XP, xp = i % XP;
    cp_async16(buf + yy * RS + 2 * xp, reinterpret_cast<const float4*>(Sitem + (size_t)yy * kBig + cb * PXC) + xp);
  }
  cp_async_commit();
  if constexpr (!SPEC) {
    // the product's spectrum chunk (thread order) streams in while forward pass A runs
    const int4 up = a.unit_param[(size_t)img * a.units + unit];
    const float4* spec_plane = a.spec + a.spec_off[up.z] + ((size_t)k * (kBig / kBigCols) + cb) * (R * kBigColsNT / 2);
    float4* sb4 = reinterpret_cast<float4*>(sbuf);
#pragma unroll
    for (int q = 0; q < R / 2; ++q) cp_async16(sb4 + q * kBigColsNT + tid, spec_plane + q * kBigColsNT + tid);
    cp_async_commit();
    cp_async_wait<1>();   // the tile (first group)
  } else {
    cp_async_wait<0>();
  }
  __syncthreads();
  const int x = tid & (PXC - 1), j = tid >> 4;
  float2* col = buf + x;
  // ---- forward y pass A: thread (x, n2 = j)
  {
    float2 w[R];
#pragma unroll
    for (int n1 = 0; n1 < R; ++n1) w[n1] = col[(j + R * n1) * RS];
    dft<R, false>(w);
    col[j * RS] = w[0];
#pragma unroll
    for (int k1 = 1; k1 < R; ++k1) col[(j + R * k1) * RS] = cmul(w[k1], c_tw[TwOff<PY>::v + j * k1]);
  }
  if constexpr (!SPEC) cp_async_wait<0>();   // the spectrum chunk (other threads' copies: published by the barrier)
  __syncthreads();
  // ---- forward y pass B (+ product + inverse y pass B): thread (x, k1 = j)
  {
    float2 w[R];
#pragma unroll
    for (int n2 = 0; n2 < R; ++n2) w[n2] = col[(n2 + R * j) * RS];
    dft<R, false>(w);
    if constexpr (SPEC) {
      float2* so = reinterpret_cast<float2*>(const_cast<float4*>(a.spec)) + ((size_t)k * (kBig / kBigCols) + cb) * (R * kBigColsNT);
      const float s = a.spec_scale;
#pragma unroll
      for (int q = 0; q < R; ++q) so[q * kBigColsNT + tid] = make_float2(w[q].x * s, w[q].y * s);
    } else {
#pragma unroll
      for (int q = 0; q < R; ++q) w[q] = cmul(w[q], sbuf[q * kBigColsNT + tid]);
      dft<R, true>(w);
#pragma unroll
      for (int n2 = 0; n2 < R; ++n2) col[(n2 + R * j) * RS] = w[n2];
    }
  }
  if constexpr (SPEC) return;
  __syncthreads();
  // ---- inverse y pass A: thread (x, n2 = j)
  {
    float2 w[R];
    w[0] = col[j * RS];
#pragma unroll
    for (int k1 = 1; k1 < R; ++k1) w[k1] = cmulc(col[(j + R * k1) * RS], c_tw[TwOff<PY>::v + j * k1]);
    dft<R, true>(w);
#pragma unroll
    for (int n1 = 0; n1 < R; ++n1) col[(j + R * n1) * RS] = w[n1];
  }
  __syncthreads();
  // store the valid rows back (row-inverse kernel reads rows >= my-1)
  for (int i = tid; i < PY * XP; i += kBigColsNT) {
    const int yy = i / XP, xp = i % XP;
    if (yy < a.my - 1) continue;
    reinterpret_cast<float4*>(Sitem + (size_t)yy * kBig + cb * PXC)[xp] = *reinterpret_cast<const float4*>(buf + yy * RS + 2 * xp);
  }
}

constexpr int kBigRowsSmem = kBigRows * kBigRS * 8 + 2 * kBigRows * kBigTvLd * 2 + kBigR * (kBigR + 1) * 8;
constexpr int kBigColsSmem = kBig * (kBigCols + 2) * 8 + kBigR * kBigColsNT * 8;

}  // namespace fm
