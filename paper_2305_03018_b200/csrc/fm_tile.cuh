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
//       swizzled shared-memory tile);
//   (c) multiplies by the cached SE spectrum for k (fa *= fb, fft_conv.py:137),
//       fused into the last forward pass;
//   (d) runs the inverse FFT (x axis, then y axis) and writes only the
//       overlap-save valid window of the tile to the spectral scratch
//       Chat[img][k][out_y][out_x] (complex64) for the tonal kernel.
// With SPEC=true the same code computes the SE spectrum (rfftn(b),
// fft_conv.py:135-136) once per plan and stores it in thread-register order.
#pragma once
#include "fm_dft.cuh"

namespace fm {

constexpr uint16_t kSent = 0xFFFFu;  // "no one-hot entry": gap or outside the grid

template <int P> struct Split;
template <> struct Split<16> { static constexpr int R1 = 4, R2 = 4; };
template <> struct Split<32> { static constexpr int R1 = 8, R2 = 4; };
template <> struct Split<64> { static constexpr int R1 = 8, R2 = 8; };
template <> struct Split<128> { static constexpr int R1 = 16, R2 = 8; };
template <> struct Split<256> { static constexpr int R1 = 16, R2 = 16; };

// Twiddle tables W_P^j = exp(-2 pi i j / P) for P = 16..256, concatenated.
// Offsets: 16 -> 0, 32 -> 16, 64 -> 48, 128 -> 112, 256 -> 240 (496 entries).
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
  int k_chunk;
  int enc_sign, enc_bias;     // v = enc_sign * f + enc_bias (CONV) / v = b - se_min (SPEC)
  int vmax;                   // largest legal v
  int copies;                 // tonal-table replication (power of 2, <= 16)
  const float2* tabT;         // [T] exp(-2 pi i r / T)
  const float2* spec;         // [K][thread order] SE spectrum (CONV reads, SPEC writes)
  float2* spec_out;           // SPEC
  float spec_scale;           // SPEC: 1 / (PY_eff * PX * T)
  float2* chat;               // CONV: [imgs][K][OH*OW]
  int* err;                   // value-range error flag
};

__constant__ float2 c_tw[kTwTotal];

template <int PY, int PX, int NT, bool TWO_D>
struct TileCfg {
  static constexpr int R1x = Split<PX>::R1, R2x = Split<PX>::R2;
  static constexpr int R1y = TWO_D ? Split<PY>::R1 : 1;
  static constexpr int R2y = TWO_D ? Split<PY>::R2 : 1;
  static constexpr int NPTS = PY * PX;
  static constexpr int E = NPTS / NT;
  static constexpr int G_yA = TWO_D ? PX * R2y / NT : 0;
  static constexpr int G_yB = TWO_D ? PX * R1y / NT : 0;
  static constexpr int G_xA = PY * R2x / NT;
  static constexpr int G_xB = PY * R1x / NT;
  static constexpr int SWZ = 15;
  static_assert(NPTS % NT == 0, "tile points must divide among threads");
  static_assert(G_xA * R1x == E && G_xB * R2x == E, "x-axis item split");
  static_assert(!TWO_D || (G_yA * R1y == E && G_yB * R2y == E), "y-axis item split");
  static_assert(PX >= 16, "min tile edge 16");
  // shared memory bytes excluding the tonal table
  static constexpr int kSmemFixed = NPTS * 8 + ((NPTS * 2 + 15) / 16) * 16;
};

// swizzled position of tile element (y, x): XOR the low 4 bits of x with y
// so that 16 consecutive rows at one x hit 16 distinct 8-byte bank pairs.
template <int PX>
__device__ __forceinline__ int sidx(int y, int x) { return y * PX + (x ^ (y & 15)); }

__device__ __forceinline__ int load_img(const void* img, int dtype, int64_t i) {
  if (dtype == 0) return (int)__ldg(reinterpret_cast<const uint8_t*>(img) + i);
  if (dtype == 1) return (int)__ldg(reinterpret_cast<const uint16_t*>(img) + i);
  return __ldg(reinterpret_cast<const int32_t*>(img) + i);
}

template <int PY, int PX, int NT, bool TWO_D, bool SPEC>
__global__ void __launch_bounds__(NT, 1) tile_conv_kernel(const TileArgs a) {
  using C = TileCfg<PY, PX, NT, TWO_D>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* buf = reinterpret_cast<float2*>(smem_raw);
  uint16_t* tv = reinterpret_cast<uint16_t*>(smem_raw + C::NPTS * 8);
  float2* tab = reinterpret_cast<float2*>(smem_raw + C::kSmemFixed);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int img = SPEC ? 0 : blockIdx.z;
  const int T = a.T;
  const int copies = a.copies;
  const int cmask = copies - 1;

  // ---- tonal twiddle table, replicated `copies` times for conflict-free lookups
  for (int i = tid; i < T * copies; i += NT) tab[i] = a.tabT[i / copies];

  // ---- stage the tile's tonal indices v(x) (kSent = no entry)
  int ty = 0, tx = 0;
  if (TWO_D) {
    ty = blockIdx.x / a.tiles_x;
    tx = blockIdx.x - ty * a.tiles_x;
  }
  int bad = 0;
  for (int p = tid; p < C::NPTS; p += NT) {
    const int py = p / PX, px = p - (p / PX) * PX;
    uint16_t t = kSent;
    if (SPEC) {
      const int sy = TWO_D ? py : 0;
      if (sy < a.my && px < a.mx) {
        const int si = sy * a.mx + px;
        if (a.se_def == nullptr || a.se_def[si]) t = (uint16_t)(a.se_vals[si] + a.enc_bias);
      }
    } else {
      int iy, ix;
      bool rowok;
      if (TWO_D) {
        iy = ty * a.QY + a.DY + py;
        ix = tx * a.QX + a.DX + px;
        rowok = true;
      } else {
        const int tile = blockIdx.x * PY + py;
        iy = 0;
        ix = tile * a.QX + a.DX + px;
        rowok = tile < a.tiles_total;
      }
      if (rowok && iy >= 0 && iy < a.H && ix >= 0 && ix < a.W) {
        const int64_t gi = ((int64_t)img * a.H + iy) * a.W + ix;
        if (a.img_def == nullptr || a.img_def[gi]) {
          const int v = a.enc_sign * load_img(a.img, a.img_dtype, gi) + a.enc_bias;
          if (v < 0 || v > a.vmax) bad = 1;
          else t = (uint16_t)v;
        }
      }
    }
    tv[p] = t;
  }
  if (!SPEC && bad) atomicOr(a.err, 1);
  __syncthreads();

  const int k_begin = blockIdx.y * a.k_chunk;
  const int k_end = min(a.K, k_begin + a.k_chunk);

  for (int k = k_begin; k < k_end; ++k) {
    // encode helper: w_T^{k v} from the replicated table
    auto enc = [&](uint32_t t) -> float2 {
      if (t == kSent) return make_float2(0.f, 0.f);
      const uint32_t n = (uint32_t)k * t;
      uint32_t r = n - __umulhi(n, a.magicT) * (uint32_t)T;
      if (r >= (uint32_t)T) r -= (uint32_t)T;
      return tab[r * copies + (lane & cmask)];
    };

    if constexpr (TWO_D) {
      // ---------------- forward y, pass A (with encode)
#pragma unroll
      for (int g = 0; g < C::G_yA; ++g) {
        const int i = tid + NT * g;
        const int x = i % PX, n2 = i / PX;
        float2 w[C::R1y];
#pragma unroll
        for (int n1 = 0; n1 < C::R1y; ++n1) w[n1] = enc(tv[(n2 + C::R2y * n1) * PX + x]);
        dft<C::R1y, false>(w);
#pragma unroll
        for (int k1 = 0; k1 < C::R1y; ++k1) {
          const float2 z = (k1 == 0) ? w[k1] : cmul(w[k1], c_tw[TwOff<PY>::v + n2 * k1]);
          buf[sidx<PX>(n2 + C::R2y * k1, x)] = z;
        }
      }
      __syncthreads();
      // ---------------- forward y, pass B
#pragma unroll
      for (int g = 0; g < C::G_yB; ++g) {
        const int i = tid + NT * g;
        const int x = i % PX, k1 = i / PX;
        float2 w[C::R2y];
#pragma unroll
        for (int n2 = 0; n2 < C::R2y; ++n2) w[n2] = buf[sidx<PX>(n2 + C::R2y * k1, x)];
        dft<C::R2y, false>(w);
#pragma unroll
        for (int k2 = 0; k2 < C::R2y; ++k2) buf[sidx<PX>(k2 + C::R2y * k1, x)] = w[k2];
      }
      __syncthreads();
      // ---------------- forward x, pass A
#pragma unroll
      for (int g = 0; g < C::G_xA; ++g) {
        const int i = tid + NT * g;
        const int y = i % PY, n2 = i / PY;
        float2 w[C::R1x];
#pragma unroll
        for (int n1 = 0; n1 < C::R1x; ++n1) w[n1] = buf[sidx<PX>(y, n2 + C::R2x * n1)];
        dft<C::R1x, false>(w);
#pragma unroll
        for (int k1 = 0; k1 < C::R1x; ++k1) {
          const float2 z = (k1 == 0) ? w[k1] : cmul(w[k1], c_tw[TwOff<PX>::v + n2 * k1]);
          buf[sidx<PX>(y, n2 + C::R2x * k1)] = z;
        }
      }
      __syncthreads();
    } else {
      // ---------------- 1-D: forward x, pass A with encode (row y = independent tile)
#pragma unroll
      for (int g = 0; g < C::G_xA; ++g) {
        const int i = tid + NT * g;
        const int y = i % PY, n2 = i / PY;
        float2 w[C::R1x];
#pragma unroll
        for (int n1 = 0; n1 < C::R1x; ++n1) w[n1] = enc(tv[y * PX + n2 + C::R2x * n1]);
        dft<C::R1x, false>(w);
#pragma unroll
        for (int k1 = 0; k1 < C::R1x; ++k1) {
          const float2 z = (k1 == 0) ? w[k1] : cmul(w[k1], c_tw[TwOff<PX>::v + n2 * k1]);
          buf[sidx<PX>(y, n2 + C::R2x * k1)] = z;
        }
      }
      __syncthreads();
    }

    // ---------------- forward x, pass B (+ spectral product + inverse x pass B)
    {
      const float2* sk = a.spec + (size_t)k * C::NPTS;
      float2* so = SPEC ? a.spec_out + (size_t)k * C::NPTS : nullptr;
#pragma unroll
      for (int g = 0; g < C::G_xB; ++g) {
        const int i = tid + NT * g;
        const int y = i % PY, k1 = i / PY;
        float2 w[C::R2x];
#pragma unroll
        for (int n2 = 0; n2 < C::R2x; ++n2) w[n2] = buf[sidx<PX>(y, n2 + C::R2x * k1)];
        dft<C::R2x, false>(w);
        if constexpr (SPEC) {
#pragma unroll
          for (int e = 0; e < C::R2x; ++e) so[(g * C::R2x + e) * NT + tid] = cscale(w[e], a.spec_scale);
        } else {
#pragma unroll
          for (int e = 0; e < C::R2x; ++e) w[e] = cmul(w[e], __ldg(sk + (g * C::R2x + e) * NT + tid));
          dft<C::R2x, true>(w);
#pragma unroll
          for (int n2 = 0; n2 < C::R2x; ++n2) buf[sidx<PX>(y, n2 + C::R2x * k1)] = w[n2];
        }
      }
    }
    if constexpr (SPEC) {
      __syncthreads();
      continue;
    } else {
      __syncthreads();
      // ---------------- inverse x, pass A
#pragma unroll
      for (int g = 0; g < C::G_xA; ++g) {
        const int i = tid + NT * g;
        const int y = i % PY, n2 = i / PY;
        float2 w[C::R1x];
#pragma unroll
        for (int k1 = 0; k1 < C::R1x; ++k1) {
          const float2 z = buf[sidx<PX>(y, n2 + C::R2x * k1)];
          w[k1] = (k1 == 0) ? z : cmulc(z, c_tw[TwOff<PX>::v + n2 * k1]);
        }
        dft<C::R1x, true>(w);
        if constexpr (TWO_D) {
#pragma unroll
          for (int n1 = 0; n1 < C::R1x; ++n1) buf[sidx<PX>(y, n2 + C::R2x * n1)] = w[n1];
        } else {
          // 1-D output: row y is tile (blockIdx.x*PY + y); positions x >= mx-1 are valid
          const int tile = blockIdx.x * PY + y;
          if (tile < a.tiles_total) {
            float2* dst = a.chat + ((size_t)img * a.K + k) * (size_t)a.OW;
#pragma unroll
            for (int n1 = 0; n1 < C::R1x; ++n1) {
              const int x = n2 + C::R2x * n1;
              const int ox = tile * a.QX + x - (a.mx - 1);
              if (x >= a.mx - 1 && ox < a.OW) dst[ox] = w[n1];
            }
          }
        }
      }
      __syncthreads();
      if constexpr (TWO_D) {
        // ---------------- inverse y, pass B
#pragma unroll
        for (int g = 0; g < C::G_yB; ++g) {
          const int i = tid + NT * g;
          const int x = i % PX, k1 = i / PX;
          float2 w[C::R2y];
#pragma unroll
          for (int k2 = 0; k2 < C::R2y; ++k2) w[k2] = buf[sidx<PX>(k2 + C::R2y * k1, x)];
          dft<C::R2y, true>(w);
#pragma unroll
          for (int n2 = 0; n2 < C::R2y; ++n2) buf[sidx<PX>(n2 + C::R2y * k1, x)] = w[n2];
        }
        __syncthreads();
        // ---------------- inverse y, pass A + store of the valid window
        float2* dst = a.chat + ((size_t)img * a.K + k) * (size_t)a.OH * a.OW;
#pragma unroll
        for (int g = 0; g < C::G_yA; ++g) {
          const int i = tid + NT * g;
          const int x = i % PX, n2 = i / PX;
          float2 w[C::R1y];
#pragma unroll
          for (int k1 = 0; k1 < C::R1y; ++k1) {
            const float2 z = buf[sidx<PX>(n2 + C::R2y * k1, x)];
            w[k1] = (k1 == 0) ? z : cmulc(z, c_tw[TwOff<PY>::v + n2 * k1]);
          }
          dft<C::R1y, true>(w);
          const int ox = tx * a.QX + x - (a.mx - 1);
          if (x >= a.mx - 1 && ox < a.OW) {
#pragma unroll
            for (int n1 = 0; n1 < C::R1y; ++n1) {
              const int y = n2 + C::R2y * n1;
              const int oy = ty * a.QY + y - (a.my - 1);
              if (y >= a.my - 1 && oy < a.OH) dst[(size_t)oy * a.OW + ox] = w[n1];
            }
          }
        }
        __syncthreads();
      }
    }
  }
}

}  // namespace fm
