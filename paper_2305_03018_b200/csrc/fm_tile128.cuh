// fm_tile128.cuh — three-pass 128x128 overlap-save tile convolution (2-D).
//
// Same job as tile_conv_kernel<128,128,512> (fm_tile.cuh: encode the tonal
// twiddles w_T^{k v(x)} of one tile, forward 2-D FFT, product with the cached
// SE spectrum, inverse 2-D FFT, store of the overlap-save window), but the
// 2^14-point 2-D transform runs as THREE shared-memory passes per direction
// instead of four, with every thread holding 32 points:
//
//   F1  y: 32-point DFT over n1 (y = n2 + 4 n1)                           thread (x, n2)
//   F2  y: twiddle W_128^{n2 k1}, 4-point DFT over n2 -> k2;  x: 8-point DFT over m1 -> j1
//       (x = m2 + 16 m1), twiddle W_128^{m2 j1}                             thread (k1, m2)
//   F3  x: 16-point DFT over m2 -> j2; product; inverse 16-point DFT         thread (k1, k2, j1)
//   I2  inverse of F2 (conjugate twiddles)                                 thread (k1, m2)
//   I1  inverse 32-point DFT, store of the window rows                      thread (x, n2)
//
// so frequency (ky, kx) = (k1 + 32 k2, j1 + 8 j2).  F2 -> F3 -> I2 exchange
// only data inside the warp's own shared-memory region (warp w owns k1 in
// {2w, 2w+1}); F1 -> F2 and I2 -> I1 are the two CTA barriers per plane, and
// I1 -> the next plane's F1 needs none (same thread partition and slots).
// All butterflies, twiddles and the product are packed f32x2 instructions
// (fm_dft.cuh).  I1's columns start at the window (x = c + mx - 1), and the plan
// trims the window to a multiple of 32 columns when that leaves one I1 warp per
// scheduler without output columns: it builds the encode table of plane k + 2
// (double-buffered per-plane tables) and runs ahead into the next plane's F1.
//
// SE spectrum of the product (thread order, four 32 KB chunks per plane): slot
// 0's two chunks arrive by bulk async copies into shared memory a whole plane
// ahead (issued by the last warp to release the buffer), slot 1's go straight
// from L2 into registers, loaded at the start of the plane.
//
// Shared-memory layouts (float2 slots, per-warp regions of 1088):
//   B1 (F1/I1 <-> F2/I2): (k1, n2, x) -> (k1>>1)*1088 + ((k1&1)*4 + n2)*128 + x
//   B2 (F2/I2 <-> F3):    (k1, k2, j1, m2) -> (k1>>1)*1088 + ((k2*2 + (k1&1))*8 + j1)*17 + m2
// Half-warps read/write 16 consecutive slots (or 16 slots with distinct
// residues mod 16 through the 17-stride), so every 64-bit access is
// conflict-free; all per-element offsets are compile-time immediates.
//
// Tonal indices are staged as uint8 (T <= 254, sentinel T reads the zero
// entry of the per-plane encode table), which is what frees the room for the
// padded B2 layout beside two 32 KB SE-spectrum buffers; longer tonal axes
// (8-bit data: c3) stage uint16 indices beside one buffer.
#pragma once
#include "fm_fused.cuh"
#include "fm_tile.cuh"

namespace fm {

template <typename TV>
struct T128 {
  static constexpr int P = 128, NT = 512, NW = NT / 32;
  static constexpr int REG = 1088;                        // per-warp region (float2 slots)
  static constexpr int kBufBytes = NW * REG * 8;          // 139264
  static constexpr int kChunkF4 = 4 * NT;                 // 32 KB spectrum chunk: 4 float4 per thread
  static constexpr uint32_t kChunkBytes = kChunkF4 * 16;
  static constexpr int kSpecPairs = P * P / 2;            // float4 per tonal plane (4 chunks)
  // uint8 indices leave room for two spectrum buffers (slot 0's chunks both a
  // plane ahead); uint16 (long tonal axes) for one: chunk 1 follows chunk 0
  // through it by per-thread cp.async
  static constexpr int kNSB = sizeof(TV) == 1 ? 2 : 1;
  static constexpr int kSpecBytes = kNSB * kChunkF4 * 16;
  // tonal indices, column-major with the rows of one F1 thread (y = n2 + 4 n1,
  // n1 = 0..31) contiguous: (y, x) -> x * kTvLd + (y & 3) * 32 + (y >> 2); the
  // 16-byte column pad keeps a warp's 16-byte loads (consecutive x) conflict-free
  static constexpr int kTvLd = P + 16 / (int)sizeof(TV);
  static constexpr int kTvBytes = P * kTvLd * (int)sizeof(TV);
  static constexpr int kTvVec = 32 * (int)sizeof(TV) / 16;   // uint4 per F1 thread
  static constexpr int kTwBytes = 8 * 16 * 8;             // W_128^{m2 j1}, [j1][m2]
  static constexpr int kSmemFixed = kBufBytes + kSpecBytes + kTvBytes + kTwBytes;
  static constexpr int kEncSlots = (227 * 1024 - kSmemFixed - 256) / 8;   // two per-plane tables
  static constexpr int kSmemTotal = kSmemFixed + kEncSlots * 8;
  static constexpr int kTMax = sizeof(TV) == 1 ? 254 : (kEncSlots / 2 - 1) & ~1;
  static_assert(2 * (kTMax + 1) <= kEncSlots, "encode tables");
};

// y twiddles W_128^{n2 k1} laid out [n2][k1] (applied in F2 / I2: three per thread)
__constant__ float2 c_twy[4 * 32];

template <typename TV, bool SPEC>
__global__ void __launch_bounds__(512, 1) tile128_kernel(const TileArgs a) {
  using C = T128<TV>;
  constexpr int P = C::P, NT = C::NT, REG = C::REG;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* buf = reinterpret_cast<float2*>(smem_raw);
  float4* sbuf = reinterpret_cast<float4*>(smem_raw + C::kBufBytes);
  TV* tv = reinterpret_cast<TV*>(smem_raw + C::kBufBytes + C::kSpecBytes);
  float2* twt = reinterpret_cast<float2*>(smem_raw + C::kBufBytes + C::kSpecBytes + C::kTvBytes);
  float2* enc_s = twt + 128;

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  UnitJob job;
  if (!decode_job<SPEC>(a, job)) return;
  const int img = job.img, unit = job.unit, kchunk_idx = job.kchunk;
  const int T = job.T, K = job.K, enc_bias = job.enc_bias;
  const bool skip0 = job.skip0;
  const float4* spec_base = job.spec_base;
  const float2* enc_g = SPEC ? a.enc_tab : a.enc_tab + a.enc_off[job.unit_li];
  // per-plane encode tables M_k[t] = w_T^{(k t) mod T}, M_k[T] = 0 (double-buffered)
  auto build_mtab = [&](int kk) {
    float2* M = enc_s + (kk & 1) * (T + 1);
    for (int j = tid; j <= T; j += NT) M[j] = j < T ? enc_g[(kk * j) % T] : make_float2(0.f, 0.f);
  };

  const int ty = SPEC ? 0 : unit / a.tiles_x;
  const int tx = SPEC ? 0 : unit - ty * a.tiles_x;
  // ---- stage the tile's tonal indices (sentinel T = no entry)
  {
    int bad = 0;
    if constexpr (SPEC) {
      for (int p = tid; p < P * P; p += NT) {
        const int py = p / P, px = p - (p / P) * P;
        int t = T;
        if (py < a.my && px < a.mx) {
          const int si = py * a.mx + px;
          // ladder entries shorter than the SE's own range are never used by a
          // unit; reduce so their (unused) spectra stay finite
          if (a.se_def == nullptr || a.se_def[si]) t = (a.se_vals[si] + a.enc_bias) % T;
        }
        tv[px * C::kTvLd + (py & 3) * 32 + (py >> 2)] = (TV)t;
      }
    } else {
      // thread (x, n2) stages rows y = n2 + 4 n1 of column x (a warp reads 32
      // consecutive x of one row) and stores them as packed 16-byte words
      constexpr int GB = 16, VPW = 4 / (int)sizeof(TV);
      const int sx = tid & (P - 1), sn2 = tid >> 7;
      const int ix = tx * a.QX + a.DX + sx;
      const bool okx = ix >= 0 && ix < a.W;
      uint4* trow = reinterpret_cast<uint4*>(tv + sx * C::kTvLd + sn2 * 32);
#pragma unroll 1
      for (int g0 = 0; g0 < 32; g0 += GB) {
        int raw[GB];
        bool ok[GB];
#pragma unroll
        for (int u = 0; u < GB; ++u) {
          const int iy = ty * a.QY + a.DY + sn2 + 4 * (g0 + u);
          ok[u] = okx && iy >= 0 && iy < a.H;
          raw[u] = 0;
          if (ok[u]) {
            const int64_t gi = ((int64_t)img * a.H + iy) * a.W + ix;
            raw[u] = load_img(a.img, a.img_dtype, gi);
            if (a.img_def != nullptr) ok[u] = a.img_def[gi] != 0;
          }
        }
        uint32_t pk[GB / VPW];
#pragma unroll
        for (int i = 0; i < GB / VPW; ++i) pk[i] = 0;
#pragma unroll
        for (int u = 0; u < GB; ++u) {
          int t = T;
          if (ok[u]) {
            // values below the unit's clamp level encode as the clamp (fm_range.cuh)
            const int v = max(a.enc_sign * raw[u] + enc_bias, 0);
            if (v >= T) bad = 1;
            else t = v;
          }
          pk[u / VPW] |= (uint32_t)t << (8 * (int)sizeof(TV) * (u % VPW));
        }
#pragma unroll
        for (int i = 0; i < GB / VPW / 4; ++i)
          trow[g0 / (16 / (int)sizeof(TV)) + i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
      }
      if (bad) atomicOr(a.err, 1);
    }
  }
  if (tid < 128) twt[tid] = c_tw[TwOff<128>::v + (tid & 15) * (tid >> 4)];
  const int k_begin = kchunk_idx * job.k_chunk;
  const int k_first = k_begin + ((skip0 && kchunk_idx == 0) ? 1 : 0);
  // with a trimmed window (QX <= 96) the inverse-y warps of column block 3 have
  // no output columns: they build the encode table two planes ahead while the
  // others run I1 (slack they would otherwise spend at the next F1 barrier), so
  // both buffers start filled; otherwise the table of plane k + 1 is built after
  // plane k's F1 barrier
  const bool tab_in_i1 = !SPEC && a.QX <= 96;
  build_mtab(k_first);
  if (tab_in_i1 && k_first + 1 < min(K, k_begin + job.k_chunk)) build_mtab(k_first + 1);
  __shared__ __align__(8) uint64_t s_full[2];   // spectrum buffers: bulk-copy completion
  __shared__ int s_rel[2];                       // warps that released the buffer
  __shared__ int s_kend;
  if (tid == 0) {
    s_kend = min(K, k_begin + job.k_chunk);
    if constexpr (!SPEC) {
#pragma unroll
      for (int b = 0; b < C::kNSB; ++b) mbar_init(&s_full[b], 1);
      s_rel[0] = 0;
      s_rel[1] = 0;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if (k_first < min(K, k_begin + job.k_chunk)) {
#pragma unroll
        for (int b = 0; b < C::kNSB; ++b) {
          mbar_expect_tx(&s_full[b], C::kChunkBytes);
          bulk_g2s_nohint(sbuf + b * C::kChunkF4, spec_base + (size_t)k_first * C::kSpecPairs + (size_t)b * C::kChunkF4,
                          C::kChunkBytes, &s_full[b]);
        }
      }
    }
  }
  __syncthreads();
  // the plane loop bound lives in shared memory (a register copy would be spilled)
  const volatile int* kend_s = &s_kend;
  // the unit's planes (8-byte complex64 elements, or 4-byte int16 pairs with chat16)
  float2* chat_unit = SPEC ? nullptr
                           : reinterpret_cast<float2*>(reinterpret_cast<char*>(a.chat) +
                                                       ((size_t)img * a.upl + (unit - a.unit0)) * a.K_max *
                                                           (size_t)a.wpx * (a.chat16 ? 4 : 8));

  // thread roles
  // F1 / I1: column x = (c + mx - 1) mod 128 for c = 32 (warp>>2) + lane, so the
  // window columns c < QX come first and a warp with 32 (warp>>2) >= QX has no
  // output column (the plan trims QX to a multiple of 32 when that idles a warp)
  // Warps w = s + 4j share scheduler s: (n2, column block) = (j, (j + s) mod 4) is
  // a Latin square, so every scheduler gets one warp of each n2 (n2 = 0 skips
  // the twiddles) and one of each column block (the idle inverse-y block)
  const int f_n2 = warp >> 2, f_xb = ((warp >> 2) + (warp & 3)) & 3;
  const int f_c = f_xb * 32 + lane, f_x = (f_c + a.mx - 1) & (P - 1);
  const bool i1_idle = f_xb * 32 >= a.QX;
  const int hi = lane >> 4, m2 = lane & 15;                                  // F2 / I2 (k1 = 2 warp + hi)
  float2* const b1_col = buf + f_n2 * P + f_x;                               // F1 / I1 slots
  float2* const b1_row = buf + warp * REG + hi * 4 * P + m2;                 // F2 reads, I2 writes
  float2* const b2_row = buf + warp * REG + hi * 8 * 17 + m2;                // F2 writes, I2 reads
  float2* const b2_grp = buf + warp * REG + (lane & 15) * 17 + hi * 16 * 17; // F3 (+ 32*17 per slot)

  int pord = 0;   // planes done: phase parity of the bulk-copied buffers
  for (int k = k_begin; k < *kend_s; ++k) {
    if (k == 0 && skip0) continue;   // plane 0 of a full unit: the tonal pass knows it
    const float2* Mk = enc_s + (k & 1) * (T + 1);

    // slot 1's SE spectrum (chunks 2, 3: this thread's 8 float4), L2 -> registers,
    // in flight through F1, F2 and slot 0 of F3
    float4 sp1[8];
    if constexpr (!SPEC) {
      const float4* src = spec_base + (size_t)k * C::kSpecPairs + (size_t)2 * C::kChunkF4 + tid;
#pragma unroll
      for (int i = 0; i < 8; ++i) sp1[i] = __ldcg(src + (i >> 2) * C::kChunkF4 + (i & 3) * NT);
    }
    // ---------------- F1: encode + y DFT32 + twiddle W^{n2 k1}
    {
      float2 v[32];
      // table entry t at byte address mkb + 8 t: one LEA per pixel (indexing Mk
      // directly adds the plane's table offset to t first)
      // (the thread's 32 indices are two / four 16-byte words: one byte permute each)
      const uint32_t mkb = smem_addr(Mk);
      const uint4* tq = reinterpret_cast<const uint4*>(tv + f_x * C::kTvLd + f_n2 * 32);
#pragma unroll
      for (int h = 0; h < C::kTvVec; ++h) {
        const uint4 q = tq[h];
        const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
        constexpr int VPW = 4 / (int)sizeof(TV), PER = 16 / (int)sizeof(TV);
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int n1 = h * PER + j, e = j % VPW;
          const uint32_t t = sizeof(TV) == 1 ? __byte_perm(w4[j / VPW], 0, 0x4440 + e)
                                             : __byte_perm(w4[j / VPW], 0, e ? 0x4432 : 0x4410);
          asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v[n1].x), "=f"(v[n1].y) : "r"(mkb + (t << 3)));
        }
      }
      dft32p_fwd<false>(v);   // the y twiddle W^{n2 k1} is applied in F2 (same work on every warp)
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int k1 = dft32p_freq(r);
        b1_col[(k1 >> 1) * REG + (k1 & 1) * 4 * P] = v[r];
      }
    }
    __syncthreads();
    // next plane's table into the other buffer (its last reader, the previous
    // plane's F1, finished before this barrier)
    if (!tab_in_i1 && k + 1 < *kend_s) build_mtab(k + 1);

    // ---------------- F2: y DFT4 over n2, x DFT8 over m1, twiddle W^{m2 j1}
    {
      float2 c[4][8];
#pragma unroll
      for (int n2 = 0; n2 < 4; ++n2)
#pragma unroll
        for (int m1 = 0; m1 < 8; ++m1) c[n2][m1] = b1_row[n2 * P + 16 * m1];
      __syncwarp();   // the warp's region is rewritten in the B2 layout below
      // y twiddle W_128^{n2 k1} of the DFT32 outputs (k1 = 2 warp + hi: three
      // runtime twiddles, each applied to the thread's 8 values of that n2)
      {
        const int k1 = 2 * warp + hi;
#pragma unroll
        for (int n2 = 1; n2 < 4; ++n2) {
          const float2 w = c_twy[n2 * 32 + k1];
#pragma unroll
          for (int m1 = 0; m1 < 8; ++m1) c[n2][m1] = cmul(c[n2][m1], w);
        }
      }
#pragma unroll
      for (int m1 = 0; m1 < 8; ++m1) {
        float2 t[4] = {c[0][m1], c[1][m1], c[2][m1], c[3][m1]};
        dft4_<false>(t);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) c[k2][m1] = t[k2];
      }
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) {
        dft8_<false>(c[k2]);
#pragma unroll
        for (int j1 = 1; j1 < 8; ++j1) c[k2][j1] = cmul(c[k2][j1], twt[j1 * 16 + m2]);
      }
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2)
#pragma unroll
        for (int j1 = 0; j1 < 8; ++j1) b2_row[k2 * 2 * 8 * 17 + j1 * 17] = c[k2][j1];
    }
    __syncwarp();

    // ---------------- F3: x DFT16 over m2 (+ product + inverse DFT16)
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      float2* g = b2_grp + s * 32 * 17;
      float2 u[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) u[q] = g[q];
      dft16_<false>(u);
      if constexpr (SPEC) {
        float4* so = a.spec_out + (size_t)k * C::kSpecPairs;
        const float sc = a.spec_scale;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float2 p0 = u[8 * h + 2 * q], p1 = u[8 * h + 2 * q + 1];
            so[(size_t)((2 * s + h) * 4 + q) * NT + tid] = make_float4(p0.x * sc, p0.y * sc, p1.x * sc, p1.y * sc);
          }
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int ch = 2 * s + h;   // chunk: slot s, frequencies j2 in [8h, 8h+8)
          float4 s4[4];
          if (ch < 2) {
            const int b = C::kNSB == 2 ? ch : 0;
            if (C::kNSB == 2 || ch == 0) mbar_wait(&s_full[b], (uint32_t)(pord & 1));
            else cp_async_wait<0>();
            const float4* sp = sbuf + b * C::kChunkF4 + tid;
#pragma unroll
            for (int q = 0; q < 4; ++q) s4[q] = sp[q * NT];
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) s4[q] = sp1[(ch - 2) * 4 + q];
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            u[8 * h + 2 * q] = cmul(u[8 * h + 2 * q], make_float2(s4[q].x, s4[q].y));
            u[8 * h + 2 * q + 1] = cmul(u[8 * h + 2 * q + 1], make_float2(s4[q].z, s4[q].w));
          }
          if (C::kNSB == 1 && ch == 0) {
            // one buffer: this thread's slots of chunk 0 are consumed, its part of chunk 1 follows
            const float4* src = spec_base + (size_t)k * C::kSpecPairs + (size_t)C::kChunkF4 + tid;
#pragma unroll
            for (int q = 0; q < 4; ++q) cp_async16(sbuf + tid + q * NT, src + q * NT);
            cp_async_commit();
          } else if (ch < 2) {
            // slot 0's chunks: the last warp to release the buffer refills it with
            // the next plane's chunk (a bulk copy a whole plane ahead); slot 1's
            // chunks come straight from L2 into registers (loaded at the plane start)
            __syncwarp();
            if (lane == 0) {
              __threadfence_block();
              const int b = C::kNSB == 2 ? ch : 0;
              int prev;
              asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(prev) : "r"(smem_addr(&s_rel[b])) : "memory");
              if (prev == C::NW - 1) {
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
          }
        }
        dft16_<true>(u);
#pragma unroll
        for (int q = 0; q < 16; ++q) g[q] = u[q];
      }
    }
    if constexpr (SPEC) continue;
    __syncwarp();

    // ---------------- I2: conjugate twiddle, inverse x DFT8 over j1, inverse y DFT4 over k2
    {
      float2 c[4][8];
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2)
#pragma unroll
        for (int j1 = 0; j1 < 8; ++j1) c[k2][j1] = b2_row[k2 * 2 * 8 * 17 + j1 * 17];
      __syncwarp();   // the warp's region is rewritten in the B1 layout below
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) {
#pragma unroll
        for (int j1 = 1; j1 < 8; ++j1) c[k2][j1] = cmulc(c[k2][j1], twt[j1 * 16 + m2]);
        dft8_<true>(c[k2]);
      }
#pragma unroll
      for (int m1 = 0; m1 < 8; ++m1) {
        float2 t[4] = {c[0][m1], c[1][m1], c[2][m1], c[3][m1]};
        dft4_<true>(t);
#pragma unroll
        for (int n2 = 0; n2 < 4; ++n2) c[n2][m1] = t[n2];
      }
      {
        const int k1 = 2 * warp + hi;
#pragma unroll
        for (int n2 = 1; n2 < 4; ++n2) {
          const float2 w = c_twy[n2 * 32 + k1];
#pragma unroll
          for (int m1 = 0; m1 < 8; ++m1) c[n2][m1] = cmulc(c[n2][m1], w);
        }
      }
#pragma unroll
      for (int n2 = 0; n2 < 4; ++n2)
#pragma unroll
        for (int m1 = 0; m1 < 8; ++m1) b1_row[n2 * P + 16 * m1] = c[n2][m1];
    }
    __syncthreads();

    // ---------------- I1: conjugate twiddle, inverse y DFT32, store of the window
    if (!i1_idle) {
      float2 v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int k1 = dft32p_freq(r);
        v[r] = b1_col[(k1 >> 1) * REG + (k1 & 1) * 4 * P];
      }
      dft32p_inv<true>(v);   // its conjugate y twiddle was applied in I2
      // window pixel (y - (my-1)) * QX + (x - (mx-1)); rows y = n2 + 4 n1 in
      // [my-1, y_end) are stored: a per-thread row mask (bit n1) and a running
      // pointer keep the unrolled store loop at one predicate test and one
      // 64-bit add per row
      const int ox = tx * a.QX + f_c;
      if (f_c < a.QX && ox < a.OW) {
        const int y_end = min(P, a.OH - ty * a.QY + (a.my - 1));
        const int lo = (max(0, a.my - 1 - f_n2) + 3) >> 2;
        const int hi = min(32, (max(0, y_end - f_n2) + 3) >> 2);
        const uint32_t below_hi = hi >= 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u);
        const uint32_t rows = hi > lo ? below_hi & ~((1u << lo) - 1u) : 0u;
        const ptrdiff_t e0 = (ptrdiff_t)k * a.wpx + (ptrdiff_t)(f_n2 - (a.my - 1)) * a.QX + f_c;
        if (a.chat16) {
          // 16-bit planes: int16 pairs at the unit's fixed-point scale (half the bytes)
          const float q = a.chat_q_T * (float)T;
          uint64_t pa = reinterpret_cast<uint64_t>(reinterpret_cast<uint32_t*>(chat_unit) + e0);
          const uint64_t step_b = (uint64_t)(4 * a.QX) * sizeof(uint32_t);
#pragma unroll
          for (int n1 = 0; n1 < 32; ++n1) {
            if ((rows >> n1) & 1u)
              asm volatile("st.global.b32 [%0], %1;" ::"l"(pa), "r"(pack16(v[n1], q)) : "memory");
            asm("add.s64 %0, %0, %1;" : "+l"(pa) : "l"(step_b));
          }
        } else {
        float2* dst = chat_unit + e0;
        // the running row address is kept in a register by inline PTX (left to
        // itself the compiler re-derives it from the kernel parameter every row)
        uint64_t pa = reinterpret_cast<uint64_t>(dst);
        const uint64_t step_b = (uint64_t)(4 * a.QX) * sizeof(float2);
#pragma unroll
        for (int n1 = 0; n1 < 32; ++n1) {
          if ((rows >> n1) & 1u)
            asm volatile("st.global.v2.f32 [%0], {%1, %2};" ::"l"(pa), "f"(v[n1].x), "f"(v[n1].y) : "memory");
          asm("add.s64 %0, %0, %1;" : "+l"(pa) : "l"(step_b));
        }
        }
      }
      // no barrier: the next plane's F1 writes exactly the slots this thread read
    } else if (tab_in_i1 && f_xb == 3 && k + 2 < *kend_s) {
      // plane k + 2's table into this plane's buffer (its F1 reads ended at the
      // F1 barrier; plane k + 1's barriers publish it)
      float2* M = enc_s + (k & 1) * (T + 1);
      const int kk = k + 2;
      for (int j = f_n2 * 32 + lane; j <= T; j += 128) M[j] = j < T ? enc_g[(kk * j) % T] : make_float2(0.f, 0.f);
    }
    ++pord;
  }
  if constexpr (!SPEC)
    fused_tail<NT>(a, chat_unit, img, unit, K, T, job.k_chunk, reinterpret_cast<float2*>(smem_raw),
                   (C::kBufBytes + C::kSpecBytes) / 8);
}

}  // namespace fm
