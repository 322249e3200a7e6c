// fm_abi.cu — plan construction, launch dispatch and the extern "C" ABI
// declared in include/fftmorph_b200.h.
//
// Host-side bookkeeping restates the reference's plan/range logic:
//   required_lr            umbra.py:172-174   (here with both data minima removed)
//   make_plan / ranges     fft_conv.py:80-91, tensor.py:76-101
//   reflect / negate       morphology.py:147-163 (erosion duality, l' = max f)
//   crop / _paste          morphology.py:51-62,131-140
// Kernels: fm_tile.cuh (encode + spatial FFT conv), fm_tonal.cuh (inverse
// tonal FFT + threshold + degree), fm_naive.cuh (exact direct oracle).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <functional>
#include <vector>

#include "fftmorph_b200.h"
#include "fm_bigtile.cuh"
#include "fm_direct.cuh"
#include "fm_fft64.cuh"
#include "fm_naive.cuh"
#include "fm_range.cuh"
#include "fm_tile.cuh"
#include "fm_tile128.cuh"
#include "fm_tonal.cuh"
#include "fm_tonal_coop.cuh"

using namespace fm;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};
std::mutex g_tw_mu;
unsigned long long g_tw_init_mask = 0;  // devices whose c_tw is initialised

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define FM_CUDA(call)                                                               \
  do {                                                                              \
    cudaError_t e_ = (call);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return fail(FM_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
  } while (0)

constexpr double kPi = 3.14159265358979323846;
constexpr int64_t kFp32CountBudget = 1 << 17;   // fm_plan_desc.count_budget default
constexpr int kChat16MaxCount = 2048;            // 16-bit spectral planes up to this many SE entries

int set_all_smem_attrs();

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled_fn() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(f);
  }
  return fn;
}
// [rows][wpx] float2 spectral scratch as a 2-D tensor of 8-byte elements; box {bx, by}
bool encode_chat_map(CUtensorMap* m, void* chat, int64_t wpx, int64_t rows, int bx, int by, int esz = 8) {
  EncodeTiledFn fn = encode_tiled_fn();
  if (!fn || bx < 1 || by < 1 || bx > 256 || by > 256) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)wpx, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)wpx * esz};
  const cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by};
  const cuuint32_t estr[2] = {1, 1};
  // 8-byte complex64 elements, or 4-byte int16 pairs (16-bit planes): the map only moves bytes
  return fn(m, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, chat, dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int ensure_twiddles(int device) {
  std::lock_guard<std::mutex> lk(g_tw_mu);
  if (device < 64 && (g_tw_init_mask >> device) & 1ull) return FM_OK;
  std::vector<float2> tw(kTwTotal);
  const int sizes[5] = {16, 32, 64, 128, 256};
  const int offs[5] = {0, 16, 48, 112, 240};
  for (int s = 0; s < 5; ++s)
    for (int j = 0; j < sizes[s]; ++j) {
      const double ang = -2.0 * kPi * j / sizes[s];
      tw[offs[s] + j] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    }
  FM_CUDA(cudaMemcpyToSymbol(c_tw, tw.data(), sizeof(float2) * kTwTotal));
  std::vector<float2> twy(4 * 32);
  for (int n2 = 0; n2 < 4; ++n2)
    for (int k1 = 0; k1 < 32; ++k1) {
      const double ang = -2.0 * kPi * (n2 * k1) / 128.0;
      twy[n2 * 32 + k1] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    }
  FM_CUDA(cudaMemcpyToSymbol(c_twy, twy.data(), sizeof(float2) * twy.size()));
  std::vector<float2> tt(kTonalTabTotal);
  for (int i = 0; i < kTonalCount; ++i) {
    const int n = kTonalNs[i], off = tonal_off(n);
    for (int j = 0; j < 2 * n; ++j) {
      const double ang = 2.0 * kPi * j / (2.0 * n);
      tt[off + j] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    }
  }
  FM_CUDA(cudaMemcpyToSymbol(c_ttw, tt.data(), sizeof(float2) * kTonalTabTotal));
  int rc = set_all_smem_attrs();
  if (rc) return rc;
  if (device < 64) g_tw_init_mask |= (1ull << device);
  return FM_OK;
}

bool smooth235(int n) {
  if (n < 1) return false;
  for (int p : {2, 3, 5})
    while (n % p == 0) n /= p;
  return n == 1;
}

std::vector<int> radix_plan(int n) {
  std::vector<int> r;
  while (n % 8 == 0) { r.push_back(8); n /= 8; }
  while (n % 4 == 0) { r.push_back(4); n /= 4; }
  while (n % 2 == 0) { r.push_back(2); n /= 2; }
  while (n % 3 == 0) { r.push_back(3); n /= 3; }
  while (n % 5 == 0) { r.push_back(5); n /= 5; }
  return r;
}

// ---- kernel variants ------------------------------------------------------
typedef void (*tile_launch_fn)(dim3, size_t, cudaStream_t, const TileArgs&);

template <int PY, int PX, int NT, bool TWO_D, bool SPEC>
void launch_tile(dim3 grid, size_t smem, cudaStream_t s, const TileArgs& a) {
  tile_conv_kernel<PY, PX, NT, TWO_D, SPEC><<<grid, NT, smem, s>>>(a);
}

template <int PY, int PX, int NT, bool TWO_D, bool SPEC>
cudaError_t set_smem_attr(size_t smem) {
  // the opt-in limit covers static + dynamic shared memory
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, tile_conv_kernel<PY, PX, NT, TWO_D, SPEC>);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(tile_conv_kernel<PY, PX, NT, TWO_D, SPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(smem - fa.sharedSizeBytes));
}

template <typename TV, bool SPEC>
void launch_tile128(dim3 grid, size_t smem, cudaStream_t s, const TileArgs& a) {
  tile128_kernel<TV, SPEC><<<grid, T128<TV>::NT, smem, s>>>(a);
}
template <typename TV, bool SPEC>
cudaError_t set_smem_attr128(size_t smem) {
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, tile128_kernel<TV, SPEC>);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(tile128_kernel<TV, SPEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(smem - fa.sharedSizeBytes));
}

struct Variant {
  int two_d, py, px, nt;
  int smem_fixed;
  tile_launch_fn conv, spec;
  cudaError_t (*attr_conv)(size_t);
  cudaError_t (*attr_spec)(size_t);
  int tmax;   // largest global tonal length the variant encodes (uint8 indices: 254)
};

#define FM_VARIANT(TD, PY, PX, NT)                                                        \
  Variant {                                                                               \
    TD, PY, PX, NT, TileCfg<PY, PX, NT, TD>::kSmemTotal, &launch_tile<PY, PX, NT, TD, false>, \
        &launch_tile<PY, PX, NT, TD, true>, &set_smem_attr<PY, PX, NT, TD, false>,          \
        &set_smem_attr<PY, PX, NT, TD, true>, 1 << 30                                       \
  }

#define FM_VARIANT128(TV)                                                                              \
  Variant {                                                                                            \
    true, 128, 128, T128<TV>::NT, T128<TV>::kSmemTotal, &launch_tile128<TV, false>, &launch_tile128<TV, true>, \
        &set_smem_attr128<TV, false>, &set_smem_attr128<TV, true>, T128<TV>::kTMax                      \
  }

// the three-pass 128x128 kernels (fm_tile128.cuh) come first: at equal cost the
// plan takes the uint8-index one when the tonal length fits it, else the
// uint16 one, else the four-pass kernel
const Variant kVariants[] = {
    FM_VARIANT128(uint8_t), FM_VARIANT128(uint16_t),
    FM_VARIANT(true, 16, 16, 32),   FM_VARIANT(true, 32, 32, 64),   FM_VARIANT(true, 64, 64, 256),
    FM_VARIANT(true, 128, 128, 512), FM_VARIANT(false, 8, 256, 64), FM_VARIANT(false, 16, 256, 128),
    FM_VARIANT(false, 32, 16, 64),  FM_VARIANT(false, 32, 32, 64),
    FM_VARIANT(false, 32, 64, 128),  FM_VARIANT(false, 32, 128, 128), FM_VARIANT(false, 32, 256, 256),
};

typedef void (*tonal_launch_fn)(dim3, int, size_t, cudaStream_t, const TonalArgs&);
template <int N, bool SM, int NT>
void launch_tonal(dim3 grid, int nt, size_t smem, cudaStream_t s, const TonalArgs& a) {
  tonal_kernel_t<N, SM, NT><<<grid, NT, smem, s>>>(a);
}
// long tonal axes: the cooperative kernel (fm_tonal_coop.cuh), several threads per pixel
template <int N>
void launch_tonal_coop(dim3 grid, int nt, size_t smem, cudaStream_t s, const TonalArgs& a) {
  if constexpr (coop_ok(N)) tonal_kernel_coop<N><<<grid, coop_threads(N), smem, s>>>(a);
}
template <int N>
constexpr bool tonal_sm() { return N > kTonalRegMax; }
template <int N>
constexpr int tonal_nt() { return N > kTonalRegMax ? 64 : 128; }

typedef void (*tonal_pipe_launch_fn)(dim3, int, size_t, cudaStream_t, const TonalArgs&, const CUtensorMap*);
struct TonalVariant {
  int n, nt, smem;
  tonal_launch_fn fn;
  // cooperative kernel (coop_ok(n)): threads, dynamic smem, launcher; 32 pixels per CTA
  int coop_nt, coop_smem;
  tonal_launch_fn coop_fn;
  cudaError_t (*attr)();
  // pipelined persistent kernel (register variants): threads, dynamic smem, launcher
  int pipe_nt, pipe_smem;
  tonal_pipe_launch_fn pipe_fn;
  cudaError_t (*pipe_attr)(int*);   // sets the smem attribute, returns CTAs per SM
};
template <int N>
void launch_tonal_pipe(dim3 grid, int nt, size_t smem, cudaStream_t s, const TonalArgs& a, const CUtensorMap* tms) {
  if constexpr (N <= kTonalRegMax)
    tonal_kernel_pipe<N, tonal_pipe_nt<N>(), tonal_pipe_st<N>()><<<grid, tonal_pipe_nt<N>() + 32, smem, s>>>(a, tms[0],
                                                                                                             tms[1]);
}
template <int N>
cudaError_t tonal_pipe_attr(int* occ) {
  occ[0] = occ[1] = 0;
  if constexpr (N <= kTonalRegMax) {
    auto k = tonal_kernel_pipe<N, tonal_pipe_nt<N>(), tonal_pipe_st<N>()>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, tonal_pipe_smem<N>());
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k, tonal_pipe_nt<N>() + 32, tonal_pipe_smem<N>());
    if (e != cudaSuccess) return e;
    // 16-bit planes: the stages hold 4-byte values, half the ring
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ + 1, k, tonal_pipe_nt<N>() + 32, tonal_pipe_smem<N>() / 2);
  }
  return cudaSuccess;
}
template <int N>
cudaError_t tonal_attr() {
  return cudaFuncSetAttribute(tonal_kernel_t<N, tonal_sm<N>(), tonal_nt<N>()>,
                              cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
}
#define FM_TV(N)                                                                                             \
  TonalVariant {                                                                                             \
    N, tonal_nt<N>(), tonal_sm<N>() ? 2 * N * tonal_nt<N>() * 8 : 0, &launch_tonal<N, tonal_sm<N>(), tonal_nt<N>()>, \
        coop_ok(N) ? coop_threads(N) : 0, coop_smem(N), &launch_tonal_coop<N>, &tonal_attr<N>, tonal_pipe_nt<N>(), tonal_pipe_smem<N>(), &launch_tonal_pipe<N>, &tonal_pipe_attr<N>      \
  }
const TonalVariant kTonal[] = {
    FM_TV(1),  FM_TV(2),  FM_TV(3),  FM_TV(4),  FM_TV(5),   FM_TV(6),   FM_TV(8),   FM_TV(9),   FM_TV(10),
    FM_TV(12), FM_TV(15), FM_TV(16), FM_TV(18), FM_TV(20),  FM_TV(24),  FM_TV(25),  FM_TV(27),  FM_TV(30),
    FM_TV(32), FM_TV(36), FM_TV(40), FM_TV(45), FM_TV(48),  FM_TV(50),  FM_TV(54),  FM_TV(60),  FM_TV(64),
    FM_TV(72), FM_TV(75), FM_TV(80), FM_TV(81), FM_TV(90),  FM_TV(96),  FM_TV(100), FM_TV(108), FM_TV(120),
    FM_TV(125), FM_TV(128), FM_TV(135), FM_TV(144), FM_TV(150), FM_TV(160)};
static_assert(sizeof(kTonal) / sizeof(TonalVariant) == kTonalCount, "tonal variant table");

constexpr int kAuxStreams = 7;
int g_tonal_pipe_occ[kTonalCount][2];   // CTAs per SM of each pipelined variant (0: not pipelined); [1]: 16-bit planes
int g_num_sms = 148;
const bool g_tonal_nopipe = std::getenv("FM_TONAL_NOPIPE") != nullptr;  // A/B switch for measurements
const bool g_no_skip0 = std::getenv("FM_NO_SKIP0") != nullptr;         // A/B: always compute plane 0
// pipelined tonal CTAs per SM (persistent grid); below the occupancy limit it
// leaves room for the next chunk's range CTAs
const int g_tonal_occ_cap = std::getenv("FM_TONAL_OCC") ? std::atoi(std::getenv("FM_TONAL_OCC")) : 64;
// fused tonal step (fm_fused.cuh): FM_FUSE=1 runs it (default: the separate tonal
// kernels, faster while both passes are FP32-issue-bound);
// FM_FUSE_KCH=<n> splits every unit's planes into chunks of n (0 = plan default);
// FM_DISCARD=0 keeps the consumed spectral lines in L2 (they are then written back)
const bool g_fuse = std::getenv("FM_FUSE") && std::getenv("FM_FUSE")[0] == '1';
const int g_fuse_kch = std::getenv("FM_FUSE_KCH") ? std::atoi(std::getenv("FM_FUSE_KCH")) : 0;
const bool g_discard = !(std::getenv("FM_DISCARD") && std::getenv("FM_DISCARD")[0] == '0');
// FM_DEVDISPATCH=0: small launches also wait on the host for the per-ladder counts (A/B)
const bool g_devdispatch = !(std::getenv("FM_DEVDISPATCH") && std::getenv("FM_DEVDISPATCH")[0] == '0');
// FM_BIG_JOBS=0: the 256^2 kernels launch a (plane, unit x image) grid instead of the compact job list (A/B)
const bool g_big_jobs = !(std::getenv("FM_BIG_JOBS") && std::getenv("FM_BIG_JOBS")[0] == '0');
// FM_BIG_PAIR=0: no Nyquist-plane pairing of neighbouring units on the 256^2 path (A/B)
const bool g_big_pair = !(std::getenv("FM_BIG_PAIR") && std::getenv("FM_BIG_PAIR")[0] == '0');
const int g_big_steps = std::getenv("FM_BIG_STEPS") ? std::atoi(std::getenv("FM_BIG_STEPS")) : 1;
// 256^2 path: L2 budget (MiB) of one unit batch's scratch items (FM_BIG_L2_MB; default 0 = one
// batch: measured slower at 96 / 48 / 24 MiB, the passes are latency bound, not HBM bound)
const int g_big_l2_mb = std::getenv("FM_BIG_L2_MB") ? std::atoi(std::getenv("FM_BIG_L2_MB")) : 0;
// FM_CHAT16=0 keeps complex64 spectral planes (A/B)
const bool g_chat16 = !(std::getenv("FM_CHAT16") && std::getenv("FM_CHAT16")[0] == '0');
// FM_OVERLAP=0: the tonal pass of a launch step and the next step's conv stay serialised (A/B)
const bool g_overlap = !(std::getenv("FM_OVERLAP") && std::getenv("FM_OVERLAP")[0] == '0');
// FM_GRAPH=0: small calls launch their kernels one by one instead of replaying a graph (A/B)
const bool g_graph = !(std::getenv("FM_GRAPH") && std::getenv("FM_GRAPH")[0] == '0');
// FM_RANGE_ALIGNED=0: the range kernel stages uint8 windows pixel by pixel (A/B)
const bool g_range_aligned = !(std::getenv("FM_RANGE_ALIGNED") && std::getenv("FM_RANGE_ALIGNED")[0] == '0');
// FM_RANGE_WIN8=0: the range kernel always stages int16 windows (A/B)
const bool g_range_win8 = !(std::getenv("FM_RANGE_WIN8") && std::getenv("FM_RANGE_WIN8")[0] == '0');
const int g_range_splits = std::getenv("FM_RANGE_SPLITS") ? std::atoi(std::getenv("FM_RANGE_SPLITS")) : 0;   // A/B: CTAs per unit
const int g_range_sync = std::getenv("FM_RANGE_SYNC") ? std::atoi(std::getenv("FM_RANGE_SYNC")) : 0;
// largest N served by the pipelined tonal kernel (beyond it the register
// pressure of the per-pixel FFT leaves too few warps to cover the stream)
// FM_TONAL_COOP=0: long tonal axes (40 < N <= 160) by the one-thread-per-pixel kernels (A/B)
const bool g_tonal_coop = !(std::getenv("FM_TONAL_COOP") && std::getenv("FM_TONAL_COOP")[0] == '0');
// largest number of 128-pixel items for which the N <= 40 ladder entries of a launch step go in
// one device-dispatched launch (FM_TONAL_DISP_MAX; 0 = always one pipelined launch per entry)
const int g_tonal_disp_max = std::getenv("FM_TONAL_DISP_MAX") ? std::atoi(std::getenv("FM_TONAL_DISP_MAX")) : 16384;
// smallest N served by the cooperative kernel (FM_TONAL_COOP_MIN), conv grid target in CTAs per SM slot
const int g_tonal_coop_min = std::getenv("FM_TONAL_COOP_MIN") ? std::atoi(std::getenv("FM_TONAL_COOP_MIN")) : 41;
const int g_conv_waves = std::getenv("FM_CONV_WAVES") ? std::atoi(std::getenv("FM_CONV_WAVES")) : 4;
// smallest N served by the pipelined tonal kernel (FM_TONAL_PIPE_MIN; measured at c4, N = 1:
// the one-thread-per-pixel kernel is slower, 0.065 vs 0.038 ms, so the default keeps every N)
const int g_tonal_pipe_min = std::getenv("FM_TONAL_PIPE_MIN") ? std::atoi(std::getenv("FM_TONAL_PIPE_MIN")) : 0;
// longest tonal axis (N) served by tonal_kernel_rows instead of the pipelined kernel (FM_TONAL_ROWS_MAX; 0 = off)
const int g_tonal_rows_max = std::getenv("FM_TONAL_ROWS_MAX") ? std::atoi(std::getenv("FM_TONAL_ROWS_MAX")) : 4;
// FM_TONAL_HALF_RING=0: the pipelined tonal kernel keeps the complex64-sized ring with 16-bit planes (A/B)
const bool g_tonal_half_ring = !(std::getenv("FM_TONAL_HALF_RING") && std::getenv("FM_TONAL_HALF_RING")[0] == '0');
const int g_tonal_pipe_max = std::getenv("FM_TONAL_PIPE_MAX") ? std::atoi(std::getenv("FM_TONAL_PIPE_MAX")) : 40;

const TonalVariant* find_tonal(int n) {
  for (const TonalVariant& v : kTonal)
    if (v.n == n) return &v;
  return nullptr;
}

int dtype_size(int dt) { return dt == FM_U8 ? 1 : dt == FM_U16 ? 2 : 4; }

constexpr int kSmemLimit = 227 * 1024;

int set_all_smem_attrs() {
  for (const Variant& v : kVariants) {
    FM_CUDA(v.attr_conv(kSmemLimit));
    FM_CUDA(v.attr_spec(kSmemLimit));
  }
  for (int i = 0; i < kTonalCount; ++i) {
    FM_CUDA(kTonal[i].attr());
    FM_CUDA(kTonal[i].pipe_attr(g_tonal_pipe_occ[i]));
  }
  {
    int dev = 0;
    FM_CUDA(cudaGetDevice(&dev));
    FM_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  FM_CUDA(cudaFuncSetAttribute(tonal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
  FM_CUDA(cudaFuncSetAttribute(range_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRangeSmemMax));
  FM_CUDA(cudaFuncSetAttribute(range_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRangeSmemMax));
  FM_CUDA(cudaFuncSetAttribute(range_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRangeSmemMax));
  FM_CUDA(cudaFuncSetAttribute(range_kernel<0, int8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRangeSmemMax));
  FM_CUDA(cudaFuncSetAttribute(range_kernel<1, int8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRangeSmemMax));
  FM_CUDA(cudaFuncSetAttribute(range_kernel<2, int8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRangeSmemMax));
  FM_CUDA(cudaFuncSetAttribute(big_rows_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
  FM_CUDA(cudaFuncSetAttribute(big_rows_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
  FM_CUDA(cudaFuncSetAttribute(big_rows_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
  FM_CUDA(cudaFuncSetAttribute(big_cols_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
  FM_CUDA(cudaFuncSetAttribute(big_cols_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
  return FM_OK;
}

}  // namespace

struct fm_plan {
  fm_plan_desc d{};
  int device = 0;
  bool two_d = true;
  int64_t H = 1, W = 1, batch = 1;
  int my = 1, mx = 1;
  int64_t lo_y = 0, lo_x = 0;  // lo of the SE actually convolved (reflected for erosion)
  int se_min = 0, se_max = 0, se_count = 0;
  int lr = 0, T = 0, N = 0, K = 0;
  std::vector<int> radix;
  const Variant* var = nullptr;
  int PY = 1, PX = 16, QY = 1, QX = 1, tiles_y = 1, tiles_x = 1, tiles_total = 1, tile_ctas = 1;
  int DY = 0, DX = 0;
  int64_t OH = 1, OW = 1, off_y = 0, off_x = 0;
  int k_chunk = 1, kchunks = 1;
  int conv_occ = 1;  // conv CTAs per SM
  int64_t ipc = 1;  // images per launch
  size_t conv_smem = 0, tonal_smem = 0;
  int tonal_threads = 128, tonal_stride = 1;
  int enc_sign = 1, enc_bias = 0, vmax = 0;
  int out_sign = 1;
  // device buffers
  float4* spec = nullptr;
  float2* twN = nullptr;
  float2* wT = nullptr;
  float2* chat = nullptr;
  int* stats = nullptr;  // [0] = deviation bits, [1] = value error
  int32_t* se_vals_d = nullptr;
  uint8_t* se_def_d = nullptr;
  // host-buffer path staging
  void* h_img = nullptr;
  uint8_t* h_def = nullptr;
  int32_t* h_out = nullptr;
  uint8_t* h_valid = nullptr;
  cudaStream_t last_stream = nullptr;
  // event timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;                  // reusable events
  std::vector<std::pair<int, int>> pending_conv, pending_tonal, pending_range;  // (start, stop) indices into ev_pool
  size_t ev_next = 0;
  fm_timing acc{};
  double conv_flops_per_plane = 0;  // per unit and plane
  // per-unit tonal length: ladder of supported N (ascending), one SE spectrum each
  std::vector<int> ladder;
  std::vector<int64_t> spec_off;          // float4 offsets into spec
  std::vector<const TonalVariant*> ladder_var;
  // per ladder entry: 2-D tensor maps of the spectral scratch for the pipelined
  // tonal kernel (box {pipe_nt pixels, K planes} and {pipe_nt, K-1}); empty: per-plane copies
  std::vector<CUtensorMap> tmaps;
  int units = 1, wpx = 1, npx = 1, win_y = 1, win_x = 1, unit_step_x = 0;  // wpx: even plane stride
  std::vector<int2> taps;                 // clamp-bound taps of fm_range.cuh, best first
  std::vector<int> full_prefix;           // prefix count of "full" units (window inside the image)
  // range outputs are double-buffered so the range kernel of the next launch
  // chunk runs on its own low-priority stream while this chunk's conv / tonal
  // kernels still read the current set
  int* range_part[2] = {};                // [ipc*units][8] split partials of fm_range.cuh
  bool counts = false;                    // FM_FLAG_COUNTS: count-volume output
  float2* enc_tab = nullptr;              // per ladder entry: exp(-2 pi i j / T), j < T, then 0
  int* d_enc_off = nullptr;               // [L] offsets into enc_tab
  std::vector<int> enc_off;
  int upl = 1;                            // units per launch (chat slots per image)
  int* d_ladder = nullptr;
  int64_t* d_spec_off = nullptr;
  int4* unit_param[2] = {};               // [ipc][units]
  int* bucket_count[2] = {};              // [L]
  int2* bucket_list[2] = {};              // [L][ipc*units]
  int* h_counts[2] = {};                  // mapped pinned [L], written by publish_counts
  int* h_counts_dev[2] = {};              // their device aliases
  cudaEvent_t count_ev[2] = {};           // range + counts of a buffer set done (on range_stream)
  cudaEvent_t free_ev[2] = {};            // conv + tonal done with a buffer set (on the caller's stream)
  cudaEvent_t entry_ev = nullptr;
  cudaStream_t range_stream = nullptr;
  cudaStream_t aux[kAuxStreams] = {};     // tonal launches side by side
  cudaEvent_t ev_fork = nullptr, ev_join[kAuxStreams] = {};
  int64_t planes_done = 0, units_done = 0; // for the plan's mean planes per unit
  // 256x256 tiles through an HBM scratch (fm_bigtile.cuh) for wide SEs
  bool big = false;
  float2* S = nullptr;
  int2* big_jobs = nullptr;        // 256^2 path: compact (image, unit, plane) job list + counter
  int* big_njobs = nullptr;
  int64_t big_jobs_cap = 0;
  // composite plan (SE wider than one tile, fm_plan_create): dilation by B = U B_i is the
  // max over the parts' dilations (erosion: min), validity OR-ed
  std::vector<fm_plan*> parts;
  void* part_out = nullptr;               // [batch][OH][OW] of out_dtype
  uint8_t* part_valid = nullptr;          // [batch][OH][OW]
  uint8_t* acc_valid = nullptr;           // [batch][OH][OW] when the caller passes no validity
  // one-launch-step calls sized on the device replay a captured CUDA graph (keyed on the
  // buffers and the stream): no per-kernel host launches, smaller gaps between the kernels
  bool graphable = false, capturing = false;
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t gstream = nullptr;
  cudaEvent_t gev_in = nullptr, gev_out = nullptr;
  int gmiss = 0;                          // captures so far (new buffer sets)
  bool gstaged = false;                   // graph on plan-owned staging buffers
  void* g_img = nullptr;
  uint8_t* g_def = nullptr;
  void* g_out = nullptr;
  uint8_t* g_valid = nullptr;
  const void* gkey[5] = {};
  int64_t graph_kernels = 0;
  // conv of launch step i+1 overlapping the tonal pass of step i: two spectral buffer sets
  // (chat16 keeps their sum within the scratch budget), the tonal passes on their own stream
  bool overlap = false;
  size_t chat_set_bytes = 0;
  cudaStream_t tstream = nullptr;
  cudaEvent_t conv_ev[2] = {}, tjoin_ev = nullptr;
  // 16-bit spectral planes (chat16): int16 pairs at scale q = chat_q_T * T (see fm_plan_create)
  bool chat16 = false;
  float chat_q_T = 0.f, chat_invq_T = 0.f;
  // fused tonal step (fm_fused.cuh): ladder entries with N <= fuse_nmax finish in the conv kernel
  int fuse_nmax = 0;
  int* unit_done = nullptr;               // [ipc][upl] plane-chunk completion counters
  // host-buffer pipeline
  cudaStream_t copy_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_done = nullptr;
  std::vector<cudaEvent_t> ev_chunks;     // per chunk: input landed, compute done
};

namespace {

void free_plan(fm_plan* p) {
  if (!p) return;
  for (fm_plan* q : p->parts) free_plan(q);
  p->parts.clear();
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  cudaFree(p->part_out);
  cudaFree(p->part_valid);
  cudaFree(p->acc_valid);
  cudaFree(p->spec);
  cudaFree(p->twN);
  cudaFree(p->wT);
  cudaFree(p->chat);
  cudaFree(p->stats);
  cudaFree(p->se_vals_d);
  cudaFree(p->se_def_d);
  cudaFree(p->h_img);
  cudaFree(p->h_def);
  cudaFree(p->h_out);
  cudaFree(p->h_valid);
  for (cudaEvent_t e : p->ev_pool) cudaEventDestroy(e);
  cudaFree(p->d_ladder);
  cudaFree(p->d_spec_off);
  for (int b = 0; b < 2; ++b) {
    cudaFree(p->range_part[b]);
    cudaFree(p->unit_param[b]);
    cudaFree(p->bucket_count[b]);
    cudaFree(p->bucket_list[b]);
    if (p->h_counts[b]) cudaFreeHost(p->h_counts[b]);
    if (p->count_ev[b]) cudaEventDestroy(p->count_ev[b]);
    if (p->free_ev[b]) cudaEventDestroy(p->free_ev[b]);
  }
  if (p->entry_ev) cudaEventDestroy(p->entry_ev);
  if (p->range_stream) cudaStreamDestroy(p->range_stream);
  cudaFree(p->enc_tab);
  cudaFree(p->d_enc_off);
  cudaFree(p->unit_done);
  if (p->gexec) cudaGraphExecDestroy(p->gexec);
  cudaFree(p->g_img);
  cudaFree(p->g_def);
  cudaFree(p->g_out);
  cudaFree(p->g_valid);
  if (p->gstream) cudaStreamDestroy(p->gstream);
  if (p->gev_in) cudaEventDestroy(p->gev_in);
  if (p->gev_out) cudaEventDestroy(p->gev_out);
  if (p->tstream) cudaStreamDestroy(p->tstream);
  for (int b = 0; b < 2; ++b)
    if (p->conv_ev[b]) cudaEventDestroy(p->conv_ev[b]);
  if (p->tjoin_ev) cudaEventDestroy(p->tjoin_ev);
  cudaFree(p->S);
  cudaFree(p->big_jobs);
  cudaFree(p->big_njobs);
  if (p->copy_stream) cudaStreamDestroy(p->copy_stream);
  if (p->d2h_stream) cudaStreamDestroy(p->d2h_stream);
  for (cudaEvent_t e : p->ev_chunks) cudaEventDestroy(e);
  if (p->ev_in) cudaEventDestroy(p->ev_in);
  if (p->ev_done) cudaEventDestroy(p->ev_done);
  if (p->ev_fork) cudaEventDestroy(p->ev_fork);
  for (int i = 0; i < kAuxStreams; ++i) {
    if (p->aux[i]) cudaStreamDestroy(p->aux[i]);
    if (p->ev_join[i]) cudaEventDestroy(p->ev_join[i]);
  }
  cudaSetDevice(prev);
  delete p;
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

cudaEvent_t next_event(fm_plan* p) {
  if (p->ev_next == p->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    p->ev_pool.push_back(e);
  }
  return p->ev_pool[p->ev_next++];
}

int validate_common(const fm_plan_desc* d) {
  if (!d) return fail(FM_EINVAL, "null descriptor");
  if (d->ndim != 1 && d->ndim != 2) return fail(FM_EUNSUPPORTED, "only 1-D signals and 2-D images are supported");
  if (d->mode != FM_DILATE && d->mode != FM_ERODE) return fail(FM_EINVAL, "mode must be FM_DILATE or FM_ERODE");
  if (d->img_dtype < FM_U8 || d->img_dtype > FM_I32) return fail(FM_EINVAL, "bad image dtype");
  if (d->batch < 1) return fail(FM_EINVAL, "batch must be >= 1");
  for (int i = 0; i < d->ndim; ++i) {
    if (d->shape[i] < 1) return fail(FM_EINVAL, "empty grid");
    if (d->se_shape[i] < 1) return fail(FM_EINVAL, "empty structuring element");
    if (d->shape[i] > (1 << 30) || d->se_shape[i] > (1 << 30)) return fail(FM_EUNSUPPORTED, "extent too large");
  }
  return FM_OK;
}

}  // namespace

// validity-aware max (dilation) / min (erosion) of a part into the accumulated result
template <typename T>
__global__ void combine_kernel(T* __restrict__ out, uint8_t* __restrict__ valid, const T* __restrict__ part,
                               const uint8_t* __restrict__ pvalid, int64_t n, int erode) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!pvalid[i]) continue;
    const T v = part[i];
    if (!valid[i]) {
      out[i] = v;
      valid[i] = 1;
    } else {
      const T o = out[i];
      out[i] = erode ? (v < o ? v : o) : (v > o ? v : o);
    }
  }
}

int out_elem_size(int od) { return od == FM_OUT_U8 ? 1 : (od == FM_OUT_U16 || od == FM_OUT_I16) ? 2 : 4; }

// Largest SE extent per axis served by one plan (the 256x256 tile path); wider SEs are
// split into blocks of at most kSplitEdge (so each block keeps a useful 256-tile window).
constexpr int kMaxSeEdge = 256;
constexpr int kSplitEdge = 128;

extern "C" int fm_plan_create(fm_plan** out_plan, const fm_plan_desc* desc, const int32_t* se_values,
                              const uint8_t* se_defined);

// Composite plan: the SE is cut into blocks B_i (each with its own lo), one plan per non-empty
// block, all writing the parent's output window (crop = 2); exact because a dilation by a
// union of SEs is the max of the dilations (erosion: the min), a pixel being valid if any
// part has a pair there (morphology.py:65-113 semantics per part).
int create_composite(fm_plan** out_plan, const fm_plan_desc& d, const int32_t* se_values, const uint8_t* se_defined) {
  const bool two_d = d.ndim == 2;
  const int64_t my = two_d ? d.se_shape[0] : 1, mx = two_d ? d.se_shape[1] : d.se_shape[0];
  const int64_t H = two_d ? d.shape[0] : 1, W = two_d ? d.shape[1] : d.shape[0];
  const int64_t lo_y = two_d ? d.se_lo[0] : 0, lo_x = two_d ? d.se_lo[1] : d.se_lo[0];
  // the parent's output window, as a single plan would place it (crop / Minkowski range)
  int64_t wy = 0, wx = 0, oh = H, ow = W;
  if (d.crop == 2) {
    wy = two_d ? d.win_lo[0] : 0;
    wx = two_d ? d.win_lo[1] : d.win_lo[0];
    oh = two_d ? d.win_shape[0] : 1;
    ow = two_d ? d.win_shape[1] : d.win_shape[0];
  } else if (!d.crop) {
    const bool er = d.mode == FM_ERODE;
    wy = two_d ? (er ? -(lo_y + my - 1) : lo_y) : 0;
    wx = er ? -(lo_x + mx - 1) : lo_x;
    oh = two_d ? H + my - 1 : 1;
    ow = W + mx - 1;
  }
  const int64_t ny = (my + kSplitEdge - 1) / kSplitEdge, nx = (mx + kSplitEdge - 1) / kSplitEdge;
  const int64_t by = (my + ny - 1) / ny, bx = (mx + nx - 1) / nx;
  fm_plan* p = new fm_plan();
  p->d = d;
  p->device = d.device;
  p->two_d = two_d;
  p->batch = d.batch;
  p->H = H;
  p->W = W;
  p->my = (int)my;
  p->mx = (int)mx;
  p->OH = oh;
  p->OW = ow;
  p->off_y = wy;
  p->off_x = wx;
  int smin = INT32_MAX, smax = INT32_MIN, cnt = 0;
  for (int64_t i = 0; i < my * mx; ++i)
    if (!se_defined || se_defined[i]) {
      smin = std::min(smin, se_values[i]);
      smax = std::max(smax, se_values[i]);
      ++cnt;
    }
  if (cnt == 0) { delete p; return fail(FM_EINVAL, "grid needs at least one defined pixel"); }
  p->se_min = smin;
  p->se_max = smax;
  p->se_count = cnt;
  for (int64_t y0 = 0; y0 < my; y0 += by)
    for (int64_t x0 = 0; x0 < mx; x0 += bx) {
      const int64_t sh = std::min(by, my - y0), sw = std::min(bx, mx - x0);
      std::vector<int32_t> v((size_t)(sh * sw));
      std::vector<uint8_t> m((size_t)(sh * sw));
      bool any = false;
      for (int64_t yy = 0; yy < sh; ++yy)
        for (int64_t xx = 0; xx < sw; ++xx) {
          const int64_t src = (y0 + yy) * mx + (x0 + xx);
          v[(size_t)(yy * sw + xx)] = se_values[src];
          m[(size_t)(yy * sw + xx)] = se_defined ? (se_defined[src] ? 1 : 0) : 1;
          any = any || m[(size_t)(yy * sw + xx)];
        }
      if (!any) continue;
      fm_plan_desc c = d;
      c.crop = 2;
      if (two_d) {
        c.se_shape[0] = sh;
        c.se_shape[1] = sw;
        c.se_lo[0] = lo_y + y0;
        c.se_lo[1] = lo_x + x0;
        c.win_lo[0] = wy;
        c.win_lo[1] = wx;
        c.win_shape[0] = oh;
        c.win_shape[1] = ow;
      } else {
        c.se_shape[0] = sw;
        c.se_lo[0] = lo_x + x0;
        c.win_lo[0] = wx;
        c.win_shape[0] = ow;
      }
      fm_plan* q = nullptr;
      const int rc = fm_plan_create(&q, &c, v.data(), m.data());
      if (rc) {
        const std::string msg = g_err;
        free_plan(p);
        return fail(rc, "SE block plan: " + msg);
      }
      p->parts.push_back(q);
    }
  DeviceGuard dg(p->device);
  const size_t n = (size_t)p->batch * oh * ow;
  cudaError_t e = cudaMalloc(&p->part_out, n * out_elem_size(d.out_dtype));
  if (e == cudaSuccess) e = cudaMalloc(&p->part_valid, n);
  if (e == cudaSuccess) e = cudaMalloc(&p->acc_valid, n);
  if (e != cudaSuccess) {
    free_plan(p);
    return fail(FM_ENOMEM, std::string("composite buffers: ") + cudaGetErrorString(e));
  }
  *out_plan = p;
  return FM_OK;
}

extern "C" {

int fm_abi_version(void) { return FM_ABI_VERSION; }
const char* fm_last_error(void) { return g_err.c_str(); }
int64_t fm_kernel_launches(void) { return (int64_t)g_launches.load(); }

int fm_plan_create(fm_plan** out_plan, const fm_plan_desc* desc, const int32_t* se_values,
                   const uint8_t* se_defined) {
  if (!out_plan) return fail(FM_EINVAL, "null plan pointer");
  *out_plan = nullptr;
  int rc = validate_common(desc);
  if (rc) return rc;
  if (!se_values) return fail(FM_EINVAL, "null SE values");
  const fm_plan_desc& d = *desc;
  if (d.img_min > d.img_max) return fail(FM_EINVAL, "img_min > img_max");

  if (d.flags & ~FM_FLAG_COUNTS) return fail(FM_EINVAL, "unknown flags");
  if ((d.flags & FM_FLAG_COUNTS) && (d.mode != FM_DILATE || d.crop))
    return fail(FM_EINVAL, "count volumes need mode=dilate and crop=0");
  if (d.crop < 0 || d.crop > 2) return fail(FM_EINVAL, "crop must be 0, 1 or 2");
  if (d.crop == 2)
    for (int i = 0; i < d.ndim; ++i)
      if (d.win_shape[i] < 1 || d.win_shape[i] > (1 << 30) || d.win_lo[i] < -(1 << 30) || d.win_lo[i] > (1 << 30))
        return fail(FM_EINVAL, "crop=2 needs a non-empty output window within +-2^30");
  {
    const bool wide = d.ndim == 2 ? (d.se_shape[0] > kMaxSeEdge || d.se_shape[1] > kMaxSeEdge)
                                  : d.se_shape[0] > kMaxSeEdge;
    if (wide && (d.flags & FM_FLAG_COUNTS))
      return fail(FM_EUNSUPPORTED, "count volumes need an SE within one tile (<= 256 per axis)");
    if (wide) return create_composite(out_plan, d, se_values, se_defined);
  }
  fm_plan* p = new fm_plan();
  p->d = d;
  p->counts = (d.flags & FM_FLAG_COUNTS) != 0;
  p->device = d.device;
  p->two_d = d.ndim == 2;
  p->batch = d.batch;
  if (p->two_d) {
    p->H = d.shape[0];
    p->W = d.shape[1];
    p->my = (int)d.se_shape[0];
    p->mx = (int)d.se_shape[1];
  } else {
    p->H = 1;
    p->W = d.shape[0];
    p->my = 1;
    p->mx = (int)d.se_shape[0];
  }
  const int64_t se_n = (int64_t)p->my * p->mx;
  // SE as convolved: reflected for erosion (reflect(b), morphology.py:147-152)
  std::vector<int32_t> sv(se_n);
  std::vector<uint8_t> sd(se_n);
  for (int64_t i = 0; i < se_n; ++i) {
    const int64_t src = (d.mode == FM_ERODE) ? (se_n - 1 - i) : i;
    sv[i] = se_values[src];
    sd[i] = se_defined ? (se_defined[src] ? 1 : 0) : 1;
  }
  int64_t lo_y = p->two_d ? d.se_lo[0] : 0, lo_x = p->two_d ? d.se_lo[1] : d.se_lo[0];
  if (d.mode == FM_ERODE) {
    lo_y = -(lo_y + p->my - 1);
    lo_x = -(lo_x + p->mx - 1);
  }
  p->lo_y = lo_y;
  p->lo_x = lo_x;
  int smin = INT32_MAX, smax = INT32_MIN, cnt = 0;
  for (int64_t i = 0; i < se_n; ++i)
    if (sd[i]) {
      smin = std::min(smin, sv[i]);
      smax = std::max(smax, sv[i]);
      ++cnt;
    }
  if (cnt == 0) { free_plan(p); return fail(FM_EINVAL, "grid needs at least one defined pixel"); }
  if (smin < 0) { free_plan(p); return fail(FM_EINVAL, "tonal lift needs non-negative values"); }
  p->se_min = smin;
  p->se_max = smax;
  p->se_count = cnt;
  {
    // a-priori precision budget (fft_conv.py:114-125 restated for FP32): a count is the
    // number of (image, SE) pairs meeting at one degree, at most the defined SE entries
    // (and the image pixels).  The FP32 pipeline's measured worst deviation grows ~2e-7 per
    // unit of count (c4: 9.8e-4 at 5123), so below 2^17 it stays < 0.03, a 10x margin to
    // the reference's 0.25 abort threshold.
    const int64_t budget = d.count_budget > 0 ? d.count_budget : kFp32CountBudget;
    const int64_t npx = (p->two_d ? p->H : 1) * p->W;
    const int64_t bound = std::min<int64_t>(cnt, npx);
    if (bound >= budget) {
      free_plan(p);
      char buf[200];
      std::snprintf(buf, sizeof buf, "count bound %lld >= FP32 budget %lld; split the structuring element",
                    (long long)bound, (long long)budget);
      return fail(FM_EPRECISION, buf);
    }
  }

  // tonal extent: only the spread of values matters (dilation commutes with
  // constant shifts of f and b); l_R of the reference is max f + max b.
  const int64_t lr64 = (int64_t)(d.img_max - d.img_min) + (smax - smin);
  if (lr64 > 100000) { free_plan(p); return fail(FM_EUNSUPPORTED, "tonal range too large for the FFT path"); }
  p->lr = (int)lr64;
  // encode / decode
  if (d.mode == FM_DILATE) {
    p->enc_sign = 1;
    p->enc_bias = -d.img_min;
    p->out_sign = 1;
  } else {
    p->enc_sign = -1;
    p->enc_bias = d.img_max;
    p->out_sign = -1;
  }
  p->vmax = d.img_max - d.img_min;
  {
    // every possible output value must fit the requested output type
    const int64_t lo = d.mode == FM_DILATE ? (int64_t)d.img_min + smin : (int64_t)d.img_min - smax;
    const int64_t hi = d.mode == FM_DILATE ? (int64_t)d.img_max + smax : (int64_t)d.img_max - smin;
    const int64_t vlo = std::min<int64_t>(lo, d.fill), vhi = std::max<int64_t>(hi, d.fill);
    int64_t tlo = INT32_MIN, thi = INT32_MAX;
    if (d.out_dtype == FM_OUT_U8) { tlo = 0; thi = 255; }
    else if (d.out_dtype == FM_OUT_U16) { tlo = 0; thi = 65535; }
    else if (d.out_dtype == FM_OUT_I16) { tlo = -32768; thi = 32767; }
    else if (d.out_dtype != FM_OUT_I32) { free_plan(p); return fail(FM_EINVAL, "bad out_dtype"); }
    if (vlo < tlo || vhi > thi) { free_plan(p); return fail(FM_EINVAL, "output values do not fit out_dtype"); }
  }

  // tonal length: even, > l_R, with T/2 5-smooth
  int T = d.tonal_len;
  if (T > 0) {
    if (T % 2 || T < p->lr + 1 || !smooth235(T / 2)) {
      free_plan(p);
      return fail(FM_EINVAL, "forced tonal_len must be even, > l_R and have a 2-3-5-smooth half");
    }
  } else {
    T = std::max(2, p->lr + 1);
    if (T % 2) ++T;
    while (!smooth235(T / 2)) T += 2;
  }
  p->T = T;
  p->N = T / 2;
  p->K = p->N + 1;
  p->radix = radix_plan(p->N);
  if (p->radix.size() > 12) { free_plan(p); return fail(FM_EUNSUPPORTED, "tonal radix plan too deep"); }

  // output region and overlap-save offsets (tensor.py:76-101, morphology.py:131-140)
  const int64_t hi_y = lo_y + p->my - 1, hi_x = lo_x + p->mx - 1;
  if (d.crop == 2) {
    // explicit output window (row strips): any placement relative to the image
    p->off_y = p->two_d ? d.win_lo[0] : 0;
    p->off_x = p->two_d ? d.win_lo[1] : d.win_lo[0];
    p->OH = p->two_d ? d.win_shape[0] : 1;
    p->OW = p->two_d ? d.win_shape[1] : d.win_shape[0];
  } else if (d.crop) {
    p->off_y = 0;
    p->off_x = 0;
    p->OH = p->H;
    p->OW = p->W;
  } else {
    p->off_y = p->two_d ? lo_y : 0;
    p->off_x = lo_x;
    p->OH = p->two_d ? p->H + p->my - 1 : 1;
    p->OW = p->W + p->mx - 1;
  }
  const int64_t DY = p->off_y - hi_y, DX = p->off_x - hi_x;
  if (DY < -(1 << 30) || DY > (1 << 30) || DX < -(1 << 30) || DX > (1 << 30)) {
    free_plan(p);
    return fail(FM_EUNSUPPORTED, "SE offset too large");
  }
  p->DY = p->two_d ? (int)DY : 0;
  p->DX = (int)DX;

  // tile choice: minimise the estimated time over the built variants.  Per (tile, plane) a
  // CTA costs c(P) = P^2 (log2 P^2 + 2) + overhead; a launch of J such jobs with `occ` CTAs
  // per SM takes ceil(J / (SMs occ)) waves of occ * c(P): the throughput form J c(P) / SMs
  // for large batches (c5, c3), and for small images (latency bound: fewer jobs than the
  // GPU holds) the per-CTA latency, where smaller tiles win.  Planes per tile after the
  // clamp are not known yet: estimated as K / 3.
  const double kest = std::max(1.0, std::ceil((double)p->K / 3.0));
  double best = 1e300;
  const Variant* bv = nullptr;
  // FM_TILE3=0 disables the three-pass 128x128 kernel (A/B measurements)
  const char* t3env = std::getenv("FM_TILE3");
  const bool allow_t3 = !(t3env && t3env[0] == '0');
  for (const Variant& v : kVariants) {
    if ((bool)v.two_d != p->two_d) continue;
    if (v.tmax < (1 << 30) && (!allow_t3 || p->T > v.tmax)) continue;
    const int P = v.px;
    if (d.tile > 0 && d.tile != P) continue;
    if (P < p->mx || (p->two_d && P < p->my)) continue;
    const int qx = P - p->mx + 1, qy = p->two_d ? P - p->my + 1 : 1;
    const double tx = std::ceil((double)p->OW / qx), ty = p->two_d ? std::ceil((double)p->OH / qy) : 1.0;
    const double pts = p->two_d ? (double)P * P : (double)P;
    const double occ = std::max(1, std::min(kSmemLimit / (v.smem_fixed + 1024), 2048 / v.nt));
    const double units = p->two_d ? tx * ty : std::ceil(tx / v.py);   // 1-D: py tiles per CTA
    const double jobs = units * (double)p->batch * kest;
    const double per = (p->two_d ? 1.0 : (double)v.py) * (pts * (std::log2(pts) + 2.0) + 2048.0);
    // CTAs actually sharing an SM in a wave (a lone CTA gets the SM to itself)
    const double resident = std::min(occ, std::ceil(jobs / (double)g_num_sms));
    const double cost = std::ceil(jobs / ((double)g_num_sms * occ)) * resident * per;
    if (cost < best) {
      best = cost;
      bv = &v;
    }
  }
  // 256x256 tiles (three kernels through HBM) pay ~1.7x per point but win for wide SEs
  if (p->two_d && p->my <= kBig && p->mx <= kBig && (d.tile == 0 || d.tile == kBig)) {
    const int q = kBig - p->mx + 1, qy = kBig - p->my + 1;
    const double tx = std::ceil((double)p->OW / q), ty = std::ceil((double)p->OH / qy);
    const double pts = (double)kBig * kBig;
    const double cost = 1.7 * tx * ty * (double)p->batch * kest * (pts * (std::log2(pts) + 2.0) + 2048.0) /
                        (double)g_num_sms;
    if (cost < best || d.tile == kBig) {
      best = cost;
      p->big = true;
    }
  }
  if (!bv && !p->big) {
    free_plan(p);
    return fail(FM_EUNSUPPORTED, "structuring element larger than the largest FFT tile (" +
                                     std::string(p->two_d ? "256x256" : "256") + ")");
  }
  if (p->big) bv = nullptr;
  p->var = bv;
  if (std::getenv("FM_PLAN_DEBUG"))
    std::fprintf(stderr, "[fm plan] %s %lldx%lld se %dx%d T=%d K=%d tile %s%dx%d nt=%d batch=%lld\n",
                 p->two_d ? "2-D" : "1-D", (long long)p->H, (long long)p->W, p->my, p->mx, p->T, p->K,
                 p->big ? "big " : "", bv ? bv->py : kBig, bv ? bv->px : kBig, bv ? bv->nt : 0, (long long)p->batch);
  p->PY = p->big ? kBig : bv->py;
  p->PX = p->big ? kBig : bv->px;
  p->QX = p->PX - p->mx + 1;
  // three-pass 128 kernel: its inverse y pass runs one warp per 32 window
  // columns; a window a few columns past a multiple of 32 is trimmed to it
  // (c5: 98 -> 96, 2% more tiles, a quarter of that pass saved)
  {
    const char* tq = std::getenv("FM_TRIM_QX");   // A/B switch: FM_TRIM_QX=0 keeps the full window
    const bool trim = !(tq && tq[0] == '0');
    if (trim && bv && bv->tmax < (1 << 30) && p->QX > 32 && p->QX % 32 != 0 && p->QX % 32 <= 4) p->QX -= p->QX % 32;
  }
  p->QY = p->two_d ? p->PY - p->my + 1 : 1;
  p->tiles_x = (int)((p->OW + p->QX - 1) / p->QX);
  p->tiles_y = p->two_d ? (int)((p->OH + p->QY - 1) / p->QY) : 1;
  p->tiles_total = p->tiles_x * p->tiles_y;
  p->tile_ctas = p->two_d ? p->tiles_total : (p->tiles_total + p->PY - 1) / p->PY;

  // shared memory (tile buffer + spectrum staging + tonal indices)
  p->conv_smem = p->big ? kBigColsSmem : bv->smem_fixed;
  if (p->conv_smem > kSmemLimit) { free_plan(p); return fail(FM_EUNSUPPORTED, "tile too large for shared memory"); }

  // tonal ladder: each conv unit uses the smallest N_t of the ladder with
  // 2 N_t > its own l_R (fm_range.cuh); a forced tonal_len pins a single entry
  if (d.tonal_len > 0 || p->counts) {
    p->ladder = {p->N};
  } else {
    for (int i = 0; i < kTonalCount; ++i)
      if (kTonalNs[i] < p->N) p->ladder.push_back(kTonalNs[i]);
    p->ladder.push_back(p->N);
  }
  for (int n : p->ladder) p->ladder_var.push_back(find_tonal(n));
  // generic tonal kernel (N beyond the compiled set): geometry for N_global
  p->tonal_stride = (p->N + 1) | 1;
  int nt = 128;
  // long tonal axes (10-11-bit data): fewer pixels per CTA, down to 8 (T up to ~3200)
  while (nt > 8 && (size_t)(2 * p->N + 2 * (size_t)nt * p->tonal_stride) * 8 > 200 * 1024) nt = nt > 32 ? nt - 32 : nt / 2;
  p->tonal_threads = nt;
  p->tonal_smem = (size_t)(2 * p->N + 2 * (size_t)nt * p->tonal_stride) * 8;
  if (!p->ladder_var.back() && p->tonal_smem > kSmemLimit) {
    free_plan(p);
    return fail(FM_EUNSUPPORTED, "tonal length too large for the tonal kernel");
  }

  // conv units: one 2-D tile, or PY consecutive 1-D tiles (one CTA)
  if (p->two_d) {
    p->units = p->tiles_total;
    p->npx = p->QY * p->QX;
    p->win_y = p->PY;
    p->win_x = p->PX;
  } else {
    p->units = p->tile_ctas;
    p->npx = p->PY * p->QX;
    p->win_y = 1;
    p->win_x = (p->PY - 1) * p->QX + p->PX;
    p->unit_step_x = p->PY * p->QX;
  }

  p->wpx = (p->npx + 3) & ~3;  // plane stride a multiple of 4 pixels: 16-byte aligned bulk / TMA copies of pixel blocks for both element sizes (8 B, and 4 B with 16-bit planes)
  // units whose input window lies inside the image (the "full" test of fm_range.cuh)
  p->full_prefix.assign(p->units + 1, 0);
  for (int u = 0; u < p->units; ++u) {
    bool full;
    if (p->two_d) {
      const int ty = u / p->tiles_x, tx = u - ty * p->tiles_x;
      const int64_t y0 = (int64_t)ty * p->QY + p->DY, x0 = (int64_t)tx * p->QX + p->DX;
      full = y0 >= 0 && y0 + p->win_y <= p->H && x0 >= 0 && x0 + p->win_x <= p->W;
    } else {
      const int64_t x0 = (int64_t)u * p->unit_step_x + p->DX;
      full = x0 >= 0 && x0 + p->win_x <= p->W;
    }
    p->full_prefix[u + 1] = p->full_prefix[u] + (full ? 1 : 0);
  }

  // clamp-bound taps (fm_range.cuh): the highest SE entries, ties spread over
  // the SE by a multiplicative hash; offsets index the staged input window;
  // padded to a multiple of 8 with taps that never win.
  // FM_RANGE_TAPS=<n> caps the count (0 disables the clamp).
  {
    int cap_taps = kMaxBoundTaps;
    if (const char* env = std::getenv("FM_RANGE_TAPS")) cap_taps = std::max(0, std::min(kMaxBoundTaps, std::atoi(env)));
    const size_t wsm = (size_t)p->win_y * p->win_x * sizeof(int16_t);
    const bool fits = p->vmax <= 32767 && (p->se_max - p->se_min) < 32768 && wsm <= kRangeSmemMax;
    if (fits && cap_taps > 0 && !p->counts) {
      std::vector<std::pair<int64_t, int2>> cand;
      for (int py = 0; py < p->my; ++py)
        for (int px = 0; px < p->mx; ++px) {
          const int64_t i = (int64_t)py * p->mx + px;
          if (!sd[i]) continue;
          const int off = (p->my - 1 - py) * p->win_x + (p->mx - 1 - px);
          const int bv = sv[i] - p->se_min;
          const uint32_t h = (uint32_t)(i * 2654435761u);
          cand.push_back({((int64_t)(p->se_max - sv[i]) << 32) | h, make_int2(off, bv)});
        }
      std::sort(cand.begin(), cand.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
      for (size_t i = 0; i < cand.size() && (int)i < cap_taps; ++i) p->taps.push_back(cand[i].second);
      while (p->taps.size() % 8) p->taps.push_back(make_int2(0, kTapPadB));
    }
  }

  // spectral scratch and launch chunking
  // scratch per unit: its K_max spectral planes (+ the 256^2 tile slab on the big path).
  // Whole images per launch when they fit the budget, else chunks of units of one image.
  const int64_t per_unit = (int64_t)p->K * p->wpx * 8 + (p->big ? (int64_t)p->K * kBig * kBig * 8 : 0);
  // default budget 16 GiB: large launches keep the per-launch tail small (B200: 180 GB HBM)
  const int64_t budget = d.scratch_bytes > 0 ? d.scratch_bytes : (int64_t)16 << 30;
  p->upl = (int)std::max<int64_t>(1, std::min<int64_t>(p->units, budget / std::max<int64_t>(per_unit, 1)));
  // one image on the 256^2 path: split its units into a few launch steps so the range
  // kernel of step i+1 (its own low-priority stream) overlaps the conv / tonal of step i
  // instead of preceding them (FM_BIG_STEPS=<n>, default 3; 1 = one step)
  if (p->big && d.batch == 1 && g_big_steps > 1 && p->units >= 4 * g_big_steps)
    p->upl = std::min(p->upl, (p->units + g_big_steps - 1) / g_big_steps);
  if (p->upl < p->units) {
    p->ipc = 1;
  } else {
    p->ipc = std::max<int64_t>(1, std::min<int64_t>(p->batch, budget / std::max<int64_t>(per_unit * p->units, 1)));
    if (p->ipc > 65535) p->ipc = 65535;
    // equal launches: the largest divisor of the batch within the budget when it
    // is at least half of it, else balanced sizes (c5, 64 images: 8 x 8 instead
    // of 5 x 12 + 4 -- no short last launch, and earlier output copies)
    int64_t div = 0;
    for (int64_t c = p->ipc; c >= 1 && 2 * c >= p->ipc; --c)
      if (p->batch % c == 0) {
        div = c;
        break;
      }
    if (div > 0) {
      p->ipc = div;
    } else {
      const int64_t nl = (p->batch + p->ipc - 1) / p->ipc;
      p->ipc = (p->batch + nl - 1) / nl;
    }
  }
  // the 256x256 path launches gridDim.z = units x images of a launch (<= 65535)
  if (p->big && (int64_t)p->upl * p->ipc > 65535) {
    if (p->upl > 65535) p->upl = 65535;
    p->ipc = std::max<int64_t>(1, 65535 / p->upl);
  }
  const int64_t slots = p->ipc * p->upl;
  const int occ = p->two_d ? std::max(1, (kSmemLimit) / (int)(p->conv_smem + 1024)) : 2;
  const int64_t target = 148LL * 2 * occ;
  const int64_t base = (int64_t)p->upl * p->ipc;
  int kch = (int)std::min<int64_t>(p->K, std::max<int64_t>(1, (target + base - 1) / base));
  p->k_chunk = (p->K + kch - 1) / kch;
  // fused tonal step: three-pass 128x128 kernels (register budget of 128 per thread),
  // value outputs (not count volumes)
  if (g_fuse && !p->counts && !p->big && p->two_d && bv && bv->tmax < (1 << 30)) {
    p->fuse_nmax = kFuseNMax;
    if (g_fuse_kch > 0) p->k_chunk = std::min(p->K, g_fuse_kch);
  }
  // 16-bit spectral planes.  A plane value is X_k = (1/T) sum_t c(t) w^{kt} with
  // sum_t c(t) <= C = defined SE entries, so |Re X_k|, |Im X_k| <= C / T: stored as int16
  // at q = 32000 T / C the rounding error is <= C / (64000 T) per component, and the
  // inverse tonal transform (2N terms, |weights| <= 1 after the c2r packing) recovers
  // every count within sqrt(2) C / 64000 (C = 961 at c5: 0.021; the reference aborts at
  // 0.25).  Enabled for C <= 2048 (bound <= 0.045) on the three-pass 128^2 kernels;
  // the measured deviation (fm_read_stats) includes it.  Halves the spectral volume's
  // bytes (conv writes, tonal reads).
  if (g_chat16 && !p->counts && !p->big && p->two_d && bv && bv->tmax < (1 << 30) &&
      p->se_count <= kChat16MaxCount) {
    p->chat16 = true;
    p->chat_q_T = (float)(32000.0 / (double)p->se_count);
    p->chat_invq_T = (float)((double)p->se_count / 32000.0);
  }
  p->kchunks = (p->K + p->k_chunk - 1) / p->k_chunk;
  p->conv_occ = occ;
  {
    const double pts = p->two_d ? (double)p->PY * p->PX : (double)p->PX;
    const double tiles_per_unit = p->two_d ? 1.0 : (double)p->PY;
    p->conv_flops_per_plane = tiles_per_unit * (2.0 * 5.0 * pts * std::log2(pts) + 6.0 * pts);
  }
  DeviceGuard dg(p->device);
  rc = ensure_twiddles(p->device);
  if (rc) { free_plan(p); return rc; }
  auto cfail = [&](cudaError_t e, const char* what) {
    free_plan(p);
    return fail(FM_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  };
  cudaError_t e;

  const size_t npts = (size_t)p->PY * p->PX;
  const int L = (int)p->ladder.size();
  int64_t spec_f4 = 0;
  for (int n : p->ladder) {
    p->spec_off.push_back(spec_f4);
    spec_f4 += (int64_t)(n + 1) * (int64_t)(npts / 2);
  }
  const int64_t cap = slots;
  if ((e = cudaMalloc(&p->spec, sizeof(float4) * spec_f4)) != cudaSuccess) return cfail(e, "spec alloc");
  if ((e = cudaMalloc(&p->d_ladder, sizeof(int) * L)) != cudaSuccess) return cfail(e, "ladder alloc");
  if ((e = cudaMalloc(&p->d_spec_off, sizeof(int64_t) * L)) != cudaSuccess) return cfail(e, "ladder alloc");
  for (int b = 0; b < 2; ++b) {
    if ((e = cudaMalloc(&p->unit_param[b], sizeof(int4) * p->ipc * p->units)) != cudaSuccess) return cfail(e, "unit alloc");
    if ((e = cudaMalloc(&p->bucket_count[b], sizeof(int) * L)) != cudaSuccess) return cfail(e, "bucket alloc");
    if ((e = cudaMalloc(&p->bucket_list[b], sizeof(int2) * cap * L)) != cudaSuccess) return cfail(e, "bucket alloc");
    if ((e = cudaHostAlloc(&p->h_counts[b], sizeof(int) * L, cudaHostAllocMapped)) != cudaSuccess) return cfail(e, "pinned alloc");
    if ((e = cudaHostGetDevicePointer(&p->h_counts_dev[b], p->h_counts[b], 0)) != cudaSuccess) return cfail(e, "pinned map");
    if ((e = cudaEventCreateWithFlags(&p->count_ev[b], cudaEventDisableTiming)) != cudaSuccess) return cfail(e, "event");
    if ((e = cudaEventCreateWithFlags(&p->free_ev[b], cudaEventDisableTiming)) != cudaSuccess) return cfail(e, "event");
  }
  if ((e = cudaEventCreateWithFlags(&p->entry_ev, cudaEventDisableTiming)) != cudaSuccess) return cfail(e, "event");
  {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if ((e = cudaStreamCreateWithPriority(&p->range_stream, cudaStreamNonBlocking, least)) != cudaSuccess)
      return cfail(e, "stream");
  }
  if ((e = cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming)) != cudaSuccess) return cfail(e, "event");
  for (int i = 0; i < kAuxStreams; ++i) {
    if ((e = cudaStreamCreateWithFlags(&p->aux[i], cudaStreamNonBlocking)) != cudaSuccess) return cfail(e, "stream");
    if ((e = cudaEventCreateWithFlags(&p->ev_join[i], cudaEventDisableTiming)) != cudaSuccess) return cfail(e, "event");
  }
  {
    const size_t np = (size_t)p->ipc * p->units;
    for (int b = 0; b < 2; ++b)
      if ((e = cudaMalloc(&p->range_part[b], sizeof(int) * 8 * np)) != cudaSuccess) return cfail(e, "range alloc");
    std::vector<int> init(8 * np, 0);
    for (size_t i = 0; i < np; ++i) {
      init[8 * i + 0] = INT32_MAX;
      init[8 * i + 1] = INT32_MIN;
      init[8 * i + 2] = INT32_MAX;
    }
    for (int b = 0; b < 2; ++b) cudaMemcpy(p->range_part[b], init.data(), sizeof(int) * 8 * np, cudaMemcpyHostToDevice);
  }
  {
    // encode tables, FP64-rounded: entry j = exp(-2 pi i j / T), entry T = 0
    std::vector<float2> tab;
    for (int li = 0; li < L; ++li) {
      const int Tl = 2 * p->ladder[li];
      p->enc_off.push_back((int)tab.size());
      for (int j = 0; j < Tl; ++j) {
        const double ang = -2.0 * kPi * j / Tl;
        tab.push_back(make_float2((float)std::cos(ang), (float)std::sin(ang)));
      }
      tab.push_back(make_float2(0.f, 0.f));
    }
    if ((e = cudaMalloc(&p->enc_tab, sizeof(float2) * tab.size())) != cudaSuccess) return cfail(e, "table alloc");
    if ((e = cudaMalloc(&p->d_enc_off, sizeof(int) * L)) != cudaSuccess) return cfail(e, "table alloc");
    cudaMemcpy(p->enc_tab, tab.data(), sizeof(float2) * tab.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(p->d_enc_off, p->enc_off.data(), sizeof(int) * L, cudaMemcpyHostToDevice);
  }
  cudaMemcpy(p->d_ladder, p->ladder.data(), sizeof(int) * L, cudaMemcpyHostToDevice);
  cudaMemcpy(p->d_spec_off, p->spec_off.data(), sizeof(int64_t) * L, cudaMemcpyHostToDevice);
  if ((e = cudaMalloc(&p->twN, sizeof(float2) * std::max(1, p->N))) != cudaSuccess) return cfail(e, "table alloc");
  if ((e = cudaMalloc(&p->wT, sizeof(float2) * std::max(1, p->N))) != cudaSuccess) return cfail(e, "table alloc");
  if ((e = cudaMalloc(&p->stats, sizeof(int) * 4)) != cudaSuccess) return cfail(e, "stats alloc");
  if ((e = cudaMalloc(&p->se_vals_d, sizeof(int32_t) * se_n)) != cudaSuccess) return cfail(e, "se alloc");
  if ((e = cudaMalloc(&p->se_def_d, se_n)) != cudaSuccess) return cfail(e, "se alloc");
  if (p->big &&
      (e = cudaMalloc(&p->S, (size_t)slots * p->K * kBig * kBig * 8 + (size_t)p->K * kBig * kBig * 8)) !=
          cudaSuccess) {
    free_plan(p);
    return fail(FM_ENOMEM, std::string("tile scratch alloc: ") + cudaGetErrorString(e));
  }
  if (p->big) {
    p->big_jobs_cap = std::min<int64_t>((int64_t)slots * p->K, (int64_t)4 << 20);
    if ((e = cudaMalloc(&p->big_jobs, sizeof(int2) * (size_t)p->big_jobs_cap)) != cudaSuccess) return cfail(e, "job list alloc");
    if ((e = cudaMalloc(&p->big_njobs, sizeof(int))) != cudaSuccess) return cfail(e, "job list alloc");
  }
  if (p->fuse_nmax > 0) {
    if ((e = cudaMalloc(&p->unit_done, sizeof(int) * (size_t)slots)) != cudaSuccess) return cfail(e, "counter alloc");
    cudaMemset(p->unit_done, 0, sizeof(int) * (size_t)slots);
  }
  p->chat_set_bytes = (size_t)slots * p->K * p->wpx * (p->chat16 ? 4 : 8);
  p->overlap = g_overlap && p->chat16 && !p->counts && !p->big && p->fuse_nmax == 0;
  if (p->overlap) {
    if ((e = cudaStreamCreateWithFlags(&p->tstream, cudaStreamNonBlocking)) != cudaSuccess) return cfail(e, "stream");
    for (int b = 0; b < 2; ++b)
      if ((e = cudaEventCreateWithFlags(&p->conv_ev[b], cudaEventDisableTiming)) != cudaSuccess) return cfail(e, "event");
    if ((e = cudaEventCreateWithFlags(&p->tjoin_ev, cudaEventDisableTiming)) != cudaSuccess) return cfail(e, "event");
  }
  if ((e = cudaMalloc(&p->chat, p->chat_set_bytes * (p->overlap ? 2 : 1))) != cudaSuccess) {
    free_plan(p);
    return fail(FM_ENOMEM, std::string("spectral scratch alloc: ") + cudaGetErrorString(e));
  }
  // FM_TONAL_TMA=0: per-plane bulk copies in the pipelined tonal kernel (A/B)
  {
    const char* te = std::getenv("FM_TONAL_TMA");
    bool ok = !(te && te[0] == '0') && !p->counts;
    std::vector<CUtensorMap> maps(2 * L);
    for (int li = 0; li < L && ok; ++li) {
      const TonalVariant* tv = p->ladder_var[li];
      const int K = p->ladder[li] + 1;
      const int bx = tv ? tv->pipe_nt : 128;
      const int esz = p->chat16 ? 4 : 8;
      const int64_t rows = slots * p->K * (p->overlap ? 2 : 1);
      ok = encode_chat_map(&maps[2 * li], p->chat, p->wpx, rows, bx, K, esz) &&
           encode_chat_map(&maps[2 * li + 1], p->chat, p->wpx, rows, bx, std::max(1, K - 1), esz);
    }
    if (ok) p->tmaps = std::move(maps);
  }
  std::vector<float2> tn(std::max(1, p->N)), wt(std::max(1, p->N));
  for (int j = 0; j < p->N; ++j) {
    const double a1 = 2.0 * kPi * j / p->N, a2 = 2.0 * kPi * j / T;
    tn[j] = make_float2((float)std::cos(a1), (float)std::sin(a1));
    wt[j] = make_float2((float)std::cos(a2), (float)std::sin(a2));
  }
  cudaMemcpy(p->twN, tn.data(), sizeof(float2) * tn.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(p->wT, wt.data(), sizeof(float2) * wt.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(p->se_vals_d, sv.data(), sizeof(int32_t) * se_n, cudaMemcpyHostToDevice);
  cudaMemcpy(p->se_def_d, sd.data(), se_n, cudaMemcpyHostToDevice);
  cudaMemset(p->stats, 0, sizeof(int) * 4);

  // SE spectra, one per ladder entry: same encode + forward passes as the image
  // tiles, scaled by 1/(PY_eff * PX * T) so the inverse transforms need no
  // normalisation.
  for (int li = 0; li < L && p->big; ++li) {
    // 256x256 tiles: forward x (rows kernel) then forward y + scaled store (cols kernel)
    const int Tl = 2 * p->ladder[li];
    BigArgs b{};
    b.se_vals = p->se_vals_d;
    b.se_def = p->se_def_d;
    b.my = p->my;
    b.mx = p->mx;
    b.T = Tl;
    b.K = p->ladder[li] + 1;
    b.enc_sign = 1;
    b.enc_bias = -smin;
    b.units = 1;
    b.nu = 1;
    b.nub = 1;
    b.K_max = b.K;
    b.S = p->S + (size_t)slots * p->K * kBig * kBig;   // spare slab after the batch scratch
    b.spec = p->spec + p->spec_off[li];
    b.spec_scale = (float)(1.0 / ((double)kBig * kBig * Tl));
    b.err = p->stats + 1;
    big_rows_kernel<true, true><<<dim3(kBig / kBigRows, b.K, 1), kBigNT, kBigRowsSmem>>>(b);
    big_cols_kernel<true><<<dim3(kBig / kBigCols, b.K, 1), kBigColsNT, kBigColsSmem>>>(b);
    g_launches += 2;
    if ((e = cudaGetLastError()) != cudaSuccess) return cfail(e, "SE spectrum launch");
  }
  for (int li = 0; li < L && !p->big; ++li) {
    const int Tl = 2 * p->ladder[li];
    TileArgs a{};
    a.se_vals = p->se_vals_d;
    a.se_def = p->se_def_d;
    a.H = 1;
    a.W = 1;
    a.my = p->my;
    a.mx = p->mx;
    a.T = Tl;
    a.K = p->ladder[li] + 1;
    a.magicT = (uint32_t)((1ull << 32) / (uint64_t)Tl);
    a.k_chunk = 1;
    a.enc_sign = 1;
    a.enc_bias = -smin;
    a.spec = p->spec + p->spec_off[li];
    a.spec_out = p->spec + p->spec_off[li];
    a.spec_scale = (float)(1.0 / ((double)(p->two_d ? p->PY : 1) * p->PX * Tl));
    a.enc_tab = p->enc_tab + p->enc_off[li];
    a.tiles_x = 1;
    a.tiles_total = 1;
    a.err = p->stats + 1;
    bv->spec(dim3(1, a.K, 1), p->conv_smem, 0, a);
    g_launches++;
    if ((e = cudaGetLastError()) != cudaSuccess) return cfail(e, "SE spectrum launch");
  }
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cfail(e, "SE spectrum");
  // a whole call is one device-dispatched launch step (run_images' devdisp): capturable
  p->graphable = g_graph && !p->big && !p->counts && p->fuse_nmax == 0 && p->N <= kDispatchNMax &&
                 p->ipc >= p->batch && p->upl >= p->units &&
                 (int64_t)p->units * p->batch < (int64_t)g_num_sms * p->conv_occ * 2 && g_devdispatch;
  *out_plan = p;
  return FM_OK;
}

int fm_plan_query(const fm_plan* p, fm_plan_info* info) {
  if (!p || !info) return fail(FM_EINVAL, "null argument");
  if (!p->parts.empty()) {
    // composite: geometry of the first block, output / SE facts of the whole plan
    int rc = fm_plan_query(p->parts[0], info);
    if (rc) return rc;
    int64_t scratch = 0;
    for (const fm_plan* q : p->parts) {
      fm_plan_info qi;
      fm_plan_query(q, &qi);
      scratch += qi.scratch_bytes;
      info->tonal_len = std::max(info->tonal_len, qi.tonal_len);
      info->planes = std::max(info->planes, qi.planes);
      info->l_r = std::max(info->l_r, qi.l_r);
    }
    info->out_shape[0] = p->two_d ? p->OH : p->OW;
    info->out_shape[1] = p->two_d ? p->OW : 0;
    info->out_lo_offset[0] = p->two_d ? p->off_y : p->off_x;
    info->out_lo_offset[1] = p->two_d ? p->off_x : 0;
    info->scratch_bytes = scratch + (int64_t)p->batch * p->OH * p->OW * (out_elem_size(p->d.out_dtype) + 2);
    info->se_min = p->se_min;
    info->se_max = p->se_max;
    info->se_count = p->se_count;
    return FM_OK;
  }
  std::memset(info, 0, sizeof(*info));
  info->tonal_len = p->T;
  info->planes = p->K;
  info->l_r = p->lr;
  info->tile_y = p->two_d ? p->PY : 1;
  info->tile_x = p->PX;
  info->valid_y = p->QY;
  info->valid_x = p->QX;
  info->tiles_y = p->tiles_y;
  info->tiles_x = p->tiles_x;
  info->k_chunk = p->k_chunk;
  info->out_shape[0] = p->two_d ? p->OH : p->OW;
  info->out_shape[1] = p->two_d ? p->OW : 0;
  info->out_lo_offset[0] = p->two_d ? p->off_y : p->off_x;
  info->out_lo_offset[1] = p->two_d ? p->off_x : 0;
  info->images_per_launch = p->ipc;
  info->scratch_bytes = (int64_t)p->upl * p->K * p->wpx * 8 * p->ipc +
                        (p->big ? (int64_t)p->upl * p->K * kBig * kBig * 8 * p->ipc : 0);
  info->se_min = p->se_min;
  info->se_max = p->se_max;
  info->se_count = p->se_count;
  info->count_len = p->counts ? p->lr + 1 : 0;
  return FM_OK;
}

int fm_reset_stats(fm_plan* p, void* stream) {
  if (!p) return fail(FM_EINVAL, "null plan");
  for (fm_plan* q : p->parts) {
    int rc = fm_reset_stats(q, stream);
    if (rc) return rc;
  }
  if (!p->parts.empty()) return FM_OK;
  DeviceGuard dg(p->device);
  FM_CUDA(cudaMemsetAsync(p->stats, 0, sizeof(int) * 4, (cudaStream_t)stream));
  return FM_OK;
}

// Images [cbeg, cend) of the batch (device pointers address image 0), in
// launch chunks of ipc images and upl units.
static int out_size(int od) { return od == FM_OUT_U8 ? 1 : (od == FM_OUT_U16 || od == FM_OUT_I16) ? 2 : 4; }

// chunks (optional): explicit image chunks (first image, images <= ipc), else
// chunks of ipc images; in_ready (optional): one event per chunk, recorded when
// that chunk's input is in place; after_chunk (optional): called with the chunk
// index once its last kernels are enqueued on s (the host-buffer path queues
// its D2H there).
static int run_images(fm_plan* p, const void* img, const uint8_t* img_defined, void* out, uint8_t* valid,
                      cudaStream_t s, int64_t cbeg, int64_t cend,
                      const std::vector<std::pair<int64_t, int>>* chunks = nullptr, const cudaEvent_t* in_ready = nullptr,
                      const std::function<int(size_t, int64_t, int, cudaStream_t)>& after_chunk = nullptr) {
  p->last_stream = s;
  const int64_t npix = p->OH * p->OW;
  const int64_t img_elems = p->H * p->W;
  const int dsz = dtype_size(p->d.img_dtype);
  const int L = (int)p->ladder.size();
  const int64_t cap = p->ipc * p->upl;
  // launch steps: (image chunk, unit chunk)
  struct Step {
    int64_t c0;
    int n, u0, nu;
    size_t chunk;
  };
  std::vector<Step> steps;
  std::vector<std::pair<int64_t, int>> plan_chunks;
  if (chunks) {
    plan_chunks = *chunks;
  } else {
    // balanced launch chunks (16 images with room for 12: 8 + 8, not 12 + 4)
    const int64_t nimg = cend - cbeg;
    const int64_t nch = (nimg + p->ipc - 1) / std::max<int64_t>(p->ipc, 1);
    for (int64_t i = 0, c0 = cbeg; i < nch; ++i) {
      const int64_t n = (nimg - (c0 - cbeg) + (nch - i) - 1) / (nch - i);
      plan_chunks.push_back({c0, (int)n});
      c0 += n;
    }
  }
  for (size_t ci = 0; ci < plan_chunks.size(); ++ci)
    for (int u0 = 0; u0 < p->units; u0 += p->upl)
      steps.push_back({plan_chunks[ci].first, plan_chunks[ci].second, u0, std::min(p->upl, p->units - u0), ci});
  if (steps.empty()) return FM_OK;
  bool used_tstream = false;
  // range kernels run one step ahead on a low-priority stream (double-buffered
  // outputs): they fill the conv tail and overlap the tonal kernels
  cudaStream_t rs = p->range_stream;
  // Device dispatch (small launches, latency bound): the conv grid and the tonal pass are
  // sized on the device from the range kernel's per-ladder counts (decode_job with
  // k_chunk = 0, tonal_kernel_dispatch), so the call never waits on the host for them.
  const int64_t conv_target_all = (int64_t)g_num_sms * p->conv_occ * 2;
  auto devdisp = [&](const Step& st) {
    return g_devdispatch && !p->big && !p->counts && p->fuse_nmax == 0 && p->N <= kDispatchNMax &&
           (int64_t)st.nu * st.n < conv_target_all;
  };
  FM_CUDA(cudaEventRecord(p->entry_ev, s));          // inputs / prior work on s
  FM_CUDA(cudaStreamWaitEvent(rs, p->entry_ev, 0));
  auto launch_range = [&](const Step& st, int buf) -> int {
    const int64_t c0 = st.c0;
    const int n = st.n, u0 = st.u0, nu = st.nu;
    // the previous user of this buffer set (a graph replay is ordered on its stream as a whole,
    // and a capture may not wait on events recorded outside it)
    if (!p->capturing) FM_CUDA(cudaStreamWaitEvent(rs, p->free_ev[buf], 0));
    if (in_ready) FM_CUDA(cudaStreamWaitEvent(rs, in_ready[st.chunk], 0));
    // ---- per-unit tonal range -> ladder entry + work lists (fm_range.cuh)
    FM_CUDA(cudaMemsetAsync(p->bucket_count[buf], 0, sizeof(int) * L, rs));
    RangeArgs r{};
    r.img = reinterpret_cast<const char*>(img) + (size_t)c0 * img_elems * dsz;
    r.img_def = img_defined ? img_defined + (size_t)c0 * img_elems : nullptr;
    r.H = (int)p->H;
    r.W = (int)p->W;
    r.two_d = p->two_d ? 1 : 0;
    r.DY = p->DY;
    r.DX = p->DX;
    r.QY = p->QY;
    r.QX = p->QX;
    r.win_y = p->win_y;
    r.win_x = p->win_x;
    r.my = p->my;
    r.mx = p->mx;
    r.tiles_x = p->tiles_x;
    r.units = p->units;
    r.unit0 = u0;
    r.unit_step_x = p->unit_step_x;
    r.OH = (int)p->OH;
    r.OW = (int)p->OW;
    r.enc_sign = p->enc_sign;
    r.enc_bias = p->enc_bias;
    r.vmax = p->vmax;
    r.lr_se = p->se_max - p->se_min;
    r.cy = p->two_d ? (p->my - 1) / 2 : 0;
    r.cx = (p->mx - 1) / 2;
    r.ntaps = (int)p->taps.size();
    for (int i = 0; i < r.ntaps; ++i) r.taps[i] = p->taps[i];
    r.flat_taps = r.ntaps > 0 ? 1 : 0;
    for (int i = 0; i < r.ntaps; ++i)
      if (p->taps[i].y != 0) r.flat_taps = 0;
    // split units between CTAs when there are too few of them to fill the GPU
    int S = 1;
    if (r.ntaps > 0) {
      const int64_t ctas = (int64_t)nu * n;
      const int max_s = p->two_d ? std::max(1, p->QY / 4) : std::max(1, p->unit_step_x / 256);
      S = (int)std::min<int64_t>(std::min(max_s, 32), std::max<int64_t>(1, (4 * 148 + ctas - 1) / ctas));
    }
    if (g_range_splits > 0 && r.ntaps > 0) S = std::max(1, std::min(g_range_splits, p->two_d ? std::max(1, p->QY / 4) : std::max(1, p->unit_step_x / 256)));
    r.splits = S;
    r.skip0 = g_no_skip0 ? 0 : 1;
    r.warp_sync = g_range_sync;
    // chunk-aligned staging (fm_range.cuh): uint8 rows 16-byte aligned, no mask, 2-D
    r.aligned = g_range_aligned && p->two_d && p->d.img_dtype == FM_U8 && img_defined == nullptr && p->W % 16 == 0 &&
                (reinterpret_cast<uintptr_t>(r.img) % 16) == 0;
    // window elements: int8 when every encoded value fits 7 bits (half the shared memory)
    const bool win8 = g_range_win8 && p->vmax <= 127;
    const size_t wsz = win8 ? 1 : 2;
    size_t rsm = 0;
    if (r.ntaps > 0) {
      const size_t stride = r.aligned ? (size_t)((p->win_x + 15) & ~15) + 16 : (size_t)p->win_x;
      rsm = p->two_d ? (size_t)((p->QY + S - 1) / S + p->my - 1) * stride * wsz
                     : (size_t)((p->unit_step_x + S - 1) / S + p->mx - 1) * wsz;
      rsm = (rsm + 15) & ~(size_t)15;
      if (rsm > (size_t)kRangeSmemMax) {   // (the plan sized the window for the plain stride)
        r.aligned = 0;
        rsm = ((size_t)((p->QY + S - 1) / S + p->my - 1) * p->win_x * wsz + 15) & ~(size_t)15;
      }
    }
    r.part = p->range_part[buf];
    r.ladder = p->d_ladder;
    r.L = L;
    r.unit_param = p->unit_param[buf];
    r.bucket_count = p->bucket_count[buf];
    r.bucket_list = p->bucket_list[buf];
    r.cap = (int)cap;
    r.err = p->stats + 1;
    int er = -1;
    if (p->timing) { er = (int)p->ev_next; FM_CUDA(cudaEventRecord(next_event(p), rs)); }
    {
      const dim3 rg((unsigned)(nu * S), n);
      if (win8) {
        if (p->d.img_dtype == FM_U8) range_kernel<0, int8_t><<<rg, kRangeNT, rsm, rs>>>(r);
        else if (p->d.img_dtype == FM_U16) range_kernel<1, int8_t><<<rg, kRangeNT, rsm, rs>>>(r);
        else range_kernel<2, int8_t><<<rg, kRangeNT, rsm, rs>>>(r);
      } else if (p->d.img_dtype == FM_U8) range_kernel<0><<<rg, kRangeNT, rsm, rs>>>(r);
      else if (p->d.img_dtype == FM_U16) range_kernel<1><<<rg, kRangeNT, rsm, rs>>>(r);
      else range_kernel<2><<<rg, kRangeNT, rsm, rs>>>(r);
    }
    g_launches++;
    FM_CUDA(cudaGetLastError());
    if (p->timing) {
      FM_CUDA(cudaEventRecord(next_event(p), rs));
      p->pending_range.push_back({er, er + 1});
    }
    // the counts reach the host through a kernel store to mapped memory, not a
    // copy-engine D2H: a D2H copy would queue behind any large D2H transfer in
    // flight on the device (e.g. the previous chunk's outputs)
    if (!devdisp(st) || p->timing) {   // (timing mode accounts the planes on the host)
      publish_counts<<<1, 64, 0, rs>>>(p->bucket_count[buf], p->h_counts_dev[buf], L);
      g_launches++;
      FM_CUDA(cudaGetLastError());
    }
    FM_CUDA(cudaEventRecord(p->count_ev[buf], rs));

    return FM_OK;
  };
  {
    int rc = launch_range(steps[0], 0);
    if (rc) return rc;
  }
  for (size_t si = 0; si < steps.size(); ++si) {
    const int buf = (int)(si & 1);
    if (si + 1 < steps.size()) {
      int rc = launch_range(steps[si + 1], buf ^ 1);
      if (rc) return rc;
    }
    const int64_t c0 = steps[si].c0;
    const int n = steps[si].n, u0 = steps[si].u0, nu = steps[si].nu;
    FM_CUDA(cudaStreamWaitEvent(s, p->count_ev[buf], 0));
    // this step's spectral buffer set (two sets alternate when the tonal pass of a step
    // overlaps the next step's conv)
    float2* chat_set = reinterpret_cast<float2*>(reinterpret_cast<char*>(p->chat) +
                                                 (p->overlap ? (size_t)buf * p->chat_set_bytes : 0));
    cudaStream_t tsm = p->overlap ? p->tstream : s;   // where this step's tonal pass runs
    TileArgs a{};
    a.img = reinterpret_cast<const char*>(img) + (size_t)c0 * img_elems * dsz;
    a.img_def = img_defined ? img_defined + (size_t)c0 * img_elems : nullptr;
    a.img_dtype = p->d.img_dtype;
    a.H = (int)p->H;
    a.W = (int)p->W;
    a.OH = (int)p->OH;
    a.OW = (int)p->OW;
    a.DY = p->DY;
    a.DX = p->DX;
    a.QY = p->QY;
    a.QX = p->QX;
    a.my = p->my;
    a.mx = p->mx;
    a.tiles_x = p->tiles_x;
    a.tiles_total = p->tiles_total;
    a.T = p->T;
    a.K = p->K;
    a.magicT = (uint32_t)((1ull << 32) / (uint64_t)p->T);
    a.k_chunk = p->k_chunk;
    a.enc_sign = p->enc_sign;
    a.enc_bias = p->enc_bias;
    a.spec = p->spec;
    a.chat = chat_set;
    a.err = p->stats + 1;
    a.unit_param = p->unit_param[buf];
    a.spec_off = p->d_spec_off;
    a.units = p->units;
    a.unit0 = u0;
    a.upl = p->upl;
    a.K_max = p->K;
    a.wpx = p->wpx;
    a.bucket_count = p->bucket_count[buf];
    a.bucket_list = p->bucket_list[buf];
    a.ladder = p->d_ladder;
    a.enc_tab = p->enc_tab;
    a.enc_off = p->d_enc_off;
    a.cap = (int)cap;
    a.L = L;
    a.chat16 = p->chat16 ? 1 : 0;
    a.chat_q_T = p->chat_q_T;
    if (p->fuse_nmax > 0) {
      a.fuse_nmax = p->fuse_nmax;
      a.discard = g_discard ? 1 : 0;
      a.unit_done = p->unit_done;
      a.out = reinterpret_cast<char*>(out) + (size_t)c0 * npix * out_size(p->d.out_dtype);
      a.out_dtype = p->d.out_dtype;
      a.valid = valid ? valid + (size_t)c0 * npix : nullptr;
      a.out_sign = p->out_sign;
      a.se_min = p->se_min;
      a.fill = p->d.fill;
      a.se_count = p->se_count;
      a.dev_max = reinterpret_cast<float*>(p->stats);
    }
    // Few units (one small image): split every unit's planes into chunks so the
    // conv grid fills the GPU; that needs the per-ladder counts first.  Many
    // units: one CTA per unit (all its planes), launched before the host waits.
    // (device-sized small launches: 2 CTAs per slot; host-sized ones, whose units carry many
    // planes, split finer -- the tail of the last wave is at most one chunk long)
    const int64_t conv_target = (int64_t)g_num_sms * p->conv_occ * (devdisp(steps[si]) ? 2 : g_conv_waves);
    const bool dyn = !p->big && (int64_t)nu * n < conv_target && p->k_chunk > 1;
    int e0 = -1;
    auto launch_conv = [&](unsigned grid) -> int {
      if (p->timing) { e0 = (int)p->ev_next; FM_CUDA(cudaEventRecord(next_event(p), s)); }
      p->var->conv(dim3(grid), p->conv_smem, s, a);
      g_launches++;
      FM_CUDA(cudaGetLastError());
      if (p->timing) {
        FM_CUDA(cudaEventRecord(next_event(p), s));
        p->pending_conv.push_back({e0, e0 + 1});
      }
      return FM_OK;
    };
    // 256x256 path: launched after the host has the per-ladder counts, with a
    // plane grid of the largest tonal length in use (not the plan's K: most
    // units need a few planes, the rest of the grid would only exit)
    bool jobs_listed = false;
    auto big_args = [&]() -> BigArgs {
      BigArgs b{};
      b.img = a.img;
      b.img_def = a.img_def;
      b.img_dtype = a.img_dtype;
      b.H = a.H;
      b.W = a.W;
      b.OH = a.OH;
      b.OW = a.OW;
      b.DY = a.DY;
      b.DX = a.DX;
      b.QY = a.QY;
      b.QX = a.QX;
      b.my = a.my;
      b.mx = a.mx;
      b.tiles_x = a.tiles_x;
      b.enc_sign = a.enc_sign;
      b.unit_param = p->unit_param[buf];
      b.units = p->units;
      b.unit0 = u0;
      b.upl = p->upl;
      b.nu = nu;
      b.K_max = p->K;
      b.S = p->S;
      b.spec = p->spec;
      b.spec_off = p->d_spec_off;
      b.chat = p->chat;
      b.wpx = p->wpx;
      b.err = p->stats + 1;
      b.pair = g_big_pair ? 1 : 0;
      b.lu0 = 0;
      b.nub = nu;
      return b;
    };
    // the job list needs nothing from the host: built as soon as the range kernel is done,
    // while the host still waits for the counts
    auto list_big_jobs = [&]() -> int {
      BigArgs b = big_args();
      FM_CUDA(cudaMemsetAsync(p->big_njobs, 0, sizeof(int), s));
      big_jobs_kernel<<<(unsigned)((nu * n + 255) / 256), 256, 0, s>>>(b, n, p->big_jobs, p->big_njobs, (int)p->big_jobs_cap);
      g_launches++;
      FM_CUDA(cudaGetLastError());
      jobs_listed = true;
      return FM_OK;
    };
    auto launch_big = [&](int kmax) -> int {
      if (p->timing) { e0 = (int)p->ev_next; FM_CUDA(cudaEventRecord(next_event(p), s)); }
      BigArgs b = big_args();
      const unsigned inv_blocks = (unsigned)((kBig - (p->my - 1) + kBigRows - 1) / kBigRows);
      // units in batches whose 256^2 scratch items (written and re-read by the three
      // kernels) fit in L2, so the passes read back from L2 instead of HBM
      int ub = nu;
      if (g_big_l2_mb > 0) {
        const int64_t item = (int64_t)kBig * kBig * 8 * kmax * n;
        ub = (int)std::max<int64_t>(1, std::min<int64_t>(nu, ((int64_t)g_big_l2_mb << 20) / item));
      }
      // compact job list (fm_bigtile.cuh): an upper bound of the live items sizes the grid -- the
      // per-ladder counts give the planes, the "full" units of the launch drop their plane 0
      // (the pairing of Nyquist planes is only known on the device); CTAs past the device
      // count exit
      int64_t jobs_upper = 0;
      for (int li = 0; li < L; ++li)
        jobs_upper += (int64_t)reinterpret_cast<volatile int*>(p->h_counts[buf])[li] * (p->ladder[li] + 1);
      if (!g_no_skip0 && img_defined == nullptr) jobs_upper -= (int64_t)n * (p->full_prefix[u0 + nu] - p->full_prefix[u0]);
      bool nu_done = false;
      if (jobs_listed && jobs_upper > 0 && jobs_upper <= p->big_jobs_cap) {
        b.jobs = p->big_jobs;
        b.njobs = p->big_njobs;
        const unsigned gy = (unsigned)std::min<int64_t>(jobs_upper, 65535), gz = (unsigned)((jobs_upper + gy - 1) / gy);
        big_rows_kernel<true, false><<<dim3(kBig / kBigRows, gy, gz), kBigNT, kBigRowsSmem, s>>>(b);
        big_cols_kernel<false><<<dim3(kBig / kBigCols, gy, gz), kBigColsNT, kBigColsSmem, s>>>(b);
        big_rows_kernel<false, false><<<dim3(inv_blocks, gy, gz), kBigNT, kBigRowsSmem, s>>>(b);
        g_launches += 3;
        FM_CUDA(cudaGetLastError());
        nu_done = true;
      }
      for (int b0 = 0; b0 < nu && !nu_done; b0 += ub) {
        b.lu0 = b0;
        b.nub = std::min(ub, nu - b0);
        const unsigned z = (unsigned)(b.nub * n);
        big_rows_kernel<true, false><<<dim3(kBig / kBigRows, kmax, z), kBigNT, kBigRowsSmem, s>>>(b);
        big_cols_kernel<false><<<dim3(kBig / kBigCols, kmax, z), kBigColsNT, kBigColsSmem, s>>>(b);
        big_rows_kernel<false, false><<<dim3(inv_blocks, kmax, z), kBigNT, kBigRowsSmem, s>>>(b);
        g_launches += 3;
        FM_CUDA(cudaGetLastError());
      }
      if (p->timing) {
        FM_CUDA(cudaEventRecord(next_event(p), s));
        p->pending_conv.push_back({e0, e0 + 1});
      }
      return FM_OK;
    };
    if (devdisp(steps[si])) {
      // ---- device-dispatched small launch: no host round trip
      a.k_chunk = 0;
      a.conv_target = (int)conv_target;
      int rc = launch_conv((unsigned)(conv_target + (int64_t)nu * n));
      if (rc) return rc;
      TonalArgs t{};
      t.chat = chat_set;
      t.K_max = p->K;
      t.unit_param = p->unit_param[buf];
      t.units = p->units;
      t.unit0 = u0;
      t.upl = p->upl;
      t.wpx = p->wpx;
      t.npx = p->npx;
      t.qx_magic = p->QX > 1 ? (uint32_t)((0x100000000ull + p->QX - 1) / p->QX) : 0u;
      t.tx_magic = p->tiles_x > 1 ? (uint32_t)((0x100000000ull + p->tiles_x - 1) / p->tiles_x) : 0u;
      t.two_d = p->two_d ? 1 : 0;
      t.QY = p->QY;
      t.QX = p->QX;
      t.OH = (int)p->OH;
      t.OW = (int)p->OW;
      t.tiles_x = p->tiles_x;
      t.unit_step_x = p->unit_step_x;
      t.out = reinterpret_cast<char*>(out) + (size_t)c0 * npix * out_size(p->d.out_dtype);
      t.out_dtype = p->d.out_dtype;
      t.valid = valid ? valid + (size_t)c0 * npix : nullptr;
      t.out_sign = p->out_sign;
      t.se_min = p->se_min;
      t.fill = p->d.fill;
      t.dev_max = reinterpret_cast<float*>(p->stats);
      t.chat16 = p->chat16 ? 1 : 0;
      t.chat_invq_T = p->chat_invq_T;
      t.bucket_count = p->bucket_count[buf];
      t.ladder = p->d_ladder;
      t.lists = p->bucket_list[buf];
      t.L = L;
      t.cap = (int)cap;
      t.se_count = p->se_count;
      constexpr int kDispNT = 128;
      const int64_t blocks = (int64_t)nu * n * ((p->npx + kDispNT - 1) / kDispNT);
      int e1 = -1;
      if (p->timing) { e1 = (int)p->ev_next; FM_CUDA(cudaEventRecord(next_event(p), s)); }
      if (p->N <= 10) tonal_kernel_dispatch<kDispNT, 10><<<(unsigned)blocks, kDispNT, 0, s>>>(t);
      else if (p->N <= 16) tonal_kernel_dispatch<kDispNT, 16><<<(unsigned)blocks, kDispNT, 0, s>>>(t);
      else tonal_kernel_dispatch<kDispNT, kDispatchNMax><<<(unsigned)blocks, kDispNT, 0, s>>>(t);
      g_launches++;
      FM_CUDA(cudaGetLastError());
      if (p->timing) {
        FM_CUDA(cudaEventRecord(next_event(p), s));
        p->pending_tonal.push_back({e1, e1 + 1});
      }
      p->units_done += (int64_t)n * nu;
      if (p->timing) {
        // measurement mode: the per-ladder counts (published for it) give the planes
        FM_CUDA(cudaEventSynchronize(p->count_ev[buf]));
        double planes = 0, tonal_b = 0;
        for (int li = 0; li < L; ++li) {
          const int cnt = reinterpret_cast<volatile int*>(p->h_counts[buf])[li];
          planes += (double)cnt * (p->ladder[li] + 1);
          tonal_b += (double)cnt * ((p->ladder[li] + 1) * (double)p->npx * (p->chat16 ? 4.0 : 8.0) +
                                    (double)p->npx * (out_size(p->d.out_dtype) + (valid ? 1.0 : 0.0)));
        }
        if (!g_no_skip0 && img_defined == nullptr) {
          const double skipped = (double)n * (double)(p->full_prefix[u0 + nu] - p->full_prefix[u0]);
          planes -= skipped;
          tonal_b -= skipped * (double)p->npx * (p->chat16 ? 4.0 : 8.0);
        }
        p->planes_done += (int64_t)planes;
        p->acc.conv_bytes += (double)n * img_elems * dsz * nu / p->units + planes * (double)p->npx * (p->chat16 ? 4.0 : 8.0);
        p->acc.conv_flops += planes * p->conv_flops_per_plane;
        p->acc.tonal_bytes += tonal_b;
      }
      // (a capture records no persistent event: one recorded inside a graph cannot be
      // waited on by a later direct call; replays are ordered through the caller's stream)
      if (!p->capturing) FM_CUDA(cudaEventRecord(p->free_ev[buf], s));
      if (after_chunk && u0 + nu >= p->units) {
        int rc2 = after_chunk(steps[si].chunk, c0, n, s);
        if (rc2) return rc2;
      }
      continue;
    }
    if (p->big) {
      if (g_big_jobs && g_big_l2_mb <= 0 && nu <= 65535) {
        int rc = list_big_jobs();
        if (rc) return rc;
      }
    } else if (!dyn) {
      // plan-time chunking (one chunk per unit for large launches); CTAs past
      // the actual job count exit at once
      a.k_chunk = p->k_chunk;
      int rc = launch_conv((unsigned)(nu * n * p->kchunks));
      if (rc) return rc;
    }

    // ---- the tonal kernels need the per-ladder unit counts (ready long before
    // the conv kernel finishes; the host waits only for the small copy)
    FM_CUDA(cudaEventSynchronize(p->count_ev[buf]));
    if (p->big) {
      int kmax = 0;
      for (int li = 0; li < L; ++li)
        if (reinterpret_cast<volatile int*>(p->h_counts[buf])[li] > 0) kmax = std::max(kmax, p->ladder[li] + 1);
      if (kmax > 0) {
        int rc = launch_big(kmax);
        if (rc) return rc;
      }
    }
    if (dyn) {
      int64_t planes_tot = 0;
      for (int li = 0; li < L; ++li)
        planes_tot += (int64_t)reinterpret_cast<volatile int*>(p->h_counts[buf])[li] * (p->ladder[li] + 1);
      const int kc = (int)std::max<int64_t>(1, (planes_tot + conv_target - 1) / conv_target);
      int64_t jobs = 0;
      for (int li = 0; li < L; ++li)
        jobs += (int64_t)reinterpret_cast<volatile int*>(p->h_counts[buf])[li] * ((p->ladder[li] + kc) / kc);
      a.k_chunk = kc;
      if (jobs > 0) {
        int rc = launch_conv((unsigned)jobs);
        if (rc) return rc;
      }
    }
    TonalArgs t{};
    t.chat = chat_set;
    t.K_max = p->K;
    t.unit_param = p->unit_param[buf];
    t.units = p->units;
    t.unit0 = u0;
    t.upl = p->upl;
    t.wpx = p->wpx;
    t.npx = p->npx;
    t.qx_magic = p->QX > 1 ? (uint32_t)((0x100000000ull + p->QX - 1) / p->QX) : 0u;
    t.tx_magic = p->tiles_x > 1 ? (uint32_t)((0x100000000ull + p->tiles_x - 1) / p->tiles_x) : 0u;
    t.two_d = p->two_d ? 1 : 0;
    t.QY = p->QY;
    t.QX = p->QX;
    t.OH = (int)p->OH;
    t.OW = (int)p->OW;
    t.tiles_x = p->tiles_x;
    t.unit_step_x = p->unit_step_x;
    t.out = reinterpret_cast<char*>(out) + (size_t)c0 * npix * out_size(p->d.out_dtype);
    t.out_dtype = p->d.out_dtype;
    t.valid = valid ? valid + (size_t)c0 * npix : nullptr;
    t.out_sign = p->out_sign;
    t.se_min = p->se_min;
    t.fill = p->d.fill;
    t.dev_max = reinterpret_cast<float*>(p->stats);
    t.chat16 = p->chat16 ? 1 : 0;
    t.chat_invq_T = p->chat_invq_T;
    if (p->counts) {
      t.counts = reinterpret_cast<int32_t*>(out) + (size_t)c0 * npix * (size_t)(p->lr + 1);
      t.count_len = p->lr + 1;
      t.count_base = p->d.img_min;
    }
    // the tonal pass runs on tsm after this step's conv (with overlap, beside the next
    // step's conv on s)
    used_tstream = used_tstream || p->overlap;
    if (p->overlap) {
      FM_CUDA(cudaEventRecord(p->conv_ev[buf], s));
      FM_CUDA(cudaStreamWaitEvent(tsm, p->conv_ev[buf], 0));
    }
    int e1 = -1;
    if (p->timing) { e1 = (int)p->ev_next; FM_CUDA(cudaEventRecord(next_event(p), tsm)); }
    double planes = 0, tonal_b = 0;
    // one launch per ladder entry in use, spread over the aux streams so the
    // small ones (few units each) run side by side; joined back into s
    int nlaunch = 0;
    double fused_b = 0;   // logical bytes of the tonal steps run inside the conv kernel
    for (int li = 0; li < L; ++li) {
      const int cnt = reinterpret_cast<volatile int*>(p->h_counts[buf])[li];
      if (cnt <= 0) continue;
      if (p->ladder[li] <= p->fuse_nmax) {
        const int N = p->ladder[li];
        planes += (double)cnt * (N + 1);
        fused_b += (double)cnt * ((N + 1) * (double)p->npx * (p->chat16 ? 4.0 : 8.0) +
                                  (double)p->npx * (out_size(p->d.out_dtype) + (valid ? 1.0 : 0.0)));
        continue;
      }
      ++nlaunch;
    }
    // few units per ladder entry (one mid-sized image: c3): the register-kernel entries
    // (N <= 40) go in ONE device-dispatched launch instead of one small launch each
    int disp_nmax = 0;
    if (!p->counts && p->fuse_nmax <= 0 && g_tonal_disp_max > 0) {
      constexpr int kDispNT = 128;
      const int bpj = (p->npx + kDispNT - 1) / kDispNT;
      int64_t items = 0;
      int entries = 0;
      for (int li = 0; li < L && p->ladder[li] <= kDispatchNMax; ++li) {
        const int cnt = reinterpret_cast<volatile int*>(p->h_counts[buf])[li];
        items += (int64_t)cnt * bpj;
        entries += cnt > 0;
      }
      if (entries > 1 && items <= g_tonal_disp_max) {
        disp_nmax = kDispatchNMax;
        nlaunch -= entries - 1;
      }
    }
    const int nstreams = std::min(nlaunch, 1 + kAuxStreams);
    if (nstreams > 1) {
      FM_CUDA(cudaEventRecord(p->ev_fork, tsm));
      for (int i = 0; i < nstreams - 1; ++i) FM_CUDA(cudaStreamWaitEvent(p->aux[i], p->ev_fork, 0));
    }
    int launch_i = 0;
    if (disp_nmax > 0) {
      constexpr int kDispNT = 128;
      const int bpj = (p->npx + kDispNT - 1) / kDispNT;
      int64_t items = 0;
      for (int li = 0; li < L && p->ladder[li] <= disp_nmax; ++li) {
        const int cnt = reinterpret_cast<volatile int*>(p->h_counts[buf])[li];
        const int N = p->ladder[li];
        items += (int64_t)cnt * bpj;
        planes += (double)cnt * (N + 1);
        tonal_b += (double)cnt * ((N + 1) * (double)p->npx * (p->chat16 ? 4.0 : 8.0) +
                                  (double)p->npx * (out_size(p->d.out_dtype) + (valid ? 1.0 : 0.0)));
      }
      t.bucket_count = p->bucket_count[buf];
      t.ladder = p->d_ladder;
      t.lists = p->bucket_list[buf];
      t.L = L;
      t.cap = (int)cap;
      t.se_count = p->se_count;
      // the last stream of the round robin: the long entries start first on the others
      const int si = nstreams - 1;
      tonal_kernel_dispatch<kDispNT, kDispatchNMax><<<(unsigned)items, kDispNT, 0, si == 0 ? tsm : p->aux[si - 1]>>>(t);
      g_launches++;
      FM_CUDA(cudaGetLastError());
    }
    for (int li = L - 1; li >= 0; --li) {
      const int cnt = reinterpret_cast<volatile int*>(p->h_counts[buf])[li];
      if (cnt <= 0 || p->ladder[li] <= p->fuse_nmax || p->ladder[li] <= disp_nmax) continue;
      const int N = p->ladder[li];
      const int si = launch_i++ % nstreams;
      cudaStream_t ts = si == 0 ? tsm : p->aux[si - 1];
      t.N = N;
      t.T = 2 * N;
      t.x0_full = (float)((double)p->se_count / (2.0 * N));
      t.list = p->bucket_list[buf] + (size_t)li * cap;
      const TonalVariant* tv = p->counts ? nullptr : p->ladder_var[li];
      const bool half_ring = p->chat16 && g_tonal_half_ring;
      const int occ = tv ? g_tonal_pipe_occ[tv - kTonal][half_ring ? 1 : 0] : 0;
      if (tv && N <= kRowsNMax && N <= g_tonal_rows_max) {
#ifndef FM_ROWS_PPT
#define FM_ROWS_PPT 8
#endif
#ifndef FM_ROWS_NT
#define FM_ROWS_NT 128
#endif
        constexpr int kRowsNT = FM_ROWS_NT, kRowsPPT = FM_ROWS_PPT;
        t.se_count = p->se_count;
        tonal_kernel_rows<kRowsNT, kRowsPPT><<<dim3((unsigned)cnt, (unsigned)((p->npx + kRowsNT * kRowsPPT - 1) / (kRowsNT * kRowsPPT))),
                                               kRowsNT, 0, ts>>>(t);
      } else if (tv && occ > 0 && !g_tonal_nopipe && N <= g_tonal_pipe_max && N >= g_tonal_pipe_min) {
        t.njobs = cnt;
        const int64_t items = (int64_t)cnt * ((p->npx + tv->pipe_nt - 1) / tv->pipe_nt);
        const int grid = (int)std::min<int64_t>(items, (int64_t)g_num_sms * std::min(occ, g_tonal_occ_cap));
        static const CUtensorMap kNoMap[2] = {};
        t.use_tma = p->tmaps.empty() ? 0 : 1;
        t.tma_row0 = p->overlap ? buf * (int)(cap * p->K) : 0;
        tv->pipe_fn(dim3((unsigned)grid), tv->pipe_nt, half_ring ? tv->pipe_smem / 2 : tv->pipe_smem, ts, t,
                    t.use_tma ? &p->tmaps[2 * li] : kNoMap);
      } else if (tv && tv->coop_nt > 0 && g_tonal_coop && N >= g_tonal_coop_min) {
        tv->coop_fn(dim3((unsigned)cnt, (unsigned)((p->npx + kCoopPix - 1) / kCoopPix)), tv->coop_nt, tv->coop_smem, ts, t);
      } else if (tv) {
        const int nt = tv->nt;
        tv->fn(dim3((unsigned)cnt, (unsigned)((p->npx + nt - 1) / nt)), nt, tv->smem, ts, t);
      } else {
        t.nstages = (int)p->radix.size();
        for (size_t i = 0; i < p->radix.size(); ++i) t.radix[i] = p->radix[i];
        t.twN = p->twN;
        t.wT = p->wT;
        t.stride = p->tonal_stride;
        const int nt = p->tonal_threads;
        tonal_kernel<<<dim3((unsigned)cnt, (unsigned)((p->npx + nt - 1) / nt)), nt, p->tonal_smem, ts>>>(t);
      }
      g_launches++;
      FM_CUDA(cudaGetLastError());
      planes += (double)cnt * (N + 1);
      tonal_b += (double)cnt * ((N + 1) * (double)p->npx * (p->chat16 ? 4.0 : 8.0) +
                                (double)p->npx * (out_size(p->d.out_dtype) + (valid ? 1.0 : 0.0)));
    }
    for (int i = 0; i < nstreams - 1; ++i) {
      FM_CUDA(cudaEventRecord(p->ev_join[i], p->aux[i]));
      FM_CUDA(cudaStreamWaitEvent(tsm, p->ev_join[i], 0));
    }
    // full units (fm_range.cuh) skip plane 0: fewer planes computed, stored and read
    if (!g_no_skip0 && img_defined == nullptr) {
      const double skipped = (double)n * (double)(p->full_prefix[u0 + nu] - p->full_prefix[u0]);
      planes -= skipped;
      // (per-ladder counts of full units are not known here: with the fused step the
      // skipped planes are charged to it, else to the tonal kernels)
      if (p->fuse_nmax > 0) fused_b -= skipped * (double)p->npx * (p->chat16 ? 4.0 : 8.0);
      else tonal_b -= skipped * (double)p->npx * (p->chat16 ? 4.0 : 8.0);
    }
    p->planes_done += (int64_t)planes;
    p->units_done += (int64_t)n * nu;
    if (p->timing) {
      FM_CUDA(cudaEventRecord(next_event(p), tsm));
      p->pending_tonal.push_back({e1, e1 + 1});
      p->acc.conv_bytes += (double)n * img_elems * dsz * nu / p->units + planes * (double)p->npx * (p->chat16 ? 4.0 : 8.0) + fused_b;
      p->acc.conv_flops += planes * p->conv_flops_per_plane;
      p->acc.tonal_bytes += tonal_b;
    }
    FM_CUDA(cudaEventRecord(p->free_ev[buf], tsm));
    if (after_chunk && u0 + nu >= p->units) {
      int rc = after_chunk(steps[si].chunk, c0, n, tsm);
      if (rc) return rc;
    }
  }
  if (p->overlap && used_tstream) {   // the caller's stream sees every step's outputs
    FM_CUDA(cudaEventRecord(p->tjoin_ev, p->tstream));
    FM_CUDA(cudaStreamWaitEvent(s, p->tjoin_ev, 0));
  }
  return FM_OK;
}

static int execute_composite(fm_plan* p, const void* img, const uint8_t* img_defined, void* out, uint8_t* valid,
                      cudaStream_t s) {
  p->last_stream = s;
  uint8_t* acc = valid ? valid : p->acc_valid;
  const int64_t n = p->batch * p->OH * p->OW;
  for (size_t i = 0; i < p->parts.size(); ++i) {
    fm_plan* q = p->parts[i];
    if (i == 0) {
      const int rc = run_images(q, img, img_defined, out, acc, s, 0, q->batch);
      if (rc) return rc;
      continue;
    }
    int rc = run_images(q, img, img_defined, p->part_out, p->part_valid, s, 0, q->batch);
    if (rc) return rc;
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)g_num_sms * 8));
    const int er = p->d.mode == FM_ERODE ? 1 : 0;
    switch (p->d.out_dtype) {
      case FM_OUT_U8:
        combine_kernel<uint8_t><<<g, 256, 0, s>>>((uint8_t*)out, acc, (const uint8_t*)p->part_out, p->part_valid, n, er);
        break;
      case FM_OUT_U16:
        combine_kernel<uint16_t><<<g, 256, 0, s>>>((uint16_t*)out, acc, (const uint16_t*)p->part_out, p->part_valid, n, er);
        break;
      case FM_OUT_I16:
        combine_kernel<int16_t><<<g, 256, 0, s>>>((int16_t*)out, acc, (const int16_t*)p->part_out, p->part_valid, n, er);
        break;
      default:
        combine_kernel<int32_t><<<g, 256, 0, s>>>((int32_t*)out, acc, (const int32_t*)p->part_out, p->part_valid, n, er);
        break;
    }
    g_launches++;
    FM_CUDA(cudaGetLastError());
  }
  return FM_OK;
}

int fm_execute(fm_plan* p, const void* img, const uint8_t* img_defined, void* out, uint8_t* valid,
               void* stream) {
  if (!p || !img || !out) return fail(FM_EINVAL, "null argument");
  DeviceGuard dg(p->device);
  if (!p->parts.empty()) return execute_composite(p, img, img_defined, out, valid, (cudaStream_t)stream);
  if (p->counts)
    FM_CUDA(cudaMemsetAsync(out, 0, (size_t)p->batch * p->OH * p->OW * (size_t)(p->lr + 1) * sizeof(int32_t),
                            (cudaStream_t)stream));
  cudaStream_t cs = (cudaStream_t)stream;
  if (p->graphable && !p->timing) {
    // the graph is captured and replayed on the plan's own stream, ordered after the
    // caller's stream by an event and back (the legacy default stream cannot be captured)
    if (!p->gstream) {
      FM_CUDA(cudaStreamCreateWithFlags(&p->gstream, cudaStreamNonBlocking));
      FM_CUDA(cudaEventCreateWithFlags(&p->gev_in, cudaEventDisableTiming));
      FM_CUDA(cudaEventCreateWithFlags(&p->gev_out, cudaEventDisableTiming));
    }
    cudaStream_t s = p->gstream;
    FM_CUDA(cudaEventRecord(p->gev_in, cs));
    FM_CUDA(cudaStreamWaitEvent(s, p->gev_in, 0));
    const void* key[5] = {img, img_defined, out, valid, nullptr};
    // Callers that pass new buffers every call (the drop-in API) would force a capture per
    // call: after the second distinct buffer set the graph runs on plan-owned staging
    // buffers instead, with device-to-device copies in and out around each replay.
    const bool match = p->gexec && std::memcmp(key, p->gkey, sizeof(key)) == 0;
    const size_t in_b = (size_t)p->batch * p->H * p->W * dtype_size(p->d.img_dtype);
    const size_t def_b = (size_t)p->batch * p->H * p->W;
    const size_t out_b = (size_t)p->batch * p->OH * p->OW * out_size(p->d.out_dtype);
    const size_t val_b = (size_t)p->batch * p->OH * p->OW;
    if (!match && !p->gstaged && ++p->gmiss >= 2) {
      FM_CUDA(cudaMalloc(&p->g_img, in_b));
      FM_CUDA(cudaMalloc(&p->g_def, def_b));
      FM_CUDA(cudaMalloc(&p->g_out, out_b));
      FM_CUDA(cudaMalloc(&p->g_valid, val_b));
      p->gstaged = true;
    }
    const void* gi = img;
    const uint8_t* gd = img_defined;
    void* go = out;
    uint8_t* gv = valid;
    if (p->gstaged) {
      FM_CUDA(cudaMemcpyAsync(p->g_img, img, in_b, cudaMemcpyDeviceToDevice, s));
      if (img_defined) FM_CUDA(cudaMemcpyAsync(p->g_def, img_defined, def_b, cudaMemcpyDeviceToDevice, s));
      gi = p->g_img;
      gd = img_defined ? p->g_def : nullptr;
      go = p->g_out;
      gv = valid ? p->g_valid : nullptr;
      key[0] = gi;
      key[1] = gd;
      key[2] = go;
      key[3] = gv;
    }
    if (!p->gexec || std::memcmp(key, p->gkey, sizeof(key)) != 0) {
      // (re)capture the whole call: memset, range, conv and tonal kernels on s and the
      // range stream, joined back into s
      if (p->gexec) {
        cudaGraphExecDestroy(p->gexec);
        p->gexec = nullptr;
      }
      FM_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      p->capturing = true;
      const long long l0 = g_launches.load();
      const int rc = run_images(p, gi, gd, go, gv, s, 0, p->batch);
      p->capturing = false;
      cudaGraph_t g = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(s, &g);
      if (rc || ec != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();   // a failed capture leaves its error behind: not this plan's next call's
        if (rc) return rc;
        return fail(FM_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ec));
      }
      const cudaError_t ei = cudaGraphInstantiate(&p->gexec, g, 0);
      cudaGraphDestroy(g);
      if (ei != cudaSuccess) {
        p->gexec = nullptr;
        return fail(FM_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ei));
      }
      p->graph_kernels = g_launches.load() - l0;
      g_launches -= p->graph_kernels;   // counted when replayed
      std::memcpy(p->gkey, key, sizeof(key));
    }
    FM_CUDA(cudaGraphLaunch(p->gexec, s));
    g_launches += p->graph_kernels;
    if (p->gstaged) {
      FM_CUDA(cudaMemcpyAsync(out, p->g_out, out_b, cudaMemcpyDeviceToDevice, s));
      if (valid) FM_CUDA(cudaMemcpyAsync(valid, p->g_valid, val_b, cudaMemcpyDeviceToDevice, s));
    }
    FM_CUDA(cudaEventRecord(p->gev_out, s));
    FM_CUDA(cudaStreamWaitEvent(cs, p->gev_out, 0));
    p->last_stream = s;
    return FM_OK;
  }
  return run_images(p, img, img_defined, out, valid, cs, 0, p->batch);
}

int fm_set_timing(fm_plan* p, int enable) {
  if (!p) return fail(FM_EINVAL, "null plan");
  for (fm_plan* q : p->parts) fm_set_timing(q, enable);
  p->timing = enable != 0;
  return FM_OK;
}

int fm_get_timing(fm_plan* p, fm_timing* out, int reset) {
  if (!p) return fail(FM_EINVAL, "null plan");
  if (!p->parts.empty()) {
    fm_timing sum{};
    for (fm_plan* q : p->parts) {
      fm_timing t{};
      int rc = fm_get_timing(q, &t, reset);
      if (rc) return rc;
      sum.conv_ms += t.conv_ms;
      sum.tonal_ms += t.tonal_ms;
      sum.conv_launches += t.conv_launches;
      sum.tonal_launches += t.tonal_launches;
      sum.conv_bytes += t.conv_bytes;
      sum.tonal_bytes += t.tonal_bytes;
      sum.conv_flops += t.conv_flops;
      sum.range_ms += t.range_ms;
      sum.range_launches += t.range_launches;
    }
    if (out) *out = sum;
    return FM_OK;
  }
  DeviceGuard dg(p->device);
  FM_CUDA(cudaStreamSynchronize(p->last_stream));
  FM_CUDA(cudaDeviceSynchronize());
  for (auto& pr : p->pending_conv) {
    float ms = 0.f;
    FM_CUDA(cudaEventElapsedTime(&ms, p->ev_pool[pr.first], p->ev_pool[pr.second]));
    p->acc.conv_ms += ms;
    p->acc.conv_launches++;
  }
  for (auto& pr : p->pending_tonal) {
    float ms = 0.f;
    FM_CUDA(cudaEventElapsedTime(&ms, p->ev_pool[pr.first], p->ev_pool[pr.second]));
    p->acc.tonal_ms += ms;
    p->acc.tonal_launches++;
  }
  for (auto& pr : p->pending_range) {
    float ms = 0.f;
    FM_CUDA(cudaEventElapsedTime(&ms, p->ev_pool[pr.first], p->ev_pool[pr.second]));
    p->acc.range_ms += ms;
    p->acc.range_launches++;
  }
  p->pending_conv.clear();
  p->pending_tonal.clear();
  p->pending_range.clear();
  p->ev_next = 0;
  if (out) *out = p->acc;
  if (reset) p->acc = fm_timing{};
  return FM_OK;
}

int fm_read_stats(fm_plan* p, fm_stats* st) {
  if (!p) return fail(FM_EINVAL, "null plan");
  if (!p->parts.empty()) {
    fm_stats acc{0.0, 0};
    int worst = FM_OK;
    std::string msg;
    for (fm_plan* q : p->parts) {
      fm_stats qs{};
      const int rc = fm_read_stats(q, &qs);
      acc.max_abs_deviation = std::max(acc.max_abs_deviation, qs.max_abs_deviation);
      acc.value_error |= qs.value_error;
      if (rc && !worst) {
        worst = rc;
        msg = g_err;
      }
    }
    if (st) *st = acc;
    return worst ? fail(worst, msg) : FM_OK;
  }
  DeviceGuard dg(p->device);
  FM_CUDA(cudaStreamSynchronize(p->last_stream));
  int h[2] = {0, 0};
  FM_CUDA(cudaMemcpy(h, p->stats, sizeof(int) * 2, cudaMemcpyDeviceToHost));
  float dev;
  std::memcpy(&dev, &h[0], sizeof(float));
  if (st) {
    st->max_abs_deviation = dev;
    st->value_error = h[1];
  }
  if (h[1]) return fail(FM_EINVAL, "image value outside the plan's [img_min, img_max] range");
  if (dev >= 0.25f) {
    char buf[160];
    std::snprintf(buf, sizeof buf, "pre-rounding deviation %.3g >= 0.25; precision budget logic is broken", dev);
    return fail(FM_EDEVIATION, buf);
  }
  return FM_OK;
}

int fm_execute_host(fm_plan* p, const void* img_host, const uint8_t* def_host, void* out_host_v,
                    uint8_t* valid_host, void* stream) {
  if (!p || !img_host || !out_host_v) return fail(FM_EINVAL, "null argument");
  if (p->counts) return fail(FM_EUNSUPPORTED, "count-volume plans run on device buffers (fm_execute)");
  DeviceGuard dg(p->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (!p->parts.empty()) {
    // composite plan: one staged round trip (no chunk pipeline)
    const size_t in_b = (size_t)p->batch * p->H * p->W * dtype_size(p->d.img_dtype);
    const size_t n = (size_t)p->batch * p->OH * p->OW, ob = n * out_elem_size(p->d.out_dtype);
    char* buf = nullptr;
    FM_CUDA(cudaMallocAsync(&buf, in_b + (def_host ? (size_t)p->batch * p->H * p->W : 0) + ob + n, s));
    char* di = buf;
    uint8_t* dd = def_host ? reinterpret_cast<uint8_t*>(buf + in_b) : nullptr;
    char* dout = buf + in_b + (def_host ? (size_t)p->batch * p->H * p->W : 0);
    uint8_t* dv = reinterpret_cast<uint8_t*>(dout + ob);
    int rc = FM_OK;
    cudaError_t e = cudaMemcpyAsync(di, img_host, in_b, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && dd) e = cudaMemcpyAsync(dd, def_host, (size_t)p->batch * p->H * p->W, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) rc = execute_composite(p, di, dd, dout, dv, s);
    if (e == cudaSuccess && !rc) e = cudaMemcpyAsync(out_host_v, dout, ob, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && !rc && valid_host) e = cudaMemcpyAsync(valid_host, dv, n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && !rc) e = cudaStreamSynchronize(s);
    cudaFreeAsync(buf, s);
    if (rc) return rc;
    if (e != cudaSuccess) return fail(FM_ECUDA, std::string("composite host path: ") + cudaGetErrorString(e));
    return FM_OK;
  }
  const size_t in_n = (size_t)p->batch * p->H * p->W;
  const size_t out_n = (size_t)p->batch * p->OH * p->OW;
  const size_t dsz = dtype_size(p->d.img_dtype);
  const size_t osz = out_size(p->d.out_dtype);
  char* out_host = reinterpret_cast<char*>(out_host_v);
  if (!p->h_img) {
    // allocate into locals and commit to the plan only when every call succeeded (a
    // partial failure leaves the plan without staging, so the next call retries)
    void* hi = nullptr;
    uint8_t *hd = nullptr, *hv = nullptr;
    int32_t* ho = nullptr;
    cudaStream_t cs = nullptr, ds2 = nullptr;
    cudaEvent_t evi = nullptr;
    const int64_t nchunks = (p->batch + p->ipc - 1) / p->ipc;
    std::vector<cudaEvent_t> evs(2 * nchunks, nullptr);
    cudaError_t e = cudaMalloc(&hi, in_n * dsz);
    if (e == cudaSuccess) e = cudaMalloc(&hd, in_n);
    if (e == cudaSuccess) e = cudaMalloc(&ho, out_n * osz);
    if (e == cudaSuccess) e = cudaMalloc(&hv, out_n);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ds2, cudaStreamNonBlocking);
    for (auto& ev : evs)
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&evi, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      cudaFree(hi);
      cudaFree(hd);
      cudaFree(ho);
      cudaFree(hv);
      if (cs) cudaStreamDestroy(cs);
      if (ds2) cudaStreamDestroy(ds2);
      for (auto ev : evs)
        if (ev) cudaEventDestroy(ev);
      if (evi) cudaEventDestroy(evi);
      return fail(e == cudaErrorMemoryAllocation ? FM_ENOMEM : FM_ECUDA,
                  std::string("host-path staging: ") + cudaGetErrorString(e));
    }
    p->h_img = hi;
    p->h_def = hd;
    p->h_out = ho;
    p->h_valid = hv;
    p->copy_stream = cs;
    p->d2h_stream = ds2;
    p->ev_chunks = std::move(evs);
    p->ev_in = evi;
  }
  // Chunk pipeline: every H2D is queued up front on one copy stream, each
  // chunk's compute on `s` waits only for its own input, and its D2H runs on a
  // second copy stream while later chunks compute (pinned host memory).
  const size_t img_e = (size_t)p->H * p->W, out_e = (size_t)p->OH * p->OW;
  const char* hin = reinterpret_cast<const char*>(img_host);
  char* din = reinterpret_cast<char*>(p->h_img);
  cudaStream_t hs = p->copy_stream, ds = p->d2h_stream;
  FM_CUDA(cudaEventRecord(p->ev_in, s));          // order after prior work on s
  FM_CUDA(cudaStreamWaitEvent(hs, p->ev_in, 0));
  FM_CUDA(cudaStreamWaitEvent(ds, p->ev_in, 0));
  // every H2D is queued up front on hs (one event per chunk of ipc images);
  // one run_images call then pipelines the whole batch (the range kernels run
  // a step ahead as in fm_execute) and each chunk's D2H is queued on ds as soon
  // as its tonal kernels are
  // chunk plan: one-image chunks first and last, so the pipeline fills after one
  // image's upload and drains after one image's download
  std::vector<std::pair<int64_t, int>> chunks;
  {
    int64_t c0 = 0, left = p->batch;
    if (left > 2 && p->ipc > 1) {
      chunks.push_back({0, 1});
      c0 = 1;
      left -= 1;
    }
    while (left > 0) {
      int64_t n = std::min<int64_t>(p->ipc, left);
      if (n == left && n > 1 && p->ipc > 1 && p->batch > 2) n -= 1;
      chunks.push_back({c0, (int)n});
      c0 += n;
      left -= n;
    }
  }
  const int64_t nchunks = (int64_t)chunks.size();
  if ((int64_t)p->ev_chunks.size() < 2 * nchunks) {
    const size_t old = p->ev_chunks.size();
    p->ev_chunks.resize(2 * nchunks);
    for (size_t i = old; i < p->ev_chunks.size(); ++i)
      FM_CUDA(cudaEventCreateWithFlags(&p->ev_chunks[i], cudaEventDisableTiming));
  }
  std::vector<cudaEvent_t> in_ev(nchunks);
  for (int64_t ci = 0; ci < nchunks; ++ci) {
    const int64_t c0 = chunks[ci].first, n = chunks[ci].second;
    FM_CUDA(cudaMemcpyAsync(din + c0 * img_e * dsz, hin + c0 * img_e * dsz, n * img_e * dsz, cudaMemcpyHostToDevice, hs));
    if (def_host)
      FM_CUDA(cudaMemcpyAsync(p->h_def + c0 * img_e, def_host + c0 * img_e, n * img_e, cudaMemcpyHostToDevice, hs));
    FM_CUDA(cudaEventRecord(p->ev_chunks[2 * ci], hs));
    in_ev[ci] = p->ev_chunks[2 * ci];
  }
  auto after = [&](size_t ci, int64_t c0, int n, cudaStream_t done) -> int {
    FM_CUDA(cudaEventRecord(p->ev_chunks[2 * ci + 1], done));   // the chunk's outputs are written on `done`
    FM_CUDA(cudaStreamWaitEvent(ds, p->ev_chunks[2 * ci + 1], 0));
    FM_CUDA(cudaMemcpyAsync(out_host + c0 * out_e * osz, reinterpret_cast<char*>(p->h_out) + c0 * out_e * osz,
                            n * out_e * osz, cudaMemcpyDeviceToHost, ds));
    if (valid_host)
      FM_CUDA(cudaMemcpyAsync(valid_host + c0 * out_e, p->h_valid + c0 * out_e, n * out_e, cudaMemcpyDeviceToHost, ds));
    return FM_OK;
  };
  {
    int rc = run_images(p, p->h_img, def_host ? p->h_def : nullptr, p->h_out, valid_host ? p->h_valid : nullptr, s, 0,
                        p->batch, &chunks, in_ev.data(), after);
    if (rc) return rc;
  }
  FM_CUDA(cudaStreamSynchronize(ds));
  FM_CUDA(cudaStreamSynchronize(s));
  return FM_OK;
}

void fm_plan_destroy(fm_plan* p) { free_plan(p); }

int fm_conv_full_direct(int ndim, const int64_t* a_shape, const int64_t* a, const int64_t* b_shape,
                        const int64_t* b, int64_t* out, void* stream) {
  if (ndim < 1 || ndim > 3) return fail(FM_EINVAL, "ndim must be 1..3");
  if (!a_shape || !b_shape || !a || !b || !out) return fail(FM_EINVAL, "null argument");
  DirectArgs d{};
  d.nout = 1;
  for (int i = 0; i < 3; ++i) {
    const int j = i - (3 - ndim);
    d.as[i] = j >= 0 ? a_shape[j] : 1;
    d.bs[i] = j >= 0 ? b_shape[j] : 1;
    if (d.as[i] < 1 || d.bs[i] < 1) return fail(FM_EINVAL, "empty array");
    d.os[i] = d.as[i] + d.bs[i] - 1;
    d.nout *= d.os[i];
  }
  d.a = a;
  d.b = b;
  d.out = out;
  const int64_t blocks = (d.nout + 255) / 256;
  if (blocks > (1ll << 31) - 1) return fail(FM_EUNSUPPORTED, "output too large");
  conv_direct_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(d);
  g_launches++;
  FM_CUDA(cudaGetLastError());
  return FM_OK;
}

// ---- count level in FP64 (fm_fft64.cuh) --------------------------------------------
}  // extern "C"

namespace {

unsigned fft64_grid(int64_t n) {
  const int64_t b = (n + kFft64NT - 1) / kFft64NT;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)g_num_sms * 16));
}

// radix order of a ladder length (2^k or 45*2^k): 4s, a 2, 3s, 5s
std::vector<int> fft64_radices(int64_t n) {
  std::vector<int> r;
  while (n % 4 == 0) { r.push_back(4); n /= 4; }
  while (n % 2 == 0) { r.push_back(2); n /= 2; }
  while (n % 3 == 0) { r.push_back(3); n /= 3; }
  while (n % 5 == 0) { r.push_back(5); n /= 5; }
  if (n != 1) r.clear();
  return r;
}
bool fft64_ok(int64_t n) { return n == 1 || !fft64_radices(n).empty(); }

// N-D complex FFT of a [d0][d1][d2][d3] volume (sign -1 forward, +1 inverse, unnormalised);
// ping-pongs between `a` and `tmp`, returns the buffer holding the result
int fft64_nd(double2* a, double2* tmp, const Shape4& s, int sign, cudaStream_t st, double2** result) {
  double2* in = a;
  double2* outb = tmp;
  const int64_t total = s.d[0] * s.d[1] * s.d[2] * s.d[3];
  for (int ax = 0; ax < 4; ++ax) {
    const int64_t n = s.d[ax];
    if (n == 1) continue;
    int64_t outer = 1, inner = 1;
    for (int k = 0; k < ax; ++k) outer *= s.d[k];
    for (int k = ax + 1; k < 4; ++k) inner *= s.d[k];
    const std::vector<int> rad = fft64_radices(n);
    if (rad.empty()) return fail(FM_EINVAL, "FFT length must factor into 2, 3 and 5");
    int64_t Ns = 1;
    for (int R : rad) {
      const unsigned g = fft64_grid(total / R);
      switch (R) {
        case 2: fft64_stage<2><<<g, kFft64NT, 0, st>>>(in, outb, outer, n, inner, Ns, sign); break;
        case 3: fft64_stage<3><<<g, kFft64NT, 0, st>>>(in, outb, outer, n, inner, Ns, sign); break;
        case 4: fft64_stage<4><<<g, kFft64NT, 0, st>>>(in, outb, outer, n, inner, Ns, sign); break;
        default: fft64_stage<5><<<g, kFft64NT, 0, st>>>(in, outb, outer, n, inner, Ns, sign); break;
      }
      g_launches++;
      FM_CUDA(cudaGetLastError());
      Ns *= R;
      std::swap(in, outb);
    }
  }
  *result = in;
  return FM_OK;
}

int shape4(int ndim, const int64_t* shape, Shape4* s) {
  if (ndim < 1 || ndim > 4) return fail(FM_EINVAL, "ndim must be 1..4");
  for (int i = 0; i < 4; ++i) {
    const int j = i - (4 - ndim);
    s->d[i] = j >= 0 ? shape[j] : 1;
    if (s->d[i] < 1) return fail(FM_EINVAL, "empty array");
  }
  return FM_OK;
}

}  // namespace

extern "C" {

int fm_conv_full_fft64(int ndim, const int64_t* a_shape, const int64_t* a, const int64_t* b_shape, const int64_t* b,
                       const int64_t* padded, int64_t* out, double* max_dev, void* stream) {
  if (!a_shape || !b_shape || !a || !b || !padded || !out) return fail(FM_EINVAL, "null argument");
  Shape4 sa, sb, sp, so;
  int rc = shape4(ndim, a_shape, &sa);
  if (!rc) rc = shape4(ndim, b_shape, &sb);
  if (!rc) rc = shape4(ndim, padded, &sp);
  if (rc) return rc;
  int64_t P = 1;
  for (int i = 0; i < 4; ++i) {
    so.d[i] = sa.d[i] + sb.d[i] - 1;
    if (sp.d[i] < so.d[i]) return fail(FM_EINVAL, "padded shape smaller than the full output");
    if (!fft64_ok(sp.d[i])) return fail(FM_EINVAL, "padded length must factor into 2, 3 and 5");
    P *= sp.d[i];
  }
  cudaStream_t st = (cudaStream_t)stream;
  double2* buf = nullptr;
  unsigned long long* dbits = nullptr;
  FM_CUDA(cudaMallocAsync(&buf, sizeof(double2) * 4 * (size_t)P, st));
  cudaError_t e = cudaMallocAsync(&dbits, sizeof(unsigned long long), st);
  if (e != cudaSuccess) {
    cudaFreeAsync(buf, st);
    return fail(FM_ENOMEM, std::string("fft64 alloc: ") + cudaGetErrorString(e));
  }
  double2 *A = buf, *At = buf + P, *Bb = buf + 2 * P, *Bt = buf + 3 * P, *ra = nullptr, *rb = nullptr, *rc2 = nullptr;
  auto run = [&]() -> int {
    FM_CUDA(cudaMemsetAsync(dbits, 0, sizeof(unsigned long long), st));
    fft64_pad<<<fft64_grid(P), kFft64NT, 0, st>>>(a, sa, sp, A);
    fft64_pad<<<fft64_grid(P), kFft64NT, 0, st>>>(b, sb, sp, Bb);
    g_launches += 2;
    FM_CUDA(cudaGetLastError());
    int r = fft64_nd(A, At, sp, -1, st, &ra);
    if (!r) r = fft64_nd(Bb, Bt, sp, -1, st, &rb);
    if (r) return r;
    fft64_product<<<fft64_grid(P), kFft64NT, 0, st>>>(ra, rb, P);
    g_launches++;
    FM_CUDA(cudaGetLastError());
    r = fft64_nd(ra, ra == A ? At : A, sp, +1, st, &rc2);
    if (r) return r;
    const int64_t O = so.d[0] * so.d[1] * so.d[2] * so.d[3];
    fft64_finish<<<fft64_grid(O), kFft64NT, 0, st>>>(rc2, sp, so, 1.0 / (double)P, out, dbits);
    g_launches++;
    FM_CUDA(cudaGetLastError());
    unsigned long long h = 0;
    FM_CUDA(cudaMemcpyAsync(&h, dbits, sizeof(h), cudaMemcpyDeviceToHost, st));
    FM_CUDA(cudaStreamSynchronize(st));
    double d;
    std::memcpy(&d, &h, sizeof(d));
    if (max_dev) *max_dev = d;
    return FM_OK;
  };
  rc = run();
  cudaFreeAsync(buf, st);
  cudaFreeAsync(dbits, st);
  return rc;
}

int fm_fft64(int ndim, const int64_t* shape, void* data, int inverse, void* stream) {
  if (!shape || !data) return fail(FM_EINVAL, "null argument");
  Shape4 s;
  int rc = shape4(ndim, shape, &s);
  if (rc) return rc;
  for (int i = 0; i < 4; ++i)
    if (!fft64_ok(s.d[i])) return fail(FM_EINVAL, "length must factor into 2, 3 and 5");
  const int64_t P = s.d[0] * s.d[1] * s.d[2] * s.d[3];
  cudaStream_t st = (cudaStream_t)stream;
  double2* tmp = nullptr;
  FM_CUDA(cudaMallocAsync(&tmp, sizeof(double2) * (size_t)P, st));
  double2* res = nullptr;
  double2* d = reinterpret_cast<double2*>(data);
  rc = fft64_nd(d, tmp, s, inverse ? +1 : -1, st, &res);
  if (!rc && res != d) {
    cudaError_t e = cudaMemcpyAsync(d, res, sizeof(double2) * (size_t)P, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) rc = fail(FM_ECUDA, cudaGetErrorString(e));
  }
  cudaFreeAsync(tmp, st);
  return rc;
}

int fm_build_umbra(int64_t npx, const int64_t* values, const uint8_t* defined, int64_t t, int64_t* bits,
                   void* stream) {
  if (!values || !bits || npx < 0 || t < 1) return fail(FM_EINVAL, "bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  FM_CUDA(cudaMemsetAsync(bits, 0, sizeof(int64_t) * (size_t)npx * (size_t)t, st));
  if (npx == 0) return FM_OK;
  umbra_kernel<<<fft64_grid(npx), kFft64NT, 0, st>>>(values, defined, npx, t, bits);
  g_launches++;
  FM_CUDA(cudaGetLastError());
  return FM_OK;
}

int fm_project(int64_t npx, int64_t t, const int64_t* window, int64_t* values, uint8_t* valid, void* stream) {
  if (!window || !values || !valid || npx < 0 || t < 1) return fail(FM_EINVAL, "bad argument");
  if (npx == 0) return FM_OK;
  project_kernel<<<fft64_grid(npx), kFft64NT, 0, (cudaStream_t)stream>>>(window, npx, t, values, valid);
  g_launches++;
  FM_CUDA(cudaGetLastError());
  return FM_OK;
}

// ---- row strips across GPUs: halo rows by NVLink peer copies ----------------------

int fm_copy_peer(void* dst, int dst_device, const void* src, int src_device, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return fail(FM_EINVAL, "bad argument");
  if (bytes == 0) return FM_OK;
  if (dst_device < 0 || src_device < 0)   // IPC-mapped peer memory: location from unified addressing
    FM_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  else
    FM_CUDA(cudaMemcpyPeerAsync(dst, dst_device, src, src_device, (size_t)bytes, (cudaStream_t)stream));
  return FM_OK;
}

int fm_ipc_get_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out) {
  if (!dev_ptr || !handle_out || !offset_out) return fail(FM_EINVAL, "null argument");
  // the handle names the whole allocation (a caching allocator may place the buffer
  // inside a larger block): report the buffer's offset from the allocation base
  typedef CUresult (*RangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
  static RangeFn range_fn = nullptr;
  if (!range_fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(FM_ECUDA, "cuMemGetAddressRange unavailable");
    range_fn = reinterpret_cast<RangeFn>(f);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) return fail(FM_ECUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  FM_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
  std::memcpy(handle_out, &h, sizeof(h));
  *offset_out = (int64_t)((CUdeviceptr)dev_ptr - base);
  return FM_OK;
}

int fm_ipc_open_handle(const void* handle, int device, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(FM_EINVAL, "null argument");
  DeviceGuard dg(device);
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  FM_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return FM_OK;
}

int fm_ipc_close_handle(void* dev_ptr) {
  if (!dev_ptr) return fail(FM_EINVAL, "null argument");
  FM_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return FM_OK;
}

int fm_naive(const fm_plan_desc* desc, const int32_t* se_values, const uint8_t* se_defined, const void* img,
             const uint8_t* img_defined, int32_t* out, uint8_t* valid, void* stream) {
  int rc = validate_common(desc);
  if (rc) return rc;
  if (!se_values || !img || !out) return fail(FM_EINVAL, "null argument");
  const fm_plan_desc& d = *desc;
  const bool two_d = d.ndim == 2;
  const int64_t H = two_d ? d.shape[0] : 1, W = two_d ? d.shape[1] : d.shape[0];
  const int64_t my = two_d ? d.se_shape[0] : 1, mx = two_d ? d.se_shape[1] : d.se_shape[0];
  const int64_t lo_y = two_d ? d.se_lo[0] : 0, lo_x = two_d ? d.se_lo[1] : d.se_lo[0];
  std::vector<int4> ent;
  for (int64_t jy = 0; jy < my; ++jy)
    for (int64_t jx = 0; jx < mx; ++jx) {
      const int64_t i = jy * mx + jx;
      if (se_defined && !se_defined[i]) continue;
      ent.push_back(make_int4((int)jy, (int)jx, se_values[i], 0));
    }
  if (ent.empty()) return fail(FM_EINVAL, "grid needs at least one defined pixel");
  const bool erode = d.mode == FM_ERODE;
  // output ranges: dilate_naive (tensor.py:76-89) / erode_naive (morphology.py:92-93)
  int64_t off_y = 0, off_x = 0, OH = H, OW = W;
  if (!d.crop) {
    off_y = two_d ? (erode ? -(lo_y + my - 1) : lo_y) : 0;
    off_x = erode ? -(lo_x + mx - 1) : lo_x;
    OH = two_d ? H + my - 1 : 1;
    OW = W + mx - 1;
  }
  NaiveArgs a{};
  a.img = img;
  a.img_def = img_defined;
  a.img_dtype = d.img_dtype;
  a.H = (int)H;
  a.W = (int)W;
  a.OH = (int)OH;
  a.OW = (int)OW;
  // dilation: i = a + (off - lo) - j ; erosion: i = a + (off + lo) + j
  a.CY = (int)(erode ? off_y + lo_y : off_y - lo_y);
  a.CX = (int)(erode ? off_x + lo_x : off_x - lo_x);
  if (!two_d) a.CY = 0;
  a.erode = erode ? 1 : 0;
  a.nent = (int)ent.size();
  a.fill = d.fill;
  a.out = out;
  a.valid = valid;
  DeviceGuard dg(d.device);
  int4* dent = nullptr;
  FM_CUDA(cudaMalloc(&dent, sizeof(int4) * ent.size()));
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemcpyAsync(dent, ent.data(), sizeof(int4) * ent.size(), cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) {
    a.ent = dent;
    naive_kernel<<<dim3((unsigned)((OW + 31) / 32), (unsigned)((OH + 7) / 8), (unsigned)d.batch), 256, 0, s>>>(a);
    g_launches++;
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  cudaFree(dent);
  if (e != cudaSuccess) return fail(FM_ECUDA, std::string("naive kernel: ") + cudaGetErrorString(e));
  return FM_OK;
}

}  // extern "C"
