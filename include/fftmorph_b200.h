/*
 * fftmorph_b200.h — C ABI of the B200-native exact grey-scale dilation/erosion
 * hot path (arXiv 2305.03018: tonal one-hot encode -> FFT convolution ->
 * highest nonzero degree; erosion by duality).
 *
 * The reference (`fftmorph`, pure Python) has no FFI; its hot path is the
 * Python call chain listed beside each entry point.  This header is what a
 * ctypes / cffi binding of that path binds.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Image / output / validity pointers given
 *    to fm_execute are DEVICE pointers owned by the caller; fm_execute_host
 *    takes HOST pointers (pinned recommended) and does the copies itself.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Every entry point returns an fm_status; fm_last_error() gives a
 *    thread-local message for the last failure on the calling thread.
 *  - Status codes map onto the reference's exception types:
 *      FM_EINVAL       -> ValueError            (umbra.py:36-59, morphology.py:119-120,158-161)
 *      FM_EPRECISION   -> PrecisionBudgetError  (fft_conv.py:37-38,114-125)
 *      FM_EDEVIATION   -> ArithmeticError       (fft_conv.py:145-148)
 *      FM_EUNSUPPORTED -> NotImplementedError   (shape outside the built tile set)
 *      FM_ECUDA        -> RuntimeError
 *  - A plan is reentrant per (plan, stream); different plans are independent.
 */
#ifndef FFTMORPH_B200_H
#define FFTMORPH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FM_ABI_VERSION 4

typedef enum fm_status {
  FM_OK = 0,
  FM_EINVAL = 1,
  FM_EPRECISION = 2,
  FM_EDEVIATION = 3,
  FM_ECUDA = 4,
  FM_EUNSUPPORTED = 5,
  FM_ENOMEM = 6
} fm_status;

typedef enum fm_mode { FM_DILATE = 0, FM_ERODE = 1 } fm_mode;

typedef enum fm_dtype { FM_U8 = 0, FM_U16 = 1, FM_I32 = 2 } fm_dtype;

/* Output element type (the plan checks that every possible output value fits). */
typedef enum fm_out_dtype { FM_OUT_I32 = 0, FM_OUT_U8 = 1, FM_OUT_U16 = 2, FM_OUT_I16 = 3 } fm_out_dtype;

/* Plan description.  1-D signals use ndim=1 and shape[0]/se_shape[0]/se_lo[0]. */
typedef struct fm_plan_desc {
  int32_t ndim;          /* 1 or 2 */
  int32_t mode;          /* fm_mode */
  int32_t crop;          /* 1: output over the image domain (reference default);
                            0: whole Minkowski range f.lo+b.lo .. f.hi+b.hi (dilation) /
                               f.lo-b.hi .. f.hi-b.lo (erosion);
                            2: the window win_lo .. win_lo+win_shape-1 (image array indices;
                               row strips of one image: each strip computes exactly its
                               owned output rows from its rows plus the SE-radius halos) */
  int32_t img_dtype;     /* fm_dtype of the image buffer */
  int64_t batch;         /* images per fm_execute call, all of `shape` */
  int64_t shape[2];      /* image array shape (row-major) */
  int64_t se_shape[2];   /* structuring-element array shape */
  int64_t se_lo[2];      /* logical index of the SE's first element (may be any sign) */
  int32_t img_min;       /* lower bound of defined image values (data minimum for exact T) */
  int32_t img_max;       /* upper bound of defined image values; values outside
                            [img_min, img_max] make fm_execute fail with FM_EINVAL */
  int32_t fill;          /* output value at pixels with no (image, SE) pair */
  int32_t device;        /* CUDA device ordinal */
  int64_t scratch_bytes; /* spectral scratch budget (0 = default 16 GiB) */
  int32_t tile;          /* 0 = auto, else forced FFT tile edge (16..256) */
  int32_t tonal_len;     /* 0 = auto, else forced tonal length T (even, > l_R) */
  int32_t out_dtype;     /* fm_out_dtype of the output values (0 = int32) */
  int32_t flags;         /* FM_FLAG_* */
  int32_t count_budget;  /* a-priori FP32 precision budget: the largest count a pixel can
                            reach (<= defined SE entries) must stay below it, else
                            fm_plan_create returns FM_EPRECISION (the FP32 analogue of
                            check_precision_budget, fft_conv.py:114-125); 0 = default 2^17 */
  int32_t reserved;      /* 0 */
  int64_t win_lo[2];     /* crop = 2: first output index per axis (image array coordinates) */
  int64_t win_shape[2];  /* crop = 2: output extent per axis */
} fm_plan_desc;

/* fm_plan_desc.flags */
enum {
  /* Count-volume mode (dilation only): fm_execute writes, instead of the dilation,
   * the count volume of umbra(f) (*) umbra(b) over the full Minkowski range
   * (crop must be 0) as int32 [batch][OH][OW][count_len], count_len = l_r + 1,
   * degree index d <-> degree d + img_min + se_min; replaces
   * conv_full_fft_with_stats(build_umbra(f), build_umbra(b)) (fft_conv.py:128-150,
   * umbra.py:177-186).  `valid` still receives "any count". */
  FM_FLAG_COUNTS = 1
};

/* Read-only facts about a plan (for stats / bench / tests). */
typedef struct fm_plan_info {
  int32_t tonal_len;       /* T */
  int32_t planes;          /* T/2+1 tonal frequency planes computed */
  int32_t l_r;             /* tonal extent actually needed: (img_max-img_min)+(se_max-se_min) */
  int32_t tile_y, tile_x;  /* FFT tile edges (tile_y = 1 for 1-D) */
  int32_t valid_y, valid_x;/* output pixels per tile per axis */
  int32_t tiles_y, tiles_x;
  int32_t k_chunk;         /* tonal planes per CTA */
  int64_t out_shape[2];    /* output array shape */
  int64_t out_lo_offset[2];/* output lo minus image lo, per axis */
  int64_t images_per_launch;
  int64_t scratch_bytes;
  int32_t se_min, se_max;  /* over defined SE entries (after reflection for erosion) */
  int32_t se_count;        /* defined SE entries */
  int32_t count_len;       /* FM_FLAG_COUNTS: degrees per output pixel (l_r + 1), else 0 */
} fm_plan_info;

typedef struct fm_stats {
  double max_abs_deviation; /* max |x - rint(x)| over all computed counts (reference
                               stats["max_abs_deviation"], morphology.py:125-127) */
  int32_t value_error;      /* nonzero: an image value fell outside [img_min, img_max] */
} fm_stats;

/* Per-kernel device time of the launches made while timing was enabled
 * (CUDA events recorded on the launch stream around every kernel), and the
 * algorithmic bytes those launches move (the roofline numerator). */
typedef struct fm_timing {
  double conv_ms;          /* encode + spatial FFT conv kernel (fm_tile.cuh) */
  double tonal_ms;         /* inverse tonal FFT + threshold kernel (fm_tonal.cuh) */
  int64_t conv_launches;
  int64_t tonal_launches;
  double conv_bytes;       /* image read + spectral volume written */
  double tonal_bytes;      /* spectral volume read + int32 values (+ validity) written */
  double conv_flops;       /* nominal FFT flops: per tile and plane 2*5*P^2*log2(P^2) + 6*P^2 */
  double range_ms;         /* per-unit range + clamp bound kernel (fm_range.cuh) */
  int64_t range_launches;
} fm_timing;

typedef struct fm_plan fm_plan;

/* Create a plan and precompute the SE spectrum (once per SE).
 * Replaces, per call of the reference: required_lr (umbra.py:172-174),
 * build_umbra(b) (umbra.py:177-186), make_plan (fft_conv.py:80-91),
 * rfftn(b) (fft_conv.py:135-136), and for erosion reflect(b) (morphology.py:147-152).
 * se_values: int32[se_shape] host array; se_defined: uint8[se_shape] host array or NULL
 * (all defined).  SE values must be >= 0 (dilate_fft, morphology.py:119-120). */
int fm_plan_create(fm_plan** plan, const fm_plan_desc* desc,
                   const int32_t* se_values, const uint8_t* se_defined);

/* Run the hot path on a device-resident batch.
 * Replaces dilate_fft (morphology.py:116-144) / erode_fft (morphology.py:166-180):
 * build_umbra(f) + rfftn(f) + product + irfftn + rint/deviation + project_with_validity
 * + _paste (umbra.py:177-205, fft_conv.py:128-150, morphology.py:51-62).
 * img: device [batch, shape] of img_dtype; img_defined: device uint8 [batch, shape] or NULL;
 * out: device [batch, out_shape] of the plan's out_dtype; valid: device uint8 [batch, out_shape] or NULL.
 * Asynchronous on `stream`; deviation/value errors are read with fm_read_stats. */
int fm_execute(fm_plan* plan, const void* img, const uint8_t* img_defined,
               void* out, uint8_t* valid, void* stream);

/* Same as fm_execute but with HOST buffers; copies in and out on `stream` and
 * synchronizes before returning (the reference-facing call with host memory). */
int fm_execute_host(fm_plan* plan, const void* img_host, const uint8_t* img_defined_host,
                    void* out_host, uint8_t* valid_host, void* stream);

/* Synchronize the plan's last stream, return the stats accumulated since the last
 * fm_reset_stats, and map them to a status: FM_EINVAL on a value error,
 * FM_EDEVIATION if max_abs_deviation >= 0.25 (fft_conv.py:22,145-148). */
int fm_read_stats(fm_plan* plan, fm_stats* stats);
int fm_reset_stats(fm_plan* plan, void* stream);

int fm_plan_query(const fm_plan* plan, fm_plan_info* info);

/* Enable/disable per-kernel event timing on a plan; fm_get_timing synchronizes,
 * accumulates all recorded event pairs and optionally resets the totals. */
int fm_set_timing(fm_plan* plan, int enable);
int fm_get_timing(fm_plan* plan, fm_timing* timing, int reset);
void fm_plan_destroy(fm_plan* plan);

/* Exact direct max-plus dilation / min-plus erosion on the GPU with the
 * reference's naive semantics (dilate_naive / erode_naive, morphology.py:65-113):
 * verification path and method="naive".  Same desc fields as a plan
 * (img_min/img_max unused; fill = neutral value).  Synchronous. */
int fm_naive(const fm_plan_desc* desc, const int32_t* se_values, const uint8_t* se_defined,
             const void* img, const uint8_t* img_defined, int32_t* out, uint8_t* valid,
             void* stream);

/* Number of CUDA kernels this library launched since load (evidence counter). */
int64_t fm_kernel_launches(void);

const char* fm_last_error(void);

/* Exact full-mode N-D (ndim 1..3) integer convolution on the device:
 * out[k] = sum_i a[i] b[k-i], shapes sa + sb - 1 (direct_full, fft_conv.py:94-106;
 * conv_full_direct, fft_conv.py:109-111).  int64 device buffers, row-major. */
int fm_conv_full_direct(int ndim, const int64_t* a_shape, const int64_t* a, const int64_t* b_shape,
                        const int64_t* b, int64_t* out, void* stream);
/* Full-mode N-D (ndim 1..4) convolution of int64 volumes by FP64 FFTs on the device,
 * zero-padded to `padded` (every length 2^k or 45*2^k, fft_conv.py:61-91), then slice,
 * rint and the max pre-rounding deviation (written to *max_dev, host): replaces
 * conv_full_fft_with_stats for operands that are not tonal one-hot volumes
 * (fft_conv.py:128-150; precision budget 2^52 as fft_conv.py:114-125, checked by the
 * caller).  a, b, out: device buffers, row-major; out has shape a_shape + b_shape - 1.
 * Synchronous on `stream`. */
int fm_conv_full_fft64(int ndim, const int64_t* a_shape, const int64_t* a, const int64_t* b_shape,
                       const int64_t* b, const int64_t* padded, int64_t* out, double* max_dev, void* stream);

/* In-place N-D (ndim 1..4) complex FP64 DFT of a device volume of interleaved (re, im)
 * doubles: forward exp(-2 pi i jk/n) unnormalised, or inverse (1/n not applied):
 * transform_forward / transform_inverse (fft_conv.py:157-170).  Lengths 2, 3, 5-smooth. */
int fm_fft64(int ndim, const int64_t* shape, void* data, int inverse, void* stream);

/* build_umbra (umbra.py:177-186) on the device: bits[npx][t] int64 = 1 at (x, values[x])
 * for defined x (defined may be NULL), 0 elsewhere.  Values must lie in [0, t). */
int fm_build_umbra(int64_t npx, const int64_t* values, const uint8_t* defined, int64_t t, int64_t* bits,
                   void* stream);

/* project_with_validity's reduction (umbra.py:189-205) over a contiguous count window
 * [npx][t]: values[x] = highest k with window[x][k] >= 1 (0 if none), valid[x] = any. */
int fm_project(int64_t npx, int64_t t, const int64_t* window, int64_t* values, uint8_t* valid, void* stream);

/* Row strips of one image across GPUs: the SE-radius halo rows a strip
 * needs from its neighbours move by NVLink peer copies, no collective.
 * fm_copy_peer: cudaMemcpyPeerAsync of `bytes` from src (on src_device) to dst (on
 * dst_device), asynchronous on `stream` (same-device copies allowed; a negative device
 * means IPC-mapped peer memory, copied by unified addressing).
 * fm_ipc_get_handle / fm_ipc_open_handle / fm_ipc_close_handle: one process per GPU --
 * export a device buffer as a 64-byte CUDA IPC handle plus the buffer's byte offset in its
 * allocation, map a peer's handle into this process (peer access enabled), unmap it. */
int fm_copy_peer(void* dst, int dst_device, const void* src, int src_device, int64_t bytes, void* stream);
int fm_ipc_get_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out);
int fm_ipc_open_handle(const void* handle, int device, void** dev_ptr);
int fm_ipc_close_handle(void* dev_ptr);

int fm_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FFTMORPH_B200_H */
