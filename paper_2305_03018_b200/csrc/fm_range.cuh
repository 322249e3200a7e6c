// fm_range.cuh — per-unit tonal range (the local l_R of each tile).
//
// The reference sizes the tonal axis from the global data maxima
// (required_lr, umbra.py:172-174).  Exactness only needs, for every output
// pixel, a tonal length larger than the spread of the degrees that can meet
// there: (max f - min f over the pixel's input window) + (max b - min b).
// This kernel computes min/max of the defined values over every conv unit's
// input window (one 2-D tile, or a group of 1-D tiles), picks the smallest
// tonal length T_t = 2 N_t of the plan's ladder with T_t > l_R,t, records the
// unit's anchor value (min f for dilation, max f for erosion), and appends the
// unit to the work list of its ladder entry (the tonal kernel is specialised
// per N).  Values outside the plan's [img_min, img_max] raise the error flag.
#pragma once
#include <stdint.h>
#include <cuda_runtime.h>

namespace fm {

struct RangeArgs {
  const void* img;
  const uint8_t* img_def;
  int img_dtype;
  int H, W;
  int two_d;
  int DY, DX, QY, QX;
  int win_y, win_x;       // input window extent of one unit
  int tiles_x;            // 2-D tile grid width
  int units;              // units per image
  int unit0;              // first unit of this launch
  int unit_step_x;        // 1-D: output pixels per unit (tiles_per_unit * QX)
  int img_min, img_max;
  int enc_sign;           // +1 dilation, -1 erosion
  int lr_se;              // se_max - se_min
  const int* ladder;      // ascending N values
  int L;
  int4* unit_param;       // [imgs][units]
  int* bucket_count;      // [L]
  int2* bucket_list;      // [L][cap]
  int cap;
  int* err;
};

__device__ __forceinline__ int range_load(const void* img, int dtype, int64_t i) {
  if (dtype == 0) return (int)__ldg(reinterpret_cast<const uint8_t*>(img) + i);
  if (dtype == 1) return (int)__ldg(reinterpret_cast<const uint16_t*>(img) + i);
  return __ldg(reinterpret_cast<const int32_t*>(img) + i);
}

__global__ void __launch_bounds__(256) range_kernel(const RangeArgs a) {
  const int unit = a.unit0 + blockIdx.x, img = blockIdx.y;
  int y0, x0;
  if (a.two_d) {
    const int ty = unit / a.tiles_x, tx = unit - (unit / a.tiles_x) * a.tiles_x;
    y0 = ty * a.QY + a.DY;
    x0 = tx * a.QX + a.DX;
  } else {
    y0 = 0;
    x0 = unit * a.unit_step_x + a.DX;
  }
  const int ya = max(y0, 0), yb = min(y0 + a.win_y, a.H);
  const int xa = max(x0, 0), xb = min(x0 + a.win_x, a.W);
  int lo = INT32_MAX, hi = INT32_MIN, bad = 0;
  // warps stride over rows, lanes over columns: coalesced, no index division
  const int nw = blockDim.x >> 5, lane = threadIdx.x & 31;
  for (int yy = ya + (int)(threadIdx.x >> 5); yy < yb; yy += nw) {
    const int64_t rowbase = ((int64_t)img * a.H + yy) * a.W;
#pragma unroll 4
    for (int xx = xa + lane; xx < xb; xx += 32) {
      const int64_t gi = rowbase + xx;
      if (a.img_def && !a.img_def[gi]) continue;
      const int v = range_load(a.img, a.img_dtype, gi);
      lo = min(lo, v);
      hi = max(hi, v);
      bad |= (v < a.img_min) | (v > a.img_max);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  __shared__ int slo[8], shi[8], sbad[8];
  const int wid = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    slo[wid] = lo;
    shi[wid] = hi;
    sbad[wid] = bad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
      lo = min(lo, slo[i]);
      hi = max(hi, shi[i]);
      bad |= sbad[i];
    }
    if (bad) atomicOr(a.err, 1);
    const bool any = lo <= hi;
    if (!any) lo = hi = 0;
    const int lr = (hi - lo) + a.lr_se;
    int li = a.L - 1;
    for (int i = 0; i < a.L; ++i)
      if (2 * a.ladder[i] >= lr + 1) {
        li = i;
        break;
      }
    const int anchor = a.enc_sign > 0 ? lo : hi;
    a.unit_param[(size_t)img * a.units + unit] = make_int4(anchor, a.ladder[li], li, any ? 1 : 0);
    const int slot = atomicAdd(&a.bucket_count[li], 1);
    a.bucket_list[(size_t)li * a.cap + slot] = make_int2(img, unit);
  }
}

}  // namespace fm
