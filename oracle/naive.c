/*
 * ORACLE — test infrastructure only (never linked into the product library).
 *
 * Plain-C restatement of the reference's exact direct operators, used to check
 * the GPU FFT path at sizes where the numpy restatement (oracle/port.py) is too
 * slow (c3..c5 of BASELINE.json):
 *   dilate_naive  morphology.py:65-85  — acc = max over defined SE entries y of
 *                 f(x-y)+b(y); no pair -> 0 and invalid; crop pastes the
 *                 Minkowski-range result into f's domain (_paste, morphology.py:51-62)
 *   erode_naive   morphology.py:88-113 — acc = min of f(x+y)-b(y); no pair -> neutral
 * Row-parallel over pthreads; the inner loop is a contiguous max/min over one
 * image row, so it auto-vectorises.  Arithmetic is int32 with +-2^30
 * sentinels (the reference uses int64 and +-2^40, morphology.py:27): valid for
 * |f| + |b| < 2^29, which every test input respects.
 *
 * Build: make -C oracle   ->   oracle/_build/libmorph_oracle.so
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NEG_SENT (-(1 << 30))
#define POS_SENT (1 << 30)

typedef struct {
  int64_t H, W, OH, OW, CY, CX;
  const int32_t* img;  /* prepared: undefined -> sentinel */
  int nent;
  const int32_t* ent;  /* (jy, jx, v) triples */
  int erode;
  int32_t fill;
  int32_t* out;
  uint8_t* valid;
  int64_t row0, row1;
} job_t;

static void* run_rows(void* arg) {
  job_t* j = (job_t*)arg;
  int32_t* acc = (int32_t*)malloc(sizeof(int32_t) * (size_t)j->OW);
  for (int64_t oy = j->row0; oy < j->row1; ++oy) {
    const int32_t init = j->erode ? POS_SENT : NEG_SENT;
    for (int64_t x = 0; x < j->OW; ++x) acc[x] = init;
    for (int e = 0; e < j->nent; ++e) {
      const int64_t jy = j->ent[3 * e], jx = j->ent[3 * e + 1];
      const int32_t v = j->ent[3 * e + 2];
      /* dilation: i = o + C - jj ; erosion: i = o + C + jj */
      const int64_t iy = j->erode ? oy + j->CY + jy : oy + j->CY - jy;
      if (iy < 0 || iy >= j->H) continue;
      const int64_t dx = j->erode ? j->CX + jx : j->CX - jx; /* ix = ox + dx */
      int64_t x0 = -dx > 0 ? -dx : 0;
      int64_t x1 = j->W - dx < j->OW ? j->W - dx : j->OW;
      if (x1 <= x0) continue;
      const int32_t* src = j->img + iy * j->W + dx;
      if (j->erode) {
        for (int64_t x = x0; x < x1; ++x) {
          const int32_t c = src[x] - v;
          acc[x] = c < acc[x] ? c : acc[x];
        }
      } else {
        for (int64_t x = x0; x < x1; ++x) {
          const int32_t c = src[x] + v;
          acc[x] = c > acc[x] ? c : acc[x];
        }
      }
    }
    for (int64_t x = 0; x < j->OW; ++x) {
      const int ok = j->erode ? acc[x] < (POS_SENT >> 1) : acc[x] > (NEG_SENT >> 1);
      j->out[oy * j->OW + x] = ok ? acc[x] : j->fill;
      if (j->valid) j->valid[oy * j->OW + x] = (uint8_t)ok;
    }
  }
  free(acc);
  return NULL;
}

/* ndim 1 or 2; shapes row-major; se_lo = logical origin of the SE; image lo = 0.
 * Values must satisfy |v| < 2^28.  Returns 0 on success. */
int oracle_naive(int ndim, const int64_t* shape, const int32_t* img, const uint8_t* img_def,
                 const int64_t* se_shape, const int32_t* se, const uint8_t* se_def,
                 const int64_t* se_lo, int erode, int crop, int32_t fill, int32_t* out,
                 uint8_t* valid, int nthreads) {
  const int two = ndim == 2;
  const int64_t H = two ? shape[0] : 1, W = two ? shape[1] : shape[0];
  const int64_t my = two ? se_shape[0] : 1, mx = two ? se_shape[1] : se_shape[0];
  const int64_t lo_y = two ? se_lo[0] : 0, lo_x = two ? se_lo[1] : se_lo[0];
  int64_t off_y = 0, off_x = 0, OH = H, OW = W;
  if (!crop) {
    off_y = two ? (erode ? -(lo_y + my - 1) : lo_y) : 0;
    off_x = erode ? -(lo_x + mx - 1) : lo_x;
    OH = two ? H + my - 1 : 1;
    OW = W + mx - 1;
  }
  int32_t* prep = (int32_t*)malloc(sizeof(int32_t) * (size_t)(H * W));
  if (!prep) return 1;
  const int32_t sent = erode ? POS_SENT : NEG_SENT;
  for (int64_t i = 0; i < H * W; ++i) prep[i] = (img_def && !img_def[i]) ? sent : img[i];
  int32_t* ent = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)(my * mx));
  int n = 0;
  for (int64_t jy = 0; jy < my; ++jy)
    for (int64_t jx = 0; jx < mx; ++jx) {
      const int64_t i = jy * mx + jx;
      if (se_def && !se_def[i]) continue;
      ent[3 * n] = (int32_t)jy;
      ent[3 * n + 1] = (int32_t)jx;
      ent[3 * n + 2] = se[i];
      ++n;
    }
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  pthread_t th[256];
  job_t jobs[256];
  const int64_t CY = erode ? off_y + lo_y : off_y - lo_y;
  const int64_t CX = erode ? off_x + lo_x : off_x - lo_x;
  for (int t = 0; t < nthreads; ++t) {
    job_t* j = &jobs[t];
    j->H = H; j->W = W; j->OH = OH; j->OW = OW; j->CY = two ? CY : 0; j->CX = CX;
    j->img = prep; j->nent = n; j->ent = ent; j->erode = erode; j->fill = fill;
    j->out = out; j->valid = valid;
    j->row0 = OH * t / nthreads;
    j->row1 = OH * (t + 1) / nthreads;
    pthread_create(&th[t], NULL, run_rows, j);
  }
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(prep);
  free(ent);
  return 0;
}
