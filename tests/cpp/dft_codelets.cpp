// Host-side check of the register DFT codelets of fm_dft.cuh (compiled by
// tests/test_dft_codelets.py with g++): every radix against an FP64 DFT.
#include <cuda_runtime.h>
#include <cstdio>
#include <cmath>
#include <complex>
#include "fm_dft.cuh"
using namespace fm;
template <int R, bool INV> double check() {
  double worst = 0;
  for (int trial = 0; trial < 50; ++trial) {
    float2 x[R]; std::complex<double> xd[R];
    for (int i = 0; i < R; ++i) { float re = std::sin(1.3*i + trial), im = std::cos(0.7*i*i + 2*trial); x[i] = make_float2(re, im); xd[i] = {re, im}; }
    dft<R, INV>(x);
    for (int k = 0; k < R; ++k) {
      std::complex<double> acc = 0;
      for (int n = 0; n < R; ++n) acc += xd[n] * std::polar(1.0, (INV ? 2 : -2) * M_PI * n * k / R);
      worst = std::max(worst, std::abs(acc - std::complex<double>(x[k].x, x[k].y)));
    }
  }
  return worst;
}
// dft32p_fwd (permuted output order, dft32p_freq) and dft32p_inv (that order in, natural out)
template <bool INV> double check32() {
  double worst = 0;
  for (int trial = 0; trial < 50; ++trial) {
    float2 x[32], y[32]; std::complex<double> xd[32];
    for (int i = 0; i < 32; ++i) { float re = std::sin(1.3*i + trial), im = std::cos(0.7*i*i + 2*trial); x[i] = make_float2(re, im); xd[i] = {re, im}; }
    for (int r = 0; r < 32; ++r) y[r] = x[dft32p_freq(r)];   // input of the inverse in permuted order
    dft32p_fwd<INV>(x);
    dft32p_inv<INV>(y);
    for (int k = 0; k < 32; ++k) {
      std::complex<double> acc = 0;
      for (int n = 0; n < 32; ++n) acc += xd[n] * std::polar(1.0, (INV ? 2 : -2) * M_PI * n * k / 32);
      // forward: register r holds frequency dft32p_freq(r)
      for (int r = 0; r < 32; ++r)
        if (dft32p_freq(r) == k) worst = std::max(worst, std::abs(acc - std::complex<double>(x[r].x, x[r].y)));
      worst = std::max(worst, std::abs(acc - std::complex<double>(y[k].x, y[k].y)));
    }
  }
  return worst;
}
// tw128: v * W_128^j (and conjugate) for every j
double check_tw128() {
  double worst = 0;
  for (int j = 0; j < 128; ++j) {
    const float2 v = make_float2(0.37f, -1.21f);
    const std::complex<double> vd(0.37, -1.21);
    const float2 f = tw128<false>(v, j), b = tw128<true>(v, j);
    const std::complex<double> wf = vd * std::polar(1.0, -2 * M_PI * j / 128), wb = vd * std::polar(1.0, 2 * M_PI * j / 128);
    worst = std::max(worst, std::abs(wf - std::complex<double>(f.x, f.y)));
    worst = std::max(worst, std::abs(wb - std::complex<double>(b.x, b.y)));
  }
  return worst;
}
int main() {
  printf("%g %g %g %g %g %g %g %g %g %g %g %g %g\n", check<2, false>(), check<3, false>(), check<4, false>(), check<5, false>(),
         check<8, false>(), check<16, false>(), check<3, true>(), check<5, true>(), check<8, true>(), check<16, true>(),
         check32<false>(), check32<true>(), check_tw128());
}
