"""CPU model of two round-2 kernel ideas (numpy only; the GPU parity tests exercise the kernels).

* Nyquist-plane pairing (csrc/fm_bigtile.cuh): plane k = T/2 of a unit is real, (-1)^v, and so is the SE's;
  two units then share one complex transform, z = a + i a', because the kernel h is real.
* The cooperative tonal kernel's index split (csrc/fm_tonal_coop.cuh): k = N2 a + b, n = c + N1 d gives
  W_N^{kn} = W_N1^{ac} W_N^{bc} W_N2^{bd}, i.e. N2 transforms of length N1, a twiddle, N1 transforms of
  length N2 -- and every split in the table has G | N1 and G | N2.
"""
import re
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]


def test_nyquist_planes_of_two_units_share_one_complex_transform():
    rng = np.random.default_rng(3)
    P = 32
    for T in (2, 4, 6, 10):
        N = T // 2
        v1 = rng.integers(0, T, (P, P))
        v2 = rng.integers(0, T, (P, P))
        gap = rng.random((P, P)) < 0.1                       # undefined pixels encode as 0
        a1 = np.where(gap, 0.0, np.exp(-2j * np.pi * N * v1 / T))
        a2 = np.exp(-2j * np.pi * N * v2 / T)
        assert np.allclose(a1.imag, 0, atol=1e-12) and np.allclose(a2.imag, 0, atol=1e-12)
        b = rng.integers(0, 3, (5, 7))
        h = np.zeros((P, P), complex)
        h[:5, :7] = np.exp(-2j * np.pi * N * b / T)          # the SE's plane N: real as well
        assert np.allclose(h.imag, 0, atol=1e-12)
        H = np.fft.fft2(h)
        sep1 = np.fft.ifft2(np.fft.fft2(a1.real) * H)
        sep2 = np.fft.ifft2(np.fft.fft2(a2.real) * H)
        z = np.fft.ifft2(np.fft.fft2(a1.real + 1j * a2.real) * H)
        assert np.allclose(z.real, sep1.real, atol=1e-9) and np.allclose(z.imag, sep2.real, atol=1e-9)
        assert np.allclose(sep1.imag, 0, atol=1e-9)          # the shared plane splits exactly


def _coop_table():
    src = (ROOT / "paper_2305_03018_b200" / "csrc" / "fm_tonal_coop.cuh").read_text()
    return [tuple(int(x) for x in m) for m in re.findall(r"case (\d+): return \{(\d+), (\d+), (\d+)\};", src)]


def test_cooperative_tonal_split_table_and_index_identity():
    table = _coop_table()
    assert len(table) >= 20
    ns_src = (ROOT / "paper_2305_03018_b200" / "csrc" / "fm_tonal.cuh").read_text()
    block = re.search(r"#define FM_TONAL_NS(.*?)\nconstexpr", ns_src, re.S).group(1)
    lengths = {int(x) for x in re.findall(r"\d+", block)}
    rng = np.random.default_rng(5)
    for n, n1, n2, g in table:
        assert n1 * n2 == n and n1 % g == 0 and n2 % g == 0 and 2 <= g <= 5
        assert n in lengths and n1 in lengths and n2 in lengths   # compile-time register FFTs exist
        # two-pass inverse DFT as the kernel runs it == the length-N inverse DFT
        z = rng.standard_normal(n) + 1j * rng.standard_normal(n)
        ref = np.fft.ifft(z) * n
        s = np.empty(n, complex)
        for b in range(n2):                                   # pass 1, in place over k = n2*a + b
            y = np.fft.ifft(z[b::n2]) * n1                    # length n1 over a
            s[b::n2] = y * np.exp(2j * np.pi * b * np.arange(n1) / n)
        out = np.empty(n, complex)
        for c in range(n1):                                   # pass 2: contiguous block n2*c .. n2*c + n2
            out[c::n1] = np.fft.ifft(s[n2 * c:n2 * c + n2]) * n2
        assert np.allclose(out, ref, atol=1e-9), n
