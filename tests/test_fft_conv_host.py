"""Host logic of the count-level API (paper_2305_03018_b200.fft_conv): no GPU calls.

Mirrors test_fft_conv.py:21-36 (next_fast_size), :60-64 (offset ranges) and
:110-114 (precision budget) of the reference."""

import numpy as np
import pytest


def test_next_fast_size_smooth_and_flat():
    from paper_2305_03018_b200.fft_conv import next_fast_size
    for n in list(range(1, 200)) + [271, 351, 1021, 5000]:
        s = next_fast_size(n)
        assert s >= n
        for p in (2, 3, 5):
            while s % p == 0:
                s //= p
        assert s == 1
    assert next_fast_size(256 + 16 - 1) == next_fast_size(256 + 96 - 1)
    with pytest.raises(ValueError):
        next_fast_size(0)


def test_make_plan_ranges():
    from paper_2305_03018_b200.fft_conv import OffsetArray, make_plan
    plan = make_plan(OffsetArray(np.ones(9, np.int64), (-1,)), OffsetArray(np.ones(9, np.int64), (-3,)))
    assert (plan.out_lo, plan.out_hi) == ((-4,), (12,))
    assert plan.padded_shape == (32,)   # min(2^5, 45)
    with pytest.raises(ValueError):
        make_plan(OffsetArray(np.ones((2, 2))), OffsetArray(np.ones(3)))


def test_precision_budget():
    from paper_2305_03018_b200 import PrecisionBudgetError
    from paper_2305_03018_b200.fft_conv import check_precision_budget
    big = np.full(32, 1 << 32, dtype=np.int64)
    with pytest.raises(PrecisionBudgetError):
        check_precision_budget(big, big)
    check_precision_budget(np.ones(10), np.ones(10))


def test_umbra_detection():
    from paper_2305_03018_b200.fft_conv import _as_umbra
    bits = np.zeros((4, 6), np.int64)
    bits[0, 3] = bits[2, 5] = bits[3, 0] = 1
    v, d = _as_umbra(bits)
    assert v.tolist() == [3, 0, 5, 0] and d.tolist() == [True, False, True, True]
    bits[1, 1] = 2
    assert _as_umbra(bits) is None
    assert _as_umbra(np.ones((3, 3), np.int64)) is None
