"""CPU: host-side logic of the drop-in boundary (no kernel calls).

GridFunction semantics (umbra.py:23-133), range helpers (tensor.py:76-101),
MorphMethod parsing, reflect / negate (morphology.py:147-163), validation
errors raised before any device work, and the sharding geometry.
"""

import numpy as np
import pytest

from conftest import flat_se
from paper_2305_03018_b200 import (GridFunction, MorphMethod, dilate_fft, erode_fft,
                                   full_output_range, intersect_ranges, negate, reflect)
from paper_2305_03018_b200 import sharding


class TestGrid:
    def test_validation(self):
        with pytest.raises(ValueError):
            GridFunction(np.zeros(0))
        with pytest.raises(ValueError):
            GridFunction(np.array([1, 2]), defined=np.array([False, False]))
        with pytest.raises(ValueError):
            GridFunction(np.array([1, 300]))
        with pytest.raises(ValueError):
            GridFunction(np.array([-1, 2]))
        with pytest.raises(ValueError):
            GridFunction(np.array([1, 2]), lo=(0, 0))
        with pytest.raises(ValueError):
            GridFunction(np.array([1, 2]), tonal_max=0)
        g = GridFunction(np.array([-1, 2]), signed=True)
        assert g.min_defined() == -1

    def test_properties_and_tokens(self):
        g = GridFunction.from_tokens([1, 2, None, 0], lo=(-1,), tonal_max=2)
        assert g.ranges == ((-1, 2),) and g.hi == (2,)
        assert g.to_list() == [1, 2, None, 0]
        assert g.at(0) == 2 and g.at(1) is None
        assert not g.gap_free and g.max_defined() == 2
        with pytest.raises(IndexError):
            g.at(3)
        assert not g.values.flags.writeable

    def test_equality_rule(self):
        a = GridFunction(np.array([1, 5]), defined=np.array([True, False]), tonal_max=9)
        b = GridFunction(np.array([1, 7]), defined=np.array([True, False]), tonal_max=3, signed=True)
        assert a == b                      # gap values, tonal_max and signed are ignored
        c = GridFunction(np.array([1, 7]), defined=np.array([True, False]), lo=(1,), tonal_max=7)
        assert a != c

    def test_duck_typed_foreign_grid(self):
        class Foreign:
            values = np.array([3, 4])
            defined = np.array([True, True])
            lo = (0,)
            tonal_max = 4
            signed = False
        g = GridFunction.coerce(Foreign())
        assert g == Foreign() and Foreign() == g or g == Foreign()


def test_ranges():
    assert full_output_range(((-1, 7),), ((-3, 5),)) == ((-4, 12),)
    assert intersect_ranges(((0, 5),), ((6, 9),)) is None
    assert intersect_ranges(((0, 5), (1, 2)), ((3, 9), (0, 9))) == ((3, 5), (1, 2))


def test_method_parse():
    assert MorphMethod.parse("fft") is MorphMethod.FFT_UMBRA
    assert MorphMethod.parse("NAIVE") is MorphMethod.NAIVE
    with pytest.raises(ValueError):
        MorphMethod.parse("quick")


def test_reflect_negate(example_image, example_se):
    r = reflect(example_se)
    assert r.lo == (-2,) and r.to_list() == [0, None, 2, 1]
    assert reflect(reflect(example_se)) == example_se
    assert reflect(flat_se(5)) == flat_se(5)
    assert negate(example_image, 7).to_list() == [4, 7, 0, 1, 5, 0]
    assert negate(negate(example_image, 7), 7) == example_image
    with pytest.raises(ValueError):
        negate(example_image, 5)


def test_validation_errors_before_device(example_image):
    neg = GridFunction(np.array([-1, 2]), tonal_max=3, signed=True)
    with pytest.raises(ValueError):
        dilate_fft(neg, flat_se(3))
    with pytest.raises(ValueError):
        erode_fft(example_image, flat_se(3), l=5)
    bneg = GridFunction(np.array([-1, 0]), tonal_max=1, signed=True)
    with pytest.raises(ValueError):
        dilate_fft(example_image, bneg)
    with pytest.raises(ValueError):
        dilate_fft(example_image, flat_se(3, ndim=2))


def test_shard_range_partition():
    for n in (0, 1, 7, 64, 65):
        for w in (1, 2, 3, 8):
            parts = [sharding.shard_range(n, r, w) for r in range(w)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [e - s for s, e in parts]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("mode", ["dilate", "erode"])
def test_strip_windows_cover_dependency_cone(mode):
    rng = np.random.default_rng(4)
    for _ in range(50):
        H = int(rng.integers(1, 60))
        w = int(rng.integers(1, 6))
        my = int(rng.integers(1, 12))
        lo = int(rng.integers(-14, 4))
        plan = sharding.strips(H, w, lo, my, mode)
        for s in plan:
            for y in range(s.out0, s.out1):
                for j in range(my):
                    yy = y - (lo + j) if mode == "dilate" else y + (lo + j)
                    if 0 <= yy < H:
                        assert s.in0 <= yy < s.in1
            assert s.in0 <= s.out0 and s.out1 <= s.in1
        for src, dst, r0, r1 in sharding.halo_transfers(plan):
            assert plan[src].out0 <= r0 < r1 <= plan[src].out1


def test_umulhi_division_magic():
    """fm_tonal.cuh divides by QX / tiles_x with ceil(2^32/d) and a high multiply:
    exact for every divisor 2..4096 and every quotient input below 2^16."""
    p = np.arange(1 << 16, dtype=np.uint64)
    for d in list(range(2, 300)) + [511, 1000, 4095, 4096]:
        magic = np.uint64(((1 << 32) + d - 1) // d)
        q = (p * magic) >> np.uint64(32)
        assert np.array_equal(q, p // np.uint64(d)), d


def test_reference_file_formats_interoperate(tmp_path):
    """SURVEY 8(f) row 3 (data formats either side of the path): the reference's own
    PGM / SE readers and writers (pgmio.py:62-183) exchange grids with the drop-in
    without conversion — reference grids are accepted as inputs (duck typing) and the
    drop-in's grids are written by the reference writers.  Skipped where the
    reference is absent (the GPU box)."""
    import sys
    ref_src = "/root/reference/pkg/src"
    import os
    if not os.path.isdir(ref_src):
        pytest.skip("reference package not present")
    sys.path.insert(0, ref_src)
    try:
        from fftmorph import pgmio
        from fftmorph.umbra import GridFunction as RefGrid
    finally:
        sys.path.remove(ref_src)
    from paper_2305_03018_b200 import GridFunction
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (7, 9))
    ours = GridFunction(img, tonal_max=255)
    pgmio.write_pgm(ours, tmp_path / "a.pgm")
    back = pgmio.read_pgm(tmp_path / "a.pgm")
    assert isinstance(back, RefGrid)
    assert ours == back and back == ours
    se_vals = rng.integers(0, 5, (3, 5))
    se_def = rng.random((3, 5)) > 0.3
    se_def[1, 2] = True
    se = GridFunction(se_vals, se_def, lo=(-1, -2), tonal_max=4)
    pgmio.write_se(se, tmp_path / "b.se")
    se_back = pgmio.read_se(tmp_path / "b.se")
    assert se == se_back and se_back == se


def test_grid_cached_extrema_and_trusted_constructor():
    """Grids cache min / max / gap-free at construction (gap-free grids skip the
    boolean-indexed copy); the device-result constructor keeps __init__'s checks."""
    from paper_2305_03018_b200 import GridFunction
    v = np.array([[3, 9], [0, 4]])
    g = GridFunction(v, tonal_max=9)
    assert (g.min_defined(), g.max_defined(), g.gap_free) == (0, 9, True)
    d = np.array([[True, False], [True, True]])
    h = GridFunction(v, d, tonal_max=9)
    assert (h.min_defined(), h.max_defined(), h.gap_free) == (0, 4, False)
    t = GridFunction._from_device(v, (0, 0), 9, False, 0, 9)
    assert t == g and t.gap_free and not t.values.flags.writeable
    with pytest.raises(ValueError):
        GridFunction._from_device(v, (0, 0), 8, False, 0, 9)      # exceeds tonal_max
    with pytest.raises(ValueError):
        GridFunction._from_device(v - 5, (0, 0), 9, False, -5, 4)  # negative, unsigned
    s = GridFunction._from_device(v - 5, (1, -2), 9, True, -5, 4)
    assert s.lo == (1, -2) and s.signed and s.min_defined() == -5


def test_committed_bench_line_contract():
    """The newest committed bench line carries every key the driver and the judge
    read (metric/value/unit/..., roofline, e2e, cpu_baseline, clocks, gpu_launches)."""
    import json
    from pathlib import Path
    prof = Path(__file__).resolve().parents[1] / "profiles"
    lines = sorted(prof.glob("r*_bench_line.json"), key=lambda f: (f.stem[:2], len(f.stem), f.stem))
    assert lines, "no committed bench line"
    d = json.loads(lines[-1].read_text())
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
                "clocks", "cpu_baseline"):
        assert key in d, key
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-6
    for key in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert key in d["e2e"], key
    for key in ("value", "unit", "cores", "kind", "sample"):
        assert key in d["cpu_baseline"], key
    assert d["gpu_launches"] > 0 and d["steps"] >= 1 and d["warmup"] >= 3
    assert not set(d["clocks"].get("reasons", [])) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if lines[-1].name.startswith("r2"):
        # round 2: the timed output is parity-checked image by image, erosion measured too
        assert d["parity"]["ok"] and d["parity"]["images"] == 64
        assert d["erode"]["parity"]["ok"] and r["bound"] == "fp32"
