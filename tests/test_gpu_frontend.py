"""GPU: the ``morph`` command line and the CSV bench harness on the B200 path
(test_cli.py semantics of the reference): PGM / SE files in,
device computation, PGM / CSV out."""

import csv

import numpy as np
import pytest

from conftest import EXAMPLE_DILATION
from oracle import cnaive

pytestmark = pytest.mark.gpu


@pytest.fixture
def example_files(tmp_path):
    img = tmp_path / "f.pgm"
    img.write_bytes(b"P2\n6 1\n7\n3 0 7 6 2 7\n")
    se = tmp_path / "b.se"
    se.write_text("origin: 0 1\n1 2 X 0\n")
    return img, se


@pytest.mark.parametrize("method", ["naive", "fft", "gpu"])
def test_dilate_worked_example(example_files, tmp_path, method, capsys):
    from paper_2305_03018_b200 import pgmio
    from paper_2305_03018_b200.cli import main
    img, se = example_files
    out = tmp_path / "out.pgm"
    assert main(["dilate", "--image", str(img), "--se", str(se), "--method", method, "--out", str(out)]) == 0
    assert pgmio.read_pgm(out).values[0].tolist() == EXAMPLE_DILATION
    text = capsys.readouterr().out
    assert "dilate" in text and ("deviation" in text) == (method != "naive")


def test_verbs_identity_gradient_open_close(example_files, tmp_path):
    from paper_2305_03018_b200 import GridFunction, pgmio
    from paper_2305_03018_b200.cli import main
    rng = np.random.default_rng(8)
    img = tmp_path / "f.pgm"
    pgmio.write_pgm(GridFunction(rng.integers(0, 256, (8, 8)), tonal_max=255), img)
    se = tmp_path / "id.se"
    se.write_text("origin: 0 0\n0\n")
    a, b = tmp_path / "a.pgm", tmp_path / "b.pgm"
    assert main(["erode", "--image", str(img), "--se", str(se), "--method", "gpu", "--out", str(a)]) == 0
    assert main(["dilate", "--image", str(a), "--se", str(se), "--method", "fft", "--out", str(b)]) == 0
    assert b.read_bytes() == img.read_bytes()
    c = tmp_path / "c.pgm"
    pgmio.write_pgm(GridFunction(np.full((6, 6), 9), tonal_max=15), c)
    flat = tmp_path / "flat.se"
    flat.write_text("origin: 1 1\n0 0 0\n0 0 0\n0 0 0\n")
    g = tmp_path / "g.pgm"
    assert main(["gradient", "--image", str(c), "--se", str(flat), "--method", "fft", "--out", str(g)]) == 0
    assert not pgmio.read_pgm(g).values.any()
    fimg, fse = example_files
    for op in ("open", "close"):
        o = tmp_path / f"{op}.pgm"
        assert main([op, "--image", str(fimg), "--se", str(fse), "--method", "gpu", "--out", str(o), "--clamp"]) == 0
        o2 = tmp_path / f"{op}_n.pgm"
        assert main([op, "--image", str(fimg), "--se", str(fse), "--method", "naive", "--out", str(o2), "--clamp"]) == 0
        assert o.read_bytes() == o2.read_bytes()


def test_larger_file_against_oracle(tmp_path):
    """A 300x260 8-bit P5 file and a gapped 9x7 SE file through `morph dilate --method gpu`."""
    from paper_2305_03018_b200 import GridFunction, pgmio
    from paper_2305_03018_b200.cli import main
    rng = np.random.default_rng(3)
    v = rng.integers(0, 256, (300, 260))
    img = tmp_path / "big.pgm"
    pgmio.write_pgm(GridFunction(v, tonal_max=255), img)
    se_v = rng.integers(0, 9, (9, 7))
    se_d = rng.random((9, 7)) < 0.7
    se_d[4, 3] = True
    se = tmp_path / "s.se"
    pgmio.write_se(GridFunction(se_v, se_d, lo=(-4, -3), tonal_max=8), se)
    out = tmp_path / "o.pgm"
    assert main(["dilate", "--image", str(img), "--se", str(se), "--method", "gpu", "--out", str(out),
                 "--clamp"]) == 0
    ref, _ = cnaive.naive(v, None, se_v, se_d, (-4, -3), erode=False, crop=True, fill=0)
    assert np.array_equal(pgmio.read_pgm(out).values, np.clip(ref, 0, 255))


def test_read_pgm_device_and_batch(tmp_path):
    import torch
    from paper_2305_03018_b200 import GridFunction, pgmio
    rng = np.random.default_rng(2)
    paths = []
    for i in range(3):
        p = tmp_path / f"{i}.pgm"
        pgmio.write_pgm(GridFunction(rng.integers(0, 64, (20, 30)), tonal_max=63), p)
        paths.append(p)
    t, m = pgmio.read_pgm_device(paths[0])
    assert t.is_cuda and t.dtype == torch.uint8 and m == 63
    assert np.array_equal(t.cpu().numpy(), pgmio.read_pgm(paths[0]).values)
    bt, m = pgmio.read_pgm_batch(paths)
    assert tuple(bt.shape) == (3, 20, 30) and bt.is_cuda


def test_bench_csv_gpu_rows(tmp_path):
    from paper_2305_03018_b200.cli import main
    out_csv = tmp_path / "bench.csv"
    assert main(["bench", "--mode", "filter-sweep", "--bits", "4", "--seed", "1", "--sizes", "24:3,24:5",
                 "--repeats", "2", "--csv", str(out_csv)]) == 0
    with open(out_csv) as fh:
        rows = list(csv.DictReader(fh))
    assert len(rows) == 2 * 2 * 2
    for r in rows:
        assert float(r["seconds"]) > 0 and len(r["input_digest"]) == 16 and "B200" in r["device"]
    fft_rows = [r for r in rows if r["method"] == "fft"]
    assert fft_rows and all(r["max_abs_diff_vs_naive"] == "0" for r in fft_rows)
