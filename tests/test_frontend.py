"""CPU: the reference frontend's file formats and CLI verbs that need no GPU
(SURVEY §8(f) row 3): PGM P2/P5 and SE text readers/writers with the reference's
error behaviour (test_io.py semantics), hist / diff verbs, bench configuration
validation and seeding (test_cli.py semantics), and byte-level interop with the
reference's own pgmio when /root/reference is present (build container only)."""

import csv
import sys

import numpy as np
import pytest

from paper_2305_03018_b200 import GridFunction, benchcsv, pgmio
from paper_2305_03018_b200.cli import build_parser, main


def test_read_pgm_ascii_binary_comments(tmp_path):
    p = tmp_path / "a.pgm"
    p.write_bytes(b"P2\n2 1\n255\n3 0\n")
    g = pgmio.read_pgm(p)
    assert g.shape == (1, 2) and g.tonal_max == 255 and g.values.tolist() == [[3, 0]]
    p.write_bytes(b"P2 # graymap\n# dims\n3 2\n15\n0 1 2\n3 4 5\n")
    g = pgmio.read_pgm(p)
    assert g.values.tolist() == [[0, 1, 2], [3, 4, 5]] and g.tonal_max == 15
    rng = np.random.default_rng(0)
    for binary in (True, False):
        g = GridFunction(rng.integers(0, 16, (5, 7)), tonal_max=15)
        pgmio.write_pgm(g, p, binary=binary)
        assert pgmio.read_pgm(p) == g


@pytest.mark.parametrize("blob", [b"P6\n1 1\n255\n\x00", b"P2\n0 1\n255\n", b"P2\n1 1\n300\n5\n",
                                  b"P2\n2 1\n255\n3\n", b"P2\n1 1\n15\n99\n", b"P5\n2 2\n255\n\x00\x01",
                                  b"P2\n1 1\nhello\n0\n", b"P5\n2 1\n3\n\x00\x09"])
def test_read_pgm_malformed(tmp_path, blob):
    p = tmp_path / "bad.pgm"
    p.write_bytes(blob)
    with pytest.raises(pgmio.ParseError):
        pgmio.read_pgm(p)


def test_parse_error_offset(tmp_path):
    p = tmp_path / "bad.pgm"
    p.write_bytes(b"P2\n1 1\nhello\n0\n")
    with pytest.raises(pgmio.ParseError) as e:
        pgmio.read_pgm(p)
    assert e.value.offset == 7 and isinstance(e.value, ValueError)


def test_write_pgm_rejects_and_clamp(tmp_path):
    p = tmp_path / "x.pgm"
    with pytest.raises(ValueError):
        pgmio.write_pgm(GridFunction(np.array([[1, 2]]), np.array([[True, False]]), tonal_max=2), p)
    with pytest.raises(ValueError):
        pgmio.write_pgm(GridFunction(np.array([[-1, 2]]), tonal_max=2, signed=True), p)
    g = pgmio.clamp(GridFunction(np.array([[-3, 5, 300]]), tonal_max=300, signed=True), 0, 255)
    assert g.values.tolist() == [[0, 5, 255]]


def test_read_se_formats(tmp_path):
    p = tmp_path / "b.se"
    p.write_text("# worked example\norigin: 0 1\n1 2 X 0\n")
    b = pgmio.read_se(p)
    assert b.lo == (0, -1) and b.defined.tolist() == [[True, True, False, True]]
    b2 = GridFunction.from_tokens([[3, None, 1], [0, 2, None]], lo=(-1, 0), tonal_max=3)
    pgmio.write_se(b2, p)
    assert pgmio.read_se(p) == b2


@pytest.mark.parametrize("text", ["1 2 3\n", "origin: 0\n1\n", "origin: 0 0\n", "origin: 0 0\n1 2\n3\n",
                                  "origin: 5 0\n1 2\n", "origin: 0 0\n1 -2\n", "origin: 0 0\nX X\n",
                                  "origin: 0 0\n1 q\n"])
def test_read_se_malformed(tmp_path, text):
    p = tmp_path / "bad.se"
    p.write_text(text)
    with pytest.raises(pgmio.ParseError):
        pgmio.read_se(p)


def test_requantize_histogram(tmp_path):
    q = pgmio.requantize(GridFunction(np.array([[0, 128, 255]]), tonal_max=255), 4)
    assert q.tonal_max == 15 and q.values.tolist() == [[0, 7, 15]]
    with pytest.raises(ValueError):
        pgmio.requantize(GridFunction(np.array([0]), tonal_max=1), 9)
    assert pgmio.histogram(GridFunction(np.array([[0, 1, 1], [3, 1, 0]]), tonal_max=3)).tolist() == [2, 3, 0, 1]
    c = tmp_path / "h.csv"
    pgmio.write_histogram_csv(np.array([2, 0, 1]), c)
    assert c.read_text() == "value,count\n0,2\n1,0\n2,1\n"


def test_cli_hist_diff_and_errors(tmp_path, capsys):
    img = tmp_path / "f.pgm"
    img.write_bytes(b"P2\n3 1\n3\n0 1 1\n")
    out_csv = tmp_path / "h.csv"
    assert main(["hist", "--image", str(img), "--csv", str(out_csv)]) == 0
    assert out_csv.read_text() == "value,count\n0,1\n1,2\n2,0\n3,0\n"
    a, b = tmp_path / "a.pgm", tmp_path / "b.pgm"
    pgmio.write_pgm(GridFunction(np.full((3, 4), 3), tonal_max=255), a)
    pgmio.write_pgm(GridFunction(np.full((3, 4), 5), tonal_max=255), b)
    neg = tmp_path / "d.pgm"
    assert main(["diff", str(a), str(b), "--out", str(neg)]) == 0
    out = capsys.readouterr().out
    assert "max abs difference:  2" in out and "mean abs difference: 2.000000" in out
    assert (pgmio.read_pgm(neg).values == 253).all()
    pgmio.write_pgm(GridFunction(np.full((2, 2), 1), tonal_max=255), b)
    assert main(["diff", str(a), str(b)]) == 2
    assert "shape mismatch" in capsys.readouterr().err
    # unreadable input: reference exit code 1 and an "error:" line, before any device work
    rc = main(["dilate", "--image", str(tmp_path / "nope.pgm"), "--se", str(tmp_path / "nope.se"),
               "--method", "gpu", "--out", str(tmp_path / "o.pgm")])
    assert rc == 1 and "error:" in capsys.readouterr().err


def test_cli_parser_and_bench_config():
    args = build_parser().parse_args(["erode", "--image", "a", "--se", "b", "--method", "gpu", "--out", "c",
                                      "--tonal-max", "63"])
    assert args.method == "gpu" and args.tonal_max == 63
    with pytest.raises(ValueError):
        benchcsv.BenchConfig(mode="zigzag", bits=[4], seed=0, sizes=[(16, 3)])
    with pytest.raises(ValueError):
        benchcsv.BenchConfig(mode="filter-sweep", bits=[12], seed=0, sizes=[(16, 3)])
    with pytest.raises(ValueError):
        benchcsv.BenchConfig(mode="filter-sweep", bits=[4], seed=0, sizes=[(8, 16)])
    with pytest.raises(ValueError):
        benchcsv.BenchConfig(mode="image-sweep", bits=[8], seed=0, sizes=[(4096, 5)], memory_ceiling_bytes=2**20)
    d1 = [benchcsv.case_inputs(9, 4, 16, 3, r)[2] for r in range(3)]
    assert d1 == [benchcsv.case_inputs(9, 4, 16, 3, r)[2] for r in range(3)] and len(set(d1)) == 3


def test_csv_schema(tmp_path):
    rows = [benchcsv.BenchRow("filter-sweep", 4, 24, 3, "fft", 0, 0.01, 0, "0123456789abcdef", 1, "NVIDIA B200")]
    p = tmp_path / "b.csv"
    benchcsv.write_csv(rows, p)
    with open(p) as fh:
        r = list(csv.DictReader(fh))
    assert list(r[0].keys()) == list(benchcsv.CSV_COLUMNS) + ["device"]
    assert r[0]["device"] == "NVIDIA B200" and r[0]["max_abs_diff_vs_naive"] == "0"


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not __import__("os").path.isdir(REF), reason="reference not present (GPU box)")
def test_interop_with_reference_pgmio(tmp_path):
    """Files written by either package read back identically in the other."""
    sys.path.insert(0, REF)
    try:
        from fftmorph import pgmio as rp
        from fftmorph.umbra import GridFunction as RG
    finally:
        sys.path.remove(REF)
    rng = np.random.default_rng(5)
    vals = rng.integers(0, 200, (9, 13))
    for binary in (True, False):
        p = tmp_path / "x.pgm"
        rp.write_pgm(RG(vals, tonal_max=255), p, binary=binary)
        ours = p.read_bytes()
        assert pgmio.read_pgm(p) == rp.read_pgm(p)
        pgmio.write_pgm(GridFunction(vals, tonal_max=255), p, binary=binary)
        assert p.read_bytes() == ours
    b = RG.from_tokens([[3, None, 1], [0, 2, None]], lo=(-1, 0), tonal_max=3)
    s = tmp_path / "b.se"
    rp.write_se(b, s)
    txt = s.read_text()
    assert pgmio.read_se(s) == rp.read_se(s)
    pgmio.write_se(pgmio.read_se(s), s)
    assert s.read_text() == txt
