"""CPU: the register DFT codelets (fm_dft.cuh, host-compilable, radix 2..16 and the
permuted-order 32-point pair) against an FP64 DFT."""

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_codelets_match_fp64_dft(tmp_path):
    if shutil.which("g++") is None:
        pytest.skip("g++ unavailable")
    exe = tmp_path / "dft"
    cuda_inc = "/usr/local/cuda/include"
    subprocess.run(["g++", "-std=c++17", "-O1", f"-I{cuda_inc}", f"-I{ROOT / 'paper_2305_03018_b200' / 'csrc'}",
                    str(ROOT / "tests" / "cpp" / "dft_codelets.cpp"), "-o", str(exe)], check=True)
    errs = [float(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert len(errs) == 13
    assert max(errs[:10]) < 2e-6, errs
    assert max(errs[10:12]) < 6e-6, errs   # 32 points: outputs up to ~32 in magnitude
    assert errs[12] < 1e-6, errs           # W_128^j twiddles
