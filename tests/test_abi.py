"""CPU: the C-ABI library builds, loads and exports every symbol of
include/fftmorph_b200.h; the ctypes structs match the C layout.  No compute
calls (no GPU here)."""

import ctypes
import re
import subprocess
import textwrap

import pytest

from conftest import ROOT
from paper_2305_03018_b200 import _lib
from paper_2305_03018_b200 import build as B

HEADER = ROOT / "include" / "fftmorph_b200.h"


def _declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fm_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    B.build()
    return _lib.load()


def test_header_and_binding_agree():
    assert sorted(_lib.EXPORTED) == _declared_functions()


def test_library_exports_every_symbol(lib):
    for name in _declared_functions():
        assert hasattr(lib, name), name
    assert lib.fm_abi_version() == _lib.ABI_VERSION == 4


def test_dynamic_symbol_table():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("nm unavailable")
    syms = set(re.findall(r"\bT (fm_\w+)", out.stdout))
    assert set(_declared_functions()) <= syms


def test_sm100a_code_in_library():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_struct_layouts_match_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text(textwrap.dedent("""
        #include <stdio.h>
        #include <stddef.h>
        #include "fftmorph_b200.h"
        int main(void) {
          printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\\n", sizeof(fm_plan_desc), sizeof(fm_plan_info),
                 sizeof(fm_stats), offsetof(fm_plan_desc, img_min), offsetof(fm_plan_desc, scratch_bytes),
                 offsetof(fm_plan_info, se_count), offsetof(fm_plan_desc, flags), offsetof(fm_plan_info, count_len),
                 sizeof(fm_timing), offsetof(fm_timing, range_launches), offsetof(fm_plan_desc, count_budget),
                 offsetof(fm_plan_desc, win_lo), offsetof(fm_plan_desc, win_shape));
          return 0;
        }
    """))
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_lib.PlanDesc), ctypes.sizeof(_lib.PlanInfo), ctypes.sizeof(_lib.Stats),
            _lib.PlanDesc.img_min.offset, _lib.PlanDesc.scratch_bytes.offset, _lib.PlanInfo.se_count.offset,
            _lib.PlanDesc.flags.offset, _lib.PlanInfo.count_len.offset, ctypes.sizeof(_lib.Timing),
            _lib.Timing.range_launches.offset, _lib.PlanDesc.count_budget.offset,
            _lib.PlanDesc.win_lo.offset, _lib.PlanDesc.win_shape.offset]
    assert got == want


def test_error_string_without_gpu(lib):
    # validation happens before any CUDA call: a null descriptor is FM_EINVAL
    h = ctypes.c_void_p()
    rc = lib.fm_plan_create(ctypes.byref(h), None, None, None)
    assert rc == _lib.FM_EINVAL
    assert b"null" in lib.fm_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_no_cpu_fallback(tmp_path):
    """The operators never compute on the CPU: without a usable library / device they raise."""
    import os
    import subprocess
    import sys
    code = ("import paper_2305_03018_b200 as fm\n"
            "f = fm.GridFunction.from_tokens([3, 0, 7, 6, 2, 7], tonal_max=7)\n"
            "b = fm.GridFunction.from_tokens([1, 2, None, 0], lo=(-1,), tonal_max=2)\n"
            "try:\n"
            "    fm.dilate_fft(f, b)\n"
            "    print('computed')\n"
            "except RuntimeError as e:\n"
            "    print('raised')\n")
    env = dict(os.environ, FM_LIB=str(tmp_path / "missing.so"), CUDA_VISIBLE_DEVICES="")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.stdout.strip().splitlines()[-1] == "raised", out.stdout + out.stderr
