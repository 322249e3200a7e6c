"""Build the sm_100a C-ABI library in-tree (no JIT cache, no site-packages).

    python -m paper_2305_03018_b200.build          # -> paper_2305_03018_b200/_build/libfftmorph_b200.so
"""
from __future__ import annotations

import fcntl
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT_DIR = PKG / "_build"
LIB = OUT_DIR / "libfftmorph_b200.so"
SOURCES = [CSRC / "fm_abi.cu"]
HEADERS = sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "fftmorph_b200.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile the library if a source is newer than it.  Safe under concurrent callers
    (ranks of one node, parallel test workers): an exclusive file lock serialises the
    build, and each process writes its own temporary file before the atomic rename."""
    if not force and not needs_build():
        return LIB
    OUT_DIR.mkdir(parents=True, exist_ok=True)
    with open(OUT_DIR / ".build.lock", "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if not force and not needs_build():   # another process built it meanwhile
                return LIB
            tmp = LIB.with_name(f"{LIB.name}.{os.getpid()}.tmp")
            cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-shared", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-v" if verbose else "-O3",
                   *os.environ.get("FM_NVCC_EXTRA", "").split(),
                   "-I", str(ROOT / "include"), "-I", str(CSRC),
                   *[str(s) for s in SOURCES], "-o", str(tmp), "-lcudart"]
            res = subprocess.run(cmd, capture_output=True, text=True)
            if res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
                try:
                    tmp.unlink()
                except FileNotFoundError:
                    pass
                raise RuntimeError(f"nvcc failed ({res.returncode})")
            if verbose:
                sys.stderr.write(res.stderr)
            os.replace(tmp, LIB)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)
    return LIB


def build_rank_safe(rank: int = 0, world: int = 1) -> Path:
    """Multi-process launch (torchrun): rank 0 builds, every rank waits at a barrier of the
    already-initialised process group, then checks the library exists."""
    import torch.distributed as dist
    multi = world > 1 and dist.is_available() and dist.is_initialized()
    if not multi or rank == 0:
        build()
    if multi:
        dist.barrier()
    if not LIB.exists():
        raise RuntimeError(f"{LIB} missing after the build")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
