"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``.

The golden vectors below restate the reference's own fixtures
(/root/reference/pkg/tests/conftest.py:10-61): the paper's worked 1-D
example (image [3 0 7 6 2 7], SE [1 2 X 0] with origin at its second entry).
"""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
TESTS = Path(__file__).resolve().parent
if str(TESTS) not in sys.path:
    sys.path.insert(0, str(TESTS))
GOLDEN = TESTS / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs on the GPU box)")


def pytest_collection_modifyitems(config, items):
    # on a CPU-only box, gpu tests are skipped only if the user did not ask for them
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


EXAMPLE_IMAGE = [3, 0, 7, 6, 2, 7]
EXAMPLE_SE = [1, 2, None, 0]
EXAMPLE_SE_LO = (-1,)
EXAMPLE_DILATION = [5, 8, 9, 8, 8, 9]

# Rows are tonal values 9..0 (umbra convention); columns are spatial indices.
RESULT_COUNT_MATRIX = [
    [0, 0, 1, 0, 0, 1],
    [0, 1, 0, 1, 1, 0],
    [0, 0, 1, 0, 1, 0],
    [0, 0, 0, 0, 0, 1],
    [1, 0, 0, 0, 0, 0],
    [0, 0, 0, 0, 1, 0],
    [0, 0, 1, 1, 0, 0],
    [0, 1, 0, 0, 0, 0],
    [1, 0, 0, 0, 0, 0],
    [0, 0, 0, 1, 0, 0],
]


@pytest.fixture
def example_image():
    from paper_2305_03018_b200 import GridFunction
    return GridFunction.from_tokens(EXAMPLE_IMAGE, tonal_max=7)


@pytest.fixture
def example_se():
    from paper_2305_03018_b200 import GridFunction
    return GridFunction.from_tokens(EXAMPLE_SE, lo=EXAMPLE_SE_LO, tonal_max=2)


def load_cases():
    meta = json.loads((GOLDEN / "cases.json").read_text())
    arr = np.load(GOLDEN / "cases.npz")
    return meta, arr


def flat_se(width, ndim=1):
    from paper_2305_03018_b200 import GridFunction
    r = width // 2
    return GridFunction(np.zeros((width,) * ndim, dtype=np.int64), lo=(-r,) * ndim, tonal_max=1)


def identity_se(ndim=1):
    from paper_2305_03018_b200 import GridFunction
    return GridFunction(np.zeros((1,) * ndim, dtype=np.int64), lo=(0,) * ndim, tonal_max=1)


def random_grid(rng, shape, top, gap_p=0.0, lo=None):
    """Same draw order as the reference's helper (test_morphology.py:23-28)."""
    from paper_2305_03018_b200 import GridFunction
    defined = rng.random(shape) >= gap_p
    if not defined.any():
        defined.flat[0] = True
    return GridFunction(rng.integers(0, top + 1, shape), defined, lo=lo, tonal_max=top)
