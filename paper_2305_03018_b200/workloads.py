"""Seeded synthetic inputs for the five BASELINE.json configurations.

The recipes (RNG streams, call order, SE shapes) follow SURVEY.md §8(d);
the reference harness's seeding style is ``np.random.default_rng([seed, ...])``
(bench.py:86-95).  No public dataset is involved.  Digests are sha256 of the
raw bytes, first 16 hex characters (images as uint8, c1 as int32; SEs as
``int32 values || uint8 mask``).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

SEED = 230503018


@dataclass
class Workload:
    name: str
    images: np.ndarray          # [B, *shape] (uint8, or int32 for c1)
    se_values: np.ndarray       # int64 [*se_shape]
    se_defined: np.ndarray      # bool [*se_shape]
    se_lo: tuple
    tonal_max: int              # 2^bits - 1 of the images
    bits: int

    @property
    def shape(self):
        return self.images.shape[1:]

    @property
    def se_tonal_max(self) -> int:
        return max(int(self.se_values[self.se_defined].max()), 1)


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def se_digest(values: np.ndarray, defined: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(values.astype(np.int32)).tobytes()
                          + np.ascontiguousarray(defined.astype(np.uint8)).tobytes()).hexdigest()[:16]


def _centered_lo(shape):
    return tuple(-(s // 2) for s in shape)


def c1() -> Workload:
    r = np.random.default_rng([SEED, 1])
    img = r.integers(0, 16, 4096, dtype=np.int32)
    se = r.integers(0, 4, 31).astype(np.int64)
    return Workload("c1", img[None], se, np.ones(31, bool), _centered_lo(se.shape), 15, 4)


def c2() -> Workload:
    r = np.random.default_rng([SEED, 2])
    img = r.integers(0, 32, (512, 512)).astype(np.uint8)
    se = np.zeros((15, 15), np.int64)
    return Workload("c2", img[None], se, np.ones((15, 15), bool), _centered_lo(se.shape), 31, 5)


def c3_image() -> np.ndarray:
    r = np.random.default_rng([SEED, 3])
    n = 1024
    yy, xx = np.mgrid[0:n, 0:n].astype(np.float64)
    canvas = np.full((n, n), 128.0)
    for _ in range(32):
        cy = r.uniform(0, n)
        cx = r.uniform(0, n)
        s = r.uniform(10, 80)
        a = r.uniform(-128, 128)
        canvas += a * np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2.0 * s * s))
    canvas += r.uniform(-8, 8, (n, n))
    return np.clip(np.rint(canvas), 0, 255).astype(np.uint8)


def c3_se():
    d = np.arange(-10, 11)
    r2 = d[:, None] ** 2 + d[None, :] ** 2
    defined = r2 <= 100
    vals = np.where(defined, 7 - np.rint(7 * r2 / 100.0), 0).astype(np.int64)
    return vals, defined


def c3() -> Workload:
    v, m = c3_se()
    return Workload("c3", c3_image()[None], v, m, (-10, -10), 255, 8)


def c4() -> Workload:
    r = np.random.default_rng([SEED, 4])
    img = r.integers(0, 16, (2048, 2048)).astype(np.uint8)
    mask = r.random((101, 101)) < 0.5
    mask[50, 50] = True
    return Workload("c4", img[None], np.zeros((101, 101), np.int64), mask, (-50, -50), 15, 4)


def c5_image(i: int) -> np.ndarray:
    from scipy.ndimage import gaussian_filter
    r = np.random.default_rng([SEED, 5, i])
    g = gaussian_filter(r.standard_normal((2048, 2048)), 4.0)
    g = (g - g.min()) / (g.max() - g.min())
    return np.rint(g * 63).astype(np.uint8)


def c5_se():
    r = np.random.default_rng([SEED, 5, 1000])
    return r.integers(0, 16, (31, 31)).astype(np.int64)


def c5(n_images: int = 64, first: int = 0) -> Workload:
    imgs = np.stack([c5_image(i) for i in range(first, first + n_images)])
    se = c5_se()
    return Workload("c5", imgs, se, np.ones((31, 31), bool), (-15, -15), 63, 6)


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5}

# SURVEY.md §8(d) input digests (numpy 2.3.5 / scipy 1.18.1)
EXPECTED_DIGESTS = {
    "c1": ("83dd871019982184", "6edab3038d82f855"),
    "c2": ("cf726c2bc1663cc1", "c3b6956ae0116e80"),
    "c3": ("ad433f4809516293", "c50fe3308f26a2fc"),
    "c4": ("d4a5caf64bb732f4", "4a1227901fe0ab36"),
    "c5": ("d9249d25b39ad57f", "07eadbd2d76128f6"),
}
C5_IMG63_DIGEST = "cb22530af0ff7f51"
