"""Host-side grid type and index-range helpers of the drop-in boundary.

``GridFunction`` is the boundary type of the reference's hot path
(``fftmorph.umbra.GridFunction``, umbra.py:23-133): an integer grid with a
per-axis logical origin ``lo`` (any sign), a ``defined`` mask (gaps), a
declared tonal ceiling ``tonal_max`` (default 255) and a ``signed`` flag.
This class keeps the same constructor, validation errors, properties and
equality rule, and additionally accepts any object with the same attributes
(duck typing), so grids built by the reference package can be passed in and
compared with ``==`` in either direction.

The range helpers restate tensor.py:76-101 (Minkowski sum and intersection
of inclusive per-axis ranges).
"""

from __future__ import annotations

import numpy as np

IndexRange = tuple[int, int]  # inclusive (lo, hi)


def full_output_range(ra, rb):
    """Minkowski sum of inclusive per-axis ranges (tensor.py:76-89)."""
    if len(ra) != len(rb):
        raise ValueError("rank mismatch")
    out = []
    for (la, ha), (lb, hb) in zip(ra, rb):
        if ha < la or hb < lb:
            raise ValueError("empty index range")
        out.append((la + lb, ha + hb))
    return tuple(out)


def intersect_ranges(ra, rb):
    """Per-axis intersection, or None if empty on some axis (tensor.py:92-101)."""
    out = []
    for (la, ha), (lb, hb) in zip(ra, rb):
        lo, hi = max(la, lb), min(ha, hb)
        if hi < lo:
            return None
        out.append((lo, hi))
    return tuple(out)


def _is_gridlike(obj) -> bool:
    return all(hasattr(obj, a) for a in ("values", "defined", "lo", "tonal_max"))


class GridFunction:
    """Integer-valued function on an N-d logical grid, with gaps.

    Same semantics as the reference (umbra.py:23-61): ``values`` is int64,
    C-contiguous and read-only; undefined entries are never read;
    ``tonal_max`` must bound the defined values; negative values need
    ``signed=True``.
    """

    __slots__ = ("values", "defined", "lo", "tonal_max", "signed", "_gap_free", "_vmin", "_vmax")

    def __init__(self, values, defined=None, lo=None, tonal_max: int = 255,
                 signed: bool = False):
        values = np.ascontiguousarray(np.asarray(values, dtype=np.int64))
        if values.size == 0:
            raise ValueError("empty grid")
        if defined is None:
            defined = np.ones(values.shape, dtype=bool)
        else:
            defined = np.ascontiguousarray(np.asarray(defined, dtype=bool))
            if defined.shape != values.shape:
                raise ValueError("defined mask shape mismatch")
        if not defined.any():
            raise ValueError("grid needs at least one defined pixel")
        if lo is None:
            lo = (0,) * values.ndim
        lo = tuple(int(x) for x in lo)
        if len(lo) != values.ndim:
            raise ValueError("lo rank mismatch")
        tonal_max = int(tonal_max)
        if tonal_max < 1:
            raise ValueError("tonal_max must be positive")
        # min / max of the defined values, computed once (the grids are immutable);
        # gap-free grids skip the boolean-indexed copy
        gap_free = bool(defined.all())
        dv = values if gap_free else values[defined]
        vmin, vmax = int(dv.min()), int(dv.max())
        if vmax > tonal_max:
            raise ValueError(f"value {vmax} exceeds tonal_max {tonal_max}")
        if not signed and vmin < 0:
            raise ValueError("negative value in an unsigned grid")
        values.flags.writeable = False
        defined.flags.writeable = False
        self.values = values
        self.defined = defined
        self.lo = lo
        self.tonal_max = tonal_max
        self.signed = bool(signed)
        self._gap_free, self._vmin, self._vmax = gap_free, vmin, vmax

    @classmethod
    def _from_device(cls, values, lo, tonal_max: int, signed: bool, vmin: int, vmax: int) -> "GridFunction":
        """Gap-free grid of freshly computed int64 values whose min / max are already
        known (reduced on the device): the same checks as __init__ without another
        pass over the host array."""
        tonal_max = int(tonal_max)
        if tonal_max < 1:
            raise ValueError("tonal_max must be positive")
        if vmax > tonal_max:
            raise ValueError(f"value {vmax} exceeds tonal_max {tonal_max}")
        if not signed and vmin < 0:
            raise ValueError("negative value in an unsigned grid")
        values = np.ascontiguousarray(values, dtype=np.int64)
        defined = np.ones(values.shape, dtype=bool)
        values.flags.writeable = False
        defined.flags.writeable = False
        g = cls.__new__(cls)
        g.values, g.defined, g.lo = values, defined, tuple(int(x) for x in lo)
        g.tonal_max, g.signed = tonal_max, bool(signed)
        g._gap_free, g._vmin, g._vmax = True, int(vmin), int(vmax)
        return g

    @classmethod
    def coerce(cls, g) -> "GridFunction":
        """Accept our own grid or any reference-shaped grid object."""
        if isinstance(g, cls):
            return g
        if _is_gridlike(g):
            return cls(np.asarray(g.values), np.asarray(g.defined), lo=tuple(g.lo),
                       tonal_max=int(g.tonal_max), signed=bool(getattr(g, "signed", False)))
        raise TypeError(f"expected a GridFunction, got {type(g).__name__}")

    @property
    def shape(self) -> tuple[int, ...]:
        return self.values.shape

    @property
    def ndim(self) -> int:
        return self.values.ndim

    @property
    def hi(self) -> tuple[int, ...]:
        return tuple(l + n - 1 for l, n in zip(self.lo, self.shape))

    @property
    def ranges(self) -> tuple[IndexRange, ...]:
        return tuple(zip(self.lo, self.hi))

    @property
    def gap_free(self) -> bool:
        return self._gap_free

    def max_defined(self) -> int:
        return self._vmax

    def min_defined(self) -> int:
        return self._vmin

    def at(self, x) -> int | None:
        """Value at logical index x, or None at a gap."""
        if isinstance(x, int):
            x = (x,)
        off = tuple(xj - lj for xj, lj in zip(x, self.lo))
        for o, n in zip(off, self.shape):
            if not 0 <= o < n:
                raise IndexError(f"index {x} outside {self.ranges}")
        if not self.defined[off]:
            return None
        return int(self.values[off])

    def to_list(self):
        """Nested lists with None at gaps (test convenience)."""
        out = np.where(self.defined, self.values, np.int64(0)).astype(object)
        out[~self.defined] = None
        return out.tolist()

    @classmethod
    def from_tokens(cls, tokens, lo=None, tonal_max: int | None = None):
        """Build from nested lists where None marks a gap."""
        arr = np.asarray(tokens, dtype=object)
        defined = np.vectorize(lambda t: t is not None)(arr).astype(bool)
        values = np.where(defined, arr, 0).astype(np.int64)
        if tonal_max is None:
            tonal_max = max(int(values[defined].max()), 1)
        return cls(values, defined, lo=lo, tonal_max=tonal_max)

    def __eq__(self, other):
        # Same rule as umbra.py:122-129; also answers for reference-shaped grids,
        # whose own __eq__ returns NotImplemented for a foreign type.
        if not isinstance(other, GridFunction):
            if not _is_gridlike(other):
                return NotImplemented
        ov = np.asarray(other.values)
        od = np.asarray(other.defined)
        return (tuple(self.lo) == tuple(other.lo)
                and self.shape == ov.shape
                and bool((self.defined == od).all())
                and bool((self.values[self.defined] == ov[od]).all()))

    __hash__ = None

    def __repr__(self):
        return (f"GridFunction(shape={self.shape}, lo={self.lo}, "
                f"tonal_max={self.tonal_max})")
