"""B200-native exact grey-scale dilation / erosion (arXiv 2305.03018).

Drop-in for the hot path of the reference package ``fftmorph``: the operator
names, signatures and semantics of ``fftmorph.morphology`` on top of a
hand-written sm_100a CUDA library (include/fftmorph_b200.h).
"""

from .grid import GridFunction, full_output_range, intersect_ranges
from .morphology import (MorphMethod, beucher_gradient, closing, dilate, dilate_fft,
                         dilate_naive, erode, erode_fft, erode_naive, negate, opening,
                         reflect)
from ._lib import PrecisionBudgetError

__version__ = "0.1.0"

__all__ = [
    "GridFunction", "MorphMethod", "PrecisionBudgetError", "beucher_gradient", "closing",
    "dilate", "dilate_fft", "dilate_naive", "erode", "erode_fft", "erode_naive",
    "full_output_range", "intersect_ranges", "negate", "opening", "reflect",
]
