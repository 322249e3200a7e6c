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
from .fft_conv import (Backend, ConvPlan, FftStats, OffsetArray, conv_full_direct, conv_full_fft,
                       conv_full_fft_with_stats, direct_full, make_plan, next_fast_size, set_fft_workers,
                       transform_forward, transform_inverse)
from .umbra import (CountVolume, UmbraVolume, build_umbra, project, project_with_validity,
                    required_lr)

__version__ = "0.1.0"

__all__ = [
    "Backend", "CountVolume", "UmbraVolume", "build_umbra", "direct_full", "make_plan", "project",
    "project_with_validity", "required_lr", "transform_forward", "transform_inverse",
    "ConvPlan", "FftStats", "GridFunction", "MorphMethod", "OffsetArray", "PrecisionBudgetError",
    "beucher_gradient", "closing", "conv_full_direct", "conv_full_fft", "conv_full_fft_with_stats",
    "next_fast_size", "set_fft_workers",
    "dilate", "dilate_fft", "dilate_naive", "erode", "erode_fft", "erode_naive",
    "full_output_range", "intersect_ranges", "negate", "opening", "reflect",
]
