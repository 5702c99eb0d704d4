"""B200-native ILS edge-preserving smoothing (drop-in for ilsmooth's smoothing path).

Public API mirrors the reference package's hot path (pkg/src/ilsmooth/
__init__.py:44-61): SmoothParams, Charbonnier, Welsch, ColorMode, MultiImage,
smooth_plane, smooth_color, make_plan, solve_ls, SolverPlan, EnergyTrace and
the error types.  Every arithmetic step runs in libils_b200.so (hand-written
sm_100a CUDA) behind the C ABI in include/ils_b200.h; there is no CPU path.
"""

from ._runtime import get_default_precision, set_default_precision
from .errors import ImageFormatError, NumericalError
from .image import GRAY, RGB, YUV, ColorMode, MultiImage, as_plane, clip01, luminance, rgb_to_yuv, yuv_to_rgb
from .applications import (DetailBoost, TonemapParams, clipart_clean, detail_enhance, gaussian_blur,
                           texture_smooth, tonemap_multi, tonemap_single)
from .hqs import HqsParams, hqs_smooth_batch, hqs_smooth_plane
from .penalty import DEFAULT_EPS, Charbonnier, Welsch, aux_update, check_curvature, huber, soft_threshold
from .smoother import EnergyTrace, SmoothParams, energy, smooth_batch, smooth_color, smooth_frames_u8, smooth_plane
from .solver import SolverPlan, adjoint_accumulate, grad_x, grad_y, make_plan, solve_ls

__version__ = "0.1.0"

__all__ = [
    "DetailBoost", "TonemapParams", "clip01", "clipart_clean", "detail_enhance", "gaussian_blur", "luminance",
    "texture_smooth", "tonemap_multi", "tonemap_single",
    "DEFAULT_EPS", "GRAY", "RGB", "YUV", "Charbonnier", "ColorMode", "EnergyTrace", "HqsParams", "ImageFormatError",
    "MultiImage", "NumericalError", "SmoothParams", "SolverPlan", "Welsch", "as_plane", "check_curvature",
    "get_default_precision", "hqs_smooth_batch", "hqs_smooth_plane", "huber", "make_plan", "rgb_to_yuv", "set_default_precision", "smooth_batch", "smooth_color", "smooth_frames_u8",
    "smooth_plane", "soft_threshold", "solve_ls", "yuv_to_rgb",
    "adjoint_accumulate", "aux_update", "energy", "grad_x", "grad_y",
]
