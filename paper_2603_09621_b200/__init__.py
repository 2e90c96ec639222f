"""paper_2603_09621_b200: B200-native brick rasterizer for MRI-tailored 3D Gaussians.

Drop-in for the hot path of the reference package ``gsvol``
(arxiv/paper_2603_09621): the render / loss / training-step API of
gsvol/__init__.py:11-44 (rasterizer, field, options, loss, Adam, fit), with
every computation in hand-written sm_100a CUDA behind the C ABI of
include/gsv.h (libgsv_b200.so).  There is no CPU fallback.
"""

__version__ = "0.1.0"

from .errors import (FormatError, GridMismatchError, GsvolError, NumericalError,
                     StaleIndexError)
from .volume import (GridSpec, Volume, downsample_grid, ensure_unit_range,
                     grid_covering_extent, load_volume, normalize_intensity,
                     resample_trilinear, save_volume)
from .field import (GaussianField, InitConfig, init_from_volume, load_field, random_field,
                    save_field)
from .render import RenderOptions, render_naive, weight
from .raster import (DEFAULT_BRICK_DIMS, BrickIndex, GradientBuffer, RenderCache, backward,
                     build_brick_index, forward, merge_gradients, set_worker_count,
                     worker_count)
from .optimize import (AdamState, FitConfig, FitReport, fit, loss_and_grad, step_optimizer)
from .train import Renderer, StepOutput, TrainStep
from .metrics import MetricReport, psnr, ssim3d

__all__ = [
    "__version__",
    "GsvolError", "FormatError", "GridMismatchError", "StaleIndexError", "NumericalError",
    "GridSpec", "Volume", "normalize_intensity", "ensure_unit_range", "resample_trilinear",
    "grid_covering_extent", "downsample_grid", "save_volume", "load_volume",
    "GaussianField", "InitConfig", "init_from_volume", "random_field", "save_field",
    "load_field",
    "RenderOptions", "render_naive", "weight",
    "DEFAULT_BRICK_DIMS", "BrickIndex", "RenderCache", "GradientBuffer", "build_brick_index",
    "forward", "backward", "merge_gradients", "set_worker_count", "worker_count",
    "FitConfig", "FitReport", "AdamState", "fit", "loss_and_grad", "step_optimizer",
    "TrainStep", "StepOutput", "Renderer",
    "psnr", "ssim3d", "MetricReport",
]
