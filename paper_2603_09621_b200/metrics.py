"""Reconstruction quality metrics on the device: PSNR and full-3D SSIM
(metrics.py:1-100 of the reference), same names, semantics and errors.

Both assume normalized volumes (data range 1.0) on identical grids.  The
arithmetic is f64 like the reference; the sums run in a fixed order on the
GPU (libgsv_b200: gsv_sq_diff_sum, gsv_ssim3d), so results are run-to-run
reproducible and equal the reference up to summation-order rounding.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import GridMismatchError
from .volume import GridSpec, Volume

_WINDOW_SIZE = 11
_WINDOW_SIGMA = 1.5


def _check_grids(x: Volume, y: Volume) -> None:
    if x.grid != y.grid:
        raise GridMismatchError(f"metric inputs on different grids: "
                                f"{x.grid.dims} vs {y.grid.dims}")


def _gaussian_window() -> np.ndarray:
    """The 11-tap sigma-1.5 window, normalised to sum 1, evaluated with numpy
    in the reference's operation order (metrics.py:45-49) -> identical bits."""
    offsets = np.arange(_WINDOW_SIZE) - (_WINDOW_SIZE - 1) / 2
    denom = 2.0 * _WINDOW_SIGMA ** 2
    taps = np.exp(-(offsets * offsets) / denom)
    return taps / taps.sum()


def _device_linear(v: Volume, dev) -> tuple[torch.Tensor, int]:
    lin = v.linear()
    if lin.dtype not in (torch.float32, torch.float64):
        lin = lin.to(torch.float64)
    lin = lin.to(dev).contiguous()
    return lin, int(lin.dtype == torch.float64)


def _device(x: Volume, y: Volume):
    for v in (x, y):
        if v.data.device.type == "cuda":
            return v.data.device
    return torch.device("cuda", torch.cuda.current_device())


def psnr(x: Volume, y: Volume) -> float:
    """10*log10(1/MSE) in dB against data range 1.0; inf when identical."""
    _check_grids(x, y)
    lib = _lib.lib()
    dev = _device(x, y)
    a, af = _device_linear(x, dev)
    b, bf = _device_linear(y, dev)
    v = a.numel()
    part = torch.empty(lib.gsv_metric_blocks(v), dtype=torch.float64, device=dev)
    out = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.check(lib.gsv_sq_diff_sum(a.data_ptr(), af, b.data_ptr(), bf, v, part.data_ptr(),
                                   out.data_ptr(), _lib.stream_ptr()), "sq_diff_sum")
    mse = float(out.item()) / v
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(1.0 / mse)


def ssim3d(x: Volume, y: Volume) -> float:
    """Mean local SSIM over all voxels, full 3D windows."""
    _check_grids(x, y)
    if min(x.grid.dims) < _WINDOW_SIZE:
        raise ValueError(
            f"volume too small for SSIM window: dims {x.grid.dims}, "
            f"need >= {_WINDOW_SIZE} per axis"
        )
    lib = _lib.lib()
    dev = _device(x, y)
    a, af = _device_linear(x, dev)
    b, bf = _device_linear(y, dev)
    g = _lib.make_grid(x.grid)
    nbytes = ctypes.c_size_t(0)
    _lib.check(lib.gsv_ssim3d_workspace(g, ctypes.byref(nbytes)), "ssim3d_workspace")
    ws = _lib.workspace(nbytes.value, dev, "ssim")
    win = (ctypes.c_double * _WINDOW_SIZE)(*_gaussian_window().tolist())   # host array
    out = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.check(lib.gsv_ssim3d(a.data_ptr(), af, b.data_ptr(), bf, g, win,
                              ws.data_ptr(), ws.numel(), out.data_ptr(), _lib.stream_ptr()),
               "ssim3d")
    return float(out.item()) / a.numel()


@dataclass(frozen=True)
class MetricReport:
    """PSNR + SSIM of a reconstruction against its reference volume
    (metrics.py:80-100): ``identical`` when the volumes are equal (PSNR inf,
    serialised as null)."""

    psnr: float
    ssim: float
    grid: GridSpec
    identical: bool

    @classmethod
    def evaluate(cls, x: Volume, y: Volume) -> "MetricReport":
        p = psnr(x, y)
        return cls(psnr=p, ssim=ssim3d(x, y), grid=x.grid, identical=math.isinf(p))

    def to_json(self) -> dict:
        g = self.grid
        grid = {"dims": list(g.dims), "spacing": list(g.spacing), "origin": list(g.origin)}
        return {"psnr": None if self.identical else self.psnr, "ssim": self.ssim,
                "identical": self.identical, "grid": grid}
