"""Render options and the brute-force renderer (mirrors gsvol/render.py:32-127).

``RenderOptions`` is the reference dataclass unchanged.  ``render_naive`` runs
the O(N*V) explicit-Sigma^-1 route on the GPU (gsv_render_naive), kept as an
API-compatible cross-check of the brick engine.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .field import GaussianField
from .volume import GridSpec, Volume


@dataclass(frozen=True)
class RenderOptions:
    """Shared knobs for both render engines (render.py:32-64)."""
    cutoff_sigma: float = 3.0
    epsilon_w: float = 1e-8
    precision: str = "f32"
    deterministic: bool = True

    def __post_init__(self):
        if self.cutoff_sigma <= 0:
            raise ValueError("cutoff_sigma must be positive")
        if self.epsilon_w <= 0:
            raise ValueError("epsilon_w must be positive")
        if self.precision not in ("f32", "f64"):
            raise ValueError(f"precision must be 'f32' or 'f64', got {self.precision!r}")

    @property
    def dtype(self):
        return np.float32 if self.precision == "f32" else np.float64

    @property
    def torch_dtype(self):
        return torch.float32 if self.precision == "f32" else torch.float64

    @property
    def precision_code(self) -> int:
        return 0 if self.precision == "f32" else 1

    @property
    def cutoff_sq(self) -> float:
        return self.cutoff_sigma * self.cutoff_sigma


def render_naive(f: GaussianField, grid: GridSpec, opts: RenderOptions = RenderOptions()) -> Volume:
    """Render by looping all Gaussians at every voxel centre (render.py:113-127)."""
    lib = _lib.lib()
    out = torch.empty(grid.num_voxels, dtype=opts.torch_dtype, device=f.device)
    g = _lib.make_grid(grid)
    _lib.check(lib.gsv_render_naive(
        f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
        f.raw_amplitude.data_ptr(), f.raw_relax.data_ptr(), f.count, int(f.relax_enabled),
        g, opts.cutoff_sigma, opts.epsilon_w, opts.precision_code, out.data_ptr(),
        _lib.stream_ptr()), "render_naive")
    return Volume.from_linear(grid, out)


def field_sigma_inv(f: GaussianField) -> torch.Tensor:
    """Per-Gaussian inverse covariances R diag(s^-2) R^T, (N,3,3) f64 on the
    device (render.py:67-71; gsv_sigma_inv)."""
    lib = _lib.lib()
    out = torch.empty((f.count, 3, 3), dtype=torch.float64, device=f.device)
    _lib.check(lib.gsv_sigma_inv(f.log_scales.data_ptr(), f.rotations.data_ptr(), f.count,
                                 out.data_ptr(), _lib.stream_ptr()), "sigma_inv")
    return out


def weight(f: GaussianField, i: int, p, opts: RenderOptions = RenderOptions()) -> float:
    """Spatial weight of Gaussian i at world point p, truncation included
    (render.py:74-81), evaluated on the device (gsv_weight)."""
    lib = _lib.lib()
    px, py, pz = (float(v) for v in np.asarray(p, dtype=np.float64).reshape(3))
    out = torch.empty(1, dtype=torch.float64, device=f.device)
    _lib.check(lib.gsv_weight(
        f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
        f.raw_relax.data_ptr(), f.count, int(i), int(f.relax_enabled), px, py, pz,
        float(opts.cutoff_sigma), out.data_ptr(), _lib.stream_ptr()), "weight")
    return float(out.item())
