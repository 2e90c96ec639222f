"""Render options and the brute-force renderer (mirrors gsvol/render.py:32-127).

``RenderOptions`` is the reference dataclass unchanged.  ``render_naive`` runs
the O(N*V) explicit-Sigma^-1 route on the GPU (gsv_render_naive), kept as an
API-compatible cross-check of the brick engine.
"""

from __future__ import annotations

import math
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


def weight(f: GaussianField, i: int, p, opts: RenderOptions = RenderOptions()) -> float:
    """Spatial weight of Gaussian i at world point p (render.py:74-81).

    A scalar API helper (one Gaussian, one point) evaluated from that
    Gaussian's parameters; not part of the rendering path.
    """
    q = f.rotations[i].detach().cpu().numpy()
    ls = f.log_scales[i].detach().cpu().numpy()
    mu = f.positions[i].detach().cpu().numpy()
    w, x, y, z = q
    r = np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
        [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
        [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
    ])
    sigma_inv = r @ np.diag(np.exp(-2.0 * ls)) @ r.T
    delta = np.asarray(p, dtype=np.float64) - mu
    d2 = float(delta @ sigma_inv @ delta)
    if d2 > opts.cutoff_sq:
        return 0.0
    relax = 1.0 if not f.relax_enabled else 1.0 / (1.0 + math.exp(-float(f.raw_relax[i])))
    return math.exp(-0.5 * d2) * relax
