"""Synthetic benchmark inputs -- host setup.

Restates the reference's phantom generator (phantom.py:52-108) and the
degrade/init recipe with the same numpy/scipy calls, so the LR volumes and
initial fields are bit-identical to the reference's (pinned by sha256 in
tests/golden/).  This runs once per problem on the host, like the
reference's setup; it is not part of the rendering path.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np
from scipy import ndimage

from .field import init_arrays_from_volume, InitConfig
from .volume import GridSpec, grid_covering_extent, resample_trilinear_np


@dataclass(frozen=True)
class _Ellipsoid:
    center: tuple
    semi_axes: tuple
    intensity: float


def random_ellipsoids(grid: GridSpec, seed: int, components: int = 6):
    """random_phantom("ellipsoids", ...) (phantom.py:78-100)."""
    rng = np.random.default_rng(seed)
    lo, hi = grid.extent()
    lo = np.asarray(lo)
    size = np.asarray(hi) - lo
    center = lo + size / 2
    outer = size * rng.uniform(0.30, 0.38, size=3)
    prims = [_Ellipsoid(tuple(center + size * rng.uniform(-0.02, 0.02, size=3)), tuple(outer),
                        float(rng.uniform(0.55, 0.7)))]
    for _ in range(components - 1):
        c = center + size * rng.uniform(-0.18, 0.18, size=3)
        axes = size * rng.uniform(0.04, 0.14, size=3)
        prims.append(_Ellipsoid(tuple(c), tuple(axes), float(rng.uniform(0.2, 0.95))))
    return prims


def generate_ellipsoids(prims, grid: GridSpec, smooth_sigma: float = 0.0) -> np.ndarray:
    """generate_phantom for ellipsoids (phantom.py:52-75): max at overlaps,
    optional Gaussian blur, clamp, float32.  Returns the dims-shaped array."""
    cx_, cy_, cz_ = (grid.axis_coords(k) for k in range(3))
    xs, ys, zs = cx_[:, None, None], cy_[None, :, None], cz_[None, None, :]
    out = np.zeros(grid.dims, dtype=np.float64)
    for prim in prims:
        cx, cy, cz = prim.center
        ax, ay, az = prim.semi_axes
        d2 = ((xs - cx) / ax) ** 2 + ((ys - cy) / ay) ** 2 + ((zs - cz) / az) ** 2
        np.maximum(out, np.where(d2 <= 1.0, prim.intensity, 0.0), out=out)
    if smooth_sigma > 0:
        out = ndimage.gaussian_filter(out, sigma=smooth_sigma)
    np.clip(out, 0.0, 1.0, out=out)
    return out.astype(np.float32)


@dataclass(frozen=True)
class BenchConfig:
    name: str
    lr_dims: tuple
    hr_dims: tuple
    render_dims: tuple | None = None   # render grid (defaults to hr_dims)
    jitter: bool = False


# BASELINE.json "configs".
CONFIGS = {
    1: BenchConfig("c1_32^3->64^3", (32, 32, 32), (64, 64, 64)),
    2: BenchConfig("c2_128x128x64->256x256x128", (128, 128, 64), (256, 256, 128)),
    3: BenchConfig("c3_128^3->256^3", (128, 128, 128), (256, 256, 256)),
    4: BenchConfig("c4_256x256x40->256x256x160", (256, 256, 40), (256, 256, 160)),
    5: BenchConfig("c5_2M_field->512^3", (128, 128, 128), (256, 256, 256), (512, 512, 512),
                   jitter=True),
}


def make_problem(cfg: BenchConfig, seed: int = 11):
    """HR phantom -> trilinear LR -> init field (threshold 0 => N = #LR voxels).

    Returns dict(hr_grid, hr (np f32), lr_grid, lr (np f32), field arrays,
    render_grid).  Same recipe as the reference conftest (conftest.py:26-32).
    """
    hr_grid = GridSpec(cfg.hr_dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    hr = generate_ellipsoids(random_ellipsoids(hr_grid, seed), hr_grid, smooth_sigma=0.7)
    lr_grid = grid_covering_extent(hr_grid, cfg.lr_dims)
    lr = resample_trilinear_np(hr, hr_grid, lr_grid)
    arrays = list(init_arrays_from_volume(lr, lr_grid, InitConfig(background_threshold=0.0)))
    if cfg.jitter:
        arrays = jitter_field(arrays, lr_grid)
    render_grid = hr_grid if cfg.render_dims is None else grid_covering_extent(lr_grid, cfg.render_dims)
    return {"hr_grid": hr_grid, "hr": hr, "lr_grid": lr_grid, "lr": lr, "field": arrays,
            "render_grid": render_grid}


def jitter_field(arrays, grid: GridSpec, seed: int = 1234):
    """Seeded perturbation emulating a trained field:
    mu += N(0,1)*0.1*spacing, ls += N(0,1)*0.05, q += N(0,1)*0.05 then q/|q|."""
    pos, ls, rot, ra, rr = (np.array(a, dtype=np.float64, copy=True) for a in arrays)
    rng = np.random.default_rng(seed)
    n = pos.shape[0]
    pos += rng.normal(size=(n, 3)) * (0.1 * np.asarray(grid.spacing))
    ls += rng.normal(size=(n, 3)) * 0.05
    rot += rng.normal(size=(n, 4)) * 0.05
    rot /= np.linalg.norm(rot, axis=1)[:, None]
    return [pos, ls, rot, ra, rr]


def sha256(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
