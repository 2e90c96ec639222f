"""Synthetic benchmark inputs -- setup.

Restates the reference's phantom generator (phantom.py:52-108) and the
degrade/init recipe with the same numpy/scipy calls, so the LR volumes and
initial fields are bit-identical to the reference's (pinned by sha256 in
tests/golden/).  generate_phantom_device / make_problem(device=...) run the
phantom and the degrade on the GPU (gsv_phantom: scipy's gaussian_filter
order restated), bit-identical for the ellipsoid phantoms.  Setup, not the
rendering path.
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


def gaussian_kernel1d(sigma: float, truncate: float = 4.0):
    """(weights, radius) of ndimage.gaussian_filter's order-0 kernel
    (scipy _gaussian_kernel1d with radius int(truncate * sigma + 0.5))."""
    sd = float(sigma)
    radius = int(truncate * sd + 0.5)
    x = np.arange(-radius, radius + 1)
    phi = np.exp(-0.5 / (sd * sd) * x ** 2)
    return phi / phi.sum(), radius


def generate_phantom_device(prims, grid: GridSpec, smooth_sigma: float = 0.0,
                            kind: str = "ellipsoids", device=None):
    """generate_phantom (phantom.py:52-75) on the GPU (gsv_phantom): the
    float32 volume as an x-fastest linear CUDA tensor.  prims: objects with
    center, semi_axes (ellipsoids) or sigmas (gaussian mixture), intensity.
    Ellipsoids are bit-identical to generate_ellipsoids (the host path)."""
    import torch
    from . import _lib
    if kind not in ("ellipsoids", "gaussian-mixture"):
        raise ValueError(f"unknown phantom kind {kind!r}")
    if smooth_sigma < 0:
        raise ValueError("smooth_sigma must be >= 0")
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    rows = [list(q.center) + list(q.semi_axes if kind == "ellipsoids" else q.sigmas) +
            [float(q.intensity)] for q in prims]
    pr = torch.tensor(np.asarray(rows, dtype=np.float64).reshape(-1, 7), device=dev)
    radius, w = 0, None
    if smooth_sigma > 0:
        wn, radius = gaussian_kernel1d(smooth_sigma)
        w = torch.from_numpy(wn).to(dev)
    nv = grid.num_voxels
    scratch = torch.empty(2 * nv, dtype=torch.float64, device=dev)
    out = torch.empty(nv, dtype=torch.float32, device=dev)
    lib = _lib.lib()
    _lib.check(lib.gsv_phantom(_lib.make_grid(grid), 0 if kind == "ellipsoids" else 1,
                               len(rows), pr.data_ptr() if rows else None, radius,
                               None if w is None else w.data_ptr(), scratch.data_ptr(),
                               out.data_ptr(), _lib.stream_ptr()), "phantom")
    return out


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


def make_problem(cfg: BenchConfig, seed: int = 11, device=None):
    """HR phantom -> trilinear LR -> init field (threshold 0 => N = #LR voxels).

    Returns dict(hr_grid, hr (np f32), lr_grid, lr (np f32), field arrays,
    render_grid).  Same recipe as the reference conftest (conftest.py:26-32).
    device (a CUDA device): the phantom and the resampling run there
    (gsv_phantom, gsv_resample_trilinear; bit-identical), the rest as on the host.
    """
    hr_grid = GridSpec(cfg.hr_dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    lr_grid = grid_covering_extent(hr_grid, cfg.lr_dims)
    prims = random_ellipsoids(hr_grid, seed)
    if device is not None:
        from .volume import Volume, resample_trilinear
        hr_t = generate_phantom_device(prims, hr_grid, 0.7, device=device)
        hr_v = Volume.from_linear(hr_grid, hr_t)
        hr = hr_v.numpy()
        lr = resample_trilinear(hr_v, lr_grid).numpy()
    else:
        hr = generate_ellipsoids(prims, hr_grid, smooth_sigma=0.7)
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
