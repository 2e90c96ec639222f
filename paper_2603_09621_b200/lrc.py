"""LR-consistency training mode (north_star (c); not a reference feature).

The reference trains on the LR grid (optimize.py:171-173): render at the LR
grid, compare with the LR volume.  The paper's alternative renders at the HR
grid and compares its downsample with the LR volume, so the HR render itself
is what the loss constrains.  This module provides that mode as an explicit,
flagged extra -- it is NOT part of any parity claim (the reference has no
counterpart) and fit() never uses it:

  LRConsistencyStep(lr, factors).step(f, state, lrs)
    build_brick_index + forward at the HR grid (live masks, no fused loss)
    -> gsv_pool_loss: LR prediction = mean of each LR voxel's HR block, L1/L2
       loss against lr, dL/dI_HR = dL/dI_LR / |block| as the backward's
       {dL/dI / W, I}
    -> masked backward at the HR grid -> fused chain rule / Adam / renorm.

Checked in tests/test_gpu_lrc.py against the same objective composed from the
public API (forward at HR, pooling and loss in torch, backward with that
dL/dI).
"""

from __future__ import annotations

import math

import torch

from . import _lib
from .field import GaussianField
from .raster import (_forward_into, _pair_partials, _reaching, _train_mask_vpl,
                     build_brick_index, _chain_rule)
from .render import RenderOptions
from .volume import GridSpec, Volume

LOSS_KINDS = {"l1": 0, "l2": 1}


def hr_grid_for(lr_grid: GridSpec, factors) -> GridSpec:
    """The HR grid nested in lr_grid: dims x factors, spacing / factors, each
    LR voxel covering a factors-block of HR voxels (grid_covering_extent)."""
    f = tuple(int(a) for a in factors)
    sp = tuple(s / a for s, a in zip(lr_grid.spacing, f))
    org = tuple(o - 0.5 * (a - 1) * s for o, a, s in zip(lr_grid.origin, f, sp))
    return GridSpec(tuple(d * a for d, a in zip(lr_grid.dims, f)), sp, org)


class LRConsistencyStep:
    """One fit iteration with the LR-consistency loss (module docstring)."""

    def __init__(self, lr: Volume, factors=(2, 2, 2), opts: RenderOptions = RenderOptions(),
                 brick_dims=(8, 8, 4), loss: str = "l1"):
        if opts.precision != "f32":
            raise ValueError("the LR-consistency mode runs the f32 engine")
        if loss not in LOSS_KINDS:
            raise ValueError(f"unknown loss kind {loss!r}")
        self.lr, self.factors = lr, tuple(int(a) for a in factors)
        self.hr_grid = hr_grid_for(lr.grid, self.factors)
        self.opts, self.bd, self.loss_kind = opts, tuple(brick_dims), LOSS_KINDS[loss]
        lin = lr.linear()
        if lin.device.type != "cuda":
            lin = lin.to(torch.device("cuda", torch.cuda.current_device()))
        tdt = torch.float64 if lin.dtype == torch.float64 else torch.float32
        self.target = lin.to(tdt).contiguous()
        self.pool = _lib.BufferPool(self.target.device)

    def forward_backward(self, f: GaussianField):
        """HR render, pooled loss and per-pair backward; returns (mean loss,
        per-Gaussian merged partials (N, 12) f64, index)."""
        lib = _lib.lib()
        hr, opts, pool = self.hr_grid, self.opts, self.pool
        idx = build_brick_index(f, hr, opts, self.bd, pool=pool)
        aux = idx._aux
        nv = hr.num_voxels
        S = pool.get("S", (nv,), torch.float32)
        W = pool.get("W", (nv,), torch.float32)
        I = pool.get("I", (nv,), torch.float32)
        mvpl = _train_mask_vpl(self.bd, idx.pair_count, _reaching(f, idx))
        masks = pool.get("masks", (max(idx.pair_count, 1), 4, 2), torch.int32)
        _forward_into(f, hr, idx, opts, aux.rec32, aux.rec64, S, W, I, live_masks=masks)
        gl = _lib.make_grid(self.lr.grid)
        nb = lib.gsv_pool_loss_blocks(gl)
        part = pool.get("part", (nb,), torch.float64)
        ab = pool.get("ab", (nv, 2), torch.float32)
        fx, fy, fz = self.factors
        _lib.check(lib.gsv_pool_loss(
            I.data_ptr(), W.data_ptr(), self.target.data_ptr(),
            int(self.target.dtype == torch.float64), _lib.make_grid(hr), gl, fx, fy, fz,
            self.loss_kind, float(opts.epsilon_w), ab.data_ptr(), part.data_ptr(),
            _lib.stream_ptr()), "pool_loss")
        tot = pool.get("tot", (1,), torch.float64)
        _lib.check(lib.gsv_sum(part.data_ptr(), nb, tot.data_ptr(), _lib.stream_ptr()), "sum")
        loss = float(tot.item()) / self.lr.grid.num_voxels
        gsum = _pair_partials(f, hr, idx, opts, aux.rec32, aux.rec64, ab, aux.gstart, aux.box,
                              True, pool=pool, live_masks=masks, mask_vpl=mvpl)
        self.last_cache = (S, W, I)
        return loss, gsum, idx

    def gradients(self, f: GaussianField):
        """(loss, GradientBuffer) of the LR-consistency objective."""
        loss, gsum, _ = self.forward_backward(f)
        return loss, _chain_rule(f, gsum)

    def step(self, f: GaussianField, state, lrs: dict, beta1: float = 0.9,
             beta2: float = 0.999, eps: float = 1e-8) -> float:
        """One iteration; like fit(), no update when the loss is non-finite."""
        from .train import _adam_launch
        loss, gsum, _ = self.forward_backward(f)
        if math.isfinite(loss):
            _adam_launch(f, state, lrs, beta1, beta2, eps, None, None, gsum,
                         self.opts.precision_code, self.pool)
        return loss
