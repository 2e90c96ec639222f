"""Multi-GPU slab sharding of the brick grid.

Bricks are numbered x-fastest (raster.py:209), so any contiguous brick-id
range [b0, b1) is an exact slice of the global index: concatenating the
ranks' lists reproduces the reference lists bit for bit.  A slab is such a
range.  Cuts may fall anywhere inside a brick layer, so the split can be
balanced by per-brick cost (the pair count, i.e. the brick's share of the
forward/backward work) rather than by whole z-layers, which are too coarse
when a grid has few layers (config 4: 10 layers of 8x8x4 bricks over 8
ranks).  Forward and render need no communication (each rank writes only its
own bricks' voxels); the train step's single collective is the all_reduce of
the merged per-Gaussian partial sums (TrainStep.update), with the loss
partial carried in the same buffer.
"""

from __future__ import annotations

import os

import numpy as np


def brick_grid(grid, brick_dims) -> tuple:
    """Bricks per axis: ceil(dims / brick_dims) (raster.py:152-156)."""
    return tuple(-(-d // b) for d, b in zip(grid.dims, brick_dims))


def brick_layers(grid, brick_dims) -> int:
    """Number of brick layers along z: ceil(nz / bdz)."""
    return brick_grid(grid, brick_dims)[2]


def brick_count(grid, brick_dims) -> int:
    bg = brick_grid(grid, brick_dims)
    return bg[0] * bg[1] * bg[2]


def slab_ranges(nbricks: int, world_size: int, weights=None, align: int = 1):
    """Contiguous split of brick ids [0, nbricks) into ``world_size`` slabs.

    Returns a list of (b0, b1); every brick belongs to exactly one rank, in
    rank order.  Without ``weights`` the split is even by brick count; with
    per-brick ``weights`` (e.g. pair counts, ``np.diff(starts)``) the cut
    between ranks r and r+1 is the brick boundary whose weight prefix is
    nearest (r+1)/world_size of the total.  ``align`` restricts cuts to multiples of
    ``align`` bricks (``bgx*bgy`` gives whole z-layer slabs).  Ranks beyond
    the available cuts get empty slabs (b0 == b1).
    """
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    if align < 1:
        raise ValueError("align must be >= 1")
    units = -(-nbricks // align)
    if weights is None:
        w = np.ones(units, dtype=np.float64)
    else:
        wb = np.asarray(weights, dtype=np.float64).reshape(-1)
        if wb.shape[0] != nbricks:
            raise ValueError(f"weights has {wb.shape[0]} entries, expected {nbricks}")
        if (wb < 0).any() or not np.isfinite(wb).all():
            raise ValueError("weights must be finite and >= 0")
        pad = np.zeros(units * align, dtype=np.float64)
        pad[:nbricks] = wb
        w = pad.reshape(units, align).sum(axis=1)
        if w.sum() <= 0:
            w = np.ones(units, dtype=np.float64)
    prefix = np.concatenate([[0.0], np.cumsum(w)])
    total = prefix[-1]
    cuts = [0]
    for r in range(1, world_size):
        c = int(np.searchsorted(prefix, total * r / world_size, side="left"))
        # the boundary nearer the target of the two around it
        if c > 0 and abs(prefix[c - 1] - total * r / world_size) <= abs(
                prefix[min(c, units)] - total * r / world_size):
            c -= 1
        cuts.append(min(max(c, cuts[-1]), units))
    cuts.append(units)
    return [(min(a * align, nbricks), min(b * align, nbricks)) for a, b in zip(cuts, cuts[1:])]


def layer_slab_ranges(grid, brick_dims, world_size: int):
    """Whole z-layer slabs as brick-id ranges, balanced by layer count."""
    bg = brick_grid(grid, brick_dims)
    return slab_ranges(bg[0] * bg[1] * bg[2], world_size, align=bg[0] * bg[1])


def slab_for_rank(grid, brick_dims, rank: int, world_size: int, weights=None):
    """This rank's (b0, b1), or None for a single-rank run (whole grid)."""
    if world_size <= 1:
        return None
    return slab_ranges(brick_count(grid, brick_dims), world_size, weights)[rank]


def pair_weights(f, grid, opts=None, brick_dims=(8, 8, 4)):
    """Per-brick pair counts of the whole-grid index (numpy int64): the cost
    weights for a balanced split.  One binning pass on the device; every rank
    computes the same numbers (binning is deterministic)."""
    from .raster import build_brick_index
    from .render import RenderOptions
    idx = build_brick_index(f, grid, opts or RenderOptions(), brick_dims)
    return np.diff(idx.starts.cpu().numpy())


def slab_voxel_mask(grid, brick_dims, slab):
    """Boolean mask over linear (x-fastest) voxels: those of the slab's bricks."""
    nx, ny, nz = grid.dims
    if slab is None:
        return np.ones(nx * ny * nz, dtype=bool)
    bg = brick_grid(grid, brick_dims)
    bx = np.arange(nx) // brick_dims[0]
    by = np.arange(ny) // brick_dims[1]
    bz = np.arange(nz) // brick_dims[2]
    b = bx[None, None, :] + bg[0] * (by[None, :, None] + bg[1] * bz[:, None, None])
    b = b.reshape(-1)
    return (b >= slab[0]) & (b < slab[1])


def init_from_env(backend: str = "nccl"):
    """torch.distributed init from torchrun's RANK/WORLD_SIZE/LOCAL_RANK.

    Returns (dist module or None, world_size, rank, local_rank).
    """
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws <= 1:
        return None, 1, 0, 0
    import torch.distributed as dist
    if backend == "nccl":
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return dist, ws, rank, local
