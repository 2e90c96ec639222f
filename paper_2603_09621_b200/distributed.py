"""Multi-GPU z-slab sharding of the brick grid.

Bricks are numbered x-fastest (raster.py:209), so a run of whole brick layers
[bz0, bz1) is a contiguous brick-id range and a rank's index is an exact slice
of the global index: concatenating the ranks' lists reproduces the reference
lists bit for bit.  Forward and render need no communication (each rank
writes only its own voxels); the train step's single collective is the
all_reduce of the merged per-Gaussian partial sums (TrainStep.update), with
the loss partial carried in the same buffer.
"""

from __future__ import annotations

import os


def brick_layers(grid, brick_dims) -> int:
    """Number of brick layers along z: ceil(nz / bdz)."""
    return -(-grid.dims[2] // brick_dims[2])


def slab_ranges(layers: int, world_size: int):
    """Contiguous, balanced split of brick layers [0, layers) over ranks.

    Returns a list of (bz0, bz1); every layer belongs to exactly one rank.
    Ranks beyond ``layers`` get empty slabs (bz0 == bz1).
    """
    if world_size < 1:
        raise ValueError("world_size must be >= 1")
    base, rem = divmod(layers, world_size)
    out, z = [], 0
    for r in range(world_size):
        n = base + (1 if r < rem else 0)
        out.append((z, z + n))
        z += n
    return out


def slab_for_rank(grid, brick_dims, rank: int, world_size: int):
    """This rank's (bz0, bz1), or None for a single-rank run (whole grid)."""
    if world_size <= 1:
        return None
    return slab_ranges(brick_layers(grid, brick_dims), world_size)[rank]


def slab_voxel_range(grid, brick_dims, slab):
    """Linear voxel range [v0, v1) a slab owns (whole x-y planes)."""
    plane = grid.dims[0] * grid.dims[1]
    if slab is None:
        return 0, grid.num_voxels
    z0 = slab[0] * brick_dims[2]
    z1 = min(slab[1] * brick_dims[2], grid.dims[2])
    return plane * z0, plane * max(z1, z0)


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
