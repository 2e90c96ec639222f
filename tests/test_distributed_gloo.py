"""The sharded train step's host logic at world_size 2 over gloo (CPU).

Each rank owns a contiguous brick-id range (here cut mid-layer, balanced by
pairs per brick): its index is the exact slice of the
global index, it renders only its voxels, merges its pairs' partials per
Gaussian, and one all_reduce (with the loss partial in column 11, exactly as
TrainStep.update packs it) gives every rank the full gradient.  The compute is
the CPU oracle standing in for the kernels; this checks the partition, the
slice property and the reduction the CUDA path relies on.
"""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2603_09621_b200.distributed import slab_ranges, slab_voxel_mask
from paper_2603_09621_b200.field import random_field_arrays
from paper_2603_09621_b200.volume import GridSpec

from conftest import GRAD_KEYS, field_dict

GRID = GridSpec((16, 12, 20), (1.0, 1.2, 0.9), (0.5, -1.0, 2.0))
BD = (8, 8, 4)


def _problem():
    arrs = random_field_arrays(400, GRID, 5, 0.4, 2.0)
    target = np.random.default_rng(6).uniform(size=GRID.num_voxels).astype(np.float32)
    return field_dict(arrs), target


def _slabs(starts, ws):
    """Pair-balanced brick-id ranges from the global starts (what bench.py
    does with distributed.pair_weights)."""
    return slab_ranges(len(starts) - 1, ws, weights=np.diff(starts))


def _rank_main(rank, ws, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    fd, target = _problem()
    st, gi = oracle.build_index(fd, GRID.dims, GRID.spacing, GRID.origin, BD)
    b0, b1 = _slabs(st, ws)[rank]
    # the slab index is the exact slice of the global lists
    s_starts = st.copy()
    s_starts[:b0] = st[b0]
    s_starts[b1:] = st[b1]
    S, W, I = oracle.forward(fd, GRID.dims, GRID.spacing, GRID.origin, s_starts, gi, BD)
    own_v = slab_voxel_mask(GRID, BD, (b0, b1))
    d = I[own_v].astype(np.float64) - target[own_v].astype(np.float64)
    dl = np.zeros(GRID.num_voxels)
    dl[own_v] = 2.0 * d / GRID.num_voxels                      # l2 (continuous)
    pg = oracle.pair_partials(fd, GRID.dims, GRID.spacing, GRID.origin, s_starts, gi, W, I, dl,
                              BD)
    own = np.zeros(len(gi), dtype=bool)
    own[st[b0]:st[b1]] = True
    pg[~own] = 0.0
    sums = oracle.merge(fd["positions"].shape[0], gi, pg)
    buf = torch.zeros((sums.shape[0], 12), dtype=torch.float64)
    buf[:, :11] = torch.from_numpy(sums)
    buf[0, 11] = float((d * d).sum())                           # loss partial rides along
    dist.all_reduce(buf)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), buf.numpy())
    Iv = np.zeros_like(I)
    Iv[own_v] = I[own_v]
    np.save(os.path.join(out_dir, f"I{rank}.npy"), Iv)
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_gloo_allreduce_equals_single_process(tmp_path):
    port = 29500 + (os.getpid() % 1000)
    mp.spawn(_rank_main, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    fd, target = _problem()
    st, gi = oracle.build_index(fd, GRID.dims, GRID.spacing, GRID.origin, BD)
    S, W, I = oracle.forward(fd, GRID.dims, GRID.spacing, GRID.origin, st, gi, BD)
    d = I.astype(np.float64) - target.astype(np.float64)
    dl = 2.0 * d / GRID.num_voxels
    pg = oracle.pair_partials(fd, GRID.dims, GRID.spacing, GRID.origin, st, gi, W, I, dl, BD)
    sums = oracle.merge(fd["positions"].shape[0], gi, pg)
    r0 = np.load(tmp_path / "rank0.npy")
    r1 = np.load(tmp_path / "rank1.npy")
    np.testing.assert_array_equal(r0, r1)                       # replicated after all_reduce
    np.testing.assert_allclose(r0[:, :11], sums, rtol=1e-12, atol=1e-18)
    assert r0[0, 11] / GRID.num_voxels == pytest.approx(float((d * d).mean()), rel=1e-12)
    # each rank's voxels are bit-identical to the single-process render
    i_all = np.load(tmp_path / "I0.npy") + np.load(tmp_path / "I1.npy")
    np.testing.assert_array_equal(i_all, I)
    # the cut is inside a brick layer (2 x 2 bricks per layer here)
    b_cut = _slabs(st, 2)[0][1]
    assert b_cut % 4 != 0
    g_sharded = oracle.chain_rule(fd, r0[:, :11])
    g_single = oracle.chain_rule(fd, sums)
    for k in GRAD_KEYS:
        np.testing.assert_allclose(g_sharded[k], g_single[k], rtol=1e-10, atol=1e-16)
