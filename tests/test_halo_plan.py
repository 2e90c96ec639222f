"""Owner-computes / halo plan of the sharded step (paper_2603_09621_b200/halo.py)
on the CPU: ownership partitions the Gaussians, every Gaussian the exact
binning puts in a slab's brick lists is in that rank's local set, and the
exchange lists of every rank pair line up.  A two-rank gloo run moves rows
through the same all_to_all the step uses."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2603_09621_b200.distributed import slab_ranges
from paper_2603_09621_b200.field import random_field_arrays
from paper_2603_09621_b200.halo import HaloPlan, _a2a_rows, reach_and_owner
from paper_2603_09621_b200.volume import GridSpec

from conftest import field_dict

GRID = GridSpec((24, 20, 28), (1.0, 1.2, 0.9), (0.5, -1.0, 2.0))
BD = (8, 8, 4)


def _field(n=1500, seed=3):
    return random_field_arrays(n, GRID, seed, 0.4, 2.0)


def _plans(arrs, world, margin=1.0):
    st, gi = oracle.build_index(field_dict(arrs), GRID.dims, GRID.spacing, GRID.origin, BD)
    slabs = slab_ranges(len(st) - 1, world, weights=np.diff(st))
    t = [torch.from_numpy(np.ascontiguousarray(a)) for a in arrs[:3]]
    own, lo, hi = reach_and_owner(*t, GRID, BD, slabs, 3.0, margin)
    return st, gi, slabs, own, [HaloPlan(own, lo, hi, r, world) for r in range(world)]


@pytest.mark.parametrize("world", [2, 3, 5])
def test_plan_covers_every_slab_and_partitions_owners(world):
    arrs = _field()
    st, gi, slabs, own, plans = _plans(arrs, world)
    owned = [set(p.local_gids[p.owned].tolist()) for p in plans]
    assert sum(len(o) for o in owned) == len(arrs[0])
    assert set().union(*owned) == set(range(len(arrs[0])))
    for r, (b0, b1) in enumerate(slabs):
        need = set(gi[st[b0]:st[b1]].tolist())        # exact binning of the slab
        have = set(plans[r].local_gids.tolist())
        assert need <= have, (r, len(need - have))
        assert torch.all(plans[r].local_gids[1:] > plans[r].local_gids[:-1])   # ascending


@pytest.mark.parametrize("world", [2, 4])
def test_plan_exchange_lists_line_up(world):
    arrs = _field(seed=8)
    _, _, _, own, plans = _plans(arrs, world)
    for r in range(world):
        for q in range(world):
            a = plans[r].local_gids[plans[r].to_owner[q]]      # r's halo owned by q
            b = plans[q].local_gids[plans[q].from_peer[r]]     # q's owned in r's set
            assert torch.equal(a, b), (r, q)
            assert bool((own[a] == q).all())


def test_margin_only_grows_local_sets():
    arrs = _field(seed=9)
    _, _, _, _, p0 = _plans(arrs, 3, margin=0.0)
    _, _, _, _, p1 = _plans(arrs, 3, margin=2.0)
    for a, b in zip(p0, p1):
        assert set(a.local_gids.tolist()) <= set(b.local_gids.tolist())


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    arrs = _field(seed=4)
    _, _, _, own, plans = _plans(arrs, world)
    p = plans[rank]
    # every local row holds (gid, 1): after the partial exchange an owned
    # row holds 1 + the number of other ranks that have it in their local set
    rows = torch.zeros((p.n_local, 12), dtype=torch.float64)
    rows[:, 0] = p.local_gids.to(torch.float64)
    rows[:, 1] = 1.0
    got = _a2a_rows(dist, dist.group.WORLD, p.to_owner,
                    [int(t.shape[0]) for t in p.from_peer], lambda idx: rows[idx])
    for r in range(world):
        if got[r].shape[0]:
            assert torch.equal(got[r][:, 0], rows[p.from_peer[r], 0])   # same gids, same order
            rows[:, 1].index_add_(0, p.from_peer[r], got[r][:, 1])
    holders = torch.zeros(len(arrs[0]), dtype=torch.float64)
    for pl in plans:
        holders[pl.local_gids] += 1
    oi = torch.nonzero(p.owned).view(-1)
    ok = bool(torch.equal(rows[oi, 1], holders[p.local_gids[oi]]))
    q.put((rank, ok))
    dist.destroy_process_group()


def test_partial_exchange_over_gloo_reaches_every_owner():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, 3, port, q)) for r in range(3)]
    for pr in ps:
        pr.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for pr in ps:
        pr.join(timeout=60)
    assert res == {0: True, 1: True, 2: True}
