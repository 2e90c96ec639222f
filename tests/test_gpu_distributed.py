"""The sharded train step on the GPU: two ranks (gloo, both on cuda:0 -- the
collective runs on the host, so no kernel waits on another rank) each bin,
render and back-propagate their z-slab of bricks, all_reduce the merged
per-Gaussian partials once, and apply the same Adam step.
The result equals the single-GPU step up to the f32 cast of the reduced
partial sums."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2603_09621_b200 as gs
from paper_2603_09621_b200.distributed import slab_for_rank
from paper_2603_09621_b200.synth import CONFIGS, make_problem

pytestmark = pytest.mark.gpu

STEPS = 3
F = ("positions", "log_scales", "rotations", "raw_amplitude", "raw_relax")


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(rank, world, port, cfg_id, out_dir, poison):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    p = make_problem(CONFIGS[cfg_id])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    st = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(lr.grid.spacing)
    slab = slab_for_rank(lr.grid, (8, 8, 4), rank, world)
    step = gs.TrainStep(lr, gs.RenderOptions(), (8, 8, 4), "l1", slab=slab,
                        process_group=dist.group.WORLD, world_size=world)
    losses = [step.step(f, st, lrs) for _ in range(STEPS)]
    if poison:
        bad = step.target.clone()
        bad[0] = float("nan")
        step.set_target(bad)
        losses.append(step.step(f, st, lrs))
    if rank == 0:
        np.savez(os.path.join(out_dir, "r0.npz"), losses=np.array(losses), t=st.t,
                 **{k: getattr(f, k).detach().cpu().numpy() for k in F})
    dist.barrier()
    dist.destroy_process_group()


def _single(cfg_id):
    p = make_problem(CONFIGS[cfg_id])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    st = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(lr.grid.spacing)
    step = gs.TrainStep(lr, gs.RenderOptions(), (8, 8, 4), "l1")
    losses = [step.step(f, st, lrs) for _ in range(STEPS)]
    return f, losses


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_two_rank_slab_step_matches_single_gpu(cfg_id):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_run, args=(2, _free_port(), cfg_id, d, False), nprocs=2, join=True)
        r = np.load(os.path.join(d, "r0.npz"))
        f1, l1 = _single(cfg_id)
        assert int(r["t"]) == STEPS
        np.testing.assert_allclose(r["losses"], l1, rtol=1e-6)
        for k in F:
            np.testing.assert_allclose(r[k], getattr(f1, k).cpu().numpy(), rtol=0, atol=2e-6,
                                       err_msg=k)


def test_two_rank_nonfinite_loss_skips_update():
    """A NaN target voxel in one rank's slab makes the global loss NaN after
    the all_reduce; both ranks then skip Adam (optimize.py:185-187)."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_run, args=(2, _free_port(), 1, d, True), nprocs=2, join=True)
        r = np.load(os.path.join(d, "r0.npz"))
        assert np.isnan(r["losses"][-1]) and int(r["t"]) == STEPS


def _run_nccl(rank, world, port, cfg_id, out_dir):
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world, device_id=torch.device("cuda", 0))
    torch.cuda.set_device(0)
    p = make_problem(CONFIGS[cfg_id])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    st = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(lr.grid.spacing)
    step = gs.TrainStep(lr, gs.RenderOptions(), (8, 8, 4), "l1",
                        slab=slab_for_rank(lr.grid, (8, 8, 4), rank, world),
                        process_group=dist.group.WORLD, world_size=world)
    losses = [step.step(f, st, lrs) for _ in range(STEPS)]
    captured = getattr(step, "_graph", None) is not None
    np.savez(os.path.join(out_dir, "r0.npz"), losses=np.array(losses), t=st.t,
             captured=captured, **{k: getattr(f, k).detach().cpu().numpy() for k in F})
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_sharded_graph_step_with_captured_nccl_all_reduce(cfg_id):
    """The sharded step over an NCCL group replays one CUDA graph that holds
    the all_reduce (world size 1 here: this box has one GPU, so the reduction
    is the identity).  It equals the single-GPU step up to the f32 cast of
    the reduced partials."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_run_nccl, args=(1, _free_port(), cfg_id, d), nprocs=1, join=True)
        r = np.load(os.path.join(d, "r0.npz"))
        f1, l1 = _single(cfg_id)
        assert bool(r["captured"]) and int(r["t"]) == STEPS
        np.testing.assert_allclose(r["losses"], l1, rtol=1e-6)
        for k in F:
            np.testing.assert_allclose(r[k], getattr(f1, k).cpu().numpy(), rtol=0, atol=2e-6,
                                       err_msg=k)


# --------------------------------------------- owner-computes + halo exchange
def _run_halo(rank, world, port, cfg_id, out_dir, margin, check_margin):
    from paper_2603_09621_b200.distributed import pair_weights, slab_ranges, brick_count
    from paper_2603_09621_b200.halo import HaloTrainStep
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    torch.cuda.set_device(0)
    p = make_problem(CONFIGS[cfg_id])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    st = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(lr.grid.spacing)
    w = pair_weights(f, lr.grid)
    slabs = slab_ranges(brick_count(lr.grid, (8, 8, 4)), world, weights=w)
    step = HaloTrainStep(lr, slabs, rank, dist.group.WORLD, margin=margin,
                         check_margin=check_margin)
    step.attach(f, st)
    n_local = step.plan.n_local
    losses = [step.step(lrs) for _ in range(STEPS)]
    fg, sg = step.gather()
    if rank == 0:
        np.savez(os.path.join(out_dir, "r0.npz"), losses=np.array(losses), t=sg.t,
                 n_local=n_local, n=f.count, replans=step.replans,
                 **{k: getattr(fg, k).detach().cpu().numpy() for k in F},
                 **{"m_" + k: sg.m[k].cpu().numpy() for k in F})
    dist.barrier()
    dist.destroy_process_group()


def _single_eager(cfg_id):
    p = make_problem(CONFIGS[cfg_id])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    st = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(lr.grid.spacing)
    step = gs.TrainStep(lr, gs.RenderOptions(), (8, 8, 4), "l1")
    losses = []
    for _ in range(STEPS):
        out = step.forward(f)
        losses.append(out.loss())
        step.update(f, out, st, lrs)
    return f, st, losses


@pytest.mark.parametrize("cfg_id,world,margin,check", [(1, 2, 1.0, 1e-3), (2, 3, 1.0, 1e-3),
                                                       (1, 2, 0.0, 0.5)])
def test_halo_step_matches_single_gpu(cfg_id, world, margin, check):
    """Owner-computes + halo exchange (halo.py): each rank holds ~1/world of
    the Gaussians plus a halo, exchanges only halo rows, runs Adam on the
    Gaussians it owns.  Same losses and parameters as the single-GPU step up
    to the f64 association of the halo partial sums; a check margin above
    the plan's forces the re-plan path after every step."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_run_halo, args=(world, _free_port(), cfg_id, d, margin, check),
                 nprocs=world, join=True)
        r = np.load(os.path.join(d, "r0.npz"))
        f1, s1, l1 = _single_eager(cfg_id)
        assert int(r["t"]) == STEPS
        assert int(r["n_local"]) < int(r["n"])              # a rank holds a part only
        np.testing.assert_allclose(r["losses"], l1, rtol=1e-12)
        for k in F:
            np.testing.assert_allclose(r[k], getattr(f1, k).cpu().numpy(), rtol=0, atol=1e-9,
                                       err_msg=k)
            np.testing.assert_allclose(r["m_" + k], s1.m[k].cpu().numpy(), rtol=0,
                                       atol=1e-9, err_msg=k)
        if check > margin:
            assert int(r["replans"]) >= 2                    # re-planned after a step


def _run_halo_nccl(rank, world, port, cfg_id, out_dir):
    from paper_2603_09621_b200.distributed import brick_count, pair_weights, slab_ranges
    from paper_2603_09621_b200.halo import HaloTrainStep
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world, device_id=torch.device("cuda", 0))
    torch.cuda.set_device(0)
    p = make_problem(CONFIGS[cfg_id])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    st = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(lr.grid.spacing)
    slabs = slab_ranges(brick_count(lr.grid, (8, 8, 4)), world,
                        weights=pair_weights(f, lr.grid))
    step = HaloTrainStep(lr, slabs, rank, dist.group.WORLD)
    step.attach(f, st)
    assert step.graph_mode
    h = step.step_async(lrs)
    losses = []
    for i in range(STEPS):                     # fit()'s loop: one step queued ahead
        nxt = step.step_async(lrs) if i + 1 < STEPS else None
        losses.append(h.loss())
        h = nxt
    captured = getattr(step.inner, "_graph", None) is not None
    fg, sg = step.gather()
    np.savez(os.path.join(out_dir, "r0.npz"), losses=np.array(losses), t=sg.t,
             captured=captured, **{k: getattr(fg, k).detach().cpu().numpy() for k in F})
    dist.destroy_process_group()


def test_halo_step_graph_over_nccl():
    """The halo step over NCCL is one captured CUDA graph per iteration: the
    halo exchanges (all_to_all_single with the plan's fixed splits) and the
    {loss, overflow} all_reduce are its collectives, the reach check writes a
    result flag.  World size 1 here (one GPU): the exchanges are empty, so it
    must equal the single-GPU graph step."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_run_halo_nccl, args=(1, _free_port(), 1, d), nprocs=1, join=True)
        r = np.load(os.path.join(d, "r0.npz"))
        f1, l1 = _single(1)
        assert bool(r["captured"]) and int(r["t"]) == STEPS
        np.testing.assert_allclose(r["losses"], l1, rtol=1e-12)
        for k in F:
            np.testing.assert_allclose(r[k], getattr(f1, k).cpu().numpy(), rtol=0, atol=1e-12,
                                       err_msg=k)


def _run_empty_slab(rank, world, port, out_dir):
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world, device_id=torch.device("cuda", 0))
    torch.cuda.set_device(0)
    p = make_problem(CONFIGS[1])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    st = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(lr.grid.spacing)
    # an empty brick range: the forward writes no loss partial at all
    step = gs.TrainStep(lr, gs.RenderOptions(), (8, 8, 4), "l1", slab=(0, 0),
                        process_group=dist.group.WORLD, world_size=world)
    losses = [step.step(f, st, lrs) for _ in range(2)]
    np.savez(os.path.join(out_dir, "r0.npz"), losses=np.array(losses),
             captured=getattr(step, "_graph", None) is not None)
    dist.destroy_process_group()


def test_empty_slab_graph_step_reports_zero_loss():
    """A rank whose slab is empty (slab_ranges allows b0 == b1) contributes an
    exact 0 to the step's loss sum in the captured graph (its loss partial
    buffer starts zeroed; the forward writes none)."""
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_run_empty_slab, args=(1, _free_port(), d), nprocs=1, join=True)
        r = np.load(os.path.join(d, "r0.npz"))
        assert bool(r["captured"])
        assert np.all(r["losses"] == 0.0), r["losses"]
