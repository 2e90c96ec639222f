#!/usr/bin/env python
"""bench.py -- B200 brick rasterizer benchmark (BASELINE.json metric).

Workload (config 3 of BASELINE.json): 128^3 LR synthetic phantom, x2 -> 256^3
HR, N = 2,097,152 Gaussians (one per LR voxel).  A step is one fit()
iteration (optimize.py:171-184): bin -> forward + fused L1 -> backward ->
merge -> chain rule -> Adam -> quaternion renorm, on the 128^3 LR grid the
reference trains on.  `value` = train iterations/s (whole job), timed with
CUDA events, inputs resident in HBM.  The same line carries the 256^3 render
(bin + forward at the HR grid) in Gvoxel/s and the 512^3 render of config 5.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: launched by torch.distributed.run, one rank per GPU; each rank owns a
contiguous brick-id range (cuts balanced by pairs per brick, mid-layer cuts
allowed); one NCCL all_reduce per train step.
--impl reference: the unmodified reference (gsvol, installed into baseline/_ref)
through its public fit-loop API on all host cores, each step a fit() iteration
on a bounded 1/8 sample of the config (its central LR z-slab), scaled to the
workload; the oracle port only if the reference is not installed.  Rank 0
only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train iters/s + render Gvoxel/s at 256^3 HR, 1/2/4/8 B200, % FP32/HBM roofline"
FWD_FLOP, BWD_FLOP = 28, 74          # per live pair-voxel


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--no-render512", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the config-2 fit and config-4 step/render extra keys")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-count", action="store_true", help="skip the CUPTI launch count "
                    "(needed under ncu)")
    ap.add_argument("--shard", default="halo", choices=["halo", "allreduce"],
                    help="N > 1: owner-computes + halo exchange (halo.py) or the "
                         "replicated step with one all_reduce (TrainStep + group)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the multi-rank path with ranks sharing a GPU")
    return ap.parse_args()


# ----------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_setup(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        local = local % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(local)
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        return dist, ws, rank, local
    if torch.cuda.is_available():
        torch.cuda.set_device(0)
    return None, 1, 0, 0


from paper_2603_09621_b200.distributed import pair_weights, slab_for_rank  # noqa: E402


def problem_for(cfg_id, device=None):
    """The benchmark problem (phantom -> degrade -> init).  With a CUDA device
    the phantom and degrade run there (bit-identical, faster setup); the
    reference arm builds its inputs on the host."""
    from paper_2603_09621_b200 import synth
    return synth.make_problem(synth.CONFIGS[cfg_id], device=device)


# ----------------------------------------------------------------- CPU arm
def host_threads() -> int:
    """Pin the oracle's OpenMP team to every usable host core and return the
    count.  torchrun exports OMP_NUM_THREADS=1 to each rank, so the CPU arm
    sets the thread count explicitly on the libgomp the oracle links."""
    try:
        n = len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        n = os.cpu_count() or 1
    os.environ["OMP_NUM_THREADS"] = str(n)
    try:
        import ctypes
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(n)
    except OSError:
        pass
    return n


def cpu_train_step_seconds(p, steps: int, warmup: int):
    """Oracle (port of the reference CPU path) train iterations on this host."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    from paper_2603_09621_b200.optimize import FitConfig
    oracle.build()
    g = p["lr_grid"]
    fd = dict(zip(("positions", "log_scales", "rotations", "raw_amplitude", "raw_relax"),
                  [np.array(a, order="C", copy=True) for a in p["field"]]))
    st = oracle.adam_state(fd)
    lrs = FitConfig().resolved_lrs(g.spacing)
    tgt = np.ascontiguousarray(p["lr"].ravel(order="F"))
    for _ in range(warmup):
        oracle.train_step_fast(fd, g.dims, g.spacing, g.origin, tgt, st, lrs)
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle.train_step_fast(fd, g.dims, g.spacing, g.origin, tgt, st, lrs)
    return (time.perf_counter() - t0) / steps


REF_DIR = os.path.join(ROOT, "baseline", "_ref")
REF_SLAB_Z = 16          # LR z-voxels of the reference arm's sample (of 128 at config 3)


def _import_gsvol(cores: int):
    """The unmodified reference (gsvol, pip-installed into baseline/_ref) with
    numba's pool sized to every host core: NUMBA_NUM_THREADS must be set
    before numba is first imported (gsvol/_numba_env.py caps it at 8
    otherwise), then set_worker_count(cores) (raster.py:55-59)."""
    os.environ["NUMBA_NUM_THREADS"] = str(cores)
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "gsv_bench_numba_cache"))
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import gsvol
    gsvol.set_worker_count(cores)
    return gsvol


def reference_sample(p, cfg_id: int):
    """A bounded sample of the workload for the reference's CPU path: the
    central z-slab of REF_SLAB_Z LR voxels of the config's LR volume (same
    phantom, same spacing), initialised like fit() (threshold 0: one
    Gaussian per voxel).  Returns (grid dims, spacing, origin, data, fraction)
    where fraction = sample Gaussians / workload Gaussians."""
    g = p["lr_grid"]
    nz = g.dims[2]
    dz = min(REF_SLAB_Z, nz)
    z0 = (nz - dz) // 2
    data = np.ascontiguousarray(p["lr"][:, :, z0:z0 + dz])
    origin = (g.origin[0], g.origin[1], g.origin[2] + z0 * g.spacing[2])
    return (g.dims[0], g.dims[1], dz), tuple(g.spacing), origin, data, dz / nz


def gsvol_train_step_seconds(p, cfg_id: int, steps: int, warmup: int, cores: int):
    """Seconds per config-size fit() iteration of the real reference, from
    `steps` timed iterations on the bounded sample (reference_sample), scaled
    by the sample's Gaussian fraction.  The loop body is fit()'s
    (optimize.py:177-197) through gsvol's public API; JIT compilation is
    warmed on a 4^3 grid first, as gsvol/bench.py:28-31 does."""
    gsvol = _import_gsvol(cores)
    from gsvol import (AdamState, FitConfig, GridSpec, InitConfig, RenderOptions, Volume,
                       backward, build_brick_index, forward, init_from_volume, loss_and_grad,
                       step_optimizer)
    dims, sp, org, data, frac = reference_sample(p, cfg_id)
    grid = GridSpec(dims, sp, org)
    lr = Volume(grid, data)
    opts = RenderOptions()

    def one(f, st, lrs, vol):
        idx = build_brick_index(f, vol.grid, opts)
        cache = forward(f, vol.grid, idx, opts)
        loss, dl = loss_and_grad(cache.volume(), vol, "l1")
        grads = backward(f, vol.grid, idx, cache, dl, opts)
        step_optimizer(f, grads, st, lrs)
        f.normalize_rotations()
        return loss

    # JIT warm-up on a tiny problem (every kernel of the loop body)
    wg = GridSpec((4, 4, 4), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    wv = Volume(wg, np.random.default_rng(0).uniform(size=(4, 4, 4)).astype(np.float32))
    wf = init_from_volume(wv, InitConfig(background_threshold=0.0))
    one(wf, AdamState.create(wf), FitConfig().resolved_lrs(wg.spacing), wv)
    f = init_from_volume(lr, InitConfig(background_threshold=0.0))
    st = AdamState.create(f)
    lrs = FitConfig().resolved_lrs(grid.spacing)
    for _ in range(warmup):
        one(f, st, lrs, lr)
    t0 = time.perf_counter()
    for _ in range(steps):
        one(f, st, lrs, lr)
    sec = (time.perf_counter() - t0) / steps
    return sec / frac, {"sample_dims": list(dims), "sample_N": int(f.count),
                        "fraction": frac, "sample_s_per_step": sec,
                        "numba_threads": int(gsvol.worker_count()),
                        "cpu": _cpu_model()}


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_available() -> str | None:
    """None if the real reference imports from baseline/_ref, else why not."""
    if not os.path.isdir(os.path.join(REF_DIR, "gsvol")):
        return "baseline/_ref/gsvol not installed"
    try:
        import numba  # noqa: F401
        import scipy  # noqa: F401
    except ImportError as e:
        return f"reference dependency missing: {e}"
    return None


def cpu_baseline_entry(p, cfg_id: int, steps: int, warmup: int) -> dict:
    """The reference's CPU path on this host: the real gsvol when it is
    installed (kind "reference"), else the oracle port (kind "port")."""
    cores = host_threads()
    why = reference_available()
    if why is None:
        sec, info = gsvol_train_step_seconds(p, cfg_id, steps, warmup, cores)
        d, n = info["sample_dims"], info["sample_N"]
        return {"value": 1.0 / sec, "unit": "it/s", "cores": cores, "kind": "reference",
                "sample": f"{steps} fit() iterations of the unmodified reference (gsvol from "
                          f"baseline/_ref, numba {info['numba_threads']} threads) on the "
                          f"central {d[0]}x{d[1]}x{d[2]} LR z-slab of config {cfg_id} "
                          f"(N={n}, {info['fraction']:.4g} of the workload), scaled by "
                          "1/fraction",
                "detail": info}
    sec = cpu_train_step_seconds(p, steps, warmup)
    return {"value": 1.0 / sec, "unit": "it/s", "cores": cores, "kind": "port",
            "sample": f"{steps} full config-{cfg_id} train iterations (oracle/: numpy binning "
                      f"+ OpenMP C loops, all cores); real reference unavailable: {why}"}


def run_reference(args, dist, rank):
    if rank != 0:
        return
    p = problem_for(args.config)
    cpu = cpu_baseline_entry(p, args.config, args.steps, args.warmup)
    v = cpu["value"]
    cfg = _config_dict(args, p, int(os.environ.get("WORLD_SIZE", "1")))
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "it/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 / v, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "cpu_baseline": cpu,
            "e2e": {"value": v, "unit": "it/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config_dict(args, p, ws):
    return {"workload": f"config {args.config}: fit step on {p['lr_grid'].dims} LR "
                        f"(x2 -> {p['hr_grid'].dims} HR), N={p['field'][0].shape[0]} Gaussians",
            "lr_dims": list(p["lr_grid"].dims), "hr_dims": list(p["hr_grid"].dims),
            "N": int(p["field"][0].shape[0]), "brick_dims": [8, 8, 4],
            "loss": "l1", "optimizer": "Adam (f64 master)",
            "parallelism": f"brick-range slabs x{ws} (pair-balanced)" + (
                "" if ws == 1 else f", {args.shard} exchange"),
            "l2": "inputs larger than L2 (f64 field + Adam moments = 0.7 GB, pairs 0.1 GB)"}


# ----------------------------------------------------------------- GPU arm
def run_ours(args, dist, ws, rank, local):
    import torch
    import paper_2603_09621_b200 as gs
    from paper_2603_09621_b200 import _lib
    from paper_2603_09621_b200.train import PhaseTimer

    dev = torch.device("cuda", local)
    lib = _lib.lib()
    p = problem_for(args.config, dev)
    lr_grid, hr_grid = p["lr_grid"], p["hr_grid"]
    lr = gs.Volume(lr_grid, p["lr"])
    opts = gs.RenderOptions()
    bd = (8, 8, 4)
    group = dist.group.WORLD if dist else None

    f = gs.GaussianField(*p["field"], device=dev)
    # slabs: contiguous brick-id ranges balanced by the pair count per brick
    # (one whole-grid binning pass at setup, identical on every rank)
    my_slab = slab_for_rank(lr_grid, bd, rank, ws, pair_weights(f, lr_grid, opts, bd)) \
        if ws > 1 else None
    my_hr_slab = slab_for_rank(hr_grid, bd, rank, ws, pair_weights(f, hr_grid, opts, bd)) \
        if ws > 1 else None
    state = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(lr_grid.spacing)
    timer = PhaseTimer()
    step = gs.TrainStep(lr, opts, bd, "l1", slab=my_slab, process_group=group, world_size=ws,
                        timer=timer)

    def eager_iter():
        out = step.forward(f)
        step.update(f, out, state, lrs)   # backward + fused merge/chain/Adam/renorm
        return out

    def run_fit_steps(k, launch):
        """k iterations of fit()'s loop body as fit() runs them: each step is a
        graph replay (or the eager sharded step) whose 16-byte loss read is
        taken after the next step is queued (optimize.py:177-197)."""
        losses = []
        h = launch()
        for i in range(k):
            nxt = launch() if i + 1 < k else None
            losses.append(h.loss())
            h = nxt
        return losses

    def train_launch():
        return step.step_async(f, state, lrs)

    set_target = step.set_target
    halo = None
    if ws > 1 and args.shard == "halo":
        # owner-computes + halo exchange: each rank steps its compact local
        # field; the replicated `f` stays at its initial values (it serves the
        # renders and the roofline census below)
        from paper_2603_09621_b200.distributed import brick_count, slab_ranges
        from paper_2603_09621_b200.halo import HaloTrainStep
        slabs = slab_ranges(brick_count(lr_grid, bd), ws,
                            weights=pair_weights(f, lr_grid, opts, bd))
        halo = HaloTrainStep(lr, slabs, rank, group, opts, bd, "l1")
        halo.attach(f, gs.AdamState.create(f))

        class _Done:
            def __init__(self, v):
                self.v = v

            def loss(self):
                return self.v

        def train_launch():                      # noqa: F811 -- the halo step
            return halo.step_async(lrs)          # a graph replay over NCCL

        def eager_iter():                        # noqa: F811
            halo.step(lrs)
            return None

        set_target = halo.inner.set_target

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    sampler = ClockSampler(local)
    sampler.start()
    # ---------------- per-phase breakdown (eager kernels, events per phase)
    for _ in range(args.warmup):
        out = eager_iter()
    barrier()
    timer.reset()
    for _ in range(max(3, min(args.steps, 10))):
        out = eager_iter()
    barrier()
    phases = timer.summary()
    if halo is not None:
        out = step.forward(f)                    # the slab index for the census below
        phases = {"halo_step": (0, float("nan"))}
    pairs = out.idx.pair_count
    step.timer = None
    # ---------------- train: warmup, then exactly K timed steps
    run_fit_steps(args.warmup, train_launch)
    barrier()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    timed_caps0 = getattr(step, "graph_captures", 0)
    e0.record(s)
    losses = run_fit_steps(args.steps, train_launch)
    e1.record(s)
    barrier()
    timed_captures = getattr(step, "graph_captures", 0) - timed_caps0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    assert all(math.isfinite(x) for x in losses), "non-finite loss in timed steps"

    # ---------------- e2e: fit()'s loop with host buffers (pinned H2D target, loss D2H),
    # right after the device-timed steps (before the renders allocate their buffers)
    e2e = None
    if not args.no_e2e:
        host_t = torch.from_numpy(np.ascontiguousarray(p["lr"].ravel(order="F"))).pin_memory()
        if halo is None:
            # the step's input is the pinned host target: every step copies it
            # H2D itself, inside the replayed graph on a branch that overlaps
            # binning (TrainStep.set_target_source)
            step.set_target_source(host_t)

            def e2e_launch():
                return step.step_async(f, state, lrs)
            h2d_note = ("pinned host target copied H2D by every step inside the replayed graph, "
                        "on a branch overlapping binning (TrainStep.set_target_source)")
            api = ("TrainStep.set_target_source + TrainStep.step_async/StepHandle.loss "
                   "(fit()'s loop body: CUDA-graph replay + 16-byte loss read, one step "
                   "queued ahead)")
        else:
            def e2e_launch():
                set_target(host_t)                 # pinned H2D, stream-ordered
                return train_launch()
            h2d_note = "pinned host target copied H2D (stream-ordered) before each halo step"
            api = "HaloTrainStep.step (eager, per rank) with TrainStep.set_target"
        run_fit_steps(min(args.warmup, 3), e2e_launch)
        barrier()
        # wall clock: at least 300 steps (~0.6 s) so host jitter averages out
        k_e2e = max(args.steps, 300)
        caps0 = getattr(step, "graph_captures", 0)
        t0 = time.perf_counter()
        loss = run_fit_steps(k_e2e, e2e_launch)[-1]   # loss device -> host each step
        barrier()
        sec = max_over_ranks((time.perf_counter() - t0) / k_e2e)
        if halo is None:
            step.set_target_source(None)
        e2e = {"value": 1.0 / sec, "unit": "it/s", "steps": k_e2e,
               "graph_captures": getattr(step, "graph_captures", 0) - caps0,
               "h2d_bytes_per_step": host_t.numel() * host_t.element_size(),
               "d2h_bytes_per_step": 16, "api": api, "h2d": h2d_note, "last_loss": loss}

    # ---------------- render at the 256^3 HR grid (bin + forward)
    hr_renderer = gs.Renderer(hr_grid, opts, bd, slab=my_hr_slab, device=dev)

    def render_iter(grid, slab):
        return hr_renderer(f)

    kr = max(1, min(args.steps, 10))
    for _ in range(min(args.warmup, 3)):
        render_iter(hr_grid, my_hr_slab)
    barrier()
    e0.record(s)
    for _ in range(kr):
        render_iter(hr_grid, my_hr_slab)
    e1.record(s)
    barrier()
    ms_r = max_over_ranks(e0.elapsed_time(e1) / kr)
    render = {"grid": list(hr_grid.dims), "value": hr_grid.num_voxels / (ms_r * 1e-3) / 1e9,
              "unit": "Gvoxel/s", "ms_per_render": ms_r, "renders": kr,
              "pairs": hr_renderer.pair_count() if ws == 1 else None,
              "path": "Renderer: one CUDA-graph replay per render (preprocess, scan, capacity "
              "binning, forward) + the 4-byte overflow-flag read"}

    render512 = None
    if not args.no_render512:
        from paper_2603_09621_b200 import synth
        arr5 = synth.jitter_field([np.asarray(a) for a in p["field"]], lr_grid)
        f5 = gs.GaussianField(*arr5, device=dev)
        g5 = gs.grid_covering_extent(lr_grid, (512, 512, 512))
        slab5 = slab_for_rank(g5, bd, rank, ws, pair_weights(f5, g5, opts, bd)) \
            if ws > 1 else None

        r5_renderer = gs.Renderer(g5, opts, bd, slab=slab5, device=dev)

        def r5():
            return r5_renderer(f5)
        r5()
        barrier()
        k5 = max(1, min(args.steps, 5))
        e0.record(s)
        for _ in range(k5):
            r5()
        e1.record(s)
        barrier()
        ms5 = max_over_ranks(e0.elapsed_time(e1) / k5)
        render512 = {"grid": [512, 512, 512], "value": g5.num_voxels / (ms5 * 1e-3) / 1e9,
                     "unit": "Gvoxel/s", "ms_per_render": ms5, "renders": k5,
                     "pairs": r5_renderer.pair_count() if ws == 1 else None,
                     "field": "config-5 jittered"}
        del f5, r5_renderer
    # ---------------- the other BASELINE configs (N = 1): config 2 as a
    # fixed-iteration fit() through the public API, config 4 as train steps
    # plus its HR render (BASELINE.json configs[1] and [3])
    other = None
    if ws == 1 and not args.no_configs:
        other = {"2": config2_fit(gs, dev, 200), "4": config4_step_render(gs, dev, args)}
    clocks = sampler.stop()

    # ---------------- roofline of the dominant pair kernel (live pair-voxels)
    cnt = torch.zeros(4, dtype=torch.int64, device=dev)
    out_idx = out.idx
    _lib.check(lib.gsv_diag_count_live(
        f.positions.data_ptr(), out_idx._aux.rec32.data_ptr(), f.log_scales.data_ptr(),
        f.rotations.data_ptr(), out_idx.starts.data_ptr(), out_idx.gids.data_ptr(),
        _lib.make_grid(lr_grid), _lib.make_bricks(lr_grid, bd, my_slab), 3.0, cnt.data_ptr(),
        _lib.stream_ptr()), "count_live")
    e_live, e_brick, e_tile, e_group = (int(x) for x in cnt.tolist())
    # the slots the train step's forward kernel evaluates: the grouped-column
    # kernel at LR densities (raster._use_grouped), else the whole-brick tiles
    from paper_2603_09621_b200.raster import _use_grouped
    grouped = _use_grouped(bd, pairs, f.count)
    e_eval = e_group if grouped else e_tile
    peak = fp32_peak(lib, dev)
    t_fwd = phases.get("forward", (0, float("nan")))[1]
    t_bwd = phases.get("backward", (0, float("nan")))[1]
    dom, t_dom, fl = ("backward", t_bwd, BWD_FLOP) if t_bwd >= t_fwd else ("forward", t_fwd, FWD_FLOP)
    t_upd = phases.get("update", (0, float("nan")))[1]
    achieved = e_live * fl / (t_dom * 1e-3) / 1e12
    n_g = f.count
    # algorithmic bytes of the train-step kernels: forward reads rec32 + mu
    # (88 B/Gaussian), gids (4 B/pair), target (4 B/voxel) and writes S, W, I,
    # {alpha, I} (20 B/voxel) and the live masks (32 B/pair); the masked
    # backward reads rec32 + mu + box + gstart (112 B/Gaussian), gids + masks
    # (36 B/pair), {alpha, I} (8 B/voxel) and writes the partials (48 B/pair)
    nv_lr = lr_grid.num_voxels
    bytes_alg = {"forward": 88 * n_g + 36 * pairs + 24 * nv_lr,
                 "backward": 112 * n_g + 84 * pairs + 8 * nv_lr}[dom]
    traffic = None
    issue = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        with open(tf) as fh:
            tj = json.load(fh)
        # measured for this workload at N=1 only (a rank of N>1 renders a slab)
        if tj.get("config") == args.config and ws == 1:
            traffic = tj.get(dom)
            issue = tj.get(dom + "_issue_active_pct")
    hbm_peak = 6552.0  # MEASURED_PEAKS.json (driver-written) when present
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        with open(mp) as fh:
            hbm_peak = float(json.load(fh).get("hbm_gbs", hbm_peak))
    roofline = {"bound": "fp32", "kernel": dom, "achieved": achieved, "peak": peak["tflops"],
                "unit": "TFLOP/s", "frac": achieved / peak["tflops"], "traffic": traffic,
                "peak_source": peak["source"],
                "evaluated": {
                    "kernel": "forward32c_kernel (grouped columns)" if grouped
                    else "forward32w_kernel (two-list whole brick)",
                    "E_evaluated": e_eval if dom == "forward" else None,
                    "E_tile_whole_brick": e_tile, "E_group": e_group if grouped else None,
                    "live_fraction": (e_live / e_eval) if (dom == "forward" and e_eval) else None,
                    "issue_active_pct": issue,
                    # the same 28 FLOP counted per evaluated slot: what the kernel
                    # sustains; frac above is that times the live fraction
                    "achieved_evaluated": (e_eval * fl / (t_dom * 1e-3) / 1e12)
                    if (dom == "forward" and e_eval) else None,
                    "frac_evaluated": (e_eval * fl / (t_dom * 1e-3) / 1e12 / peak["tflops"])
                    if (dom == "forward" and e_eval) else None,
                    "note": "E_evaluated counts the (pair, voxel) slots the forward kernel "
                            "issues, idle lanes included: 128 per chunk iteration of the "
                            "grouped kernel (E_group), or 128 per warp-tile hit of the "
                            "whole-brick kernel (E_tile_whole_brick, for comparison); frac "
                            "counts live pair-voxels only (SURVEY 8d's unit), frac_evaluated "
                            "every evaluated slot; issue_active_pct is the kernel's "
                            "issue-slot use from the ncu capture in profiles/"},
                "work": {"E_live": e_live, "E_brick": e_brick,
                "flop_per_live_pair_voxel": fl, "ms_per_launch": t_dom},
                "hbm": {"algorithmic_bytes": bytes_alg,
                        "achieved_gbs": bytes_alg / (t_dom * 1e-3) / 1e9, "peak_gbs": hbm_peak,
                        "frac": bytes_alg / (t_dom * 1e-3) / 1e9 / hbm_peak}}

    # ---------------- kernel launches per step (CUPTI, outside the timed region)
    launches = -1 if args.no_count else count_launches(lambda: step.step(f, state, lrs))

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline_entry(p, args.config, 2, 1)

    if rank == 0:
        line = {"metric": METRIC, "value": 1000.0 / ms, "unit": "it/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic", "config": _config_dict(args, p, ws),
                "pairs_lr": pairs,
                "render": render, "render512": render512, "configs": other,
                "phases_ms": {k: v[1] for k, v in phases.items()},
                "phases_note": ("eager forward()+update() with CUDA events per phase: binning "
                                "from scratch every step; the timed graph step edits last "
                                "step's lists instead (incremental binning, ~40 us)"),
                "e2e": e2e, "roofline": roofline, "cpu_baseline": cpu, "clocks": clocks,
                "gpu_launches": launches * args.steps, "gpu_launches_per_step": launches,
                "graph_captures_timed": timed_captures, "loss_last": losses[-1]}
        print(json.dumps(line), flush=True)


def config2_fit(gs, dev, iterations: int) -> dict:
    """Config 2 (128x128x64 LR -> x2, N = 1,048,576): one whole fit() of
    `iterations` iterations through the public API (init, graph capture,
    every iteration's loss read), wall clock."""
    import torch
    p = problem_for(2, dev)
    lr = gs.Volume(p["lr_grid"], p["lr"])
    gs.fit(lr, gs.InitConfig(background_threshold=0.0), gs.FitConfig(iterations=3))  # warm-up
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    f, rep = gs.fit(lr, gs.InitConfig(background_threshold=0.0),
                    gs.FitConfig(iterations=iterations))
    torch.cuda.synchronize(dev)
    sec = time.perf_counter() - t0
    return {"workload": "config 2: fit() on 128x128x64 LR (x2 -> 256x256x128), "
                        f"N={f.count}, {iterations} iterations, init and final render included",
            "value": iterations / sec, "unit": "it/s", "seconds": sec,
            "final_loss": rep.final["loss"], "timing": "wall clock around fit()"}


def config4_step_render(gs, dev, args) -> dict:
    """Config 4 (256x256x40 LR, spacing (1,1,4), x4 through-plane -> 256x256x160,
    N = 2,621,440): graph-replayed train steps (CUDA events) and the HR render
    (Renderer graph replays)."""
    import torch
    p = problem_for(4, dev)
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"], device=dev)
    st = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(lr.grid.spacing)
    step = gs.TrainStep(lr, gs.RenderOptions(), (8, 8, 4), "l1")
    for _ in range(args.warmup):
        step.step(f, st, lrs)
    torch.cuda.synchronize(dev)
    s = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    h = step.step_async(f, st, lrs)
    for i in range(args.steps):
        nxt = step.step_async(f, st, lrs) if i + 1 < args.steps else None
        h.loss()
        h = nxt
    e1.record(s)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / args.steps
    r = gs.Renderer(p["hr_grid"], gs.RenderOptions(), (8, 8, 4), device=dev)
    for _ in range(3):
        r(f)
    kr = max(1, min(args.steps, 10))
    torch.cuda.synchronize(dev)
    e0.record(s)
    for _ in range(kr):
        r(f)
    e1.record(s)
    torch.cuda.synchronize(dev)
    ms_r = e0.elapsed_time(e1) / kr
    nv = p["hr_grid"].num_voxels
    return {"workload": "config 4: fit step on 256x256x40 LR (spacing 1,1,4), "
                        f"N={f.count}; render at 256x256x160",
            "train": {"value": 1000.0 / ms, "unit": "it/s", "ms_per_step": ms,
                      "steps": args.steps},
            "render": {"value": nv / (ms_r * 1e-3) / 1e9, "unit": "Gvoxel/s",
                       "ms_per_render": ms_r, "renders": kr,
                       "pairs": r.pair_count()}}


def fp32_peak(lib, dev) -> dict:
    """Measured FP32 FMA throughput of this GPU (our probe kernel)."""
    import torch
    from paper_2603_09621_b200 import _lib
    sms = lib.gsv_device_sm_count()
    blocks, iters = sms * 8, 4096
    sink = torch.zeros(1, dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream()
    for _ in range(2):
        _lib.check(lib.gsv_diag_fma_probe(blocks, iters, sink.data_ptr(), _lib.stream_ptr()),
                   "fma_probe")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(5):
        lib.gsv_diag_fma_probe(blocks, iters, sink.data_ptr(), _lib.stream_ptr())
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    tflops = blocks * 256 * iters * 16 * 2 / (ms * 1e-3) / 1e12
    return {"tflops": tflops, "source": f"measured FFMA probe ({blocks} CTAs x 256 thr)"}


def count_launches(fn) -> int:
    """Kernel launches of one step, counted by the CUDA profiler (CUPTI)."""
    import torch
    try:
        from torch.profiler import ProfilerActivity, profile
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        n = 0
        for e in prof.events():
            if e.device_type.name == "CUDA" and ("gsv" in e.name or "cub" in e.name.lower()):
                n += 1
        return n
    except Exception:
        return -1


def main():
    args = parse()
    if args.impl == "reference":
        # the CPU reference arm needs no process group: rank 0 runs, the
        # other ranks exit 0 without work
        run_reference(args, None, int(os.environ.get("RANK", "0")))
        return
    dist, ws, rank, local = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference(args, dist, rank)
        else:
            run_ours(args, dist, ws, rank, local)
    finally:
        if dist:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
