"""Per-rank cost of the sharded train step at k ranks, measured on one GPU.

python tools/scale_model.py [--config 3] [--ranks 2 4 8]
For each k: the pair-balanced brick-id slabs, the owner-computes / halo plan
(halo.py) and, for the busiest middle rank, its local field; then CUDA-event
times of that rank's compute -- bin + forward (fused loss) + masked backward
+ per-Gaussian merge, and the fused chain rule / Adam / renorm tail on its
local rows -- next to the halo rows it exchanges.  The all_reduce design's
per-rank cost is measured the same way (slab work on the full field, the full
tail, the preprocess of all N) with its (N, 12) f32 all_reduce.  Collectives
are not run (one GPU); their time is modelled from bytes at the NVLink
all-to-all / all-reduce bandwidths of B200_PROFILING.md.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2603_09621_b200 as gs  # noqa: E402
from paper_2603_09621_b200 import synth  # noqa: E402
from paper_2603_09621_b200.distributed import brick_count, pair_weights, slab_ranges  # noqa: E402
from paper_2603_09621_b200.field import PARAM_NAMES  # noqa: E402
from paper_2603_09621_b200.halo import HaloPlan, reach_and_owner  # noqa: E402
from paper_2603_09621_b200.raster import _pair_partials  # noqa: E402
from paper_2603_09621_b200.train import _adam_launch  # noqa: E402

NVLINK_A2A_GBS = 700.0      # per-GPU all-to-all, 8x B200 over NVSwitch (modelled)
NVLINK_AR_GBS = 725.0       # 8-rank all_reduce bus bandwidth (B200_PROFILING.md figure)
COLL_LAT_US = 25.0          # per collective launch + sync (modelled)


def _events():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def time_rank(lr, f_local, slab, reps=5):
    """Device ms of one rank's step compute on its (local) field and slab."""
    st = gs.AdamState.create(f_local)
    lrs = gs.FitConfig().resolved_lrs(lr.grid.spacing)
    ts = gs.TrainStep(lr, gs.RenderOptions(), (8, 8, 4), "l1", slab=slab)
    opts = gs.RenderOptions()
    res = {"slab": [], "tail": []}
    for i in range(reps + 2):
        a, b = _events()
        c, d = _events()
        a.record()
        out = ts.forward(f_local)
        aux = out.idx._aux
        gsum = _pair_partials(f_local, lr.grid, out.idx, opts, aux.rec32, aux.rec64, out.ab,
                              aux.gstart, aux.box, True, pool=ts.pool, live_masks=ts._masks,
                              mask_vpl=ts._mask_vpl)
        b.record()
        c.record()
        _adam_launch(f_local, st, lrs, 0.9, 0.999, 1e-8, None, None, gsum, 0, ts.pool)
        d.record()
        torch.cuda.synchronize()
        if i >= 2:
            res["slab"].append(a.elapsed_time(b))
            res["tail"].append(c.elapsed_time(d))
    out = {k: sum(v) / len(v) for k, v in res.items()}
    # the same rank work as one CUDA-graph replay (bin + forward + masked
    # backward + merge/chain/Adam tail over the local rows): the per-rank
    # compute floor without host launch overhead
    g = gs.TrainStep(lr, opts, (8, 8, 4), "l1", slab=slab)
    fg = f_local.copy()
    sg = gs.AdamState.create(fg)
    for _ in range(3):
        g.step(fg, sg, lrs)
    a, b = _events()
    torch.cuda.synchronize()
    a.record()
    h = g.step_async(fg, sg, lrs)
    for i in range(10):
        nxt = g.step_async(fg, sg, lrs) if i + 1 < 10 else None
        h.loss()
        h = nxt
    b.record()
    torch.cuda.synchronize()
    out["graph_step"] = a.elapsed_time(b) / 10
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--margin", type=float, default=1.0)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    p = synth.make_problem(synth.CONFIGS[args.config])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    n = f.count
    w = pair_weights(f, lr.grid)
    out = {"config": args.config, "N": n, "ranks": {}}
    for k in args.ranks:
        slabs = slab_ranges(brick_count(lr.grid, (8, 8, 4)), k, weights=w)
        r = k // 2                                      # a middle rank: halo on both sides
        own, lo, hi = reach_and_owner(f.positions, f.log_scales, f.rotations, lr.grid,
                                      (8, 8, 4), slabs, 3.0, args.margin)
        plan = HaloPlan(own, lo, hi, r, k)
        g = plan.local_gids
        fl = gs.GaussianField(*[getattr(f, nm)[g] for nm in PARAM_NAMES])
        halo_t = time_rank(lr, fl, slabs[r] if k > 1 else None)
        to_owner, from_peer = plan.halo_counts()
        rows_out = sum(to_owner) + sum(from_peer)        # partials out + params out
        a2a_bytes = 2 * rows_out * 96                   # each direction, f64 rows of 12
        a2a_ms = (a2a_bytes / (NVLINK_A2A_GBS * 1e9)) * 1e3 + 3 * COLL_LAT_US * 1e-3
        # the all_reduce design: slab work on the full field + full tail + all N preprocess
        full_t = time_rank(lr, gs.GaussianField(*[getattr(f, nm) for nm in PARAM_NAMES]),
                           slabs[r] if k > 1 else None)
        ar_bytes = n * 12 * 4
        ar_ms = (2 * (k - 1) / k * ar_bytes / (NVLINK_AR_GBS * 1e9)) * 1e3 + COLL_LAT_US * 1e-3 \
            if k > 1 else 0.0
        out["ranks"][k] = {
            "slabs": len(slabs), "rank": r, "n_local": plan.n_local,
            "owned": int(plan.owned.sum()), "halo_rows_out": rows_out,
            "halo": {"eager_compute_ms": halo_t["slab"] + halo_t["tail"], **halo_t,
                     "a2a_ms_model": a2a_ms,
                     "step_ms_model": halo_t["graph_step"] + a2a_ms},
            "allreduce": {"eager_compute_ms": full_t["slab"] + full_t["tail"], **full_t,
                          "allreduce_ms_model": ar_ms,
                          "step_ms_model": full_t["graph_step"] + ar_ms}}
        print(k, json.dumps(out["ranks"][k]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
