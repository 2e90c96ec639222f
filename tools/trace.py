"""Kernel timeline of the train step (development tool, not the bench contract).

python tools/trace.py [--config 3] [--steps 5]
Runs the fit loop body (TrainStep.forward + update) under the torch profiler
(CUPTI activity tracing, no replay) and prints, per kernel, launches and mean
duration per step, plus the GPU-idle time per step (host syncs, launch gaps).
"""

from __future__ import annotations

import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2603_09621_b200 as gs  # noqa: E402
from paper_2603_09621_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--hr", action="store_true", help="trace the HR render instead")
    ap.add_argument("--grid512", action="store_true", help="HR render at config 5's 512^3")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    p = synth.make_problem(synth.CONFIGS[args.config])
    f = gs.GaussianField(*p["field"])
    if args.grid512:
        # bench.py's config-5 render: the jittered trained-size field at 512^3
        import numpy as np
        f = gs.GaussianField(*synth.jitter_field([np.asarray(a) for a in p["field"]],
                                                 p["lr_grid"]))
        rend = gs.Renderer(gs.grid_covering_extent(p["lr_grid"], (512, 512, 512)),
                           gs.RenderOptions(), (8, 8, 4))
        run = lambda: rend(f)  # noqa: E731
    elif args.hr:
        rend = gs.Renderer(p["render_grid"], gs.RenderOptions(), (8, 8, 4))
        run = lambda: rend(f)  # noqa: E731
    else:
        step = gs.TrainStep(gs.Volume(p["lr_grid"], p["lr"]), gs.RenderOptions(), (8, 8, 4),
                            "l1")
        state = gs.AdamState.create(f)
        lrs = gs.FitConfig().resolved_lrs(p["lr_grid"].spacing)
        run = lambda: step.step(f, state, lrs)  # noqa: E731
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            run()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    per = collections.defaultdict(lambda: [0, 0.0])
    busy = 0.0
    for e in evs:
        d = e.time_range.elapsed_us()
        name = e.name if len(e.name) < 70 else e.name[:67] + "..."
        per[name][0] += 1
        per[name][1] += d
        busy += d
    span = evs[-1].time_range.end - evs[0].time_range.start
    k = args.steps
    print(f"steps {k}: span {span / k:.1f} us/step, busy {busy / k:.1f} us/step, "
          f"idle {(span - busy) / k:.1f} us/step")
    for name, (n, t) in sorted(per.items(), key=lambda x: -x[1][1]):
        print(f"{t / k:9.1f} us  x{n / k:4.1f}  {name}")
    gaps = collections.defaultdict(float)
    for a, b in zip(evs, evs[1:]):
        g = b.time_range.start - a.time_range.end
        if g > 1.0:
            gaps[(a.name[:40], b.name[:40])] += g
    print("idle gaps (us/step), preceding -> following:")
    for (a, b), g in sorted(gaps.items(), key=lambda x: -x[1])[:12]:
        print(f"{g / k:9.1f}  {a}  ->  {b}")


if __name__ == "__main__":
    main()
