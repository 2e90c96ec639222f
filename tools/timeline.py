"""Kernel timeline of the graph-replayed train step (development tool).

python tools/timeline.py [--config 3] [--steps 5] [--out gpurun_out/timeline.json]

Replays TrainStep.step under torch.profiler (CUPTI activity tracing, which
records the kernels of replayed CUDA graphs with device timestamps), then per
step: the kernels in launch order with their durations, the busy time (sum
of kernel durations), the span (first start to last end) and the idle gaps
between consecutive kernels.  Warm caches, real clocks -- unlike an ncu
launch list, which serialises and flushes.
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


def short(name: str) -> str:
    for pre in ("void ", "gsv::", "(anonymous namespace)::", "<unnamed>::"):
        name = name.replace(pre, "")
    return name.split("(")[0][:60]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--skip", type=int, default=5, help="fit steps before the profiled ones")
    ap.add_argument("--render", action="store_true",
                    help="profile Renderer replays at the config's render grid instead")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    p = synth.make_problem(synth.CONFIGS[args.config])
    f = gs.GaussianField(*p["field"])
    if args.render:
        return render_timeline(f, p["render_grid"], args.steps)
    step = gs.TrainStep(gs.Volume(p["lr_grid"], p["lr"]), gs.RenderOptions(), (8, 8, 4), "l1")
    state = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(p["lr_grid"].spacing)
    for _ in range(args.skip):
        step.step(f, state, lrs)
    torch.cuda.synchronize()
    marks = []
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        # fit()'s loop: the next step is queued before this step's loss is read
        h = step.step_async(f, state, lrs)
        for i in range(args.steps):
            nxt = step.step_async(f, state, lrs) if i + 1 < args.steps else None
            h.loss()
            h = nxt
        torch.cuda.synchronize()
    kernels = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    rows = []
    for e in kernels:
        tr = e.time_range
        rows.append((tr.start, tr.end, e.name))
    rows.sort()
    # split into steps after each update tail (tail_tma_kernel / tail_kernel)
    steps, cur = [], []
    for r in rows:
        if cur and short(cur[-1][2]).startswith("tail"):
            steps.append(cur)
            cur = []
        cur.append(r)
    if cur:
        steps.append(cur)
    report = []
    for i, s in enumerate(steps):
        busy = sum(b - a for a, b, _ in s)
        span = s[-1][1] - s[0][0]
        gaps = [(s[j + 1][0] - s[j][1], short(s[j][2]), short(s[j + 1][2]))
                for j in range(len(s) - 1)]
        report.append({"step": i, "kernels": len(s), "busy_us": busy, "span_us": span,
                       "idle_us": span - busy,
                       "list": [(short(n), round(b - a, 2)) for a, b, n in s],
                       "gaps": [(round(g, 2), x, y) for g, x, y in gaps]})
        print(f"step {i}: {len(s)} kernels, busy {busy:.1f} us, span {span:.1f} us, "
              f"idle {span - busy:.1f} us")
    if report:
        mid = report[len(report) // 2]
        print("kernel list (middle step):")
        for (n, d), g in zip(mid["list"], [g[0] for g in mid["gaps"]] + [0.0]):
            print(f"  {d:9.2f} us  {n}   (gap after {g:.2f} us)")
    if args.out:
        with open(args.out, "w") as fh:
            json.dump({"steps": report, "raw": [(a, b, short(n)) for a, b, n in rows]}, fh,
                      indent=0)


def render_timeline(f, grid, reps):
    from torch.profiler import ProfilerActivity, profile
    r = gs.Renderer(grid)
    for _ in range(3):
        r(f)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            r(f)
        torch.cuda.synchronize()
    rows = sorted((e.time_range.start, e.time_range.end, e.name) for e in prof.events()
                  if e.device_type == torch.autograd.DeviceType.CUDA)
    tot = {}
    for a, b, n in rows:
        k = short(n)
        tot[k] = tot.get(k, 0.0) + (b - a)
    span = (rows[-1][1] - rows[0][0]) / reps
    print(f"render {grid.dims}: {reps} replays, span per render {span:.1f} us")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"  {v / reps:9.2f} us  {k}")


if __name__ == "__main__":
    main()
