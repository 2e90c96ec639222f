"""Where does the end-to-end step lose time against the device-timed step?
(development tool)

python tools/e2e_probe.py [--config 3] [--steps 100]
Wall-clocks fit()'s pipelined loop (step_async, one step queued ahead, loss
read per step) with: nothing else; set_target from a device tensor each
step; a pinned-H2D prefetch on a copy stream + set_target; the bench's
set_target_source (the H2D inside each replayed graph).
"""

from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_09621_b200 as gs  # noqa: E402
from paper_2603_09621_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--steps", type=int, default=100)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    p = synth.make_problem(synth.CONFIGS[args.config])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    state = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(p["lr_grid"].spacing)
    step = gs.TrainStep(lr, gs.RenderOptions(), (8, 8, 4), "l1")
    host_t = torch.from_numpy(np.ascontiguousarray(p["lr"].ravel(order="F"))).pin_memory()
    dev_t = host_t.to(dev)
    staging = torch.empty_like(dev_t)
    copy_s = torch.cuda.Stream(device=dev)
    ready, freed = torch.cuda.Event(), torch.cuda.Event()
    cur = torch.cuda.current_stream(dev)

    def plain():
        return step.step_async(f, state, lrs)

    def with_target():
        step.set_target(dev_t)
        return step.step_async(f, state, lrs)

    def prefetch():
        copy_s.wait_event(freed)
        with torch.cuda.stream(copy_s):
            staging.copy_(host_t, non_blocking=True)
            ready.record(copy_s)

    def with_h2d():
        cur.wait_event(ready)
        step.set_target(staging)
        freed.record(cur)
        prefetch()
        return step.step_async(f, state, lrs)

    def loop(k, launch):
        h = launch()
        for i in range(k):
            nxt = launch() if i + 1 < k else None
            h.loss()
            h = nxt

    freed.record(cur)
    prefetch()
    def source():
        return step.step_async(f, state, lrs)

    for name, fn in (("plain", plain), ("set_target", with_target), ("h2d", with_h2d),
                     ("source", source), ("plain", plain)):
        step.set_target_source(host_t if name == "source" else None)
        loop(5, fn)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        loop(args.steps, fn)
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / args.steps * 1e3
        devt = e0.elapsed_time(e1) / args.steps
        print(f"{name:11s} wall {wall:.4f} ms/step ({1e3 / wall:.1f} it/s)  "
              f"device {devt:.4f} ms/step")


if __name__ == "__main__":
    main()
