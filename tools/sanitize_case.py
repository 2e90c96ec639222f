"""Small end-to-end case for compute-sanitizer (memcheck / racecheck / synccheck).

python tools/sanitize_case.py
Runs every hot-path kernel once or twice at config 1 (32^3 LR, 64^3 HR):
binning, the whole-brick forward with fused loss and live masks, the masked
backward, the TMA optimizer tail (eager and inside the graph-replayed step),
the public span backward, the f64 engine, a Renderer graph and the metrics.
Exits 0 and prints one line when every result is finite.
"""

from __future__ import annotations

import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_09621_b200 as gs  # noqa: E402
from paper_2603_09621_b200.synth import CONFIGS, make_problem  # noqa: E402


def main():
    torch.cuda.set_device(0)
    p = make_problem(CONFIGS[1])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    st = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(lr.grid.spacing)
    # eager train step: forward (fused loss, live masks) + masked backward + TMA tail
    step = gs.TrainStep(lr, gs.RenderOptions(), (8, 8, 4), "l1")
    out = step.forward(f)
    loss0 = out.loss()
    step.update(f, out, st, lrs)
    # graph-replayed steps (fit()'s path), one queued ahead
    h = step.step_async(f, st, lrs)
    h2 = step.step_async(f, st, lrs)
    losses = [h.loss(), h2.loss()]
    # public API: index, forward, span backward, f64 engine
    idx = gs.build_brick_index(f, lr.grid)
    c = gs.forward(f, lr.grid, idx)
    _, dl = gs.loss_and_grad(c.volume(), lr, "l1")
    g = gs.backward(f, lr.grid, idx, c, dl)
    o64 = gs.RenderOptions(precision="f64")
    i64 = gs.build_brick_index(f, lr.grid, o64)
    c64 = gs.forward(f, lr.grid, i64, o64)
    g64 = gs.backward(f, lr.grid, i64, c64, dl, o64)
    # render graph at the HR grid, metrics
    r = gs.Renderer(p["hr_grid"])
    sr = r(f)
    hr = gs.Volume(p["hr_grid"], p["hr"])
    ps, ss = gs.psnr(sr.volume(), hr), gs.ssim3d(sr.volume(), hr)
    torch.cuda.synchronize()
    vals = [loss0, *losses, ps, ss] + [float(t.abs().sum()) for t in (*g.tensors(), *g64.tensors())]
    assert all(math.isfinite(v) for v in vals), vals
    print(f"sanitize case ok: loss {loss0:.6g} -> {losses[-1]:.6g}, psnr {ps:.3f}, ssim {ss:.5f},"
          f" pairs {idx.pair_count}, I64 sum {float(c64.I.sum()):.6f}")


if __name__ == "__main__":
    main()
