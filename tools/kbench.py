"""Per-kernel timing of the hot path (development tool, not the bench contract).

python tools/kbench.py [--config 3] [--iters 5] [--hr]
Times, with CUDA events on the launching stream: binning, forward (fused
loss), backward pair pass, merge, chain rule at the LR train grid, and the
binning + forward of the HR render.
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2603_09621_b200 as gs  # noqa: E402
from paper_2603_09621_b200 import synth  # noqa: E402
from paper_2603_09621_b200.raster import _forward_into  # noqa: E402
from paper_2603_09621_b200.train import PhaseTimer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--hr", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--graph", action="store_true",
                    help="also run graph-replayed train steps (TrainStep.step), e.g. under ncu")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    p = synth.make_problem(synth.CONFIGS[args.config])
    f = gs.GaussianField(*p["field"])
    opts = gs.RenderOptions()
    if not args.no_train:
        t = PhaseTimer()
        step = gs.TrainStep(gs.Volume(p["lr_grid"], p["lr"]), opts, (8, 8, 4), "l1", timer=t)
        state = gs.AdamState.create(f)
        lrs = gs.FitConfig().resolved_lrs(p["lr_grid"].spacing)
        for i in range(args.iters + 1):
            if i == 1:
                t.reset()
            out = step.forward(f)
            step.update(f, out, state, lrs)
        print("LR train phases (ms):", {k: round(v[1], 4) for k, v in t.summary().items()})
        if args.graph:
            step.timer = None
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            for i in range(args.iters + 3):
                if i == 3:
                    ev[0].record()
                step.step(f, state, lrs)
            ev[1].record()
            torch.cuda.synchronize()
            print("graph step ms:", round(ev[0].elapsed_time(ev[1]) / max(args.iters, 1), 4))
    if args.hr:
        grid = p["render_grid"]
        t = PhaseTimer()
        pool = gs._lib.BufferPool(f.device) if hasattr(gs, "_lib") else None
        from paper_2603_09621_b200 import _lib
        pool = _lib.BufferPool(f.device)
        n = grid.num_voxels
        S, W, I = (torch.empty(n, device=f.device) for _ in range(3))
        for i in range(args.iters + 1):
            if i == 1:
                t.reset()
            t("bin")
            idx = gs.build_brick_index(f, grid, opts, pool=pool)
            t("forward")
            _forward_into(f, grid, idx, opts, idx._aux.rec32, idx._aux.rec64, S, W, I)
            t(None)
        print("HR render phases (ms):", {k: round(v[1], 4) for k, v in t.summary().items()},
              "pairs", idx.pair_count)


if __name__ == "__main__":
    main()
