"""Host-side cost of the fit loop body (development tool).

python tools/hoststep.py [--config 3] [--steps 30]
cProfile of TrainStep.forward + update with the GPU left running: reports
where the host spends its time per step (the step is launch-bound when this
exceeds the GPU time of the step).
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_09621_b200 as gs  # noqa: E402
from paper_2603_09621_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--steps", type=int, default=30)
args = ap.parse_args()
torch.cuda.set_device(0)
p = synth.make_problem(synth.CONFIGS[args.config])
f = gs.GaussianField(*p["field"])
step = gs.TrainStep(gs.Volume(p["lr_grid"], p["lr"]), gs.RenderOptions(), (8, 8, 4), "l1")
state = gs.AdamState.create(f)
lrs = gs.FitConfig().resolved_lrs(p["lr_grid"].spacing)
for _ in range(5):
    step.update(f, step.forward(f), state, lrs)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(args.steps):
    step.update(f, step.forward(f), state, lrs)
torch.cuda.synchronize()
print(f"wall {1e3 * (time.perf_counter() - t0) / args.steps:.3f} ms/step")
pr = cProfile.Profile()
pr.enable()
for _ in range(args.steps):
    step.update(f, step.forward(f), state, lrs)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
