"""Long fit through the public fit() (development check): loss trace, graph
recaptures, wall time, and PSNR/SSIM of the HR render.

python tools/longfit.py [iterations] [config]"""

from __future__ import annotations

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2603_09621_b200 as gs  # noqa: E402
from paper_2603_09621_b200 import synth  # noqa: E402
import paper_2603_09621_b200.train as train_mod  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    torch.cuda.set_device(0)
    p = synth.make_problem(synth.CONFIGS[cfg])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    captures = [0]
    real = train_mod._graph_capture

    def counting(*a, **k):
        captures[0] += 1
        return real(*a, **k)

    train_mod._graph_capture = counting
    t0 = time.perf_counter()
    f, rep = gs.fit(lr, gs.InitConfig(background_threshold=0.0),
                    gs.FitConfig(iterations=iters, log_every=max(iters // 5, 1)))
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    print(f"fit {iters} iterations: {wall:.2f} s ({iters / wall:.0f} it/s incl. init), "
          f"graph captures {captures[0]}")
    print("losses:", [round(e["loss"], 6) for e in rep.entries])
    hr = gs.Volume(p["hr_grid"], p["hr"])
    sr = gs.Renderer(p["hr_grid"])(f)
    srv = gs.Volume(p["hr_grid"], sr.I.view(*reversed(p["hr_grid"].dims)).permute(2, 1, 0))
    print("PSNR", gs.psnr(srv, hr), "SSIM", gs.ssim3d(srv, hr))


if __name__ == "__main__":
    main()
