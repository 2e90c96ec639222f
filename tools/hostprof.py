"""Host-side timing of build_brick_index pieces (development tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_09621_b200 as gs
from paper_2603_09621_b200 import synth, raster, _lib
torch.cuda.set_device(0)
p = synth.make_problem(synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3])
f = gs.GaussianField(*p["field"])
grid = p["render_grid"]
opts = gs.RenderOptions()
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    bricks = _lib.make_bricks(grid, (8, 8, 4), None)
    nb = bricks.bgx * bricks.bgy * bricks.bgz
    rec32, rec64, counts, box = raster._preprocess(f, grid, 3.0, (8, 8, 4), None, True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    gstart = raster._scan(counts, nb)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    P = int(gstart[-1].item())
    t3 = time.perf_counter()
    starts, gids = raster._fill(counts, box, gstart, P, bricks, nb)
    t4 = time.perf_counter()
    torch.cuda.synchronize(); t5 = time.perf_counter()
    print(f"pre {1e3*(t1-t0):.2f} scan {1e3*(t2-t1):.2f} item {1e3*(t3-t2):.2f} fill-host {1e3*(t4-t3):.2f} fill-gpu {1e3*(t5-t4):.2f} ms  P={P}")
print(torch.cuda.memory_summary(abbreviated=True)[:1500])
