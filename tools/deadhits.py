"""Dead-hit census of the LR train forward (development tool).

python tools/deadhits.py [--config 3]
Counts (pair, warp-tile) hits the forward evaluates (E_tile / 128) against the
hits whose live mask is non-zero: the rest are hits the culls could have
rejected.  Also histograms live voxels per live hit.
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_09621_b200 as gs  # noqa: E402
from paper_2603_09621_b200 import _lib, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    p = synth.make_problem(synth.CONFIGS[args.config])
    f = gs.GaussianField(*p["field"])
    grid = p["lr_grid"]
    step = gs.TrainStep(gs.Volume(grid, p["lr"]), gs.RenderOptions(), (8, 8, 4), "l1")
    out = step.forward(f)
    torch.cuda.synchronize()
    P = out.idx.pair_count
    words = step._masks[:P].permute(1, 0, 2).cpu().numpy()    # (P, 4, 2) -> (4, P, 2)
    bits = np.unpackbits(np.ascontiguousarray(words).view(np.uint8), axis=-1)
    bits = bits.reshape(4, P, -1)
    per_tile = [bits[2 * t:2 * t + 2].transpose(1, 0, 2).reshape(P, -1).sum(1)
                for t in range(2)]                               # live voxels per (pair, tile)
    live_hits = int(sum(int((x > 0).sum()) for x in per_tile))
    cnt = torch.zeros(3, dtype=torch.int64, device=f.device)
    aux = out.idx._aux
    _lib.check(_lib.lib().gsv_diag_count_live(
        f.positions.data_ptr(), aux.rec32.data_ptr(), f.log_scales.data_ptr(),
        f.rotations.data_ptr(), out.idx.starts.data_ptr(), out.idx.gids.data_ptr(),
        _lib.make_grid(grid),
        _lib.make_bricks(grid, (8, 8, 4), None), 3.0, cnt.data_ptr(),
        _lib.stream_ptr()), "count_live")
    torch.cuda.synchronize()
    e_live, e_brick, e_tile = (int(x) for x in cnt.tolist())
    hits = e_tile // 128
    print(f"pairs {P}  pair-tiles {2 * P}  hits {hits}  live hits {live_hits}  "
          f"dead hits {hits - live_hits} ({100.0 * (hits - live_hits) / max(hits, 1):.1f}%)")
    print(f"E_live {e_live}  E_tile {e_tile}  live fraction {e_live / max(e_tile, 1):.3f}")
    lv = np.concatenate([x[x > 0] for x in per_tile])
    q = np.percentile(lv, [10, 25, 50, 75, 90])
    print(f"live voxels per live hit: mean {lv.mean():.1f}  p10/25/50/75/90 {q}")


if __name__ == "__main__":
    main()
