"""BASELINE-size parity on the GPU (configs 2-5): brick lists bit-exact vs
hashes of the reference's own lists, LR intensities at 4096 sampled voxels and
the LR loss vs the reference (tests/golden/full_configs.json)."""

import numpy as np
import pytest

import paper_2603_09621_b200 as gs
from paper_2603_09621_b200.synth import CONFIGS, make_problem, sha256

from conftest import load_json

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cid", [2, 3, 4, 5])
def test_full_size_lists_and_render(cid):
    ref = load_json("full_configs.json")["configs"][str(cid)]
    p = make_problem(CONFIGS[cid])
    assert sha256(p["lr"]) == ref["lr_volume"]
    assert sha256(*p["field"]) == ref["field"]
    f = gs.GaussianField(*p["field"])
    grids = {"render": p["render_grid"]} if cid == 5 else {"lr": p["lr_grid"], "hr": p["hr_grid"]}
    for name, grid in grids.items():
        idx = gs.build_brick_index(f, grid)
        r = ref[name]
        assert idx.pair_count == r["pairs"], (cid, name)
        assert sha256(idx.starts.cpu().numpy()) == r["starts"], (cid, name)
        assert sha256(idx.gids.cpu().numpy().astype(np.int64)) == r["gids"], (cid, name)
        if name == "lr":
            c = gs.forward(f, grid, idx)
            I = c.I.cpu().numpy()
            sel = np.asarray(r["sample_idx"])
            err = np.abs(I[sel].astype(np.float64) - np.asarray(r["sample_I"])).max()
            assert err <= 1e-5, (cid, err)
            loss, _ = gs.loss_and_grad(c.volume(), gs.Volume(grid, p["lr"]), "l1")
            assert abs(loss - r["loss"]) <= 1e-6 * max(1.0, abs(r["loss"])), (cid, loss, r["loss"])
        del idx
