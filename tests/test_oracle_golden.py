"""The oracle (oracle/) pinned to golden vectors produced by running the
reference itself (tests/golden/make_golden.py).  CPU only."""

import json
import os

import numpy as np
import pytest

import oracle
from paper_2603_09621_b200.field import random_field_arrays
from paper_2603_09621_b200.synth import CONFIGS, make_problem, sha256
from paper_2603_09621_b200.volume import GridSpec

from conftest import GOLDEN, GRAD_KEYS, SWEEP_GRIDS, field_dict, load_json


def _case_field(c):
    dims, sp, org = SWEEP_GRIDS[c["grid"]]
    grid = GridSpec(dims, sp, org)
    return grid, field_dict(random_field_arrays(c["n"], grid, c["seed"], 0.4, 2.0))


def test_golden_metadata_records_versions():
    meta = load_json("sweep.json")["meta"]["versions"]
    assert {"numpy", "numba", "scipy", "python", "reference"} <= set(meta)


def test_oracle_bit_exact_on_reference_sweep():
    """120 cases of test_acceptance.py:40-66 x brick dims x precision: binning,
    S/W/I and all five gradient groups bit-identical to the reference."""
    cases = load_json("sweep.json")["cases"]
    assert len(cases) == 120
    for c in cases:
        grid, fd = _case_field(c)
        bd = tuple(c["brick_dims"])
        st, gi = oracle.build_index(fd, grid.dims, grid.spacing, grid.origin, bd, 3.0)
        assert sha256(st) == c["starts"] and sha256(gi) == c["gids"], c
        S, W, I = oracle.forward(fd, grid.dims, grid.spacing, grid.origin, st, gi, bd,
                                 precision=c["precision"])
        assert (sha256(S), sha256(W), sha256(I)) == (c["S"], c["W"], c["I"]), c
        dl = np.random.default_rng(5).normal(size=grid.num_voxels)
        g = oracle.backward(fd, grid.dims, grid.spacing, grid.origin, st, gi, W, I, dl, bd,
                            precision=c["precision"])
        assert sha256(*(g[k] for k in GRAD_KEYS)) == c["grads"], c


def test_synth_inputs_identical_to_reference_config1():
    meta = load_json("config1.json")
    p = make_problem(CONFIGS[1])
    assert sha256(p["lr"]) == meta["lr_volume"]
    assert sha256(*p["field"]) == meta["field"]


def test_oracle_config1_bit_exact():
    meta = load_json("config1.json")
    g = np.load(os.path.join(GOLDEN, "config1.npz"))
    p = make_problem(CONFIGS[1])
    fd = field_dict(p["field"])
    for name, grid in (("lr", p["lr_grid"]), ("hr", p["hr_grid"])):
        st, gi = oracle.build_index(fd, grid.dims, grid.spacing, grid.origin)
        assert len(gi) == meta[f"{name}_pairs"]
        assert sha256(st) == meta[f"{name}_starts"] and sha256(gi) == meta[f"{name}_gids"]
    grid = p["lr_grid"]
    st, gi = oracle.build_index(fd, grid.dims, grid.spacing, grid.origin)
    S, W, I = oracle.forward(fd, grid.dims, grid.spacing, grid.origin, st, gi)
    assert sha256(I) == meta["lr_I"]
    loss, dl = oracle.loss_and_grad(I, p["lr"].ravel(order="F"))
    assert loss == meta["loss"]
    grads = oracle.backward(fd, grid.dims, grid.spacing, grid.origin, st, gi, W, I, dl)
    for k in GRAD_KEYS:
        np.testing.assert_array_equal(grads[k], g["grad_" + k])


def test_einsum_reduction_order_claim():
    """The CUDA preprocess sums Sigma_kk as (p0 + p2) + p1 because numpy's
    einsum("nkm,nm->nk") does (SURVEY.md §0 finding 2); pin that claim here."""
    rng = np.random.default_rng(0)
    for n in (1, 7, 64, 1000, 200_000):
        rr = rng.normal(size=(n, 3, 3)) ** 2
        var = np.exp(2.0 * rng.normal(size=(n, 3)))
        ein = np.einsum("nkm,nm->nk", rr, var)
        p = rr * var[:, None, :]
        mine = (p[:, :, 0] + p[:, :, 2]) + p[:, :, 1]
        np.testing.assert_array_equal(ein, mine)


@pytest.mark.slow
def test_oracle_full_size_binning_config2():
    """Bit-exact lists at a BASELINE size (config 2, LR and HR grids)."""
    ref = load_json("full_configs.json")["configs"]["2"]
    p = make_problem(CONFIGS[2])
    assert sha256(p["lr"]) == ref["lr_volume"]
    fd = field_dict(p["field"])
    for name, grid in (("lr", p["lr_grid"]), ("hr", p["hr_grid"])):
        st, gi = oracle.build_index(fd, grid.dims, grid.spacing, grid.origin)
        assert len(gi) == ref[name]["pairs"]
        assert sha256(st) == ref[name]["starts"] and sha256(gi) == ref[name]["gids"]


def test_oracle_fast_tail_equals_numpy_tail():
    """oracle.train_step_fast (the timed CPU baseline) == the pinned numpy path."""
    p = make_problem(CONFIGS[1])
    grid = p["lr_grid"]
    from paper_2603_09621_b200.optimize import FitConfig
    lrs = FitConfig().resolved_lrs(grid.spacing)
    fa, fb = field_dict(p["field"]), field_dict(p["field"])
    sa, sb = oracle.adam_state(fa), oracle.adam_state(fb)
    tgt = p["lr"].ravel(order="F")
    for _ in range(2):
        la = oracle.train_step(fa, grid.dims, grid.spacing, grid.origin, tgt, sa, lrs)
        lb = oracle.train_step_fast(fb, grid.dims, grid.spacing, grid.origin, tgt, sb, lrs)
        assert la == lb
    for k in oracle.GROUPS:
        np.testing.assert_allclose(fa[k], fb[k], rtol=0, atol=1e-13)


def test_oracle_metrics_match_reference_goldens():
    """The oracle's psnr / ssim3d (metrics.py:35-77 restated) against the
    reference's values on the seeded pairs of tests/golden/metrics.json."""
    import math
    for case in load_json("metrics.json")["cases"]:
        rng = np.random.default_rng(case["seed"])
        dims = tuple(case["dims"])
        a = rng.uniform(0.0, 1.0, size=dims)
        b = (np.clip(a + case["noise"] * rng.standard_normal(dims), 0.0, 1.0)
             if case["noise"] else a.copy())
        a, b = a.astype(case["dtype"]), b.astype(case["dtype"])
        p = oracle.psnr(a, b)
        if case["psnr"] is None:
            assert math.isinf(p)
        else:
            assert p == case["psnr"]
        assert oracle.ssim3d(a, b) == case["ssim"]
