"""CUDA path vs the oracle and the reference's golden vectors (needs a B200).

Bars (north_star): brick lists bit-exact; voxel intensities within 1e-5
(f32; the reference's own brick-vs-naive bar, test_acceptance.py:40-66) and
1e-10 (f64); gradients within 1e-5 relative, norm-wise per parameter group,
with the reference's W / I / dL/dI injected (SURVEY.md §0 finding 5).
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2603_09621_b200 as gs
from paper_2603_09621_b200.field import random_field_arrays
from paper_2603_09621_b200.raster import RenderCache
from paper_2603_09621_b200.synth import CONFIGS, make_problem, sha256

from conftest import GRAD_KEYS, SWEEP_GRIDS, field_dict, load_json

pytestmark = pytest.mark.gpu

TOL_I = {"f32": 1e-5, "f64": 1e-10}
TOL_G = {"f32": 1e-5, "f64": 1e-10}


def np_(t):
    return t.detach().cpu().numpy()


def rel_norm(got, ref):
    den = np.linalg.norm(ref)
    if den == 0.0:
        return float(np.linalg.norm(got))
    return float(np.linalg.norm(got - ref) / den)


def _sweep_field(n, gi):
    dims, sp, org = SWEEP_GRIDS[gi]
    grid = gs.GridSpec(dims, sp, org)
    arrs = random_field_arrays(n, grid, 100 * n + gi, 0.4, 2.0)
    return grid, arrs


SWEEP = [(n, gi) for n in (1, 10, 100, 1000) for gi in range(5)]


# ------------------------------------------------------------ binning
def test_sweep_binning_bit_exact_vs_reference_hashes():
    cases = load_json("sweep.json")["cases"]
    seen = set()
    for c in cases:
        key = (c["n"], c["grid"], tuple(c["brick_dims"]))
        if key in seen:
            continue
        seen.add(key)
        grid, arrs = _sweep_field(c["n"], c["grid"])
        f = gs.GaussianField(*arrs)
        idx = gs.build_brick_index(f, grid, gs.RenderOptions(), tuple(c["brick_dims"]))
        assert idx.pair_count == c["pairs"], key
        assert sha256(np_(idx.starts)) == c["starts"], key
        assert sha256(np_(idx.gids).astype(np.int64)) == c["gids"], key
    assert len(seen) == 60


def test_config1_binning_bit_exact():
    meta = load_json("config1.json")
    from paper_2603_09621_b200.synth import CONFIGS, make_problem
    p = make_problem(CONFIGS[1])
    assert sha256(*p["field"]) == meta["field"]
    f = gs.GaussianField(*p["field"])
    for name, grid in (("lr", p["lr_grid"]), ("hr", p["hr_grid"])):
        idx = gs.build_brick_index(f, grid)
        assert idx.pair_count == meta[f"{name}_pairs"]
        assert sha256(np_(idx.starts)) == meta[f"{name}_starts"]
        assert sha256(np_(idx.gids).astype(np.int64)) == meta[f"{name}_gids"]


@pytest.mark.parametrize("bd", [(8, 8, 4), (8, 8, 8), (4, 4, 4), (16, 8, 8), (3, 5, 7)])
def test_binning_matches_oracle_any_brick_dims(bd):
    grid = gs.GridSpec((21, 18, 13), (0.9, 1.1, 1.7), (-3.0, 2.0, 0.5))
    arrs = random_field_arrays(700, grid, 77, 0.3, 2.5)
    f = gs.GaussianField(*arrs)
    idx = gs.build_brick_index(f, grid, gs.RenderOptions(), bd)
    st, gi = oracle.build_index(field_dict(arrs), grid.dims, grid.spacing, grid.origin, bd, 3.0)
    np.testing.assert_array_equal(np_(idx.starts), st)
    np.testing.assert_array_equal(np_(idx.gids), gi)


@pytest.mark.parametrize("dims", [(128, 128, 256), (136, 128, 256)])
def test_binning_at_the_16_bit_key_boundary(dims):
    """Slabs of <= 65536 bricks sort 16-bit keys, larger ones 32-bit: 128x128x256
    voxels (8x8x4 bricks) is exactly 65536 bricks, 136x128x256 is 69632.  Both
    widths match the oracle bit for bit, through the eager index and through
    the capacity-mode (graph) binning of the Renderer."""
    grid = gs.GridSpec(dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    arrs = random_field_arrays(3000, grid, 5, 0.5, 2.0)
    f = gs.GaussianField(*arrs)
    idx = gs.build_brick_index(f, grid)
    st, gi = oracle.build_index(field_dict(arrs), grid.dims, grid.spacing, grid.origin,
                                (8, 8, 4), 3.0)
    assert len(st) - 1 == (dims[0] // 8) * (dims[1] // 8) * (dims[2] // 4)
    np.testing.assert_array_equal(np_(idx.starts), st)
    np.testing.assert_array_equal(np_(idx.gids), gi)
    r = gs.Renderer(grid)
    _renders_equal(r(f), gs.forward(f, grid, idx))


# ------------------------------------------------------------ forward
@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_sweep_forward_vs_oracle(precision):
    opts = gs.RenderOptions(precision=precision)
    for n, gi in SWEEP:
        grid, arrs = _sweep_field(n, gi)
        f = gs.GaussianField(*arrs)
        idx = gs.build_brick_index(f, grid, opts)
        c = gs.forward(f, grid, idx, opts)
        fd = field_dict(arrs)
        S, W, I = oracle.forward(fd, grid.dims, grid.spacing, grid.origin, np_(idx.starts),
                                 np_(idx.gids), precision=precision)
        err = np.abs(np_(c.I).astype(np.float64) - I.astype(np.float64)).max()
        assert err <= TOL_I[precision], (n, gi, precision, err)
        # coverage decisions identical: I == 0 exactly where the oracle's is
        np.testing.assert_array_equal(np_(c.I) == 0, I == 0)


def test_config1_forward_vs_reference_golden():
    g = np.load(__import__("os").path.join(__import__("conftest").GOLDEN, "config1.npz"))
    from paper_2603_09621_b200.synth import CONFIGS, make_problem
    p = make_problem(CONFIGS[1])
    f = gs.GaussianField(*p["field"])
    for grid, key in ((p["lr_grid"], "lr_I"), (p["hr_grid"], "hr_I")):
        idx = gs.build_brick_index(f, grid)
        c = gs.forward(f, grid, idx)
        err = np.abs(np_(c.I).astype(np.float64) - g[key].astype(np.float64)).max()
        assert err <= 1e-5, (key, err)
    o64 = gs.RenderOptions(precision="f64")
    idx = gs.build_brick_index(f, p["lr_grid"], o64)
    c = gs.forward(f, p["lr_grid"], idx, o64)
    assert np.abs(np_(c.I) - g["lr_I64"]).max() <= 1e-10


def test_forward_equals_naive_gpu():
    grid = gs.GridSpec((16, 16, 16), (0.7, 1.0, 1.3), (-2.0, 0.0, 1.0))
    f = gs.GaussianField(*random_field_arrays(200, grid, 9, 0.4, 2.0))
    for prec, tol in (("f32", 1e-5), ("f64", 1e-10)):
        opts = gs.RenderOptions(precision=prec)
        brick = gs.forward(f, grid, gs.build_brick_index(f, grid, opts), opts).volume()
        naive = gs.render_naive(f, grid, opts)
        assert np.abs(brick.numpy().astype(np.float64) - naive.numpy()).max() <= tol


# ------------------------------------------------------------ backward
def _backward_case(n, gi, precision, relax_enabled=True):
    grid, arrs = _sweep_field(n, gi)
    f = gs.GaussianField(*arrs)
    f.relax_enabled = relax_enabled
    fd = field_dict(arrs, relax_enabled=relax_enabled)
    opts = gs.RenderOptions(precision=precision)
    idx = gs.build_brick_index(f, grid, opts)
    st, gi_ = np_(idx.starts), np_(idx.gids)
    S, W, I = oracle.forward(fd, grid.dims, grid.spacing, grid.origin, st, gi_,
                             precision=precision)
    dl = np.random.default_rng(5).normal(size=grid.num_voxels)
    dev = f.device
    cache = RenderCache(grid, torch.from_numpy(S).to(dev), torch.from_numpy(W).to(dev),
                        torch.from_numpy(I).to(dev), f.version)
    got = gs.backward(f, grid, idx, cache, dl, opts)
    ref = oracle.backward(fd, grid.dims, grid.spacing, grid.origin, st, gi_, W, I, dl,
                          precision=precision)
    return got, ref


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_sweep_backward_vs_oracle(precision):
    for n, gi in SWEEP:
        got, ref = _backward_case(n, gi, precision)
        for k in GRAD_KEYS:
            if n == 1 and k in ("positions", "log_scales", "rotations", "raw_relax"):
                # a lone Gaussian: geometry gradients are pure rounding noise,
                # bounded relative to the one real gradient (the amplitude's)
                scale = np.linalg.norm(ref["raw_amplitude"])
                noise = np.abs(np_(getattr(got, k))).max()
                ref_noise = np.abs(ref[k]).max()   # the reference engine's own noise
                print("n=1 noise", precision, k, noise, ref_noise, scale)
                bound = max(4.0 * ref_noise, (1e-6 if precision == "f32" else 1e-12) * max(scale, 1.0))
                assert noise <= bound, (k, noise, ref_noise)
                continue
            e = rel_norm(np_(getattr(got, k)), ref[k])
            assert e <= TOL_G[precision], (n, gi, precision, k, e)


def test_config1_backward_vs_reference_golden():
    g = np.load(__import__("os").path.join(__import__("conftest").GOLDEN, "config1.npz"))
    from paper_2603_09621_b200.synth import CONFIGS, make_problem
    p = make_problem(CONFIGS[1])
    grid = p["lr_grid"]
    f = gs.GaussianField(*p["field"])
    idx = gs.build_brick_index(f, grid)
    dev = f.device
    W = torch.from_numpy(g["lr_W"]).to(dev)
    I = torch.from_numpy(g["lr_I"]).to(dev)
    cache = RenderCache(grid, torch.zeros_like(W), W, I, f.version)
    dl = g["dl"].astype(np.float64) / grid.num_voxels
    got = gs.backward(f, grid, idx, cache, dl)
    for k in GRAD_KEYS:
        e = rel_norm(np_(getattr(got, k)), g["grad_" + k])
        assert e <= 1e-5, (k, e)


def test_backward_relax_disabled_vs_oracle():
    got, ref = _backward_case(100, 1, "f32", relax_enabled=False)
    assert np.all(np_(got.raw_relax) == 0.0)
    for k in ("raw_amplitude", "positions", "log_scales", "rotations"):
        assert rel_norm(np_(getattr(got, k)), ref[k]) <= 1e-5


# ------------------------------------------------------------ KATs (test_raster / test_render)
def _point_field(position, scale):
    return gs.GaussianField(np.asarray([position], dtype=np.float64),
                            np.log(np.full((1, 3), scale)), np.asarray([[1.0, 0, 0, 0]]),
                            np.zeros(1), np.zeros(1))


def test_kat_binning_cases(unit_grid):
    idx = gs.build_brick_index(_point_field([4.0, 4.0, 1.0], 0.1), unit_grid)
    assert idx.brick_grid == (1, 1, 2) and idx.pair_count == 1
    assert int(idx.starts[1] - idx.starts[0]) == 1
    assert gs.build_brick_index(_point_field([4.0, 4.0, 4.0], 50.0), unit_grid).pair_count == 2
    assert gs.build_brick_index(_point_field([4.0, 4.0, 3.5], 0.2), unit_grid).pair_count == 2
    far = _point_field([500.0, 0.0, 0.0], 1.0)
    idx = gs.build_brick_index(far, unit_grid)
    assert idx.pair_count == 0
    v = gs.forward(far, unit_grid, idx, gs.RenderOptions(precision="f64")).volume()
    assert np.all(v.numpy() == 0.0)
    f = gs.random_field(7, unit_grid, seed=31)
    assert gs.build_brick_index(f, unit_grid, gs.RenderOptions(cutoff_sigma=np.inf)).pair_count == 14


def test_kat_infinite_cutoff_render_matches_oracle(unit_grid):
    arrs = random_field_arrays(8, unit_grid, 9)
    f = gs.GaussianField(*arrs)
    opts = gs.RenderOptions(cutoff_sigma=np.inf, precision="f64")
    c = gs.forward(f, unit_grid, gs.build_brick_index(f, unit_grid, opts), opts)
    st, gi = oracle.build_index(field_dict(arrs), unit_grid.dims, unit_grid.spacing,
                                unit_grid.origin, (8, 8, 4), np.inf)
    _, _, I = oracle.forward(field_dict(arrs), unit_grid.dims, unit_grid.spacing,
                             unit_grid.origin, st, gi, cutoff=np.inf, precision="f64")
    assert np.abs(np_(c.I) - I).max() <= 1e-10


def test_kat_single_gaussian_renders_amplitude():
    g = gs.GridSpec((4, 4, 4))
    amp = 0.7
    f = gs.GaussianField(np.asarray([[1.5, 1.5, 1.5]]), np.full((1, 3), 0.3),
                         np.asarray([[1.0, 0, 0, 0]]), np.asarray([np.log(amp / (1 - amp))]),
                         np.asarray([20.0]))
    for prec, tol in (("f64", 1e-9), ("f32", 1e-6)):
        o = gs.RenderOptions(precision=prec)
        v = gs.forward(f, g, gs.build_brick_index(f, g, o), o).volume().numpy()
        cov = v > 0
        assert cov.any()
        np.testing.assert_allclose(v[cov], amp, atol=tol)


def test_kat_two_equal_kernels_average():
    g = gs.GridSpec((1, 1, 1))
    f = gs.GaussianField(np.asarray([[-0.4, 0, 0], [0.4, 0, 0]]), np.zeros((2, 3)),
                         np.tile([1.0, 0, 0, 0], (2, 1)),
                         np.asarray([np.log(0.25), np.log(4.0)]), np.full(2, 20.0))
    for prec in ("f32", "f64"):
        o = gs.RenderOptions(precision=prec)
        v = gs.forward(f, g, gs.build_brick_index(f, g, o), o).volume().numpy()
        assert abs(float(v[0, 0, 0]) - 0.5) <= 1e-6


def test_kat_normalization_properties():
    # test_acceptance.py:86-117 (criterion 3) on the production engine
    grid = gs.GridSpec((16, 16, 16))
    opts = gs.RenderOptions()
    arrs = list(random_field_arrays(200, grid, 30))
    arrs[3] = np.full(200, 0.31)
    f = gs.GaussianField(*arrs)
    out = gs.forward(f, grid, gs.build_brick_index(f, grid, opts), opts).volume().numpy()
    amp = 1.0 / (1.0 + np.exp(-0.31))
    cov = out != 0.0
    assert cov.any() and np.abs(out[cov] - amp).max() <= 1e-6
    arrs = random_field_arrays(200, grid, 31)
    f = gs.GaussianField(*arrs)
    out = gs.forward(f, grid, gs.build_brick_index(f, grid, opts), opts).volume().numpy()
    amps = 1.0 / (1.0 + np.exp(-arrs[3]))
    cov = out != 0.0
    assert out[cov].min() >= amps.min() - 1e-6 and out[cov].max() <= amps.max() + 1e-6
    from scipy.special import logit
    r = 1.0 / (1.0 + np.exp(-arrs[4]))
    arrs2 = list(arrs)
    arrs2[4] = logit(0.37 * r)
    g2 = gs.GaussianField(*arrs2)
    scaled = gs.forward(g2, grid, gs.build_brick_index(g2, grid, opts), opts).volume().numpy()
    assert np.abs(scaled - out).max() <= 1e-6


def test_zero_upstream_is_exactly_zero(unit_grid):
    f = gs.random_field(10, unit_grid, seed=38)
    for prec in ("f32", "f64"):
        o = gs.RenderOptions(precision=prec)
        idx = gs.build_brick_index(f, unit_grid, o)
        c = gs.forward(f, unit_grid, idx, o)
        g = gs.backward(f, unit_grid, idx, c, np.zeros(unit_grid.num_voxels), o)
        for k in GRAD_KEYS:
            assert np.all(np_(getattr(g, k)) == 0.0), (prec, k)


def test_single_gaussian_geometry_gradients_vanish(unit_grid):
    f = gs.random_field(1, unit_grid, seed=15)
    o = gs.RenderOptions(precision="f64")
    idx = gs.build_brick_index(f, unit_grid, o)
    c = gs.forward(f, unit_grid, idx, o)
    g = gs.backward(f, unit_grid, idx, c, np.random.default_rng(16).normal(size=512), o)
    for k in ("positions", "log_scales", "rotations", "raw_relax"):
        assert np.abs(np_(getattr(g, k))).max() < 1e-12
    assert np.abs(np_(g.raw_amplitude)).max() > 1e-6


# ------------------------------------------------------------ errors
def test_staleness_and_upstream_errors(unit_grid):
    f = gs.random_field(5, unit_grid, seed=34)
    idx = gs.build_brick_index(f, unit_grid)
    f.bump_version()
    with pytest.raises(gs.StaleIndexError, match="version"):
        gs.forward(f, unit_grid, idx)
    f = gs.random_field(5, unit_grid, seed=35)
    idx = gs.build_brick_index(f, unit_grid)
    with pytest.raises(gs.StaleIndexError, match="grid"):
        gs.forward(f, gs.GridSpec((4, 4, 4)), idx)
    with pytest.raises(gs.StaleIndexError, match="cutoff"):
        gs.forward(f, unit_grid, idx, gs.RenderOptions(cutoff_sigma=2.0))
    cache = gs.forward(f, unit_grid, idx)
    f.bump_version()
    idx2 = gs.build_brick_index(f, unit_grid)
    with pytest.raises(gs.StaleIndexError, match="stale"):
        gs.backward(f, unit_grid, idx2, cache, np.ones(unit_grid.num_voxels))
    f = gs.random_field(4, unit_grid, seed=39)
    idx = gs.build_brick_index(f, unit_grid)
    cache = gs.forward(f, unit_grid, idx)
    with pytest.raises(ValueError, match="entries"):
        gs.backward(f, unit_grid, idx, cache, np.ones(3))
    dl = np.ones(unit_grid.num_voxels)
    dl[7] = np.nan
    with pytest.raises(gs.NumericalError, match="voxel index 7"):
        gs.backward(f, unit_grid, idx, cache, dl)


# ------------------------------------------------------------ determinism
def _shuffle(idx, seed):
    rng = np.random.default_rng(seed)
    gids = np_(idx.gids).copy()
    st = np_(idx.starts)
    for b in range(idx.brick_count):
        gids[st[b]:st[b + 1]] = rng.permutation(gids[st[b]:st[b + 1]])
    return gs.BrickIndex(idx.grid, idx.brick_dims, idx.brick_grid, st, gids,
                         idx.field_version, idx.field_count, idx.cutoff_sigma)


def test_bit_identity_across_list_order_and_runs():
    grid = gs.GridSpec((16, 16, 16))
    f = gs.random_field(500, grid, seed=40)
    dl = np.random.default_rng(41).normal(size=grid.num_voxels)
    for opts in (gs.RenderOptions(), gs.RenderOptions(precision="f64")):
        idx = gs.build_brick_index(f, grid, opts)
        ref_i = ref_g = None
        for seed in (None, 1, 2, None):
            variant = idx if seed is None else _shuffle(idx, seed)
            if seed is not None:
                assert not variant.lists_sorted()
                np.testing.assert_array_equal(np_(variant.canonicalized().gids), np_(idx.gids))
            c = gs.forward(f, grid, variant, opts)
            g = gs.backward(f, grid, variant, c, dl, opts)
            packed = np.concatenate([np_(getattr(g, k)).ravel() for k in GRAD_KEYS])
            if ref_i is None:
                ref_i, ref_g = np_(c.I), packed
            else:
                np.testing.assert_array_equal(np_(c.I), ref_i)
                np.testing.assert_array_equal(packed, ref_g)


# ------------------------------------------------------------ loss / Adam
def test_loss_kats():
    g2 = gs.GridSpec((2, 2, 2))
    data = np.zeros((2, 2, 2))
    data[1, 0, 0] = 0.1
    loss, grad = gs.loss_and_grad(gs.Volume(g2, data), gs.Volume(g2, np.zeros((2, 2, 2))), "l1")
    assert loss == pytest.approx(0.1 / 8)
    gr = np_(grad)
    assert gr[1] == pytest.approx(1.0 / 8) and np.count_nonzero(gr) == 1
    loss, grad = gs.loss_and_grad(gs.Volume(g2, np.full((2, 2, 2), 0.25)),
                                  gs.Volume(g2, np.zeros((2, 2, 2))), "l2")
    assert loss == pytest.approx(0.0625)
    np.testing.assert_allclose(np_(grad), 2 * 0.25 / 8)
    with pytest.raises(gs.GridMismatchError, match="grid"):
        gs.loss_and_grad(gs.Volume(g2, data), gs.Volume(gs.GridSpec((8, 8, 8)), np.zeros((8, 8, 8))))
    with pytest.raises(ValueError, match="loss kind"):
        gs.loss_and_grad(gs.Volume(g2, data), gs.Volume(g2, data), "huber")


def test_adam_first_step_sign_like(unit_grid):
    f = gs.random_field(3, unit_grid, seed=51)
    before = np_(f.raw_amplitude).copy()
    g = gs.GradientBuffer.zeros(3)
    g.raw_amplitude[:] = torch.tensor([0.5, -2.0, 1e-3], dtype=torch.float64)
    state = gs.AdamState.create(f)
    lrs = {k: 0.0 for k in gs.FitConfig().resolved_lrs(unit_grid.spacing)}
    lrs["raw_amplitude"] = 0.01
    gs.step_optimizer(f, g, state, lrs)
    ga = np.asarray([0.5, -2.0, 1e-3])
    np.testing.assert_allclose(np_(f.raw_amplitude), before - 0.01 * ga / (np.abs(ga) + 1e-8),
                               rtol=1e-12)
    assert state.t == 1


def test_adam_matches_oracle_bit_exact(unit_grid):
    arrs = random_field_arrays(50, unit_grid, 52)
    f = gs.GaussianField(*arrs)
    fd = field_dict(arrs)
    rng = np.random.default_rng(53)
    grads = {k: rng.normal(size=fd[k].shape) for k in GRAD_KEYS}
    gb = gs.GradientBuffer(*(torch.from_numpy(grads[k]).to(f.device) for k in GRAD_KEYS))
    st_gpu, st_cpu = gs.AdamState.create(f), oracle.adam_state(fd)
    lrs = gs.FitConfig().resolved_lrs(unit_grid.spacing)
    for _ in range(3):
        gs.step_optimizer(f, gb, st_gpu, lrs)
        f.normalize_rotations()
        oracle.adam_step(fd, grads, st_cpu, lrs)
    for k in ("positions", "log_scales", "raw_amplitude", "raw_relax"):
        np.testing.assert_array_equal(np_(getattr(f, k)), fd[k])
    np.testing.assert_allclose(np_(f.rotations), fd["rotations"], rtol=0, atol=1e-15)


# ------------------------------------------------------------ fused train step
def test_train_step_matches_unfused_api():
    from paper_2603_09621_b200.synth import CONFIGS, make_problem
    p = make_problem(CONFIGS[1])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    step = gs.TrainStep(lr, gs.RenderOptions(), (8, 8, 4), "l1")
    out = step.forward(f)
    grads = step.backward(f, out)
    idx = gs.build_brick_index(f, lr.grid)
    c = gs.forward(f, lr.grid, idx)
    loss, dl = gs.loss_and_grad(c.volume(), lr, "l1")
    g2 = gs.backward(f, lr.grid, idx, c, dl)
    assert abs(out.loss() - loss) <= 1e-12
    np.testing.assert_array_equal(np_(out.cache.I), np_(c.I))
    for k in GRAD_KEYS:  # masked (train step) vs span (public API) backward
        a, b = np_(getattr(grads, k)), np_(getattr(g2, k))
        assert np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(b) + 1e-20, k
    meta = load_json("config1.json")
    assert abs(out.loss() - meta["loss"]) <= 1e-6


# ------------------------------------------------------------ z-slab sharding
@pytest.mark.parametrize("cuts", ["layers", "balanced3", "odd"])
def test_slabs_reassemble_the_full_index_render_and_gradients(cuts):
    """Ranks emulated sequentially on one GPU, slabs = contiguous brick-id
    ranges (whole layers, pair-balanced mid-layer cuts, and odd ranges: one
    brick, empty, a layer remainder): per-slab lists are exact slices of the
    global lists, per-slab renders are bit-identical on their bricks' voxels,
    and the sum of per-slab merged partials (what the NCCL all_reduce
    computes) equals the single-index merge."""
    from paper_2603_09621_b200.distributed import (layer_slab_ranges, pair_weights,
                                                   slab_ranges, slab_voxel_mask)
    from paper_2603_09621_b200.raster import _pair_partials
    from paper_2603_09621_b200.synth import CONFIGS, make_problem
    p = make_problem(CONFIGS[1])
    grid = p["lr_grid"]
    lr = gs.Volume(grid, p["lr"])
    f = gs.GaussianField(*p["field"])
    bd = (8, 8, 4)
    full = gs.TrainStep(lr, gs.RenderOptions(), bd, "l1")
    out = full.forward(f)
    g_full = _pair_partials(f, grid, out.idx, full.opts, out.idx._aux.rec32, None, out.ab,
                            out.idx._aux.gstart, out.idx._aux.box, True,
                            live_masks=full._masks).clone()
    I_full = np_(out.cache.I).copy()
    starts_full, gids_full = np_(out.idx.starts), np_(out.idx.gids)
    nb = len(starts_full) - 1
    layer = out.idx.brick_grid[0] * out.idx.brick_grid[1]
    if cuts == "layers":
        slabs = layer_slab_ranges(grid, bd, 2)
    elif cuts == "balanced3":
        slabs = slab_ranges(nb, 3, weights=pair_weights(f, grid, gs.RenderOptions(), bd))
        assert any(b % layer for _, b in slabs[:-1]), "expected a mid-layer cut"
    else:
        c = [0, 1, 1, layer + 5, 3 * layer - 7, nb]
        slabs = list(zip(c, c[1:]))
    total = torch.zeros_like(g_full)
    loss_total = 0.0
    pieces = []
    for slab in slabs:
        st = gs.TrainStep(lr, gs.RenderOptions(), bd, "l1", slab=slab)
        o = st.forward(f)
        s0, s1 = starts_full[slab[0]], starts_full[slab[1]]
        np.testing.assert_array_equal(np_(o.idx.starts), starts_full[slab[0]:slab[1] + 1] - s0)
        np.testing.assert_array_equal(np_(o.idx.gids), gids_full[s0:s1])
        pieces.append(np_(o.idx.gids))
        own = slab_voxel_mask(grid, bd, slab)
        np.testing.assert_array_equal(np_(o.cache.I)[own], I_full[own])
        g = _pair_partials(f, grid, o.idx, st.opts, o.idx._aux.rec32, None, o.ab,
                           o.idx._aux.gstart, o.idx._aux.box, True, live_masks=st._masks)
        total += g
        loss_total += float(o.loss_sum.item())
    np.testing.assert_array_equal(np.concatenate(pieces), gids_full)
    assert abs(loss_total / grid.num_voxels - out.loss()) <= 1e-12
    a, b = np_(total[:, :11]), np_(g_full[:, :11])
    assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b) + 1e-30


def test_slab_backward_api_mid_layer():
    """The reference-shaped backward() on a mid-layer slab index: the
    backward_prep step touches only the slab's bricks (voxels outside keep
    their zero W without tripping the coverage check), and the two slabs'
    gradients sum to the whole-grid gradient."""
    from paper_2603_09621_b200.synth import CONFIGS, make_problem
    p = make_problem(CONFIGS[1])
    grid = p["lr_grid"]
    f = gs.GaussianField(*p["field"])
    opts = gs.RenderOptions()
    idx = gs.build_brick_index(f, grid, opts)
    cache = gs.forward(f, grid, idx)
    rng = np.random.default_rng(4)
    dldi = torch.as_tensor(rng.standard_normal(grid.num_voxels), device=cache.I.device)
    ref = gs.backward(f, grid, idx, cache, dldi)
    nb = idx.brick_count
    cut = (nb // 2) | 3
    acc = None
    for slab in ((0, cut), (cut, nb)):
        si = gs.build_brick_index(f, grid, opts, slab=slab)
        sc = gs.forward(f, grid, si)
        gb = [t.clone() for t in gs.backward(f, grid, si, sc, dldi).tensors()]
        acc = gb if acc is None else [x + y for x, y in zip(acc, gb)]
    for x, y in zip(acc, ref.tensors()):      # gradients are linear in the partial sums
        a, b = np_(x), np_(y)
        assert np.linalg.norm(a - b) <= 1e-9 * (np.linalg.norm(b) + 1e-30)


# ------------------------------------------------------------------ Renderer
def _renders_equal(a, b):
    for k in ("S", "W", "I"):
        assert torch.equal(getattr(a, k), getattr(b, k)), k


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_renderer_graph_equals_index_plus_forward(cfg_id):
    """The graph-replayed Renderer (capacity binning, no pair-count read) is
    bit-identical to build_brick_index + forward, follows in-place field
    updates without re-capturing, and reports the pair count."""
    p = make_problem(CONFIGS[cfg_id])
    f = gs.GaussianField(*p["field"])
    grid = p["hr_grid"]
    r = gs.Renderer(grid)
    c = r(f)
    idx = gs.build_brick_index(f, grid)
    _renders_equal(c, gs.forward(f, grid, idx))
    assert r.pair_count() == idx.pair_count
    g0 = r._graph
    with torch.no_grad():
        f.positions.add_(0.05)
        f.raw_amplitude.mul_(0.9)
    f.bump_version()
    c = r(f)
    assert r._graph is g0
    idx = gs.build_brick_index(f, grid)
    _renders_equal(c, gs.forward(f, grid, idx))


def test_renderer_recovers_from_capacity_overflow(monkeypatch):
    """A first capture with too little pair capacity overflows on the device;
    the Renderer re-captures with more room and the render is still exact."""
    import paper_2603_09621_b200.train as train_mod
    p = make_problem(CONFIGS[1])
    f = gs.GaussianField(*p["field"])
    grid = p["hr_grid"]
    r = gs.Renderer(grid)
    real = gs.Renderer._capture
    calls = []

    def capture(self, f, key, min_cap=0):
        calls.append(min_cap)
        monkeypatch.setattr(train_mod, "_RENDER_HEADROOM", 0.1 if len(calls) == 1 else 1.05)
        return real(self, f, key, min_cap)

    monkeypatch.setattr(gs.Renderer, "_capture", capture)
    c = r(f)
    assert len(calls) >= 2
    _renders_equal(c, gs.forward(f, grid, gs.build_brick_index(f, grid)))


def test_renderer_f64_is_the_eager_path():
    p = make_problem(CONFIGS[1])
    f = gs.GaussianField(*p["field"])
    opts = gs.RenderOptions(precision="f64")
    r = gs.Renderer(p["hr_grid"], opts)
    c = r(f)
    assert r.last_index is not None
    _renders_equal(c, gs.forward(f, p["hr_grid"], gs.build_brick_index(f, p["hr_grid"], opts),
                                 opts))


def test_renderer_with_no_pairs_renders_zero():
    grid = gs.GridSpec((16, 16, 16))
    n = 10
    arrs = (np.full((n, 3), 500.0), np.zeros((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)),
            np.zeros(n), np.zeros(n))
    f = gs.GaussianField(*arrs)
    c = gs.Renderer(grid)(f)
    for k in ("S", "W", "I"):
        assert float(getattr(c, k).abs().max()) == 0.0, k


def test_renderer_slabs_reassemble_the_full_render():
    """Renderer(slab=...) -- the N>1 render path -- on pair-balanced brick-id
    ranges with mid-layer cuts: each slab's voxels match the whole-grid render
    (to f32 rounding: a slab may pick the other warp tiling when its pairs per
    Gaussian sit near the whole-brick threshold), and the slabs' pair counts
    add up exactly to the whole-grid count."""
    from paper_2603_09621_b200.distributed import pair_weights, slab_ranges, slab_voxel_mask
    p = make_problem(CONFIGS[1])
    f = gs.GaussianField(*p["field"])
    grid = p["hr_grid"]
    bd = (8, 8, 4)
    full = gs.Renderer(grid)
    I_full = np_(full(f).I).copy()
    P_full = full.pair_count()
    w = pair_weights(f, grid, gs.RenderOptions(), bd)
    slabs = slab_ranges(len(w), 3, weights=w)
    layer = (-(-grid.dims[0] // 8)) * (-(-grid.dims[1] // 8))
    assert any(b % layer for _, b in slabs[:-1])
    got = np.zeros_like(I_full)
    pairs = 0
    for slab in slabs:
        r = gs.Renderer(grid, slab=slab)
        c = r(f)
        own = slab_voxel_mask(grid, bd, slab)
        np.testing.assert_allclose(np_(c.I)[own], I_full[own], rtol=4e-6, atol=1e-9)
        assert not np_(c.I)[~own].any()          # voxels outside the slab stay zero
        got[own] = np_(c.I)[own]
        pairs += r.pair_count()
    np.testing.assert_allclose(got, I_full, rtol=4e-6, atol=1e-9)
    assert pairs == P_full == int(w.sum())


def test_backward_with_cache_of_other_precision():
    """forward(f32) then backward(f64 opts): the converted W and I must stay
    distinct buffers (a freed temporary can be reused for the next
    conversion).  Equals backward on explicitly converted copies."""
    grid, arrs = _sweep_field(100, 2)
    f = gs.GaussianField(*arrs)
    o32, o64 = gs.RenderOptions(), gs.RenderOptions(precision="f64")
    idx = gs.build_brick_index(f, grid, o32)
    c32 = gs.forward(f, grid, idx, o32)
    dl = np.random.default_rng(5).normal(size=grid.num_voxels)
    got = gs.backward(f, grid, idx, c32, dl, o64)
    conv = RenderCache(grid, c32.S.to(torch.float64).clone(), c32.W.to(torch.float64).clone(),
                       c32.I.to(torch.float64).clone(), c32.field_version)
    want = gs.backward(f, grid, idx, conv, dl, o64)
    for k in GRAD_KEYS:
        assert torch.equal(getattr(got, k), getattr(want, k)), k


def test_binning_workspace_is_per_stream():
    """Two build_brick_index calls in flight on two streams use separate CUB
    scratch (the workspace is keyed by stream), and both equal the
    sequential results."""
    from paper_2603_09621_b200 import _lib
    grid = gs.GridSpec((32, 32, 32), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    fa = gs.GaussianField(*random_field_arrays(3000, grid, 7, 0.4, 2.0))
    fb = gs.GaussianField(*random_field_arrays(2000, grid, 8, 0.4, 2.0))
    ia, ib = gs.build_brick_index(fa, grid), gs.build_brick_index(fb, grid)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1):
        ja = gs.build_brick_index(fa, grid)
    with torch.cuda.stream(s2):
        jb = gs.build_brick_index(fb, grid)
    torch.cuda.synchronize()
    assert torch.equal(ia.gids, ja.gids) and torch.equal(ia.starts, ja.starts)
    assert torch.equal(ib.gids, jb.gids) and torch.equal(ib.starts, jb.starts)
    keys = {k[1] for k in _lib._ws_cache if k[2] == "bin"}
    assert {s1.cuda_stream, s2.cuda_stream} <= keys
