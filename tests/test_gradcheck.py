"""Analytic-vs-finite-difference agreement (reference tests/test_gradients.py).

The CPU half checks the harness (tests/gradcheck_fd.py) on the oracle's own
backward; the GPU half runs the same cases through the CUDA engine behind the
public API (build_brick_index -> forward -> loss_and_grad -> backward), f64
at the reference's 1e-4 bar and f32 at its 1e-2 bar (test_gradients.py:21-68).
"""

import numpy as np
import pytest

import oracle
from paper_2603_09621_b200.field import random_field_arrays
from paper_2603_09621_b200.volume import GridSpec

import gradcheck_fd as gc
from conftest import field_dict

UNIT = GridSpec((8, 8, 8), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
# all coordinates per group for N Gaussians (test_gradients.py:38-39)
SIZES = {"amplitude": 1, "relax": 1, "position": 3, "scale": 3, "rotation": 4}


def _uniform_target(seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(size=UNIT.dims).ravel(order="F")


def _oracle_analytic(fd, target, cutoff=3.0, kind="l2", precision="f64"):
    st, gi = oracle.build_index(fd, UNIT.dims, UNIT.spacing, UNIT.origin, (8, 8, 4), cutoff)
    S, W, I = oracle.forward(fd, UNIT.dims, UNIT.spacing, UNIT.origin, st, gi, cutoff=cutoff,
                             precision=precision)
    _, dl = oracle.loss_and_grad(I, target, kind)
    return oracle.backward(fd, UNIT.dims, UNIT.spacing, UNIT.origin, st, gi, W, I, dl,
                           cutoff=cutoff, precision=precision)


def _check_all(report, n=None, full=False):
    assert set(report.groups) == set(gc.PARAM_GROUPS)
    for name, g in report.groups.items():
        assert g.checked > 0, (name, report.summary())
        if full:
            assert g.excluded == 0, name
            assert g.checked + g.below_floor == SIZES[name] * n, name
    assert report.passed, report.summary()


# ------------------------------------------------------------- CPU: harness
def test_oracle_backward_agrees_with_finite_differences():
    fd = field_dict(random_field_arrays(8, UNIT, 7))
    tgt = _uniform_target(8)
    rep = gc.run(fd, UNIT, tgt, _oracle_analytic(fd, tgt), h=1e-3, rel_tol=1e-4)
    _check_all(rep)


def test_census_excludes_cutoff_crossings():
    # a wide stencil on narrow kernels must straddle the 3-sigma cutoff for
    # some coordinates; those are excluded rather than compared
    fd = field_dict(random_field_arrays(6, UNIT, 3, scale_lo=0.5))
    tgt = _uniform_target(4)
    rep = gc.run(fd, UNIT, tgt, _oracle_analytic(fd, tgt), h=5e-2, rel_tol=1.0,
                 groups=("position",))
    assert rep.groups["position"].excluded > 0


def test_harness_detects_a_wrong_gradient():
    fd = field_dict(random_field_arrays(4, UNIT, 5))
    tgt = _uniform_target(6)
    ana = _oracle_analytic(fd, tgt)
    ana["log_scales"] = ana["log_scales"] * 1.01
    rep = gc.run(fd, UNIT, tgt, ana, groups=("scale",))
    assert not rep.passed


# ------------------------------------------------------------- GPU: CUDA engine
def _cuda_analytic(fd, target, opts, kind="l2"):
    import paper_2603_09621_b200 as gs
    f = gs.GaussianField(*(fd[k] for k in ("positions", "log_scales", "rotations",
                                             "raw_amplitude", "raw_relax")))
    idx = gs.build_brick_index(f, UNIT, opts)
    cache = gs.forward(f, UNIT, idx, opts)
    tv = gs.Volume(UNIT, target.reshape(UNIT.dims, order="F"))
    _, dl = gs.loss_and_grad(cache.volume(), tv, kind)
    g = gs.backward(f, UNIT, idx, cache, dl, opts)
    return {k: getattr(g, k).detach().cpu().numpy().astype(np.float64)
            for k in ("raw_amplitude", "raw_relax", "positions", "log_scales", "rotations")}


@pytest.mark.gpu
def test_gpu_gradcheck_all_groups_within_tolerance():
    import paper_2603_09621_b200 as gs
    fd = field_dict(random_field_arrays(20, UNIT, 7))
    tgt = _uniform_target(8)
    ana = _cuda_analytic(fd, tgt, gs.RenderOptions(precision="f64"))
    _check_all(gc.run(fd, UNIT, tgt, ana, h=1e-3, rel_tol=1e-4))


@pytest.mark.gpu
def test_gpu_gradcheck_without_truncation():
    import paper_2603_09621_b200 as gs
    fd = field_dict(random_field_arrays(8, UNIT, 9))
    tgt = _uniform_target(10)
    ana = _cuda_analytic(fd, tgt, gs.RenderOptions(cutoff_sigma=np.inf, precision="f64"))
    _check_all(gc.run(fd, UNIT, tgt, ana, cutoff=np.inf), n=8, full=True)


@pytest.mark.gpu
def test_gpu_gradcheck_sharp_kernels():
    import paper_2603_09621_b200 as gs
    fd = field_dict(random_field_arrays(20, UNIT, 3, scale_lo=0.5))
    tgt = _uniform_target(4)
    ana = _cuda_analytic(fd, tgt, gs.RenderOptions(precision="f64"))
    rep = gc.run(fd, UNIT, tgt, ana)
    assert rep.passed, rep.summary()


@pytest.mark.gpu
def test_gpu_gradcheck_l1_loss():
    # offset target keeps every residual's sign fixed under the probes
    import paper_2603_09621_b200 as gs
    fd = field_dict(random_field_arrays(6, UNIT, 11))
    base = oracle.render(fd, UNIT.dims, UNIT.spacing, UNIT.origin, precision="f64")
    tgt = base + 0.2
    ana = _cuda_analytic(fd, tgt, gs.RenderOptions(precision="f64"), kind="l1")
    rep = gc.run(fd, UNIT, tgt, ana, kind="l1")
    assert rep.passed, rep.summary()


@pytest.mark.gpu
def test_gpu_gradcheck_f32_engine():
    # float32 accumulators under test, float64 finite differences as truth
    import paper_2603_09621_b200 as gs
    fd = field_dict(random_field_arrays(12, UNIT, 13))
    tgt = _uniform_target(14)
    ana = _cuda_analytic(fd, tgt, gs.RenderOptions(precision="f32"))
    rep = gc.run(fd, UNIT, tgt, ana, rel_tol=1e-2)
    assert rep.passed, rep.summary()


@pytest.mark.gpu
def test_gpu_single_gaussian_geometry_gradients_vanish():
    # one Gaussian: the normalized image is its amplitude wherever covered,
    # so geometry and relaxation cannot change the loss (test_gradients.py:71-83)
    import paper_2603_09621_b200 as gs
    fd = field_dict(random_field_arrays(1, UNIT, 15))
    f = gs.GaussianField(*(fd[k] for k in ("positions", "log_scales", "rotations",
                                             "raw_amplitude", "raw_relax")))
    opts = gs.RenderOptions(precision="f64")
    idx = gs.build_brick_index(f, UNIT, opts)
    cache = gs.forward(f, UNIT, idx, opts)
    dl = np.random.default_rng(16).normal(size=UNIT.num_voxels)
    g = gs.backward(f, UNIT, idx, cache, dl, opts)
    for k in ("positions", "log_scales", "rotations", "raw_relax"):
        assert float(getattr(g, k).abs().max()) < 1e-12, k
    assert float(g.raw_amplitude.abs().max()) > 1e-6
