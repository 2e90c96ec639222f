"""Device PSNR / SSIM3D (paper_2603_09621_b200.metrics) against the
reference's own values (tests/golden/metrics.json, from gsvol.metrics via
tests/golden/make_golden.py) and its documented properties (metrics.py:1-100)."""

import math

import numpy as np
import pytest

import paper_2603_09621_b200 as gs

from conftest import load_json

pytestmark = pytest.mark.gpu

CASES = load_json("metrics.json")["cases"]


def _pair(case):
    rng = np.random.default_rng(case["seed"])
    dims = tuple(case["dims"])
    a = rng.uniform(0.0, 1.0, size=dims)
    noise = case["noise"]
    b = np.clip(a + noise * rng.standard_normal(dims), 0.0, 1.0) if noise else a.copy()
    g = gs.GridSpec(dims)
    return gs.Volume(g, a.astype(case["dtype"])), gs.Volume(g, b.astype(case["dtype"]))


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"seed{c['seed']}")
def test_metrics_match_reference(case):
    x, y = _pair(case)
    p, s = gs.psnr(x, y), gs.ssim3d(x, y)
    if case["psnr"] is None:
        assert math.isinf(p)
    else:
        assert abs(p - case["psnr"]) <= 1e-9, (p, case["psnr"])
    # f64 like the reference; only the summation order differs
    assert abs(s - case["ssim"]) <= 1e-12, (s, case["ssim"])
    rep = gs.MetricReport.evaluate(x, y)
    assert rep.identical == (case["psnr"] is None)
    js = rep.to_json()
    assert js["grid"]["dims"] == case["dims"] and js["ssim"] == rep.ssim


def test_ssim_of_identical_volumes_is_exactly_one():
    """metrics.py:6-9: sigma_xy uses the same arithmetic as sigma_x^2."""
    rng = np.random.default_rng(5)
    v = gs.Volume(gs.GridSpec((12, 20, 15)), rng.uniform(0, 1, (12, 20, 15)).astype(np.float32))
    assert gs.ssim3d(v, v) == 1.0
    assert math.isinf(gs.psnr(v, v))


def test_metric_errors_match_reference():
    a = gs.Volume(gs.GridSpec((12, 12, 12)), np.zeros((12, 12, 12), np.float32))
    b = gs.Volume(gs.GridSpec((12, 12, 13)), np.zeros((12, 12, 13), np.float32))
    with pytest.raises(gs.GridMismatchError, match="metric inputs on different grids"):
        gs.psnr(a, b)
    with pytest.raises(gs.GridMismatchError, match="metric inputs on different grids"):
        gs.ssim3d(a, b)
    small = gs.Volume(gs.GridSpec((10, 12, 12)), np.zeros((10, 12, 12), np.float32))
    with pytest.raises(ValueError, match="volume too small for SSIM window"):
        gs.ssim3d(small, small)


def test_metrics_are_deterministic_at_256():
    rng = np.random.default_rng(9)
    g = gs.GridSpec((256, 256, 256))
    a = rng.uniform(0, 1, g.dims).astype(np.float32)
    b = np.clip(a + 0.02 * rng.standard_normal(g.dims), 0, 1).astype(np.float32)
    x, y = gs.Volume(g, a), gs.Volume(g, b)
    s1, s2 = gs.ssim3d(x, y), gs.ssim3d(x, y)
    p1, p2 = gs.psnr(x, y), gs.psnr(x, y)
    assert s1 == s2 and p1 == p2
    d = a.astype(np.float64) - b.astype(np.float64)
    assert abs(p1 - 10 * math.log10(1.0 / float((d * d).mean()))) <= 1e-9
