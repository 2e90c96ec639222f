"""Setup of a fit on the device: trilinear resampling
(volume.py:126-154) bit-identical to the reference's numpy order, and
init_from_volume (field.py:212-234) with every array but the amplitude
logit bit-identical (the logit within a few ulp: device log vs glibc)."""

import numpy as np
import pytest
import torch

import paper_2603_09621_b200 as gs
from paper_2603_09621_b200.field import init_arrays_from_volume
from paper_2603_09621_b200.synth import CONFIGS, make_problem
from paper_2603_09621_b200.volume import GridSpec, grid_covering_extent, resample_trilinear_np

pytestmark = pytest.mark.gpu


def _cases():
    p = make_problem(CONFIGS[1])
    rng = np.random.default_rng(4)
    g1 = GridSpec((13, 7, 9), (0.9, 1.3, 2.1), (-1.0, 0.5, 3.0))
    v64 = rng.uniform(size=g1.dims)
    g2 = GridSpec((29, 5, 1), (0.4, 2.0, 1.0), (-1.5, 0.0, 3.5))
    return [
        ("c1 HR->LR (the benchmark degrade)", p["hr"], p["hr_grid"], p["lr_grid"]),
        ("c1 LR->HR", p["lr"], p["lr_grid"], p["hr_grid"]),
        ("f64 anisotropic down", v64, g1, grid_covering_extent(g1, (5, 11, 4))),
        ("f64 up, one-voxel axis", v64, g1, g2),
        ("f32 single voxel source", rng.uniform(size=(1, 1, 1)).astype(np.float32),
         GridSpec((1, 1, 1)), GridSpec((3, 2, 4), (0.5, 0.5, 0.5), (-0.5, 0.0, 0.25))),
    ]


@pytest.mark.parametrize("i", range(5))
def test_resample_trilinear_bit_identical(i):
    name, data, src, dst = _cases()[i]
    want = resample_trilinear_np(data, src, dst)
    got = gs.resample_trilinear(gs.Volume(src, data), dst)
    assert got.data.dtype == (torch.float64 if data.dtype == np.float64 else torch.float32)
    np.testing.assert_array_equal(got.numpy(), want, err_msg=name)


@pytest.mark.parametrize("case", ["c1", "c4", "threshold"])
def test_init_from_volume_on_device(case):
    if case == "threshold":
        rng = np.random.default_rng(7)
        grid = GridSpec((11, 9, 6), (1.5, 1.0, 2.0), (0.0, -2.0, 1.0))
        data = rng.uniform(size=grid.dims)
        cfg = gs.InitConfig(background_threshold=0.4, scale_factor=0.6, relax_init=0.8)
    else:
        p = make_problem(CONFIGS[1 if case == "c1" else 4])
        grid, data, cfg = p["lr_grid"], p["lr"], gs.InitConfig(background_threshold=0.0)
    want = init_arrays_from_volume(data, grid, cfg)
    f = gs.init_from_volume(gs.Volume(grid, data), cfg, on_device=True)
    got = [getattr(f, k).cpu().numpy() for k in
           ("positions", "log_scales", "rotations", "raw_amplitude", "raw_relax")]
    assert f.count == want[0].shape[0]
    for k in (0, 1, 2, 4):
        np.testing.assert_array_equal(got[k], want[k])
    ulp = np.abs(got[3] - want[3]) / np.spacing(np.abs(want[3]))
    assert ulp.max() <= 4, ulp.max()


# ------------------------------------------------ phantom (phantom.py:52-75)
@pytest.mark.parametrize("dims,sigma,seed", [((64, 64, 64), 0.7, 11), ((37, 20, 9), 1.3, 3),
                                             ((256, 256, 128), 0.7, 11), ((5, 3, 2), 2.5, 7),
                                             ((24, 24, 24), 0.0, 5)])
def test_phantom_ellipsoids_bit_identical(dims, sigma, seed):
    """The device phantom (rasterization, scipy's gaussian_filter order with
    reflect edges, clip, float32) equals the host restatement bit for bit,
    which in turn equals the reference (tests/test_oracle_golden.py)."""
    from paper_2603_09621_b200.synth import (generate_ellipsoids, generate_phantom_device,
                                             random_ellipsoids)
    g = GridSpec(dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    prims = random_ellipsoids(g, seed)
    want = generate_ellipsoids(prims, g, smooth_sigma=sigma)
    got = gs.Volume.from_linear(g, generate_phantom_device(prims, g, sigma)).numpy()
    np.testing.assert_array_equal(got, want)


def test_phantom_gaussian_mixture_matches_reference_formula():
    from scipy import ndimage
    from paper_2603_09621_b200.synth import generate_phantom_device

    class Blob:
        def __init__(self, c, s, i):
            self.center, self.sigmas, self.intensity = c, s, i

    g = GridSpec((33, 21, 17), (0.8, 1.1, 1.5), (-2.0, 1.0, 0.5))
    rng = np.random.default_rng(2)
    lo, hi = (np.asarray(a) for a in g.extent())
    blobs = [Blob(tuple(lo + (hi - lo) * rng.uniform(0.2, 0.8, 3)),
                  tuple((hi - lo) * rng.uniform(0.05, 0.15, 3)), float(rng.uniform(0.3, 1.0)))
             for _ in range(5)]
    xs, ys, zs = (g.axis_coords(k) for k in range(3))
    xs, ys, zs = xs[:, None, None], ys[None, :, None], zs[None, None, :]
    want = np.zeros(g.dims)
    for b in blobs:
        (cx, cy, cz), (sx, sy, sz) = b.center, b.sigmas
        d2 = ((xs - cx) / sx) ** 2 + ((ys - cy) / sy) ** 2 + ((zs - cz) / sz) ** 2
        np.maximum(want, b.intensity * np.exp(-0.5 * d2), out=want)
    want = np.clip(ndimage.gaussian_filter(want, sigma=0.9), 0.0, 1.0).astype(np.float32)
    got = gs.Volume.from_linear(g, generate_phantom_device(blobs, g, 0.9,
                                                           kind="gaussian-mixture")).numpy()
    # exp on the device vs numpy: within an ulp before the blur
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-7)


@pytest.mark.parametrize("cid", [1, 2])
def test_make_problem_on_device_identical(cid):
    from paper_2603_09621_b200.synth import sha256
    a = make_problem(CONFIGS[cid])
    b = make_problem(CONFIGS[cid], device=torch.device("cuda", 0))
    assert sha256(a["hr"]) == sha256(b["hr"]) and sha256(a["lr"]) == sha256(b["lr"])
    assert sha256(*a["field"]) == sha256(*b["field"])
