"""Device geometry helpers of the reference API: rotation_matrices
(field.py:141-154), field_sigma_inv (render.py:67-71) and weight
(render.py:74-81), with the reference's weight KATs (test_render.py:34-57)."""

import math

import numpy as np
import pytest
import torch

import paper_2603_09621_b200 as gs
from paper_2603_09621_b200.field import random_field_arrays, rotation_matrices
from paper_2603_09621_b200.render import field_sigma_inv, weight

pytestmark = pytest.mark.gpu


def _single(mu, log_scale=0.0, amplitude_raw=0.0):
    return gs.GaussianField(np.array([mu], float), np.full((1, 3), log_scale),
                            np.array([[1.0, 0.0, 0.0, 0.0]]), np.array([amplitude_raw]),
                            np.array([20.0]))


def _np_rotation_matrices(q):
    """field.py:141-154, the reference formula."""
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    out = np.empty((q.shape[0], 3, 3))
    out[:, 0, 0] = 1 - 2 * (y * y + z * z)
    out[:, 0, 1] = 2 * (x * y - w * z)
    out[:, 0, 2] = 2 * (x * z + w * y)
    out[:, 1, 0] = 2 * (x * y + w * z)
    out[:, 1, 1] = 1 - 2 * (x * x + z * z)
    out[:, 1, 2] = 2 * (y * z - w * x)
    out[:, 2, 0] = 2 * (x * z - w * y)
    out[:, 2, 1] = 2 * (y * z + w * x)
    out[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return out


def test_rotation_matrices_bit_exact_and_verbatim():
    rng = np.random.default_rng(4)
    q = rng.normal(size=(257, 4))          # not normalised: applied verbatim
    np.testing.assert_array_equal(rotation_matrices(q).cpu().numpy(), _np_rotation_matrices(q))


def test_field_sigma_inv_matches_reference_formula():
    grid = gs.GridSpec((16, 16, 16))
    arrs = random_field_arrays(300, grid, seed=9)
    f = gs.GaussianField(*arrs)
    r = _np_rotation_matrices(arrs[2])
    ref = np.einsum("nab,nb,ncb->nac", r, np.exp(-2.0 * arrs[1]), r)
    np.testing.assert_allclose(field_sigma_inv(f).cpu().numpy(), ref, rtol=1e-14, atol=1e-15)


def test_weight_kats():
    f = _single([0.0, 0.0, 0.0])
    r = 1.0 / (1.0 + math.exp(-20.0))
    assert weight(f, 0, [0.0, 0.0, 0.0]) == pytest.approx(r, abs=1e-8)
    assert weight(f, 0, [1.0, 0.0, 0.0]) == pytest.approx(math.exp(-0.5) * r, rel=1e-8)
    assert weight(f, 0, [3.5, 0.0, 0.0], gs.RenderOptions(cutoff_sigma=3.0)) == 0.0
    assert weight(f, 0, [2.99, 0.0, 0.0], gs.RenderOptions(cutoff_sigma=3.0)) > 0.0
    with torch.no_grad():
        f.raw_relax[:] = 0.0               # r = 0.5
    assert weight(f, 0, [1.0, 0.0, 0.0]) == pytest.approx(0.5 * math.exp(-0.5), rel=1e-8)
    f.relax_enabled = False                # r = 1
    assert weight(f, 0, [1.0, 0.0, 0.0]) == pytest.approx(math.exp(-0.5), rel=1e-12)


def test_weight_anisotropic_matches_reference_formula():
    grid = gs.GridSpec((16, 16, 16))
    arrs = random_field_arrays(50, grid, seed=2)
    f = gs.GaussianField(*arrs)
    r = _np_rotation_matrices(arrs[2])
    sig = np.einsum("nab,nb,ncb->nac", r, np.exp(-2.0 * arrs[1]), r)
    rng = np.random.default_rng(1)
    for i in range(0, 50, 7):
        p = arrs[0][i] + rng.normal(scale=2.0, size=3)
        d = p - arrs[0][i]
        d2 = float(d @ sig[i] @ d)
        relax = 1.0 / (1.0 + math.exp(-arrs[4][i]))
        ref = 0.0 if d2 > 9.0 else math.exp(-0.5 * d2) * relax
        assert weight(f, i, p) == pytest.approx(ref, rel=1e-12, abs=1e-300)
    with pytest.raises(gs._lib.GsvLibraryError if hasattr(gs, "_lib") else Exception):
        weight(f, 50, [0.0, 0.0, 0.0])
