"""The LR-consistency training mode (lrc.py; the north_star's HR render +
downsample + L1 epilogue, an extra without a reference counterpart) against
the same objective composed from the public API: forward at the HR grid,
block means and the loss in torch, backward with that dL/dI."""

import numpy as np
import pytest
import torch

import paper_2603_09621_b200 as gs
from paper_2603_09621_b200.field import random_field_arrays
from paper_2603_09621_b200.lrc import LRConsistencyStep, hr_grid_for
from paper_2603_09621_b200.synth import CONFIGS, make_problem

from conftest import GRAD_KEYS

pytestmark = pytest.mark.gpu


def _composed(f, lr, factors, kind):
    hr = hr_grid_for(lr.grid, factors)
    idx = gs.build_brick_index(f, hr)
    c = gs.forward(f, hr, idx)
    fx, fy, fz = factors
    nx, ny, nz = lr.grid.dims
    I = c.I.to(torch.float64).view(nz, fz, ny, fy, nx, fx)
    pred = I.mean(dim=(1, 3, 5)).reshape(-1)
    d = pred - lr.linear().to(torch.float64)
    v = d.numel()
    if kind == "l1":
        loss, dl = float(d.abs().mean()), torch.sign(d) / v
    else:
        loss, dl = float((d * d).mean()), 2.0 * d / v
    dl_hr = dl.view(nz, 1, ny, 1, nx, 1).expand(nz, fz, ny, fy, nx, fx).reshape(-1) / (fx * fy * fz)
    return loss, gs.backward(f, hr, idx, c, dl_hr.contiguous())


@pytest.mark.parametrize("case", ["c1_x2", "aniso_z4_l2"])
def test_lr_consistency_matches_composed_objective(case):
    if case == "c1_x2":
        p = make_problem(CONFIGS[1])
        lr = gs.Volume(p["lr_grid"], p["lr"])
        arrs, factors, kind = p["field"], (2, 2, 2), "l1"
        assert hr_grid_for(lr.grid, factors) == p["hr_grid"]
    else:
        g = gs.GridSpec((16, 16, 8), (1.0, 1.0, 4.0), (0.0, 0.0, 1.5))
        rng = np.random.default_rng(2)
        lr = gs.Volume(g, rng.uniform(size=g.dims))
        arrs, factors, kind = random_field_arrays(600, g, 4, 0.5, 2.5), (1, 1, 4), "l2"
    f = gs.GaussianField(*arrs)
    step = LRConsistencyStep(lr, factors, loss=kind)
    loss, g1 = step.gradients(f)
    loss_ref, g2 = _composed(f, lr, factors, kind)
    assert abs(loss - loss_ref) <= 1e-12 * max(1.0, abs(loss_ref)), (loss, loss_ref)
    for k in GRAD_KEYS:
        a, b = getattr(g1, k).cpu().numpy(), getattr(g2, k).cpu().numpy()
        assert np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(b) + 1e-20, k


def test_lr_consistency_steps_reduce_the_loss():
    p = make_problem(CONFIGS[1])
    lr = gs.Volume(p["lr_grid"], p["lr"])
    f = gs.GaussianField(*p["field"])
    st = gs.AdamState.create(f)
    lrs = gs.FitConfig().resolved_lrs(lr.grid.spacing)
    step = LRConsistencyStep(lr, (2, 2, 2))
    losses = [step.step(f, st, lrs) for _ in range(20)]
    assert st.t == 20 and losses[-1] < 0.8 * losses[0], losses
