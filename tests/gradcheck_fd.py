"""Finite-difference gradient checker -- TEST INFRASTRUCTURE, not product.

Restates the reference's validation harness (gradcheck.py:146-196) on top of
the CPU oracle: the "truth" derivative is the fourth-order central difference
(+/-h, +/-2h) of the loss evaluated through the oracle's float64 render, a
route independent of the CUDA kernels under test.  A coordinate whose stencil
points see a different structure -- a pair crossing the cutoff or a voxel
crossing the epsilon_w coverage floor (the census, gradcheck.py:55-91) -- is
excluded and counted, exactly as the reference does.  Quaternion probes
perturb the stored values without renormalising (gradcheck.py:22-25).

Only tests import this module.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np

import oracle

# reference group name -> attribute (gradcheck.py:45-53)
GROUP_ATTR = {
    "amplitude": "raw_amplitude",
    "relax": "raw_relax",
    "position": "positions",
    "scale": "log_scales",
    "rotation": "rotations",
}
PARAM_GROUPS = tuple(GROUP_ATTR)


@dataclass
class GroupResult:
    checked: int = 0
    excluded: int = 0
    below_floor: int = 0
    max_rel_error: float = 0.0


@dataclass
class Report:
    groups: dict = dc_field(default_factory=dict)
    rel_tol: float = 1e-4

    @property
    def max_rel_error(self) -> float:
        return max((g.max_rel_error for g in self.groups.values()), default=0.0)

    @property
    def passed(self) -> bool:
        return self.max_rel_error <= self.rel_tol

    def summary(self) -> dict:
        return {k: vars(v) for k, v in self.groups.items()}


def voxel_centres(dims, spacing, origin) -> np.ndarray:
    """(V, 3) voxel centres, linear x-fastest (volume.py's layout)."""
    ix, iy, iz = np.meshgrid(*(np.arange(d) for d in dims), indexing="ij")
    lin = np.stack([ix.ravel(order="F"), iy.ravel(order="F"), iz.ravel(order="F")], axis=1)
    return np.asarray(origin) + lin * np.asarray(spacing)


def census(fd: dict, centres: np.ndarray, cutoff: float, eps_w: float):
    """Per-voxel live-pair count and coverage flag (gradcheck.py:55-91)."""
    L = oracle.whitening_factors(fd["log_scales"], fd["rotations"])   # (N, 3, 3)
    _, r = oracle.activations(fd)
    d = centres[:, None, :] - fd["positions"][None, :, :]              # (V, N, 3)
    u = np.einsum("nij,vnj->vni", L, d)
    d2 = np.einsum("vni,vni->vn", u, u)
    live = d2 <= cutoff * cutoff
    W = np.where(live, np.exp(-0.5 * d2) * r[None, :], 0.0).sum(axis=1)
    return live.sum(axis=1), W >= eps_w


def fd_loss(fd: dict, grid, target_lin: np.ndarray, cutoff: float, eps_w: float,
            kind: str) -> float:
    """Loss of the oracle's float64 render against target_lin."""
    pred = oracle.render(fd, grid.dims, grid.spacing, grid.origin, cutoff=cutoff,
                         eps_w=eps_w, precision="f64")
    return oracle.loss_and_grad(pred, target_lin, kind)[0]


def run(fd: dict, grid, target_lin: np.ndarray, analytic: dict, *, cutoff: float = 3.0,
        eps_w: float = 1e-8, h: float = 1e-3, rel_tol: float = 1e-4,
        grad_floor: float = 1e-6, kind: str = "l2", groups=PARAM_GROUPS) -> Report:
    """Compare analytic[attr] (host float64 arrays, raw-parameter gradients)
    with the finite-difference derivative, coordinate by coordinate
    (gradcheck.py:146-196)."""
    centres = voxel_centres(grid.dims, grid.spacing, grid.origin)
    report = Report(rel_tol=rel_tol)
    for name in groups:
        attr = GROUP_ATTR[name]
        ana = np.asarray(analytic[attr], dtype=np.float64)
        res = GroupResult()
        for index in np.ndindex(ana.shape):
            losses, lives, covs = [], [], []
            for step in (-2.0, -1.0, 1.0, 2.0):
                probe = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in fd.items()}
                probe[attr][index] += step * h
                lv, cv = census(probe, centres, cutoff, eps_w)
                losses.append(fd_loss(probe, grid, target_lin, cutoff, eps_w, kind))
                lives.append(lv)
                covs.append(cv)
            if (any(not np.array_equal(lives[0], x) for x in lives[1:])
                    or any(not np.array_equal(covs[0], x) for x in covs[1:])):
                res.excluded += 1
                continue
            lmm, lm, lp, lpp = losses
            fdv = (lmm - 8.0 * lm + 8.0 * lp - lpp) / (12.0 * h)
            an = float(ana[index])
            scale = max(abs(an), abs(fdv))
            if scale <= grad_floor:
                res.below_floor += 1
                continue
            res.checked += 1
            res.max_rel_error = max(res.max_rel_error, abs(an - fdv) / scale)
        report.groups[name] = res
    return report
