"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nb_golden \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz / *.json.  Every array the CUDA path must match
bit-exactly is stored as a sha256 (tiny); tolerance-compared arrays are stored
as float32 where small.  The synthetic inputs are rebuilt with this repo's
host restatement (paper_2603_09621_b200.synth) and checked against the
reference's own generator, so the GPU box (which has no reference) rebuilds
identical inputs.
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import gsvol  # noqa: E402  (the reference)
from gsvol import (GridSpec, InitConfig, RenderOptions, backward, build_brick_index,  # noqa: E402
                   forward, init_from_volume, loss_and_grad, random_field)
from gsvol.phantom import generate_phantom, random_phantom  # noqa: E402
from gsvol.volume import grid_covering_extent, resample_trilinear  # noqa: E402

from paper_2603_09621_b200 import synth  # noqa: E402
from paper_2603_09621_b200.field import random_field_arrays  # noqa: E402

sha = synth.sha256
F = ("positions", "log_scales", "rotations", "raw_amplitude", "raw_relax")
G = ("raw_amplitude", "raw_relax", "positions", "log_scales", "rotations")

SWEEP_GRIDS = [((8, 8, 8), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)),
               ((16, 16, 16), (0.7, 1.0, 1.3), (-2.0, 0.0, 1.0)),
               ((32, 24, 16), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0)),
               ((32, 32, 32), (0.5, 0.5, 0.5), (1.0, 1.0, 1.0)),
               ((24, 24, 24), (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))]


def versions():
    import numba
    import scipy
    return {"python": platform.python_version(), "numpy": np.__version__,
            "scipy": scipy.__version__, "numba": numba.__version__,
            "reference": "gsvol " + gsvol.__version__, "machine": platform.machine()}


def field_sha(f):
    return sha(*(getattr(f, k) for k in F))


def sweep():
    """test_acceptance.py:40-66 cases x precisions x brick dims: reference hashes."""
    out = []
    for n in (1, 10, 100, 1000):
        for i, (dims, sp, org) in enumerate(SWEEP_GRIDS):
            grid = GridSpec(dims, sp, org)
            seed = 100 * n + i
            f = random_field(n, grid, seed=seed, scale_lo=0.4, scale_hi=2.0)
            mine = random_field_arrays(n, grid, seed, 0.4, 2.0)
            assert sha(*mine) == field_sha(f), "random_field restatement differs"
            dl = np.random.default_rng(5).normal(size=grid.num_voxels)
            for bd in ((8, 8, 4), (8, 8, 8), (4, 4, 4)):
                for prec in ("f32", "f64"):
                    opts = RenderOptions(precision=prec)
                    idx = build_brick_index(f, grid, opts, bd)
                    c = forward(f, grid, idx, opts)
                    gr = backward(f, grid, idx, c, dl, opts)
                    out.append({"n": n, "grid": i, "seed": seed, "brick_dims": bd,
                                "precision": prec, "pairs": idx.pair_count,
                                "starts": sha(idx.starts), "gids": sha(idx.gids),
                                "S": sha(c.S), "W": sha(c.W), "I": sha(c.I),
                                "grads": sha(*(getattr(gr, k) for k in G)),
                                "I_sum": float(np.sum(c.I, dtype=np.float64))})
    return out


def problem(cfg_id):
    cfg = synth.CONFIGS[cfg_id]
    hr_grid = GridSpec(cfg.hr_dims, (1.0, 1.0, 1.0), (0.0, 0.0, 0.0))
    hr = generate_phantom(random_phantom("ellipsoids", hr_grid, seed=11), hr_grid,
                          smooth_sigma=0.7)
    lr = resample_trilinear(hr, grid_covering_extent(hr_grid, cfg.lr_dims))
    f = init_from_volume(lr, InitConfig(background_threshold=0.0))
    mine = synth.make_problem(cfg)
    assert sha(mine["hr"]) == sha(hr.data), "phantom restatement differs"
    assert sha(mine["lr"]) == sha(lr.data), "degrade restatement differs"
    assert (mine["lr_grid"].dims, mine["lr_grid"].spacing, mine["lr_grid"].origin) == (lr.grid.dims, lr.grid.spacing, lr.grid.origin)
    if cfg.jitter:
        arrs = mine["field"]
        f = gsvol.GaussianField(*arrs)
    assert sha(*mine["field"]) == field_sha(f), "init restatement differs"
    return cfg, hr, lr, f, mine


def config1():
    cfg, hr, lr, f, mine = problem(1)
    opts = RenderOptions()
    out = {}
    idx = build_brick_index(f, lr.grid, opts)
    c = forward(f, lr.grid, idx, opts)
    loss, dl = loss_and_grad(c.volume(), lr, "l1")
    gr = backward(f, lr.grid, idx, c, dl, opts)
    idx_hr = build_brick_index(f, hr.grid, opts)
    c_hr = forward(f, hr.grid, idx_hr, opts)
    arrays = {
        "lr_starts": idx.starts, "lr_gids": idx.gids.astype(np.int32),
        "lr_I": c.I, "lr_W": c.W, "hr_I": c_hr.I,
        "dl": dl.astype(np.float32) * lr.grid.num_voxels,  # sign(d) in {-1,0,1}
    }
    for k in G:
        arrays["grad_" + k] = getattr(gr, k)
    out.update({"loss": loss, "lr_pairs": idx.pair_count, "hr_pairs": idx_hr.pair_count,
                "lr_starts": sha(idx.starts), "lr_gids": sha(idx.gids),
                "hr_starts": sha(idx_hr.starts), "hr_gids": sha(idx_hr.gids),
                "lr_volume": sha(lr.data), "field": field_sha(f),
                "lr_I": sha(c.I), "hr_I": sha(c_hr.I)})
    # f64 engine on the same inputs
    o64 = RenderOptions(precision="f64")
    i64 = build_brick_index(f, lr.grid, o64)
    c64 = forward(f, lr.grid, i64, o64)
    arrays["lr_I64"] = c64.I
    return out, arrays


def fit_quality(iterations=200):
    """Reference fit on the config-1 phantom, threshold 0."""
    from gsvol.metrics import psnr, ssim3d
    from gsvol.optimize import FitConfig, fit
    cfg, hr, lr, f0, mine = problem(1)
    t0 = time.perf_counter()
    f, report = fit(lr, InitConfig(background_threshold=0.0), FitConfig(iterations=iterations))
    t = time.perf_counter() - t0
    idx = build_brick_index(f, hr.grid, RenderOptions())
    sr = forward(f, hr.grid, idx, RenderOptions()).volume()
    return {"iterations": iterations, "psnr": psnr(sr, hr), "ssim": ssim3d(sr, hr),
            "losses_head": report.losses[:20], "final_loss": report.final["loss"],
            "seconds": t, "trilinear_psnr": psnr(resample_trilinear(lr, hr.grid), hr),
            "trilinear_ssim": ssim3d(resample_trilinear(lr, hr.grid), hr)}


METRIC_CASES = [  # (seed, dims, dtype, noise): seeded volume pairs for metrics.py
    (11, (16, 16, 16), "float32", 0.05),
    (12, (11, 13, 17), "float64", 0.2),
    (13, (32, 24, 20), "float32", 0.01),
    (14, (24, 24, 24), "float64", 0.0),      # identical: PSNR inf, SSIM 1
]


def metric_pair(seed, dims, dtype, noise):
    """The inputs of one metric case, rebuilt identically on the GPU box."""
    rng = np.random.default_rng(seed)
    a = rng.uniform(0.0, 1.0, size=dims)
    b = np.clip(a + noise * rng.standard_normal(dims), 0.0, 1.0) if noise else a.copy()
    return a.astype(dtype), b.astype(dtype)


def metrics():
    """Reference psnr / ssim3d (metrics.py:35-77) on seeded volume pairs."""
    from gsvol import Volume
    from gsvol.metrics import psnr, ssim3d
    out = []
    for seed, dims, dt, noise in METRIC_CASES:
        a, b = metric_pair(seed, dims, dt, noise)
        g = GridSpec(dims)
        va, vb = Volume(g, a), Volume(g, b)
        p = psnr(va, vb)
        out.append({"seed": seed, "dims": list(dims), "dtype": dt, "noise": noise,
                    "psnr": None if p == float("inf") else p, "ssim": ssim3d(va, vb)})
    return out


IO_DIR = os.path.join(HERE, "io")


def volume_io():
    """Files written by the reference's save_volume (raw_json, NIfTI-1), and a
    big-endian int16 NIfTI with scl_slope/scl_inter read by its load_volume."""
    import hashlib
    import struct
    from gsvol import Volume
    from gsvol.volume import load_volume, save_volume
    os.makedirs(IO_DIR, exist_ok=True)
    rng = np.random.default_rng(17)
    g = GridSpec((7, 5, 4), (0.8, 1.1, 2.5), (-3.0, 0.25, 10.0))
    v = Volume(g, rng.uniform(0.0, 1.0, g.dims).astype(np.float32))
    save_volume(v, os.path.join(IO_DIR, "ref.json"))
    save_volume(v, os.path.join(IO_DIR, "ref.nii"))
    # int16, big endian, slope 0.5 intercept -2, identity qform with offsets
    h = bytearray(348)
    struct.pack_into(">i", h, 0, 348)
    struct.pack_into(">8h", h, 40, 3, 6, 4, 3, 1, 1, 1, 1)
    struct.pack_into(">h", h, 70, 4)
    struct.pack_into(">h", h, 72, 16)
    struct.pack_into(">8f", h, 76, 1.0, 1.5, 2.0, 0.5, 0, 0, 0, 0)
    struct.pack_into(">f", h, 108, 352.0)
    struct.pack_into(">f", h, 112, 0.5)
    struct.pack_into(">f", h, 116, -2.0)
    struct.pack_into(">h", h, 252, 1)
    struct.pack_into(">3f", h, 268, 1.0, -2.0, 3.0)
    struct.pack_into(">4s", h, 344, b"n+1\x00")
    vals = rng.integers(-300, 300, size=6 * 4 * 3).astype(">i2")
    with open(os.path.join(IO_DIR, "i16_be.nii"), "wb") as fh:
        fh.write(bytes(h) + bytes(4) + vals.tobytes())
    w = load_volume(os.path.join(IO_DIR, "i16_be.nii"))
    import tempfile
    from gsvol.errors import FormatError
    sys.path.insert(0, HERE)
    import io_cases
    errors, accepted = {}, {}
    with tempfile.TemporaryDirectory() as td:
        for name, make in io_cases.cases(IO_DIR).items():
            p = make(td)
            try:
                load_volume(p)
                errors[name] = None
            except FormatError as exc:
                errors[name] = str(exc).replace(p, "<path>").replace(
                    os.path.join(td, "case.bin"), "<bin>")
        for name, make in io_cases.accepted(IO_DIR).items():
            a = load_volume(make(td))
            accepted[name] = {"spacing": list(a.grid.spacing), "origin": list(a.grid.origin),
                              "sha256": hashlib.sha256(
                                  np.ascontiguousarray(a.linear(), "<f4").tobytes()).hexdigest()}
    from gsvol.field import load_field as ref_load_field, random_field as ref_random_field
    from gsvol.field import save_field as ref_save_field
    fl = ref_random_field(9, g, seed=23)
    fl.raw_relax[:] = np.linspace(-2.0, 2.0, 9)
    ref_save_field(fl, os.path.join(IO_DIR, "ref_relax.gsv"))
    fl.relax_enabled = False
    ref_save_field(fl, os.path.join(IO_DIR, "ref_norelax.gsv"))
    back = ref_load_field(os.path.join(IO_DIR, "ref_relax.gsv"))
    field_values = {k: np.asarray(getattr(back, k)).tolist() for k in
                    ("positions", "log_scales", "rotations", "raw_amplitude", "raw_relax")}
    digest = lambda p: hashlib.sha256(open(os.path.join(IO_DIR, p), "rb").read()).hexdigest()
    return {"volume_seed": 17, "dims": list(g.dims), "spacing": list(g.spacing),
            "origin": list(g.origin),
            "sha256": {n: digest(n) for n in ("ref.json", "ref.bin", "ref.nii", "ref_relax.gsv",
                                              "ref_norelax.gsv")},
            "field_seed": 23, "field_loaded": field_values,
            "i16_be": {"dims": list(w.grid.dims), "spacing": list(w.grid.spacing),
                       "origin": list(w.grid.origin), "linear": w.linear().tolist()},
            "errors": errors, "accepted": accepted}


def full_configs():
    """Bit-exact binning hashes at BASELINE sizes + sampled forward values."""
    res = {}
    opts = RenderOptions()
    for cid in (2, 3, 4, 5):
        t0 = time.perf_counter()
        cfg, hr, lr, f, mine = problem(cid)
        entry = {"lr_volume": sha(lr.data), "field": field_sha(f), "N": f.count}
        grids = {"render": mine["render_grid"]} if cid == 5 else {"lr": lr.grid, "hr": hr.grid}
        for name, grid in grids.items():
            idx = build_brick_index(f, grid, opts)
            entry[name] = {"dims": list(grid.dims), "pairs": idx.pair_count,
                           "starts": sha(idx.starts), "gids": sha(idx.gids)}
            if name == "lr":
                c = forward(f, grid, idx, opts)
                loss, _ = loss_and_grad(c.volume(), lr, "l1")
                rng = np.random.default_rng(cid)
                sel = rng.choice(grid.num_voxels, size=4096, replace=False)
                entry[name].update({"loss": loss, "sample_idx": sel.tolist(),
                                    "sample_I": c.I[sel].astype(float).tolist(),
                                    "I_sum": float(np.sum(c.I, dtype=np.float64))})
            del idx
        res[str(cid)] = entry
        print(f"config {cid}: {time.perf_counter() - t0:.1f}s", flush=True)
    return res


# ----------------------------------------------------------- full-size parity
# Size-independent fingerprints of full-size reference outputs, small enough to
# commit (tests/golden/fingerprint.py, shared with the GPU tests).
sys.path.insert(0, HERE)
from fingerprint import (SKETCH_K, grad_sample_idx, hr_sample_idx,  # noqa: E402
                         sketch)


def full_renders():
    """Reference f32 renders at the benchmarked HR grids: config 3 (256^3),
    config 4 (256x256x160) and config 5 (512^3, jittered field)."""
    opts = RenderOptions()
    out, arrays = {}, {}
    for cid in (3, 4, 5):
        t0 = time.perf_counter()
        cfg, hr, lr, f, mine = problem(cid)
        grid = mine["render_grid"]
        idx = build_brick_index(f, grid, opts)
        c = forward(f, grid, idx, opts)
        I = np.asarray(c.I)
        cov = np.asarray(c.W) >= opts.epsilon_w
        sel = hr_sample_idx(grid.num_voxels, cid)
        arrays[f"c{cid}_sample_I"] = I[sel].astype(np.float32)
        out[str(cid)] = {"dims": list(grid.dims), "pairs": idx.pair_count,
                         "field": field_sha(f), "I_sha": sha(I),
                         "coverage_sha": sha(np.packbits(cov)),
                         "covered": int(cov.sum()),
                         "I_sum": float(np.sum(I, dtype=np.float64)),
                         "I_sketch": sketch(I), "seconds": time.perf_counter() - t0}
        del idx, c, I, cov
        print(f"render config {cid}: {time.perf_counter() - t0:.1f}s", flush=True)
    return out, arrays


def full_grads():
    """Reference f32 train-step gradients at the LR grids of configs 2, 3 and
    4: forward -> loss_and_grad(l1) -> backward (optimize.py:171-183).  The
    GPU reproduces dL/dI = sign(I - T)/V from its own render; voxels where
    |I_ref - T| <= 1e-5 could flip sign within the intensity bar, so their
    reference signs are stored and injected."""
    opts = RenderOptions()
    out, arrays = {}, {}
    for cid in (2, 3, 4):
        t0 = time.perf_counter()
        cfg, hr, lr, f, mine = problem(cid)
        idx = build_brick_index(f, lr.grid, opts)
        c = forward(f, lr.grid, idx, opts)
        loss, dl = loss_and_grad(c.volume(), lr, "l1")
        d = np.asarray(c.I, dtype=np.float64) - lr.linear().astype(np.float64)
        amb = np.flatnonzero(np.abs(d) <= 1e-5)
        gr = backward(f, lr.grid, idx, c, dl, opts)
        sel = grad_sample_idx(f.count, cid)
        e = {"N": f.count, "field": field_sha(f), "loss": loss, "pairs": idx.pair_count,
             "ambiguous": int(amb.shape[0]), "groups": {}}
        arrays[f"c{cid}_amb_idx"] = amb.astype(np.int64)
        arrays[f"c{cid}_amb_sign"] = np.sign(d[amb]).astype(np.int8)
        for k in G:
            g = np.asarray(getattr(gr, k), dtype=np.float64)
            arrays[f"c{cid}_grad_{k}"] = g[sel]
            e["groups"][k] = {"norm": float(np.linalg.norm(g)), "sketch": sketch(g)}
        e["seconds"] = time.perf_counter() - t0
        out[str(cid)] = e
        del idx, c, gr
        print(f"grads config {cid}: {time.perf_counter() - t0:.1f}s", flush=True)
    return out, arrays


def main():
    meta = {"versions": versions(), "generated_by": "tests/golden/make_golden.py"}
    which = set(sys.argv[1:]) or {"sweep", "config1", "full", "fit", "metrics", "io",
                                  "renders", "grads"}
    if "sweep" in which:
        with open(os.path.join(HERE, "sweep.json"), "w") as fh:
            json.dump({"meta": meta, "cases": sweep()}, fh)
        print("sweep done", flush=True)
    if "config1" in which:
        out, arrays = config1()
        np.savez_compressed(os.path.join(HERE, "config1.npz"), **arrays)
        with open(os.path.join(HERE, "config1.json"), "w") as fh:
            json.dump({"meta": meta, **out}, fh, indent=1)
        print("config1 done", flush=True)
    if "full" in which:
        with open(os.path.join(HERE, "full_configs.json"), "w") as fh:
            json.dump({"meta": meta, "configs": full_configs()}, fh)
    if "renders" in which:
        out, arrays = full_renders()
        np.savez_compressed(os.path.join(HERE, "full_renders.npz"), **arrays)
        with open(os.path.join(HERE, "full_renders.json"), "w") as fh:
            json.dump({"meta": meta, "sketch_k": SKETCH_K, "configs": out}, fh, indent=1)
    if "grads" in which:
        out, arrays = full_grads()
        np.savez_compressed(os.path.join(HERE, "full_grads.npz"), **arrays)
        with open(os.path.join(HERE, "full_grads.json"), "w") as fh:
            json.dump({"meta": meta, "sketch_k": SKETCH_K, "configs": out}, fh, indent=1)
    if "io" in which:
        with open(os.path.join(HERE, "volume_io.json"), "w") as fh:
            json.dump({"meta": meta, **volume_io()}, fh, indent=1)
        print("io done", flush=True)
    if "metrics" in which:
        with open(os.path.join(HERE, "metrics.json"), "w") as fh:
            json.dump({"meta": meta, "cases": metrics()}, fh, indent=1)
        print("metrics done", flush=True)
    if "fit" in which:
        with open(os.path.join(HERE, "fit_quality.json"), "w") as fh:
            json.dump({"meta": meta, **fit_quality()}, fh, indent=1)
        print("fit done", flush=True)


if __name__ == "__main__":
    main()
