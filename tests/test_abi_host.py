"""C-ABI surface and host-side logic, CPU only (no kernel launches)."""

import os
import re
import subprocess

import numpy as np
import pytest
import torch

import paper_2603_09621_b200 as gs
from paper_2603_09621_b200 import _lib
from paper_2603_09621_b200.distributed import (brick_layers, layer_slab_ranges, slab_for_rank,
                                               slab_ranges, slab_voxel_mask)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADERS = [os.path.join(ROOT, "include", h) for h in ("gsv.h", "gsv_diag.h")]


def _declared():
    names = []
    for h in HEADERS:
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"\b(gsv_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _lib.EXPORTS, f"{name} has no ctypes signature"


def test_abi_version_and_error_channel_without_gpu():
    lib = _lib.load()
    header = open(os.path.join(ROOT, "include", "gsv.h")).read()
    declared = int(re.search(r"#define GSV_ABI_VERSION (\d+)", header).group(1))
    assert lib.gsv_abi_version() == declared == _lib.ABI_VERSION
    assert isinstance(lib.gsv_last_error(), bytes)


def test_binary_is_sm100a():
    so = _lib.LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_cuda():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.GsvLibraryError, match="no CPU path"):
        _lib.lib()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2603_09621_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


def test_gridspec_and_volume_contract():
    with pytest.raises(ValueError, match="dims"):
        gs.GridSpec((0, 4, 4))
    with pytest.raises(ValueError, match="spacing"):
        gs.GridSpec((4, 4, 4), (1.0, 0.0, 1.0))
    g = gs.GridSpec((3, 4, 5), (1.0, 2.0, 0.5), (1.0, 0.0, -1.0))
    data = np.arange(60, dtype=np.float32).reshape(3, 4, 5)
    v = gs.Volume(g, data)
    # x-fastest linear layout (volume.py:100-102)
    np.testing.assert_array_equal(v.linear().cpu().numpy(), data.ravel(order="F"))
    np.testing.assert_array_equal(v.numpy(), data)
    v2 = gs.Volume.from_linear(g, data.ravel(order="F"))
    np.testing.assert_array_equal(v2.numpy(), data)
    lo, hi = g.extent()
    np.testing.assert_allclose(lo, [0.5, -1.0, -1.25])


def test_options_and_config_validation():
    with pytest.raises(ValueError, match="cutoff_sigma"):
        gs.RenderOptions(cutoff_sigma=0.0)
    with pytest.raises(ValueError, match="epsilon_w"):
        gs.RenderOptions(epsilon_w=-1.0)
    with pytest.raises(ValueError, match="precision"):
        gs.RenderOptions(precision="f16")
    assert gs.RenderOptions(cutoff_sigma=3.0).cutoff_sq == 9.0
    with pytest.raises(ValueError, match="iterations"):
        gs.FitConfig(iterations=0)
    with pytest.raises(ValueError, match="loss"):
        gs.FitConfig(loss="huber")
    with pytest.raises(ValueError, match="lr_scale"):
        gs.FitConfig(lr_scale=-1.0)
    with pytest.raises(ValueError, match="background_threshold"):
        gs.InitConfig(background_threshold=1.0)
    with pytest.raises(ValueError, match=">= 1"):
        gs.set_worker_count(0)
    lrs = gs.FitConfig().resolved_lrs((2.0, 2.0, 2.0))
    assert lrs["positions"] == pytest.approx(2e-3)


def test_field_construction_rules():
    with pytest.raises(ValueError, match="positions"):
        gs.GaussianField(np.zeros((2, 2)), np.zeros((2, 3)), np.tile([1.0, 0, 0, 0], (2, 1)),
                         np.zeros(2), np.zeros(2))
    with pytest.raises(ValueError, match="zero-norm"):
        gs.GaussianField(np.zeros((1, 3)), np.zeros((1, 3)), np.zeros((1, 4)), np.zeros(1),
                         np.zeros(1))
    f = gs.GaussianField(np.zeros((1, 3)), np.zeros((1, 3)), [[2.0, 0, 0, 0]], np.zeros(1),
                         np.zeros(1))
    np.testing.assert_array_equal(f.rotations.cpu().numpy(), [[1.0, 0, 0, 0]])
    f.bump_version()
    assert f.version == 1


def test_gsv1_round_trip(tmp_path):
    g = gs.GridSpec((8, 8, 8))
    f = gs.random_field(64, g, seed=100)
    f.amplitude_enabled = False
    p = str(tmp_path / "f.gsv")
    gs.save_field(f, p)
    h = gs.load_field(p)
    gs.save_field(h, str(tmp_path / "g.gsv"))
    assert (tmp_path / "f.gsv").read_bytes() == (tmp_path / "g.gsv").read_bytes()
    assert h.amplitude_enabled is False and h.relax_enabled is True
    (tmp_path / "bad.gsv").write_bytes(b"XXXX" + b"\x00" * 16)
    with pytest.raises(gs.FormatError, match="offset 0"):
        gs.load_field(str(tmp_path / "bad.gsv"))


def test_merge_gradients_contract():
    a, b = gs.GradientBuffer.zeros(2, "cpu"), gs.GradientBuffer.zeros(2, "cpu")
    a.positions[0, 0] = 1.0
    b.positions[0, 0] = 2.0
    fwd = gs.merge_gradients([(0, a), (1, b)])
    rev = gs.merge_gradients([(1, b), (0, a)])
    assert float(fwd.positions[0, 0]) == 3.0
    assert torch.equal(fwd.positions, rev.positions)
    with pytest.raises(ValueError, match="no partials"):
        gs.merge_gradients([])


def test_brick_index_accepts_host_lists():
    g = gs.GridSpec((8, 8, 8))
    idx = gs.BrickIndex(g, (8, 8, 4), (1, 1, 2), np.array([0, 2, 3]), np.array([4, 7, 1]),
                        0, 10, 3.0)
    assert idx.pair_count == 3 and idx.brick_count == 2
    assert idx.gids.dtype == torch.int32 and idx.starts.dtype == torch.int64


def _check_partition(r, n):
    assert r[0][0] == 0 and r[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
    assert all(a <= b for a, b in r)


def test_slab_partition_covers_every_brick_once():
    for n in (1, 7, 10, 32, 128, 8192):
        for ws in (1, 2, 3, 4, 8):
            r = slab_ranges(n, ws)
            _check_partition(r, n)
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1
    g = gs.GridSpec((16, 16, 20))
    assert brick_layers(g, (8, 8, 4)) == 5
    assert slab_for_rank(g, (8, 8, 4), 0, 1) is None
    # whole-layer slabs are the aligned special case
    lay = layer_slab_ranges(g, (8, 8, 4), 2)
    _check_partition(lay, 20)
    assert sorted(b - a for a, b in lay) == [8, 12] and all(b % 4 == 0 for _, b in lay)
    # mid-layer cuts: 20 bricks over 3 ranks
    r = [slab_for_rank(g, (8, 8, 4), k, 3) for k in range(3)]
    _check_partition(r, 20)
    assert any(b % 4 for _, b in r[:-1])
    masks = [slab_voxel_mask(g, (8, 8, 4), s) for s in r]
    assert (sum(m.astype(int) for m in masks) == 1).all()


def test_slab_partition_balances_weights():
    rng = np.random.default_rng(3)
    w = rng.integers(0, 50, size=1000).astype(np.float64)
    w[:300] *= 10                                   # a heavy front
    for ws in (2, 3, 5, 8):
        r = slab_ranges(1000, ws, weights=w)
        _check_partition(r, 1000)
        loads = [w[a:b].sum() for a, b in r]
        assert max(loads) <= w.sum() / ws + w.max() + 1e-9
    # 10 layers of 64 bricks over 8 ranks: whole layers cap the balance at
    # 2 layers per rank on the heaviest; mid-layer cuts do not
    w = np.ones(640)
    lay = slab_ranges(640, 8, weights=w, align=64)
    mid = slab_ranges(640, 8, weights=w)
    assert max(b - a for a, b in lay) == 128
    assert max(b - a for a, b in mid) == 80
    with pytest.raises(ValueError):
        slab_ranges(10, 2, weights=np.ones(9))
    with pytest.raises(ValueError):
        slab_ranges(10, 2, weights=-np.ones(10))
