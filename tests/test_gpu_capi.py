"""The C ABI (include/gsv.h) from plain C: tests/capi/capi_forward.c, built
with gcc against libgsv_b200.so and cudart only (no Python, no torch), bins
and renders a field; its lists and intensities are bit-identical to the
Python API's (same kernels behind both).  It also drives the incremental
binning entry points after moving the field and checks them against a full
build."""

import os
import struct
import subprocess
import tempfile

import numpy as np
import pytest
import torch

import paper_2603_09621_b200 as gs
from paper_2603_09621_b200 import _lib
from paper_2603_09621_b200.field import random_field_arrays

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "capi", "capi_forward.c")


def _build(out_dir):
    exe = os.path.join(out_dir, "capi_forward")
    libdir = os.path.dirname(_lib.LIB_PATH)
    cmd = ["gcc", "-O2", "-std=c99", "-Wall", "-Wextra", "-Werror",
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", SRC,
           "-L", libdir, "-lgsv_b200", "-L", "/usr/local/cuda/lib64", "-lcudart",
           f"-Wl,-rpath,{libdir}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


@pytest.mark.parametrize("dims,bd", [((24, 24, 24), (8, 8, 4)), ((20, 28, 18), (4, 4, 4))])
def test_c_program_matches_python_api(dims, bd):
    grid = gs.GridSpec(dims, (0.9, 1.0, 1.2), (-1.0, 0.5, 2.0))
    arrs = random_field_arrays(400, grid, seed=21, scale_lo=0.5, scale_hi=2.0)
    with tempfile.TemporaryDirectory() as d:
        exe = _build(d)
        inp, outp = os.path.join(d, "in.bin"), os.path.join(d, "out.bin")
        n = arrs[0].shape[0]
        with open(inp, "wb") as fh:
            fh.write(struct.pack("<3i", *dims))
            fh.write(struct.pack("<7d", *grid.origin, *grid.spacing, 3.0))
            fh.write(struct.pack("<3i", *bd))
            fh.write(struct.pack("<q", n))
            for a in arrs:
                fh.write(np.ascontiguousarray(a, dtype="<f8").tobytes())
            fh.write(struct.pack("<i", 1))
        res = subprocess.run([exe, inp, outp], capture_output=True, text=True)
        assert res.returncode == 0, res.stderr
        raw = open(outp, "rb").read()
    pairs, nb = struct.unpack_from("<2q", raw, 0)
    o = 16
    starts = np.frombuffer(raw, "<i8", nb + 1, o)
    o += 8 * (nb + 1)
    gids = np.frombuffer(raw, "<i4", pairs, o)
    o += 4 * pairs
    I = np.frombuffer(raw, "<f4", grid.num_voxels, o)
    o += 4 * grid.num_voxels
    incremental_ok = struct.unpack_from("<i", raw, o)[0]

    f = gs.GaussianField(*arrs)
    idx = gs.build_brick_index(f, grid, gs.RenderOptions(), bd)
    c = gs.forward(f, grid, idx)
    assert pairs == idx.pair_count
    np.testing.assert_array_equal(starts, idx.starts.cpu().numpy())
    np.testing.assert_array_equal(gids, idx.gids.cpu().numpy())
    np.testing.assert_array_equal(I, c.I.cpu().numpy())
    # the incremental entry points (gsv_preprocess_track, gsv_bin_incremental)
    # from C: after a move, the edited lists equal a full gsv_bin_fill
    assert incremental_ok == 1
