"""Volume and field file formats against files the reference wrote
(tests/golden/make_golden.py "io"): raw_json + .bin, NIfTI-1 and GSV1 are
byte-identical on write, value-identical on read, and the loader's
FormatError messages match the reference's (volume.py:232-268,
nifti.py:90-165, field.py:262-312).  CPU only."""

import hashlib
import json
import os
import shutil
import sys

import numpy as np
import pytest

import paper_2603_09621_b200 as gs

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")
IO = os.path.join(GOLD, "io")
sys.path.insert(0, GOLD)
import io_cases  # noqa: E402

G = json.load(open(os.path.join(GOLD, "volume_io.json")))


def _sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


def _lin(v):
    return np.ascontiguousarray(v.linear().detach().cpu().numpy(), dtype="<f4")


def test_fixtures_are_the_recorded_ones():
    for name, digest in G["sha256"].items():
        assert _sha(os.path.join(IO, name)) == digest, name


@pytest.mark.parametrize("ext", ["json", "nii"])
def test_reference_volume_reads_and_rewrites_byte_identical(tmp_path, ext):
    v = gs.load_volume(os.path.join(IO, "ref." + ext))
    assert v.grid.dims == tuple(G["dims"])
    np.testing.assert_allclose(v.grid.spacing, G["spacing"], rtol=1e-6)
    np.testing.assert_allclose(v.grid.origin, G["origin"], rtol=1e-6)
    assert hashlib.sha256(_lin(v).tobytes()).hexdigest() == G["sha256"]["ref.bin"]
    out = tmp_path / ("ref." + ext)
    gs.save_volume(v, str(out))
    if ext == "json":
        assert _sha(out) == G["sha256"]["ref.json"]
        assert _sha(tmp_path / "ref.bin") == G["sha256"]["ref.bin"]
    else:
        assert _sha(out) == G["sha256"]["ref.nii"]


def test_raw_json_writer_byte_identical(tmp_path):
    v = gs.Volume.from_linear(gs.GridSpec(tuple(G["dims"]), tuple(G["spacing"]),
                                          tuple(G["origin"])),
                              np.fromfile(os.path.join(IO, "ref.bin"), dtype="<f4"))
    gs.save_volume(v, str(tmp_path / "ref.json"))
    assert _sha(tmp_path / "ref.json") == G["sha256"]["ref.json"]
    assert _sha(tmp_path / "ref.bin") == G["sha256"]["ref.bin"]
    gs.volume.save_volume(v, str(tmp_path / "x.vol"), format="nifti1")
    assert _sha(tmp_path / "x.vol") == G["sha256"]["ref.nii"]


def test_big_endian_int16_with_scaling():
    w = gs.load_volume(os.path.join(IO, "i16_be.nii"))
    ref = G["i16_be"]
    assert w.grid.dims == tuple(ref["dims"])
    assert list(w.grid.spacing) == ref["spacing"]
    assert list(w.grid.origin) == ref["origin"]
    np.testing.assert_array_equal(_lin(w), np.asarray(ref["linear"], dtype=np.float32))


@pytest.mark.parametrize("name", sorted(G["accepted"]))
def test_accepted_geometry_variants(tmp_path, name):
    a = gs.load_volume(io_cases.accepted(IO)[name](str(tmp_path)))
    ref = G["accepted"][name]
    assert list(a.grid.spacing) == ref["spacing"]
    assert list(a.grid.origin) == ref["origin"]
    assert hashlib.sha256(_lin(a).tobytes()).hexdigest() == ref["sha256"]


@pytest.mark.parametrize("name", sorted(G["errors"]))
def test_error_messages_match_reference(tmp_path, name):
    p = io_cases.cases(IO)[name](str(tmp_path))
    with pytest.raises(gs.FormatError) as exc:
        gs.load_volume(p)
    msg = str(exc.value).replace(p, "<path>").replace(str(tmp_path / "case.bin"), "<bin>")
    assert msg == G["errors"][name]


def test_format_inference_errors(tmp_path):
    v = gs.Volume.from_linear(gs.GridSpec((2, 2, 2)), np.zeros(8, np.float32))
    with pytest.raises(gs.FormatError, match=r"cannot infer volume format from extension '.vol'"):
        gs.save_volume(v, str(tmp_path / "a.vol"))
    with pytest.raises(gs.FormatError, match=r"unknown volume format 'hdf5'"):
        gs.load_volume(str(tmp_path / "a.json"), format="hdf5")


@pytest.mark.parametrize("name", ["ref_relax.gsv", "ref_norelax.gsv"])
def test_gsv1_reference_files_byte_identical(tmp_path, name):
    f = gs.load_field(os.path.join(IO, name))
    assert f.relax_enabled == (name == "ref_relax.gsv")
    if name == "ref_relax.gsv":
        for k, ref in G["field_loaded"].items():
            got = getattr(f, k)
            got = got.detach().cpu().numpy() if hasattr(got, "detach") else np.asarray(got)
            np.testing.assert_array_equal(got, np.asarray(ref), err_msg=k)
    gs.save_field(f, str(tmp_path / name))
    assert _sha(tmp_path / name) == G["sha256"][name]
