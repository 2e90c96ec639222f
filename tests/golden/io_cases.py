"""Malformed volume files for the load_volume error-path parity test.

Each case derives a broken file from the reference-written fixtures in
tests/golden/io/ by a byte edit (NIfTI) or a metadata edit (raw_json).
make_golden.py records the reference's FormatError message for each case
(path replaced by "<path>"); tests/test_volume_io.py replays the same edits
against our loader.
"""

import json
import os
import struct


def _nii(src, edit):
    def make(dst_dir):
        b = bytearray(open(src, "rb").read())
        b = edit(b)
        p = os.path.join(dst_dir, "case.nii")
        open(p, "wb").write(bytes(b))
        return p
    return make


def _pack(fmt, off, *v):
    def edit(b):
        struct.pack_into("<" + fmt, b, off, *v)
        return b
    return edit


def _raw(src_json, edit_meta=None, bin_bytes=None, text=None):
    def make(dst_dir):
        meta = json.load(open(src_json))
        p = os.path.join(dst_dir, "case.json")
        if text is not None:
            open(p, "w").write(text)
            return p
        if edit_meta:
            edit_meta(meta)
        if "data_file" in meta:
            meta["data_file"] = "case.bin"
        open(p, "w").write(json.dumps(meta))
        src_bin = os.path.join(os.path.dirname(src_json), "ref.bin")
        data = open(src_bin, "rb").read()
        open(os.path.join(dst_dir, "case.bin"), "wb").write(
            data if bin_bytes is None else data[:bin_bytes])
        return p
    return make


def _drop(key):
    return lambda m: m.pop(key)


def _set(key, value):
    return lambda m: m.__setitem__(key, value)


def cases(io_dir):
    """name -> callable(dst_dir) -> path of the broken file."""
    nii = os.path.join(io_dir, "ref.nii")
    js = os.path.join(io_dir, "ref.json")
    return {
        "nii_short_header": _nii(nii, lambda b: b[:200]),
        "nii_bad_sizeof": _nii(nii, _pack("i", 0, 540)),
        "nii_bad_magic": _nii(nii, lambda b: b[:344] + b"ni1\x00" + b[348:]),
        "nii_dim0_2": _nii(nii, _pack("h", 40, 2)),
        "nii_4d": _nii(nii, _pack("h", 48, 2)),
        "nii_float64": _nii(nii, _pack("h", 70, 64)),
        "nii_code_999": _nii(nii, _pack("h", 70, 999)),
        "nii_sform_offdiag": _nii(nii, _pack("f", 284, 0.3)),
        "nii_sform_negative": _nii(nii, _pack("f", 300, -1.1)),
        "nii_qform_rotation": _nii(nii, lambda b: _pack("h", 252, 1)(_pack("h", 254, 0)(
            _pack("f", 260, 0.2)(b)))),
        "nii_qfac_flip": _nii(nii, lambda b: _pack("h", 252, 1)(_pack("h", 254, 0)(
            _pack("f", 76, -1.0)(b)))),
        "nii_truncated_data": _nii(nii, lambda b: b[:400]),
        "raw_bad_json": _raw(js, text="{not json"),
        "raw_missing_spacing": _raw(js, _drop("spacing")),
        "raw_missing_data_file": _raw(js, _drop("data_file")),
        "raw_dtype_f64": _raw(js, _set("dtype", "f64")),
        "raw_short_bin": _raw(js, bin_bytes=100),
    }


# Geometry-only headers the loader accepts: no sform, identity qform; neither.
def accepted(io_dir):
    nii = os.path.join(io_dir, "ref.nii")
    return {
        "nii_qform_identity": _nii(nii, lambda b: _pack("h", 252, 1)(_pack("h", 254, 0)(
            _pack("3f", 268, 4.0, 5.0, 6.0)(b)))),
        "nii_no_transform": _nii(nii, lambda b: _pack("h", 252, 0)(_pack("h", 254, 0)(
            _pack("f", 80, 0.0)(b)))),
        "nii_slope_only": _nii(nii, lambda b: _pack("2f", 112, 2.0, 0.0)(b)),
        "nii_slope_zero_inter": _nii(nii, lambda b: _pack("2f", 112, 0.0, 1.5)(b)),
    }
