"""Volume files of the reference (volume.py:197-268, nifti.py:1-165): raw_json
(JSON metadata + little-endian float32 ``.bin``, x-fastest) and single-file
NIfTI-1 (``n+1``; uint8 / int16 / float32 data; identity or diagonal
qform/sform).  Same file layouts, accepted subset and error messages as the
reference, so files move between the two packages byte for byte.

Host file I/O: the voxel data lands in a device Volume (Volume.from_linear).
"""

from __future__ import annotations

import json
import os

import numpy as np

from .errors import FormatError
from .volume import GridSpec, Volume

RAW_JSON_DTYPE = "f32"

# NIfTI-1 header (348 bytes) as a structured record; fields we do not use are
# padding.  Offsets follow the NIfTI-1 standard.
_NIFTI_FIELDS = [
    ("sizeof_hdr", "i4", 0), ("dim", ("i2", 8), 40), ("datatype", "i2", 70),
    ("bitpix", "i2", 72), ("pixdim", ("f4", 8), 76), ("vox_offset", "f4", 108),
    ("scl_slope", "f4", 112), ("scl_inter", "f4", 116), ("qform_code", "i2", 252),
    ("sform_code", "i2", 254), ("quatern", ("f4", 3), 256), ("qoffset", ("f4", 3), 268),
    ("srow", ("f4", (3, 4)), 280), ("magic", "S4", 344),
]
_NIFTI_HEADER = 348
_NIFTI_MAGIC = b"n+1"
_NIFTI_DATA = {2: "u1", 4: "i2", 16: "f4"}
_NIFTI_TYPE_NAMES = {
    0: "unknown", 1: "binary", 2: "uint8", 4: "int16", 8: "int32", 16: "float32",
    32: "complex64", 64: "float64", 128: "rgb24", 256: "int8", 512: "uint16",
    768: "uint32", 1024: "int64", 1280: "uint64", 1536: "float128", 1792: "complex128",
    2048: "complex256", 2304: "rgba32",
}


def _nifti_dtype(order: str) -> np.dtype:
    names, formats, offsets = zip(*_NIFTI_FIELDS)
    formats = [(order + f[0], f[1]) if isinstance(f, tuple) else
               (f if f.startswith("S") else order + f) for f in formats]
    return np.dtype({"names": list(names), "formats": formats, "offsets": list(offsets),
                     "itemsize": _NIFTI_HEADER})


def _infer_format(path: str) -> str:
    ext = os.path.splitext(path)[1].lower()
    formats = {".json": "raw_json", ".nii": "nifti1"}
    if ext not in formats:
        raise FormatError(f"cannot infer volume format from extension {ext!r}; pass format=")
    return formats[ext]


# ------------------------------------------------------------------ raw_json
def _save_raw_json(v: Volume, path: str) -> None:
    data_file = os.path.splitext(os.path.basename(path))[0] + ".bin"
    meta = {"dims": list(v.grid.dims), "spacing": list(v.grid.spacing),
            "origin": list(v.grid.origin), "dtype": RAW_JSON_DTYPE, "data_file": data_file}
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(json.dumps(meta, indent=2) + "\n")
    flat = v.linear().detach().cpu().numpy().astype("<f4")
    flat.tofile(os.path.join(os.path.dirname(path) or ".", data_file))


def _load_raw_json(path: str) -> Volume:
    try:
        with open(path, encoding="utf-8") as fh:
            meta = json.load(fh)
    except json.JSONDecodeError as exc:
        raise FormatError(f"{path}: not valid JSON: {exc}") from exc
    missing = [k for k in ("dims", "spacing", "origin", "dtype", "data_file") if k not in meta]
    if missing:
        raise FormatError(f"{path}: missing required key {missing[0]!r}")
    if meta["dtype"] != RAW_JSON_DTYPE:
        raise FormatError(f"{path}: unsupported dtype {meta['dtype']!r} (only f32)")
    grid = GridSpec(tuple(meta["dims"]), tuple(meta["spacing"]), tuple(meta["origin"]))
    bin_path = os.path.join(os.path.dirname(path) or ".", meta["data_file"])
    flat = np.fromfile(bin_path, dtype="<f4")
    if flat.size != grid.num_voxels:
        raise FormatError(f"{bin_path}: has {flat.size} float32 values, dims {grid.dims} "
                          f"require {grid.num_voxels}")
    return Volume.from_linear(grid, flat)


# ------------------------------------------------------------------ NIfTI-1
def _nifti_geometry(h, path: str):
    """(spacing, origin) of a diagonal sform, an identity qform, or neither."""
    pixdim = [float(p) for p in h["pixdim"]]
    spacing_q = tuple(p if p > 0 else 1.0 for p in pixdim[1:4])
    if int(h["sform_code"]) > 0:
        srow = np.asarray(h["srow"], dtype=np.float64)
        lin = srow[:, :3]
        if np.abs(lin - np.diag(np.diag(lin))).max() > 1e-5 * max(np.abs(lin).max(), 1.0):
            raise FormatError(f"{path}: non-diagonal sform affine (srow_x/y/z)")
        if (np.diag(lin) <= 0).any():
            raise FormatError(f"{path}: non-positive sform diagonal (srow_x/y/z)")
        return tuple(float(d) for d in np.diag(lin)), tuple(float(t) for t in srow[:, 3])
    if int(h["qform_code"]) > 0:
        if np.abs(np.asarray(h["quatern"], dtype=np.float64)).max() > 1e-6:
            raise FormatError(f"{path}: non-identity qform rotation (quatern_b/c/d)")
        if pixdim[0] < 0:
            raise FormatError(f"{path}: qfac=-1 axis flip unsupported (pixdim[0])")
        return spacing_q, tuple(float(q) for q in h["qoffset"])
    return spacing_q, (0.0, 0.0, 0.0)


def _load_nifti(path: str) -> Volume:
    with open(path, "rb") as fh:
        raw = fh.read(_NIFTI_HEADER)
        if len(raw) < _NIFTI_HEADER:
            raise FormatError(f"{path}: file shorter than the 348-byte NIfTI-1 header")
        order = next((o for o in "<>" if np.frombuffer(raw[:4], o + "i4")[0] == _NIFTI_HEADER),
                     None)
        if order is None:
            raise FormatError(f"{path}: bad sizeof_hdr, not a NIfTI-1 file")
        h = np.frombuffer(raw, dtype=_nifti_dtype(order))[0]
        magic = bytes(raw[344:348])
        if magic != _NIFTI_MAGIC + b"\x00":
            raise FormatError(f"{path}: magic {magic!r} unsupported (need single-file 'n+1')")
        dim = [int(d) for d in h["dim"]]
        if dim[0] < 3:
            raise FormatError(f"{path}: dim[0]={dim[0]}, need a 3D volume")
        if any(d > 1 for d in dim[4:8]):
            raise FormatError(f"{path}: dim[4:]={tuple(dim[4:8])} — 4D+ volumes unsupported")
        code = int(h["datatype"])
        if code not in _NIFTI_DATA:
            name = _NIFTI_TYPE_NAMES.get(code, str(code))
            raise FormatError(f"{path}: unsupported datatype {name} (code {code}); "
                              "supported: uint8, int16, float32")
        dims = tuple(dim[1:4])
        spacing, origin = _nifti_geometry(h, path)
        count = dims[0] * dims[1] * dims[2]
        fh.seek(int(float(h["vox_offset"])))
        data = np.fromfile(fh, dtype=np.dtype(_NIFTI_DATA[code]).newbyteorder(order),
                           count=count)
        if data.size != count:
            raise FormatError(f"{path}: data truncated, got {data.size} of {count} voxels")
    data = data.astype(np.float32)
    slope, inter = float(h["scl_slope"]), float(h["scl_inter"])
    if slope not in (0.0, 1.0) or inter != 0.0:
        data = data * np.float32(slope if slope != 0.0 else 1.0) + np.float32(inter)
    return Volume.from_linear(GridSpec(dims, spacing, origin), data)


def _save_nifti(v: Volume, path: str) -> None:
    """float32 single-file .nii with a diagonal sform (data at offset 352)."""
    h = np.zeros((), dtype=_nifti_dtype("<"))
    (sx, sy, sz), (ox, oy, oz) = v.grid.spacing, v.grid.origin
    h["sizeof_hdr"] = _NIFTI_HEADER
    h["dim"] = (3, *v.grid.dims, 1, 1, 1, 1)
    h["datatype"], h["bitpix"] = 16, 32
    h["pixdim"] = (1.0, sx, sy, sz, 0, 0, 0, 0)
    h["vox_offset"], h["scl_slope"], h["scl_inter"] = 352.0, 1.0, 0.0
    h["qform_code"], h["sform_code"] = 0, 1
    h["srow"] = ((sx, 0, 0, ox), (0, sy, 0, oy), (0, 0, sz, oz))
    h["magic"] = _NIFTI_MAGIC
    with open(path, "wb") as fh:
        fh.write(h.tobytes())
        fh.write(bytes(4))                    # extension flag: none, pads to 352
        fh.write(v.linear().detach().cpu().numpy().astype("<f4").tobytes())


_WRITERS = {"raw_json": _save_raw_json, "nifti1": _save_nifti}
_READERS = {"raw_json": _load_raw_json, "nifti1": _load_nifti}


def save_volume(v: Volume, path: str, format: str | None = None) -> None:
    """Write a volume as raw_json (JSON metadata + .bin float32) or NIfTI-1."""
    fmt = format or _infer_format(path)
    if fmt not in _WRITERS:
        raise FormatError(f"unknown volume format {fmt!r}")
    _WRITERS[fmt](v, path)


def load_volume(path: str, format: str | None = None) -> Volume:
    """Read a volume written by save_volume (or by the reference)."""
    fmt = format or _infer_format(path)
    if fmt not in _READERS:
        raise FormatError(f"unknown volume format {fmt!r}")
    return _READERS[fmt](path)
