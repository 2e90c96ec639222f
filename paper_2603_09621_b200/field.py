"""Device-resident Gaussian field (mirrors gsvol/field.py:33-312).

Parameters are float64 torch tensors on the GPU in the reference's SoA layout
(field.py:33-70): positions (N,3), log_scales (N,3), rotations (N,4) w,x,y,z,
raw_amplitude (N), raw_relax (N).  The kernels read them in place.  The
mutation counter (``version``) guards brick indices exactly like the
reference (field.py:72-84, raster.py:220-230).

Construction from host arrays validates and (if needed) renormalises on the
host with numpy exactly as the reference does, so a field built from the same
inputs is bit-identical to the reference's; ``init_from_volume`` and
``random_field`` are one-time host setup restated from field.py:212-259.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch
from scipy.special import logit

from . import _lib
from .errors import FormatError
from .volume import GridSpec, Volume, default_device

IDENTITY_QUAT = (1.0, 0.0, 0.0, 0.0)

_GSV1_MAGIC = b"GSV1"
_GSV1_RECORD = 12 * 4
_FLAG_AMPLITUDE = 1
_FLAG_RELAX = 2

PARAM_NAMES = ("positions", "log_scales", "rotations", "raw_amplitude", "raw_relax")


def _host(a) -> np.ndarray:
    if isinstance(a, torch.Tensor):
        return a.detach().cpu().numpy()
    return np.asarray(a)


class GaussianField:
    """Mutable parameter container for the Gaussian mixture (field.py:33-109)."""

    def __init__(self, positions, log_scales, rotations, raw_amplitude, raw_relax,
                 amplitude_enabled: bool = True, relax_enabled: bool = True, device=None):
        dev = torch.device(device) if device is not None else default_device()
        all_dev = all(isinstance(a, torch.Tensor) and a.device.type == "cuda"
                      for a in (positions, log_scales, rotations, raw_amplitude, raw_relax))
        if all_dev:
            arrs = [a.detach().to(device=dev, dtype=torch.float64).contiguous()
                    for a in (positions, log_scales, rotations, raw_amplitude, raw_relax)]
            self._validate_shapes([tuple(a.shape) for a in arrs])
            norms = torch.linalg.vector_norm(arrs[2], dim=1)
            if bool((norms < 1e-12).any()):
                raise ValueError("zero-norm quaternion")
            if bool(((norms - 1.0).abs() > 1e-6).any()):
                arrs[2] = (arrs[2] / norms[:, None]).contiguous()
        else:
            host = [np.ascontiguousarray(_host(a), dtype=np.float64)
                    for a in (positions, log_scales, rotations, raw_amplitude, raw_relax)]
            self._validate_shapes([a.shape for a in host])
            # Renormalize only when off-unit (field.py:62-69).
            norms = np.linalg.norm(host[2], axis=1)
            if np.any(norms < 1e-12):
                raise ValueError("zero-norm quaternion")
            if np.any(np.abs(norms - 1.0) > 1e-6):
                host[2] = host[2] / norms[:, None]
            arrs = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in host]
        (self.positions, self.log_scales, self.rotations,
         self.raw_amplitude, self.raw_relax) = arrs
        self.amplitude_enabled = bool(amplitude_enabled)
        self.relax_enabled = bool(relax_enabled)
        self._version = 0

    @staticmethod
    def _validate_shapes(shapes):
        n = shapes[0][0] if len(shapes[0]) >= 1 else 0
        names = ("positions", "log_scales", "rotations")
        want = ((n, 3), (n, 3), (n, 4))
        for name, shp, w in zip(names, shapes[:3], want):
            if tuple(shp) != w:
                raise ValueError(f"{name} must be (N,{w[1]}), got {tuple(shp)}")
        if tuple(shapes[3]) != (n,):
            raise ValueError(f"raw_amplitude must be (N,), got {tuple(shapes[3])}")
        if tuple(shapes[4]) != (n,):
            raise ValueError(f"raw_relax must be (N,), got {tuple(shapes[4])}")
        if n == 0:
            raise ValueError("field must contain at least one Gaussian")

    # ---------------------------------------------------------------- state
    @property
    def count(self) -> int:
        return int(self.positions.shape[0])

    @property
    def version(self) -> int:
        return self._version

    @property
    def device(self) -> torch.device:
        return self.positions.device

    def bump_version(self) -> None:
        self._version += 1

    def activated_amplitude(self) -> torch.Tensor:
        return torch.sigmoid(self.raw_amplitude)

    def activated_relax(self) -> torch.Tensor:
        if not self.relax_enabled:
            return torch.ones(self.count, dtype=torch.float64, device=self.device)
        return torch.sigmoid(self.raw_relax)

    def scales(self) -> torch.Tensor:
        return torch.exp(self.log_scales)

    def normalize_rotations(self) -> None:
        """q /= |q| on the device (field.py:100-102), then bump the version."""
        lib = _lib.lib()
        _lib.check(lib.gsv_normalize_rotations(self.rotations.data_ptr(), self.count,
                                               _lib.stream_ptr()), "normalize_rotations")
        self._version += 1

    def copy(self) -> "GaussianField":
        f = GaussianField.__new__(GaussianField)
        for name in PARAM_NAMES:
            setattr(f, name, getattr(self, name).clone())
        f.amplitude_enabled = self.amplitude_enabled
        f.relax_enabled = self.relax_enabled
        f._version = 0
        return f

    def to_numpy(self) -> dict:
        return {name: getattr(self, name).detach().cpu().numpy() for name in PARAM_NAMES}

    def parameter_tensors(self):
        return [getattr(self, name) for name in PARAM_NAMES]


def rotation_matrices(quats) -> torch.Tensor:
    """(N,4) w,x,y,z quaternions -> (N,3,3) rotation matrices, applied
    verbatim without normalisation (field.py:141-154); f64 on the device
    (gsv_rotation_matrices)."""
    lib = _lib.lib()
    q = torch.as_tensor(quats, dtype=torch.float64)
    if q.device.type != "cuda":
        q = q.to(torch.device("cuda", torch.cuda.current_device()))
    q = q.reshape(-1, 4).contiguous()
    out = torch.empty((q.shape[0], 3, 3), dtype=torch.float64, device=q.device)
    _lib.check(lib.gsv_rotation_matrices(q.data_ptr(), q.shape[0], out.data_ptr(),
                                         _lib.stream_ptr()), "rotation_matrices")
    return out


@dataclass(frozen=True)
class InitConfig:
    """Initialization knobs (field.py:191-209)."""
    background_threshold: float = 0.01
    scale_factor: float = 0.75
    relax_init: float = 0.95

    def __post_init__(self):
        if not 0.0 <= self.background_threshold < 1.0:
            raise ValueError("background_threshold must lie in [0,1)")
        if self.scale_factor <= 0:
            raise ValueError("scale_factor must be positive")
        if not 0.0 < self.relax_init < 1.0:
            raise ValueError("relax_init must lie in (0,1)")


def init_arrays_from_volume(data: np.ndarray, grid: GridSpec, cfg: InitConfig = InitConfig()):
    """Host restatement of init_from_volume (field.py:212-234): one Gaussian per
    above-threshold voxel, gid order = np.argwhere C-order (ix slowest)."""
    data = np.asarray(data, dtype=np.float64)
    if data.min() < 0.0 or data.max() > 1.0:
        raise ValueError("LR volume must be normalized to [0,1] before init")
    mask = data >= cfg.background_threshold
    n = int(mask.sum())
    if n == 0:
        raise ValueError("empty field; lower background_threshold")
    vox = np.argwhere(mask).astype(np.float64)
    spacing = np.asarray(grid.spacing)
    positions = np.asarray(grid.origin) + vox * spacing
    log_scales = np.tile(np.log(cfg.scale_factor * spacing), (n, 1))
    rotations = np.tile(np.asarray(IDENTITY_QUAT), (n, 1))
    intensity = np.clip(data[mask], 1e-4, 1.0 - 1e-4)
    raw_amplitude = logit(intensity)
    raw_relax = np.full(n, logit(cfg.relax_init))
    return positions, log_scales, rotations, raw_amplitude, raw_relax


def init_from_volume(lr: Volume, cfg: InitConfig = InitConfig(),
                     on_device: bool = False) -> GaussianField:
    """One Gaussian per above-threshold LR voxel (field.py:212-234).

    The default is the host restatement, bit-identical to the reference.
    ``on_device=True`` builds the field with gsv_init_count / gsv_init_fill
    from the device volume (no host round trip of the volume): positions,
    scales, rotations and raw_relax are bit-identical, raw_amplitude is the
    logit by the device log (within a few ulp of scipy's)."""
    if not on_device:
        return GaussianField(*init_arrays_from_volume(lr.numpy(), lr.grid, cfg))
    import ctypes
    lin = lr.linear()
    if lin.device.type != "cuda":
        lin = lin.to(default_device())
    lin = lin.contiguous()
    if float(lin.min()) < 0.0 or float(lin.max()) > 1.0:
        raise ValueError("LR volume must be normalized to [0,1] before init")
    lib = _lib.lib()
    g = _lib.make_grid(lr.grid)
    nb = ctypes.c_size_t(0)
    _lib.check(lib.gsv_init_workspace(g, ctypes.byref(nb)), "init_workspace")
    ws = _lib.workspace(nb.value, lin.device, "init")
    slot = torch.empty(lin.numel() + 1, dtype=torch.int64, device=lin.device)
    f64 = int(lin.dtype == torch.float64)
    thr = float(cfg.background_threshold)
    _lib.check(lib.gsv_init_count(lin.data_ptr(), f64, g, thr, slot.data_ptr(), ws.data_ptr(),
                                  ws.numel(), _lib.stream_ptr()), "init_count")
    n = int(slot[-1].item())
    if n == 0:
        raise ValueError("empty field; lower background_threshold")
    spacing = np.asarray(lr.grid.spacing)
    ls3 = (ctypes.c_double * 3)(*np.log(cfg.scale_factor * spacing).tolist())
    dev = lin.device
    e = lambda *s_: torch.empty(*s_, dtype=torch.float64, device=dev)  # noqa: E731
    pos, ls, rot, ra, rr = e(n, 3), e(n, 3), e(n, 4), e(n), e(n)
    _lib.check(lib.gsv_init_fill(lin.data_ptr(), f64, g, thr, slot.data_ptr(), ls3,
                                 float(logit(cfg.relax_init)), pos.data_ptr(), ls.data_ptr(),
                                 rot.data_ptr(), ra.data_ptr(), rr.data_ptr(), _lib.stream_ptr()),
               "init_fill")
    return GaussianField(pos, ls, rot, ra, rr, device=dev)


def random_field_arrays(n: int, grid: GridSpec, seed: int, scale_lo: float = 0.7,
                        scale_hi: float = 1.6):
    """Host restatement of random_field (field.py:237-259)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    rng = np.random.default_rng(seed)
    lo, hi = grid.extent()
    lo = np.asarray(lo)
    size = np.asarray(hi) - lo
    positions = lo + size * rng.uniform(0.05, 0.95, size=(n, 3))
    mean_sp = float(np.mean(grid.spacing))
    scales = mean_sp * np.exp(rng.uniform(np.log(scale_lo), np.log(scale_hi), size=(n, 3)))
    quats = rng.normal(size=(n, 4))
    quats /= np.linalg.norm(quats, axis=1)[:, None]
    return positions, np.log(scales), quats, rng.normal(size=n), rng.normal(size=n)


def random_field(n: int, grid: GridSpec, seed: int, scale_lo: float = 0.7,
                 scale_hi: float = 1.6) -> GaussianField:
    return GaussianField(*random_field_arrays(n, grid, seed, scale_lo, scale_hi))


def save_field(f: GaussianField, path: str) -> None:
    """GSV1 container: magic, u64 count, u32 flags, N x 12 float32 LE (field.py:262-278)."""
    flags = (_FLAG_AMPLITUDE if f.amplitude_enabled else 0) | (_FLAG_RELAX if f.relax_enabled else 0)
    h = f.to_numpy()
    records = np.empty((f.count, 12), dtype="<f4")
    records[:, 0:3] = h["positions"]
    records[:, 3:6] = h["log_scales"]
    records[:, 6:10] = h["rotations"]
    records[:, 10] = h["raw_amplitude"]
    records[:, 11] = h["raw_relax"]
    with open(path, "wb") as fh:
        fh.write(_GSV1_MAGIC)
        fh.write(struct.pack("<QI", f.count, flags))
        fh.write(records.tobytes())


def load_field(path: str) -> GaussianField:
    """GSV1 reader with the reference's structured errors (field.py:281-312)."""
    with open(path, "rb") as fh:
        blob = fh.read()
    if blob[:4] != _GSV1_MAGIC:
        raise FormatError(f"{path}: bad magic {blob[:4]!r} at offset 0, expected b'GSV1'")
    if len(blob) < 16:
        raise FormatError(f"{path}: header truncated at offset {len(blob)} (need 16 bytes)")
    n, flags = struct.unpack_from("<QI", blob, 4)
    if n == 0:
        raise FormatError(f"{path}: header declares zero Gaussians at offset 4")
    if flags & ~(_FLAG_AMPLITUDE | _FLAG_RELAX):
        raise FormatError(f"{path}: unknown flag bits 0x{flags:x} at offset 12")
    expected = 16 + n * _GSV1_RECORD
    if len(blob) < expected:
        got = (len(blob) - 16) // _GSV1_RECORD
        raise FormatError(
            f"{path}: truncated at offset {len(blob)}: header declares {n} records "
            f"({expected} bytes total), only {got} complete records present")
    rec = np.frombuffer(blob, dtype="<f4", count=n * 12, offset=16).reshape(n, 12).astype(np.float64)
    return GaussianField(rec[:, 0:3], rec[:, 3:6], rec[:, 6:10], rec[:, 10], rec[:, 11],
                         amplitude_enabled=bool(flags & _FLAG_AMPLITUDE),
                         relax_enabled=bool(flags & _FLAG_RELAX))
