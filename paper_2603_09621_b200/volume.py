"""Cell-centred grids and device-resident volumes (gsvol/volume.py:16-184).

``GridSpec`` is the reference's frozen dataclass unchanged (volume.py:16-76).
``Volume`` keeps the reference's contract -- ``data`` has shape ``grid.dims``
indexed ``[ix, iy, iz]`` and ``linear()`` is the x-fastest flat layout
(volume.py:100-102) -- but ``data`` is a torch tensor that lives on the GPU:
a ``(nx, ny, nz)`` permuted view of one contiguous x-fastest buffer, so
``linear()`` is free and the kernels read it directly.

The resampling / grid helpers below run once per problem on the host
(numpy), exactly like the reference; they are setup, not the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


def default_device() -> torch.device:
    if torch.cuda.is_available():
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


@dataclass(frozen=True)
class GridSpec:
    """A cell-centered sampling lattice (volume.py:16-76).

    ``origin`` is the world coordinate of the *center* of voxel (0, 0, 0);
    voxel (i, j, k) sits at ``origin + (i, j, k) * spacing``.
    """

    dims: tuple
    spacing: tuple = (1.0, 1.0, 1.0)
    origin: tuple = (0.0, 0.0, 0.0)

    def __post_init__(self):
        dims = tuple(int(d) for d in self.dims)
        spacing = tuple(float(s) for s in self.spacing)
        origin = tuple(float(o) for o in self.origin)
        if len(dims) != 3 or len(spacing) != 3 or len(origin) != 3:
            raise ValueError("GridSpec fields must each have 3 components")
        if any(d < 1 for d in dims):
            raise ValueError(f"dims must all be >= 1, got {dims}")
        if any(not s > 0 for s in spacing):
            raise ValueError(f"spacing must all be > 0, got {spacing}")
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "spacing", spacing)
        object.__setattr__(self, "origin", origin)

    @property
    def num_voxels(self) -> int:
        nx, ny, nz = self.dims
        return nx * ny * nz

    def voxel_to_world(self, idx) -> np.ndarray:
        idx = np.asarray(idx, dtype=np.float64)
        return np.asarray(self.origin) + idx * np.asarray(self.spacing)

    def world_to_voxel(self, pts) -> np.ndarray:
        pts = np.asarray(pts, dtype=np.float64)
        return (pts - np.asarray(self.origin)) / np.asarray(self.spacing)

    def axis_coords(self, axis: int) -> np.ndarray:
        return self.origin[axis] + np.arange(self.dims[axis], dtype=np.float64) * self.spacing[axis]

    def extent(self):
        o = np.asarray(self.origin, dtype=np.float64)
        s = np.asarray(self.spacing, dtype=np.float64)
        lo = o - 0.5 * s
        return lo, lo + np.asarray(self.dims) * s


def _to_linear_tensor(data, dims, device) -> torch.Tensor:
    """x-fastest flat tensor on ``device`` from a dims-shaped array/tensor."""
    if isinstance(data, torch.Tensor):
        if tuple(data.shape) != tuple(dims):
            raise ValueError(f"data shape {tuple(data.shape)} does not match grid dims {dims}")
        if data.dtype not in (torch.float32, torch.float64):
            data = data.to(torch.float32)
        return data.to(device).permute(2, 1, 0).contiguous().reshape(-1)
    arr = np.asarray(data)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float32)
    if arr.shape != tuple(dims):
        raise ValueError(f"data shape {arr.shape} does not match grid dims {tuple(dims)}")
    flat = np.ascontiguousarray(arr.ravel(order="F"))
    return torch.from_numpy(flat).to(device)


@dataclass(frozen=True)
class Volume:
    """A dense scalar grid.  ``data`` has shape ``grid.dims``, indexed [ix, iy, iz].

    Accepts numpy arrays or torch tensors (any device); stores a device view.
    """

    grid: GridSpec
    data: object

    def __post_init__(self):
        dims = self.grid.dims
        d = self.data
        if (isinstance(d, torch.Tensor) and tuple(d.shape) == dims
                and d.dtype in (torch.float32, torch.float64) and d.dim() == 3
                and d.permute(2, 1, 0).is_contiguous()):
            return  # already an x-fastest view
        flat = _to_linear_tensor(d, dims, default_device())
        object.__setattr__(self, "data", flat.view(dims[2], dims[1], dims[0]).permute(2, 1, 0))

    @property
    def dtype(self):
        return self.data.dtype

    @property
    def device(self):
        return self.data.device

    def linear(self) -> torch.Tensor:
        """Data flattened in x-fastest order (a view, no copy)."""
        return self.data.permute(2, 1, 0).reshape(-1)

    def numpy(self) -> np.ndarray:
        """Host copy shaped ``grid.dims`` (the reference's ``Volume.data``)."""
        flat = self.linear().detach().cpu().numpy()
        return np.ascontiguousarray(flat.reshape(self.grid.dims, order="F"))

    @classmethod
    def from_linear(cls, grid: GridSpec, flat, dtype=None) -> "Volume":
        """Build from x-fastest flat data, keeping its dtype unless overridden."""
        if not isinstance(flat, torch.Tensor):
            arr = np.asarray(flat, dtype=dtype)
            if arr.dtype not in (np.float32, np.float64):
                arr = arr.astype(np.float32)
            flat = torch.from_numpy(np.ascontiguousarray(arr.reshape(-1)))
        elif dtype is not None:
            flat = flat.to(torch.float64 if np.dtype(dtype) == np.float64 else torch.float32)
        if flat.numel() != grid.num_voxels:
            raise ValueError(f"flat data has {flat.numel()} values, grid wants {grid.num_voxels}")
        if flat.device.type == "cpu" and torch.cuda.is_available():
            flat = flat.to(default_device())
        nx, ny, nz = grid.dims
        return cls(grid, flat.reshape(-1).view(nz, ny, nx).permute(2, 1, 0))


# ------------------------------------------------------------------ host setup
def normalize_intensity_np(data: np.ndarray) -> np.ndarray:
    """volume.py:115-123 on a host array."""
    d = data.astype(np.float64)
    lo, hi = float(d.min()), float(d.max())
    if hi == lo:
        return np.zeros(data.shape, dtype=data.dtype)
    return ((d - lo) / (hi - lo)).astype(data.dtype)


def resample_trilinear_np(src_data: np.ndarray, src: GridSpec, target: GridSpec) -> np.ndarray:
    """Trilinear resampling with clamp-to-edge (volume.py:126-154), host numpy.

    Same operation order as the reference so synthetic inputs are bit-identical.
    """
    src64 = src_data.astype(np.float64)
    lows, highs, fracs = [], [], []
    for axis in range(3):
        n = src.dims[axis]
        world = target.origin[axis] + np.arange(target.dims[axis]) * target.spacing[axis]
        u = (world - src.origin[axis]) / src.spacing[axis]
        u = np.clip(u, 0.0, n - 1.0)
        i0 = np.clip(np.floor(u).astype(np.intp), 0, max(n - 2, 0))
        i1 = np.minimum(i0 + 1, n - 1)
        lows.append(i0)
        highs.append(i1)
        fracs.append(u - i0)
    out = np.zeros(target.dims, dtype=np.float64)
    for cx, wx in ((lows[0], 1.0 - fracs[0]), (highs[0], fracs[0])):
        for cy, wy in ((lows[1], 1.0 - fracs[1]), (highs[1], fracs[1])):
            for cz, wz in ((lows[2], 1.0 - fracs[2]), (highs[2], fracs[2])):
                w = wx[:, None, None] * wy[None, :, None] * wz[None, None, :]
                out += w * src64[np.ix_(cx, cy, cz)]
    return out.astype(src_data.dtype)


def resample_trilinear(v: Volume, target: GridSpec) -> Volume:
    """resample_trilinear (volume.py:126-154).  On a CUDA volume this runs
    gsv_resample_trilinear (bit-identical to the reference: same f64
    operation order, result in the source dtype); a host volume takes the
    numpy restatement."""
    if v.device.type != "cuda":
        return Volume(target, resample_trilinear_np(v.numpy(), v.grid, target))
    from . import _lib
    lib = _lib.lib()
    src = v.linear().contiguous()
    out = torch.empty(target.num_voxels, dtype=src.dtype, device=src.device)
    _lib.check(lib.gsv_resample_trilinear(src.data_ptr(), int(src.dtype == torch.float64),
                                          _lib.make_grid(v.grid), out.data_ptr(),
                                          _lib.make_grid(target), _lib.stream_ptr()),
               "resample_trilinear")
    return Volume.from_linear(target, out)


def normalize_intensity(v: Volume) -> Volume:
    return Volume(v.grid, normalize_intensity_np(v.numpy()))


def ensure_unit_range(v: Volume) -> Volume:
    """volume.py:187-195."""
    d = v.linear()
    if float(d.min()) >= 0.0 and float(d.max()) <= 1.0:
        return v
    return normalize_intensity(v)


def grid_covering_extent(ref: GridSpec, dims) -> GridSpec:
    """A grid with the given dims covering exactly ``ref``'s box (volume.py:157-163)."""
    dims = tuple(int(d) for d in dims)
    lo, hi = ref.extent()
    spacing = (hi - lo) / np.asarray(dims)
    origin = lo + 0.5 * spacing
    return GridSpec(dims, tuple(spacing), tuple(origin))


def downsample_grid(ref: GridSpec, factor) -> GridSpec:
    """LR grid for an integer per-axis factor (volume.py:166-184)."""
    if np.isscalar(factor):
        factor = (factor,) * 3
    factor = tuple(int(k) for k in factor)
    if any(k < 1 for k in factor):
        raise ValueError(f"downsampling factor must be >= 1, got {factor}")
    lo, hi = ref.extent()
    dims = tuple(-(-d // k) for d, k in zip(ref.dims, factor))
    spacing = tuple(s * k for s, k in zip(ref.spacing, factor))
    size_ref = hi - lo
    size_lr = np.asarray(dims) * np.asarray(spacing)
    origin = lo + 0.5 * (size_ref - size_lr) + 0.5 * np.asarray(spacing)
    return GridSpec(dims, spacing, tuple(origin))


def save_volume(v: Volume, path: str, format: str | None = None) -> None:
    """Reference location of the volume writer (volume.py:208-217); see volume_io."""
    from .volume_io import save_volume as _save
    _save(v, path, format)


def load_volume(path: str, format: str | None = None) -> Volume:
    """Reference location of the volume reader (volume.py:220-229); see volume_io."""
    from .volume_io import load_volume as _load
    return _load(path, format)
