"""ctypes binding of libgsv_b200.so (the C ABI declared in include/gsv.h).

This is the only way the package reaches the GPU kernels.  There is no
fallback: if the library is missing or CUDA is unavailable, every entry point
raises.  Device pointers come from torch tensors (torch is plumbing here:
device memory, streams, torch.distributed).
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# GSV_LIB: an alternative build of the same ABI (measurement variants built by
# `python -m paper_2603_09621_b200.build --variant ...`); the default is the
# in-tree library __graft_entry__.build() produces
LIB_PATH = os.environ.get("GSV_LIB") or os.path.join(_HERE, "libgsv_b200.so")

c_int = ctypes.c_int
c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p
c_szp = ctypes.POINTER(ctypes.c_size_t)


class GsvGrid(ctypes.Structure):
    _fields_ = [("nx", c_i32), ("ny", c_i32), ("nz", c_i32), ("_pad", c_i32),
                ("ox", c_dbl), ("oy", c_dbl), ("oz", c_dbl),
                ("sx", c_dbl), ("sy", c_dbl), ("sz", c_dbl)]


class GsvBricks(ctypes.Structure):
    _fields_ = [("bdx", c_i32), ("bdy", c_i32), ("bdz", c_i32),
                ("bgx", c_i32), ("bgy", c_i32), ("bgz", c_i32),
                ("b0", c_i32), ("b1", c_i32)]


class GsvAdamHparams(ctypes.Structure):
    _fields_ = [("lr", c_dbl * 5), ("b1", c_dbl), ("b2", c_dbl), ("eps", c_dbl),
                ("bc1", c_dbl), ("bc2", c_dbl)]


GP = ctypes.POINTER(GsvGrid)
BP = ctypes.POINTER(GsvBricks)

# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGS = {
    "gsv_abi_version": [],
    "gsv_last_error": [],
    "gsv_device_sm_count": [],
    "gsv_preprocess": [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_dbl, GP, BP,
                       c_vp, c_vp, c_vp, c_vp, c_vp],
    "gsv_bin_workspace": [c_i64, c_i64, c_i32, c_szp],
    "gsv_bin_scan": [c_vp, c_i64, c_vp, c_vp, ctypes.c_size_t, c_vp],
    "gsv_bin_fill": [c_vp, c_vp, c_vp, c_i64, c_i64, BP, c_vp, c_vp, c_vp, c_vp, c_vp,
                     c_vp, ctypes.c_size_t, c_vp],
    "gsv_bin_fill_capacity": [c_vp, c_vp, c_vp, c_i64, c_i64, BP, c_vp, c_vp, c_vp, c_vp,
                              c_vp, c_vp, c_vp, c_vp, ctypes.c_size_t, c_vp],
    "gsv_preprocess_track": [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_dbl, GP, BP,
                             c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp],
    "gsv_bin_incremental_workspace": [c_i32, c_szp],
    "gsv_bin_incremental": [c_vp, c_vp, c_vp, c_i64, c_i64, BP, c_vp, c_vp, c_vp, c_vp, c_int,
                            c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp,
                            ctypes.c_size_t, c_vp],
    "gsv_lists_unsorted": [c_vp, c_vp, c_i32, c_i64, c_vp, c_vp],
    "gsv_canonicalize_workspace": [c_i64, c_i32, c_szp],
    "gsv_canonicalize": [c_vp, c_vp, c_vp, c_i32, c_i64, c_vp, ctypes.c_size_t, c_vp],
    "gsv_loss_bricks": [GP, BP, c_dbl, c_vp, c_vp, c_vp, c_int, c_int, c_dbl, c_int, c_vp, c_vp,
                        c_vp],
    "gsv_forward": [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, GP, BP, c_dbl, c_dbl, c_int,
                    c_vp, c_vp, c_vp, c_vp, c_int, c_int, c_dbl, c_vp, c_vp, c_vp, c_int, c_vp],
    "gsv_backward_prep": [c_vp, c_vp, c_vp, GP, BP, c_dbl, c_int, c_vp, c_vp, c_vp],
    "gsv_backward": [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, GP, BP, c_dbl,
                     c_int, c_vp, c_vp, c_int, c_vp, c_vp],
    "gsv_merge": [c_vp, c_vp, c_i64, c_int, c_vp, c_vp],
    "gsv_chain_rule": [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_vp,
                       c_vp, c_vp],
    "gsv_loss_blocks": [c_i64],
    "gsv_loss": [c_vp, c_int, c_vp, c_int, c_i64, c_int, c_vp, c_vp, c_vp],
    "gsv_sum": [c_vp, c_i64, c_vp, c_vp],
    "gsv_adam": [c_vp, c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, c_dbl,
                 c_vp],
    "gsv_normalize_rotations": [c_vp, c_i64, c_vp],
    "gsv_fused_update": [c_vp, c_vp, c_vp, c_i64, c_int, c_vp, c_vp, c_vp, c_vp, c_vp,
                         ctypes.POINTER(c_vp), c_int, c_int, ctypes.POINTER(GsvAdamHparams),
                         c_vp, c_vp],
    "gsv_step_gate": [c_vp, c_vp, c_vp, c_vp, c_vp],
    "gsv_shard_pack": [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp],
    "gsv_shard_unpack": [c_vp, c_i64, c_vp, c_vp, c_vp, c_vp],
    "gsv_fused_update_device": [c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                ctypes.POINTER(c_vp), c_int, c_int,
                                ctypes.POINTER(GsvAdamHparams), c_vp, c_vp, c_vp, GP, BP,
                                c_dbl, c_vp, c_vp, c_vp, c_vp],
    "gsv_step_advance": [c_vp, c_vp, c_vp],
    "gsv_step_advance_publish": [c_vp, c_vp, c_vp, c_vp, c_vp, c_int, c_vp],
    "gsv_metric_blocks": [c_i64],
    "gsv_sq_diff_sum": [c_vp, c_int, c_vp, c_int, c_i64, c_vp, c_vp, c_vp],
    "gsv_ssim3d_workspace": [GP, c_szp],
    "gsv_ssim3d": [c_vp, c_int, c_vp, c_int, GP, c_vp, c_vp, ctypes.c_size_t, c_vp, c_vp],
    "gsv_rotation_matrices": [c_vp, c_i64, c_vp, c_vp],
    "gsv_sigma_inv": [c_vp, c_vp, c_i64, c_vp, c_vp],
    "gsv_weight": [c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_int, c_dbl, c_dbl, c_dbl, c_dbl,
                   c_vp, c_vp],
    "gsv_render_naive": [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_int, GP, c_dbl, c_dbl, c_int,
                         c_vp, c_vp],
    "gsv_phantom": [GP, c_int, c_int, c_vp, c_int, c_vp, c_vp, c_vp, c_vp],
    "gsv_resample_trilinear": [c_vp, c_int, GP, c_vp, GP, c_vp],
    "gsv_pool_loss_blocks": [GP],
    "gsv_pool_loss": [c_vp, c_vp, c_vp, c_int, GP, GP, c_int, c_int, c_int, c_int, c_dbl, c_vp,
                      c_vp, c_vp],
    "gsv_init_workspace": [GP, c_szp],
    "gsv_init_count": [c_vp, c_int, GP, c_dbl, c_vp, c_vp, ctypes.c_size_t, c_vp],
    "gsv_init_fill": [c_vp, c_int, GP, c_dbl, c_vp, c_vp, c_dbl, c_vp, c_vp, c_vp, c_vp, c_vp,
                      c_vp],
    # include/gsv_diag.h (measurement only)
    "gsv_diag_count_live": [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, GP, BP, c_dbl, c_vp, c_vp],
    "gsv_diag_fma_probe": [c_int, c_int, c_vp, c_vp],
}
_RESTYPES = {"gsv_last_error": ctypes.c_char_p}

EXPORTS = tuple(_SIGS)
ABI_VERSION = 6        # GSV_ABI_VERSION of include/gsv.h these signatures follow

_lib = None


class GsvLibraryError(RuntimeError):
    """The CUDA extension is missing, failed to load, or a call failed."""


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the C ABI.  Raises if the library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise GsvLibraryError(
            f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    lib.gsv_abi_version.restype = c_int
    if lib.gsv_abi_version() != ABI_VERSION:
        raise GsvLibraryError(f"{path} implements ABI {lib.gsv_abi_version()}, these bindings "
                              f"expect {ABI_VERSION}: rebuild the library")
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, c_int)
    _lib = lib
    return lib


def lib() -> ctypes.CDLL:
    l = load()
    if not torch.cuda.is_available():
        raise GsvLibraryError("CUDA device not available; the B200 rasterizer has no CPU path")
    return l


def check(status: int, what: str) -> None:
    if status != 0:
        msg = load().gsv_last_error().decode(errors="replace")
        raise GsvLibraryError(f"{what} failed (status {status}): {msg}")


def ptr(t) -> int | None:
    """Raw device pointer of a tensor (None for None)."""
    if t is None:
        return None
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def make_grid(grid) -> GsvGrid:
    nx, ny, nz = grid.dims
    ox, oy, oz = grid.origin
    sx, sy, sz = grid.spacing
    return GsvGrid(nx, ny, nz, 0, ox, oy, oz, sx, sy, sz)


def make_bricks(grid, brick_dims, slab=None) -> GsvBricks:
    bdx, bdy, bdz = brick_dims
    nx, ny, nz = grid.dims
    bgx, bgy, bgz = -(-nx // bdx), -(-ny // bdy), -(-nz // bdz)
    b0, b1 = (0, bgx * bgy * bgz) if slab is None else slab
    return GsvBricks(bdx, bdy, bdz, bgx, bgy, bgz, b0, b1)


_ws_cache: dict = {}


def workspace(nbytes: int, device, key: str = "default") -> torch.Tensor:
    """Grow-only scratch buffer per (device, stream, key) for CUB temp storage.

    Keyed by the stream the work is enqueued on (the current stream), so
    two callers on different streams (two Renderers, a TrainStep beside an
    eager render) never share scratch that both may be using at once.  On
    one stream, launches are ordered and the reuse is safe.  The buffer is
    allocated while that stream is current, so the caching allocator orders
    its eventual reuse after the stream's pending work.
    """
    dev = torch.device(device)
    s = torch.cuda.current_stream(dev) if dev.type == "cuda" else None
    k = (str(dev), 0 if s is None else s.cuda_stream, key)
    buf = _ws_cache.get(k)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes * 1.25), 1 << 16), dtype=torch.uint8, device=device)
        _ws_cache[k] = buf
    return buf


class BufferPool:
    """Grow-only device buffers reused across iterations (train step / render).

    ``get(name, shape, dtype)`` returns a view of a persistent flat buffer, so
    the per-iteration allocations of the hot loop never reach cudaMalloc.
    Views stay valid until the next ``get`` of the same name.
    """

    def __init__(self, device):
        self.device = device
        self._bufs: dict = {}

    def get(self, name: str, shape, dtype, zeroed: bool = False) -> torch.Tensor:
        """``zeroed``: a newly allocated buffer starts at zero (slab outputs, whose
        voxels outside the slab are never written)."""
        shape = tuple(int(s) for s in (shape if isinstance(shape, (tuple, list)) else (shape,)))
        numel = 1
        for s in shape:
            numel *= s
        key = (name, dtype)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < max(numel, 1):
            alloc = torch.zeros if zeroed else torch.empty
            buf = alloc(int(max(numel, 1) * 1.1) + 64, dtype=dtype, device=self.device)
            self._bufs[key] = buf
        return buf[:numel].view(shape) if shape else buf[:1].view(())
