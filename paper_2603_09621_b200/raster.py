"""Brick rasterizer: the drop-in API of gsvol/raster.py on B200 kernels.

Same public names, signatures, dataclass fields and exceptions as
raster.py:55-570; every computation runs in libgsv_b200.so (include/gsv.h):

  build_brick_index  gsv_preprocess -> gsv_bin_scan -> gsv_bin_fill
                     (fused f64 AABB + count, CUB scan, emit + CUB stable radix
                     sort + CSR starts); bit-exact lists (raster.py:148-217)
  forward            gsv_preprocess (records) -> gsv_forward (CTA per brick)
  backward           gsv_backward_prep -> gsv_backward (pair partials) ->
                     gsv_merge (ascending brick order) -> gsv_chain_rule

Extensions (keyword-only, defaults keep the reference behaviour):
``slab=(b0, b1)`` restricts binning/render/backward to the contiguous brick-id
range [b0, b1) -- the sharding unit of the multi-GPU path (distributed.py).

Arrays are torch tensors on the field's CUDA device.  ``BrickIndex.gids`` is
int32 (the reference uses int64; values are identical), ``starts`` int64.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _lib
from .errors import NumericalError, StaleIndexError
from .field import GaussianField
from .render import RenderOptions
from .volume import GridSpec, Volume

DEFAULT_BRICK_DIMS = (8, 8, 4)

_WORKERS = [8]


def set_worker_count(n: int) -> None:
    """Kept for API parity (raster.py:55-59); the GPU engine has no thread pool."""
    if n < 1:
        raise ValueError("worker count must be >= 1")
    _WORKERS[0] = int(n)


def worker_count() -> int:
    return _WORKERS[0]


def _as_device_tensor(a, dtype, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=np.dtype(str(dtype).split(".")[-1]))).to(device)


@dataclass
class _Aux:
    """Per-Gaussian products of preprocessing kept with an index we built."""
    rec32: torch.Tensor
    rec64: torch.Tensor | None
    counts: torch.Tensor
    box: torch.Tensor
    gstart: torch.Tensor
    field_version: int
    canonical: bool = True
    active: int | None = None        # Gaussians with >= 1 pair (the forward's tiling choice)


@dataclass(frozen=True)
class BrickIndex:
    """CSR layout of per-brick Gaussian lists (raster.py:66-112).

    gids[starts[b]:starts[b+1]] are the Gaussians binned to brick b,
    ascending; bricks x-fastest.  With ``slab=(b0, b1)`` the index covers
    only bricks [b0, b1) and ``starts`` has one entry per slab brick.
    """
    grid: GridSpec
    brick_dims: tuple
    brick_grid: tuple
    starts: object
    gids: object
    field_version: int
    field_count: int
    cutoff_sigma: float
    slab: tuple | None = None
    _aux: object = dc_field(default=None, compare=False, repr=False)

    def __post_init__(self):
        dev = self.starts.device if isinstance(self.starts, torch.Tensor) else None
        if dev is None and isinstance(self.gids, torch.Tensor):
            dev = self.gids.device
        if dev is None:
            dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
                else torch.device("cpu")
        object.__setattr__(self, "starts", _as_device_tensor(self.starts, torch.int64, dev))
        object.__setattr__(self, "gids", _as_device_tensor(self.gids, torch.int32, dev))
        object.__setattr__(self, "brick_dims", tuple(int(b) for b in self.brick_dims))
        object.__setattr__(self, "brick_grid", tuple(int(b) for b in self.brick_grid))

    @property
    def brick_count(self) -> int:
        return int(self.starts.shape[0]) - 1

    @property
    def pair_count(self) -> int:
        return int(self.gids.shape[0])

    @property
    def slab_range(self) -> tuple:
        bg = self.brick_grid
        return self.slab if self.slab is not None else (0, bg[0] * bg[1] * bg[2])

    def lists_sorted(self) -> bool:
        """True when every brick's list is ascending (canonical order)."""
        if self._aux is not None and self._aux.canonical:
            return True
        if self.pair_count == 0:
            return True
        lib = _lib.lib()
        flag = torch.zeros(1, dtype=torch.int32, device=self.gids.device)
        _lib.check(lib.gsv_lists_unsorted(self.starts.data_ptr(), self.gids.data_ptr(),
                                          self.brick_count, self.pair_count, flag.data_ptr(),
                                          _lib.stream_ptr()), "lists_unsorted")
        return int(flag.item()) == 0

    def canonicalized(self) -> "BrickIndex":
        """An index with every brick list sorted ascending (segmented GPU sort)."""
        if self.lists_sorted():
            return self
        lib = _lib.lib()
        import ctypes
        nbytes = ctypes.c_size_t(0)
        _lib.check(lib.gsv_canonicalize_workspace(self.pair_count, self.brick_count,
                                                  ctypes.byref(nbytes)), "canonicalize_workspace")
        ws = _lib.workspace(nbytes.value, self.gids.device, "canon")
        out = torch.empty_like(self.gids)
        _lib.check(lib.gsv_canonicalize(self.starts.data_ptr(), self.gids.data_ptr(),
                                        out.data_ptr(), self.brick_count, self.pair_count,
                                        ws.data_ptr(), ws.numel(), _lib.stream_ptr()),
                   "canonicalize")
        return BrickIndex(self.grid, self.brick_dims, self.brick_grid, self.starts, out,
                          self.field_version, self.field_count, self.cutoff_sigma, self.slab,
                          None)


@dataclass(frozen=True)
class RenderCache:
    """Forward products: per-voxel numerator, denominator, render (raster.py:115-125)."""
    grid: GridSpec
    S: torch.Tensor
    W: torch.Tensor
    I: torch.Tensor
    field_version: int

    def volume(self) -> Volume:
        return Volume.from_linear(self.grid, self.I)


@dataclass
class GradientBuffer:
    """Per-Gaussian gradients w.r.t. the raw parameters (raster.py:128-145)."""
    raw_amplitude: torch.Tensor
    raw_relax: torch.Tensor
    positions: torch.Tensor
    log_scales: torch.Tensor
    rotations: torch.Tensor

    @classmethod
    def zeros(cls, n: int, device=None) -> "GradientBuffer":
        dev = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available()
            else torch.device("cpu"))
        z = lambda *s: torch.zeros(*s, dtype=torch.float64, device=dev)  # noqa: E731
        return cls(z(n), z(n), z(n, 3), z(n, 3), z(n, 4))

    @classmethod
    def empty(cls, n: int, device) -> "GradientBuffer":
        e = lambda *s: torch.empty(*s, dtype=torch.float64, device=device)  # noqa: E731
        return cls(e(n), e(n), e(n, 3), e(n, 3), e(n, 4))

    def tensors(self):
        return (self.raw_amplitude, self.raw_relax, self.positions, self.log_scales,
                self.rotations)

    def all_finite(self) -> bool:
        return all(bool(torch.isfinite(a).all()) for a in self.tensors())


# ----------------------------------------------------------------- binning
def _alloc(pool, name, shape, dtype, device):
    if pool is not None:
        return pool.get(name, shape, dtype)
    return torch.empty(shape, dtype=dtype, device=device)


def _preprocess(f: GaussianField, grid: GridSpec, cutoff_sigma: float, brick_dims, slab,
                want64: bool = True, pool=None):
    lib = _lib.lib()
    n, dev = f.count, f.device
    rec32 = _alloc(pool, "rec32", (n, 16), torch.float32, dev)
    # rec64 only for the f64 engine; the f32 engine recomputes the f64 factor
    # in its rare guard-band path
    rec64 = _alloc(pool, "rec64", (n, 12), torch.float64, dev) if want64 else None
    counts = _alloc(pool, "counts", (n,), torch.int32, dev)
    box = _alloc(pool, "box", (n, 4), torch.int32, dev)
    _lib.check(lib.gsv_preprocess(
        f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
        f.raw_amplitude.data_ptr(), f.raw_relax.data_ptr(), n, int(f.relax_enabled),
        float(cutoff_sigma), _lib.make_grid(grid), _lib.make_bricks(grid, brick_dims, slab),
        rec32.data_ptr(), _lib.ptr(rec64), counts.data_ptr(), box.data_ptr(),
        _lib.stream_ptr()), "preprocess")
    return rec32, rec64, counts, box


def _scan(counts: torch.Tensor, nbricks: int, pool=None) -> torch.Tensor:
    import ctypes
    lib = _lib.lib()
    n = counts.shape[0]
    gstart = _alloc(pool, "gstart", (n + 1,), torch.int64, counts.device)
    nbytes = ctypes.c_size_t(0)
    _lib.check(lib.gsv_bin_workspace(n, 1, nbricks, ctypes.byref(nbytes)), "bin_workspace")
    ws = _lib.workspace(nbytes.value, counts.device, "bin")
    _lib.check(lib.gsv_bin_scan(counts.data_ptr(), n, gstart.data_ptr(), ws.data_ptr(),
                                ws.numel(), _lib.stream_ptr()), "bin_scan")
    return gstart


def _fill(counts, box, gstart, pairs: int, bricks, nbricks: int, pool=None):
    import ctypes
    lib = _lib.lib()
    dev = counts.device
    n = counts.shape[0]
    nbytes = ctypes.c_size_t(0)
    _lib.check(lib.gsv_bin_workspace(n, max(pairs, 1), nbricks, ctypes.byref(nbytes)),
               "bin_workspace")
    ws = _lib.workspace(nbytes.value, dev, "bin")
    # sort scratch is never returned: always from the grow-only scratch pool
    scratch = _lib.workspace(3 * 4 * max(pairs, 1) + 64, dev, "bin_keys")
    keys_tmp = scratch[: 4 * max(pairs, 1)].view(torch.int32)
    vals_tmp = scratch[4 * max(pairs, 1): 8 * max(pairs, 1)].view(torch.int32)
    keys_out = scratch[8 * max(pairs, 1): 12 * max(pairs, 1)].view(torch.int32)
    gids = _alloc(pool, "gids", (pairs,), torch.int32, dev)
    starts = _alloc(pool, "starts", (nbricks + 1,), torch.int64, dev)
    _lib.check(lib.gsv_bin_fill(counts.data_ptr(), box.data_ptr(), gstart.data_ptr(), n, pairs,
                                bricks, keys_tmp.data_ptr(), vals_tmp.data_ptr(),
                                keys_out.data_ptr(), gids.data_ptr() if pairs else keys_out.data_ptr(),
                                starts.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr()),
               "bin_fill")
    return starts, gids


def build_brick_index(f: GaussianField, grid: GridSpec, opts: RenderOptions = RenderOptions(),
                      brick_dims=DEFAULT_BRICK_DIMS, *, slab=None, pool=None) -> BrickIndex:
    """Conservative Gaussian-to-brick binning via AABB overlap (raster.py:148-217).

    Lists are bit-identical to the reference's (same f64 bounds, same
    gid-major emission, stable sort by brick id).  ``pool`` (a
    _lib.BufferPool) makes the index's arrays views of reusable buffers --
    valid until the next build with the same pool (TrainStep / Renderer).
    """
    if any(d < 1 for d in brick_dims):
        raise ValueError(f"brick_dims must be positive, got {brick_dims}")
    brick_dims = tuple(int(d) for d in brick_dims)
    bricks = _lib.make_bricks(grid, brick_dims, slab)
    nbricks = bricks.b1 - bricks.b0
    rec32, rec64, counts, box = _preprocess(f, grid, opts.cutoff_sigma, brick_dims, slab,
                                            opts.precision == "f64", pool)
    gstart = _scan(counts, nbricks, pool)
    pairs = int(gstart[-1].item())  # the one host read binning needs (buffer sizing)
    starts, gids = _fill(counts, box, gstart, pairs, bricks, nbricks, pool)
    aux = _Aux(rec32, rec64, counts, box, gstart, f.version, True)
    return BrickIndex(grid, brick_dims, (bricks.bgx, bricks.bgy, bricks.bgz), starts, gids,
                      f.version, f.count, opts.cutoff_sigma, slab, aux)


def _check_index(f: GaussianField, grid: GridSpec, idx: BrickIndex, opts: RenderOptions) -> None:
    """Staleness guards, same messages as raster.py:220-230."""
    if idx.field_version != f.version or idx.field_count != f.count:
        raise StaleIndexError(
            f"rebuild brick index: built for field version {idx.field_version}, "
            f"field is at version {f.version}")
    if idx.grid != grid:
        raise StaleIndexError("rebuild brick index: grid changed")
    if idx.cutoff_sigma != opts.cutoff_sigma:
        raise StaleIndexError("rebuild brick index: cutoff_sigma changed")


def _records(f, grid, idx: BrickIndex, opts: RenderOptions):
    """rec32 (and rec64 for f64) for the current field state."""
    aux = idx._aux
    want64 = opts.precision == "f64"
    if aux is not None and aux.field_version == f.version and (aux.rec64 is not None or not want64):
        return aux.rec32, aux.rec64
    rec32, rec64, _, _ = _preprocess(f, grid, opts.cutoff_sigma, idx.brick_dims, idx.slab, want64)
    return rec32, rec64


# ----------------------------------------------------------------- forward
def _reaching(f: GaussianField, idx: BrickIndex) -> int:
    """Gaussians that reach the index's bricks: N for a whole-grid index
    (Gaussians outside the grid are few), counted once for a slab index."""
    aux = idx._aux
    if idx.slab is None or aux is None:
        return f.count
    if aux.active is None:
        aux.active = int(torch.count_nonzero(aux.counts).item())
    return aux.active


def _resolve_vpl(brick_dims) -> int:
    """Voxels per lane of the f32 forward's warp tiles (gsv_forward's vpl,
    the same rule as its auto mode): 4 -- columns of 4 in z, 8x4x4 tiles --
    when bdz % 4 == 0 and the brick has <= 64 columns, else 2 (4x4x4 tiles).
    GSV_VPL=2|4 forces one (measurement)."""
    forced = os.environ.get("GSV_VPL")
    if forced in ("2", "4"):
        return int(forced)
    bx, by, bz = brick_dims
    return 4 if bz % 4 == 0 and bx * by * (bz // 4) <= 64 else 2


# Pairs per reaching Gaussian up to which the grouped-column forward is used
# (LR grids: ~4.3 at configs 1-4; the 256^3 render has 11.5, 512^3 46).
_GROUPED_MAX_DENSITY = 8.0


def _use_grouped(brick_dims, pairs: int, n: int) -> bool:
    """The grouped-column forward (gsv_forward vpl 16) for 8x8x4 bricks when
    Gaussians are small against a brick (pairs <= 8 per reaching Gaussian:
    LR training grids).  There its z-runs of identical footprints make
    ~2.4x fewer (pair, column) evaluations than the two-list whole-brick
    kernel and the forward runs ~7% faster; at HR densities groups shrink to
    ~1.3 pairs and the whole-brick kernel wins (2.0 vs 3.0 ms at 256^3).
    The choice depends only on the index, so the train step, forward() and
    Renderer render bit-identically at a given grid.  GSV_FWD_COLS=0 / =1
    forces the whole-brick / grouped kernel (measurement, A-B runs)."""
    if tuple(brick_dims) != (8, 8, 4) or os.environ.get("GSV_NO_WHOLE") \
            or os.environ.get("GSV_VPL"):
        return False
    forced = os.environ.get("GSV_FWD_COLS", "")
    if forced in ("0", "1"):
        return forced == "1"
    return pairs <= _GROUPED_MAX_DENSITY * max(n, 1)


def _train_mask_vpl(brick_dims, pairs: int, n: int) -> int:
    """Mask layout of the train step's forward -> masked backward: 16 (the
    grouped forward's column-nibble masks) or, for the whole-brick and
    warp-tile forwards, their warp-tile layout (_resolve_vpl)."""
    return 16 if _use_grouped(brick_dims, pairs, n) else _resolve_vpl(brick_dims)


def _forward_vpl_arg(brick_dims, pairs: int = 0, n: int = 0, masks: bool = True) -> int:
    """gsv_forward's vpl argument.  8x8x4 bricks (the default): 16, the
    grouped-column kernel, at LR densities (_use_grouped), else 8, one warp
    per brick with two columns per lane and the pairs of each 32-pair round
    compacted into one hit list per y-half (LR train forward 0.99 -> 0.91 ms,
    256^3 render 2.26 -> 2.01 ms against the warp-tile kernels).  Either
    writes live masks for the train step.  Other bricks use the warp-tile
    kernels (_resolve_vpl); GSV_NO_WHOLE=1 or GSV_VPL=2|4 force those
    (measurement), GSV_NO_SPLIT keeps a brick's two tiles in one CTA.
    pairs / n: the index's pairs and the Gaussians reaching it."""
    del masks
    if _use_grouped(brick_dims, pairs, n):
        return 16
    if (tuple(brick_dims) == (8, 8, 4) and not os.environ.get("GSV_NO_WHOLE")
            and not os.environ.get("GSV_VPL")):
        return 8
    return _resolve_vpl(brick_dims) | (0x200 if os.environ.get("GSV_NO_SPLIT") else 0)


def _masks_fit(brick_dims, vpl: int) -> bool:
    """Live masks need a brick that fills one CTA's warp tiles exactly (4
    planes of mask words), e.g. the default 8x8x4."""
    if vpl == 16:
        return tuple(brick_dims) == (8, 8, 4)
    bx, by, bz = brick_dims
    return bx * by * (-(-bz // vpl)) == (64 if vpl == 4 else 128)


def _forward_into(f, grid, idx, opts, rec32, rec64, S, W, I, target=None, loss_kind=0,
                  ab=None, loss_part=None, live_masks=None):
    lib = _lib.lib()
    _lib.check(lib.gsv_forward(
        f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
        rec32.data_ptr(), _lib.ptr(rec64), idx.starts.data_ptr(), idx.gids.data_ptr(),
        _lib.make_grid(grid),
        _lib.make_bricks(grid, idx.brick_dims, idx.slab),
        float(opts.cutoff_sigma), float(opts.epsilon_w), opts.precision_code,
        S.data_ptr(), W.data_ptr(), I.data_ptr(), _lib.ptr(target),
        int(target is not None and target.dtype == torch.float64), int(loss_kind),
        float(grid.num_voxels), _lib.ptr(ab), _lib.ptr(loss_part), _lib.ptr(live_masks),
        _forward_vpl_arg(idx.brick_dims, idx.pair_count, _reaching(f, idx),
                         live_masks is not None),
        _lib.stream_ptr()), "forward")


def forward(f: GaussianField, grid: GridSpec, idx: BrickIndex,
            opts: RenderOptions = RenderOptions()) -> RenderCache:
    """Brick-parallel render (raster.py:296-319); equals render_naive up to
    accumulation noise.  Output arrays are linear x-fastest, opts' dtype."""
    _check_index(f, grid, idx, opts)
    if opts.deterministic:
        idx = idx.canonicalized()
    rec32, rec64 = _records(f, grid, idx, opts)
    nvox = grid.num_voxels
    dt = opts.torch_dtype
    alloc = torch.zeros if idx.slab is not None else torch.empty
    S = alloc(nvox, dtype=dt, device=f.device)
    W = alloc(nvox, dtype=dt, device=f.device)
    I = alloc(nvox, dtype=dt, device=f.device)
    _forward_into(f, grid, idx, opts, rec32, rec64, S, W, I)
    return RenderCache(grid, S, W, I, f.version)


# ----------------------------------------------------------------- backward
def _emission_layout(f, grid, idx: BrickIndex, opts: RenderOptions):
    """(gstart, box, trusted): the pair slots the backward writes into."""
    aux = idx._aux
    if aux is not None and aux.field_version == f.version:
        return aux.gstart, aux.box, True
    _, _, counts, box = _preprocess(f, grid, opts.cutoff_sigma, idx.brick_dims, idx.slab, False)
    b = _lib.make_bricks(grid, idx.brick_dims, idx.slab)
    gstart = _scan(counts, b.b1 - b.b0)
    return gstart, box, False


def _pair_partials(f, grid, idx, opts, rec32, rec64, ab, gstart, box, trusted: bool,
                   timer=None, pool=None, live_masks=None, mask_vpl: int = 0):
    lib = _lib.lib()
    n = f.count
    pdt = opts.torch_dtype
    npairs = int(gstart[-1].item()) if not trusted else idx.pair_count
    if trusted:
        partials = _alloc(pool, "partials", (max(npairs, 1), 12), pdt, f.device)
    else:
        partials = torch.zeros((max(npairs, 1), 12), dtype=pdt, device=f.device)
    if timer is not None:
        timer("backward")
    _lib.check(lib.gsv_backward(
        f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
        rec32.data_ptr(), _lib.ptr(rec64), idx.starts.data_ptr(), idx.gids.data_ptr(),
        gstart.data_ptr(),
        box.data_ptr(), _lib.make_grid(grid), _lib.make_bricks(grid, idx.brick_dims, idx.slab),
        float(opts.cutoff_sigma), opts.precision_code, ab.data_ptr(), _lib.ptr(live_masks),
        int(mask_vpl), partials.data_ptr(), _lib.stream_ptr()), "backward")
    gsum = _alloc(pool, "gsum", (n, 12), torch.float64, f.device)
    if timer is not None:
        timer("merge")
    _lib.check(lib.gsv_merge(partials.data_ptr(), gstart.data_ptr(), n, opts.precision_code,
                             gsum.data_ptr(), _lib.stream_ptr()), "merge")
    if timer is not None:
        timer(None)
    return gsum


def _chain_rule(f: GaussianField, gsum: torch.Tensor, pool=None) -> GradientBuffer:
    lib = _lib.lib()
    n = f.count
    if pool is None:
        out = GradientBuffer.empty(n, f.device)
    else:
        gb = pool.get("grads", (12 * n,), torch.float64)
        out = GradientBuffer(gb[:n], gb[n:2 * n], gb[2 * n:5 * n].view(n, 3),
                             gb[5 * n:8 * n].view(n, 3), gb[8 * n:].view(n, 4))
    _lib.check(lib.gsv_chain_rule(
        gsum.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
        f.raw_amplitude.data_ptr(), f.raw_relax.data_ptr(), f.count, int(f.relax_enabled),
        out.raw_amplitude.data_ptr(), out.raw_relax.data_ptr(), out.positions.data_ptr(),
        out.log_scales.data_ptr(), out.rotations.data_ptr(), _lib.stream_ptr()), "chain_rule")
    return out


def backward(f: GaussianField, grid: GridSpec, idx: BrickIndex, cache: RenderCache, dL_dI,
             opts: RenderOptions = RenderOptions()) -> GradientBuffer:
    """Analytic gradients through the normalized render (raster.py:470-549).

    dL_dI: per-voxel upstream gradient, linear x-fastest (numpy or torch).
    Gradients are w.r.t. the raw stored parameters; quaternion gradients are
    ambient (4-d).
    """
    _check_index(f, grid, idx, opts)
    if cache.field_version != f.version:
        raise StaleIndexError("rebuild brick index: cache is stale")
    if opts.deterministic:
        idx = idx.canonicalized()
    dl = _as_device_tensor(dL_dI, torch.float64, f.device).reshape(-1)
    nvox = grid.num_voxels
    if dl.shape[0] != nvox:
        raise ValueError(f"dL_dI has {dl.shape[0]} entries, grid has {nvox} voxels")
    lib = _lib.lib()
    pdt = opts.torch_dtype
    ab = torch.zeros((nvox, 2), dtype=pdt, device=f.device)
    bad = torch.empty(1, dtype=torch.int64, device=f.device)
    # Converted copies must stay referenced until the launch is enqueued: a
    # temporary freed after data_ptr() can be handed straight to the next
    # conversion by the caching allocator, aliasing W and I.
    Wc = cache.W if cache.W.dtype == pdt else cache.W.to(pdt)
    Ic = cache.I if cache.I.dtype == pdt else cache.I.to(pdt)
    _lib.check(lib.gsv_backward_prep(
        Wc.data_ptr(), Ic.data_ptr(),
        dl.data_ptr(), _lib.make_grid(grid), _lib.make_bricks(grid, idx.brick_dims, idx.slab),
        float(opts.epsilon_w), opts.precision_code, ab.data_ptr(), bad.data_ptr(),
        _lib.stream_ptr()), "backward_prep")
    del Wc, Ic
    k = int(bad.item())
    if k < nvox:
        raise NumericalError(f"non-finite dL_dI at voxel index {k}")
    rec32, rec64 = _records(f, grid, idx, opts)
    gstart, box, trusted = _emission_layout(f, grid, idx, opts)
    gsum = _pair_partials(f, grid, idx, opts, rec32, rec64, ab, gstart, box, trusted)
    return _chain_rule(f, gsum)


def merge_gradients(partials) -> GradientBuffer:
    """Sum per-brick GradientBuffers in ascending brick-index order (raster.py:552-570)."""
    items = sorted(partials, key=lambda kv: kv[0])
    if not items:
        raise ValueError("no partials to merge")
    first = items[0][1]
    n = first.raw_amplitude.shape[0]
    dev = first.raw_amplitude.device if isinstance(first.raw_amplitude, torch.Tensor) else None
    out = GradientBuffer.zeros(n, device=dev)
    for _, buf in items:
        for dst, src in zip(out.tensors(), buf.tensors()):
            dst += src if isinstance(src, torch.Tensor) else torch.as_tensor(src, device=dst.device)
    return out
