"""The fused training step: one iteration of fit() (optimize.py:171-184).

  forward(f):  build_brick_index -> gsv_forward with the L1/L2 loss fused into
               the epilogue (per-voxel backward inputs {dL/dI / W, I} written
               in the same pass) -> per-brick loss partials -> gsv_sum.  No
               separate loss kernel, no dL/dI round trip through HBM.
  backward(f): gsv_backward (pair partials at their gid-major emission slots)
               -> gsv_merge (ascending brick order) -> [all_reduce of the
               N x 12 partial sums, the only collective, when sharded] ->
               gsv_chain_rule.

The graph-replayed step (TrainStep.step / step_async, what fit() calls) is
the same iteration captured once and replayed; it bins incrementally from the
second replay on (see _StepGraph).

Sharding: with ``slab=(b0, b1)`` a rank bins, renders and
back-propagates only its contiguous brick-id range; the per-Gaussian
merged partials (and the loss, carried in the spare 12th column) are summed
across ranks by one NCCL all_reduce, after which every rank applies the same
chain rule and Adam step, so parameters stay replicated.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import torch

from . import _lib
from .field import GaussianField
from .raster import (BrickIndex, GradientBuffer, RenderCache, _alloc, _chain_rule,
                     _forward_vpl_arg, _masks_fit, _reaching,
                     _preprocess, _resolve_vpl, _scan, _train_mask_vpl,
                     _forward_into, _pair_partials, build_brick_index)
from .render import RenderOptions
from .volume import Volume

LOSS_KINDS = {"l1": 0, "l2": 1}

# GSV_NVTX=1 brackets every phase, capture and replay with NVTX ranges (for
# nsys / ncu --nvtx); off by default so the replay path stays host-lean
NVTX = os.environ.get("GSV_NVTX", "") == "1"


def _nvtx_push(name: str) -> None:
    if NVTX:
        torch.cuda.nvtx.range_push(name)


def _nvtx_pop() -> None:
    if NVTX:
        torch.cuda.nvtx.range_pop()


class PhaseTimer:
    """CUDA events on the launching stream around each kernel phase.

    ``mark(name)`` closes the open phase and opens ``name`` (None closes only).
    ``summary()`` synchronizes and returns {phase: (launches, mean_ms)}.
    """

    def __init__(self):
        self.events: list = []          # (name, start_event, end_event)
        self._open = None

    def __call__(self, name):
        s = torch.cuda.current_stream()
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(s)
        if self._open is not None:
            self.events.append((self._open[0], self._open[1], ev))
            _nvtx_pop()
        self._open = (name, ev) if name is not None else None
        if name is not None:
            _nvtx_push("gsv." + name)

    def reset(self):
        if self._open is not None:
            _nvtx_pop()
        self.events.clear()
        self._open = None

    def summary(self) -> dict:
        torch.cuda.synchronize()
        out: dict = {}
        for name, a, b in self.events:
            n, t = out.get(name, (0, 0.0))
            out[name] = (n + 1, t + a.elapsed_time(b))
        return {k: (n, t / n) for k, (n, t) in out.items()}


@dataclass
class StepOutput:
    idx: BrickIndex
    cache: RenderCache
    ab: torch.Tensor
    loss_sum: torch.Tensor     # (1,) float64 on device: sum of |I-T| (l1) or (I-T)^2
    nvox: int
    reduced: bool = False

    def loss(self) -> float:
        """Mean loss as a Python float (one 8-byte device->host read).  When
        sharded, valid after TrainStep.backward (the loss rides its all_reduce)."""
        if not self.reduced:
            raise RuntimeError("sharded loss is only global after backward()")
        return float(self.loss_sum.item()) / self.nvox


class TrainStep:
    """Reusable fused train step bound to one target volume and options."""

    def __init__(self, target: Volume, opts: RenderOptions = RenderOptions(),
                 brick_dims=(8, 8, 4), loss: str = "l1", slab=None, process_group=None,
                 world_size: int = 1, timer: PhaseTimer | None = None):
        if loss not in LOSS_KINDS:
            raise ValueError(f"unknown loss kind {loss!r}")
        self.grid = target.grid
        lin = target.linear()
        if lin.device.type != "cuda":
            lin = lin.to(torch.device("cuda", torch.cuda.current_device()))
        # the fused loss subtracts in f64 from the target's own values, like
        # loss_and_grad (optimize.py:97): an f64 volume keeps its f64 target
        tdt = torch.float64 if lin.dtype == torch.float64 else torch.float32
        self.target = lin.to(tdt).contiguous()
        self.opts = opts
        self.brick_dims = tuple(brick_dims)
        self.loss_kind = LOSS_KINDS[loss]
        self.slab = slab
        self.group = process_group
        self.world_size = world_size
        self.timer = timer
        # Persistent buffers: index, voxel arrays, pair partials, gradients.
        # Everything a step returns is a view valid until the next step.
        self.pool = _lib.BufferPool(self.target.device)
        self._masks = None
        self._mask_vpl = 0

    @property
    def sharded(self) -> bool:
        """A process group was given: the step all_reduces over it (also at
        world size 1, where the reduction is the identity)."""
        return self.group is not None

    def set_target(self, target_linear: torch.Tensor) -> None:
        """Load a new target volume (linear x-fastest, V values) into the step's
        persistent target buffer, stream-ordered: from a device tensor (a
        device copy) or a pinned host tensor (an asynchronous H2D).  The
        buffer's address never changes, so a captured step graph stays valid."""
        src = target_linear.reshape(-1)
        if src.numel() != self.target.numel():
            raise ValueError(f"target has {src.numel()} voxels, the grid has {self.target.numel()}")
        if src.dtype != self.target.dtype:
            src = src.to(self.target.dtype)
        self.target.copy_(src, non_blocking=True)

    def set_target_source(self, host_target) -> None:
        """Bind a pinned host tensor (linear x-fastest, the target's dtype) as
        the per-step input: every step then copies it H2D into the target
        buffer itself -- inside the replayed graph, on a branch that overlaps
        binning and joins before the forward, or first thing in an eager
        step.  Rewrite the host tensor between steps to feed a new target; a
        step that is in flight (step_async) may still be reading it.  None
        unbinds."""
        if host_target is None:
            self._target_src = None
            return
        src = host_target.reshape(-1)
        if src.device.type != "cpu" or not src.is_pinned():
            raise ValueError("the target source must be a pinned host tensor")
        if src.numel() != self.target.numel() or src.dtype != self.target.dtype:
            raise ValueError(f"the target source must hold {self.target.numel()} values of "
                             f"{self.target.dtype}")
        self._target_src = src

    def _load_target_source(self) -> None:
        src = getattr(self, "_target_src", None)
        if src is not None:
            self.target.copy_(src, non_blocking=True)

    def _mark(self, name):
        if self.timer is not None:
            self.timer(name)

    def _reduce_buffer(self, gsum: torch.Tensor, out: "StepOutput") -> torch.Tensor:
        """The single collective's buffer: the merged per-Gaussian partials
        (f32 for the f32 engine -- they are sums of f32 pair partials -- halving
        the NVLink bytes), with this rank's loss partial in column 11."""
        gsum[0, 11] = out.loss_sum[0]
        if self.opts.precision == "f32":
            return gsum.to(torch.float32)
        return gsum

    def _unpack_reduced(self, red: torch.Tensor, gsum: torch.Tensor, out: "StepOutput") -> None:
        if red.data_ptr() != gsum.data_ptr():
            gsum.copy_(red)
        out.loss_sum.copy_(gsum[0, 11:12])
        gsum[0, 11] = 0.0
        out.reduced = True

    def forward(self, f: GaussianField) -> StepOutput:
        lib = _lib.lib()
        grid, opts = self.grid, self.opts
        self._load_target_source()
        self._mark("bin")
        idx = build_brick_index(f, grid, opts, self.brick_dims, slab=self.slab, pool=self.pool)
        aux = idx._aux
        nvox = grid.num_voxels
        dt = opts.torch_dtype
        pool = self.pool
        z = self.slab is not None          # voxels outside a slab stay zero
        S = pool.get("S", (nvox,), dt, zeroed=z)
        W = pool.get("W", (nvox,), dt, zeroed=z)
        I = pool.get("I", (nvox,), dt, zeroed=z)
        ab = pool.get("ab", (nvox, 2), dt)
        nb = max(idx.brick_count, 1)
        loss_part = pool.get("loss_part", (nb,), torch.float64)
        # live-voxel masks (f32, bricks <= 256 voxels): the backward then walks
        # exactly the forward's live voxels
        bd = self.brick_dims
        masks = None
        self._mask_vpl = _train_mask_vpl(bd, idx.pair_count, _reaching(f, idx))
        if (opts.precision == "f32" and _masks_fit(bd, self._mask_vpl)
                and not os.environ.get("GSV_NO_LIVE_MASKS")):
            masks = pool.get("live_masks", (max(idx.pair_count, 1), 4, 2), torch.int32)
        self._mark("forward")
        _forward_into(f, grid, idx, opts, aux.rec32, aux.rec64, S, W, I, target=self.target,
                      loss_kind=self.loss_kind, ab=ab, loss_part=loss_part, live_masks=masks)
        self._masks = masks
        self._mark("loss_sum")
        loss_sum = pool.get("loss_sum", (1,), torch.float64)
        loss_sum.zero_()
        if idx.brick_count > 0:
            _lib.check(lib.gsv_sum(loss_part.data_ptr(), idx.brick_count, loss_sum.data_ptr(),
                                   _lib.stream_ptr()), "sum")
        self._mark(None)
        return StepOutput(idx, RenderCache(grid, S, W, I, f.version), ab, loss_sum, nvox,
                          reduced=not self.sharded)

    def backward(self, f: GaussianField, out: StepOutput) -> GradientBuffer:
        idx = out.idx
        aux = idx._aux
        gsum = _pair_partials(f, self.grid, idx, self.opts, aux.rec32, aux.rec64, out.ab,
                              aux.gstart, aux.box, True, timer=self.timer, pool=self.pool,
                              live_masks=self._masks, mask_vpl=self._mask_vpl)
        if self.sharded:
            # One collective per step: the merged per-Gaussian partials, with
            # this rank's loss partial riding in the spare 12th column.
            import torch.distributed as dist
            self._mark("allreduce")
            red = self._reduce_buffer(gsum, out)
            dist.all_reduce(red, group=self.group)
            self._unpack_reduced(red, gsum, out)
        self._mark("chain")
        g = _chain_rule(f, gsum, pool=self.pool)
        self._mark(None)
        return g


def _adam_launch(f: GaussianField, state, lrs: dict, beta1: float, beta2: float, eps: float,
                 partials, gstart, gsum, precision_code: int, pool=None) -> None:
    """gsv_fused_update: merge (or pre-reduced sums) -> chain rule -> Adam ->
    renorm.  Bumps the field version twice, like step_optimizer +
    normalize_rotations (optimize.py:148, field.py:102)."""
    import ctypes
    lib = _lib.lib()
    state.t += 1
    hp = _lib.GsvAdamHparams()
    for k, name in enumerate(("positions", "log_scales", "rotations", "raw_amplitude",
                              "raw_relax")):
        hp.lr[k] = float(lrs[name])
    hp.b1, hp.b2, hp.eps = beta1, beta2, eps
    hp.bc1 = 1.0 - beta1 ** state.t
    hp.bc2 = 1.0 - beta2 ** state.t
    groups = ("positions", "log_scales", "rotations", "raw_amplitude", "raw_relax")
    mv = (ctypes.c_void_p * 10)(*([state.m[g].data_ptr() for g in groups] +
                                  [state.v[g].data_ptr() for g in groups]))
    scratch = None
    if precision_code != 0 or os.environ.get("GSV_TAIL_SPLIT"):
        scratch = (pool.get("grad12", (f.count, 12), torch.float64) if pool is not None
                   else torch.empty((f.count, 12), dtype=torch.float64, device=f.device))
    _lib.check(lib.gsv_fused_update(
        _lib.ptr(partials), _lib.ptr(gstart), _lib.ptr(gsum), f.count, precision_code,
        f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
        f.raw_amplitude.data_ptr(), f.raw_relax.data_ptr(), mv, int(f.amplitude_enabled),
        int(f.relax_enabled), ctypes.byref(hp), _lib.ptr(scratch), _lib.stream_ptr()),
        "fused_update")
    f.bump_version()
    f.bump_version()


def _update_method(self, f: GaussianField, out: StepOutput, state, lrs: dict,
                   beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8,
                   skip_nonfinite: bool = False) -> None:
    """Backward + fused optimizer tail of one fit() iteration: pair partials ->
    [merge -> all_reduce when sharded] -> chain rule -> Adam -> renorm, without
    materialising a GradientBuffer (the public backward/step_optimizer path
    gives identical parameters)."""
    import ctypes
    lib = _lib.lib()
    idx = out.idx
    aux = idx._aux
    opts = self.opts
    if self.sharded:
        gsum = _pair_partials(f, self.grid, idx, opts, aux.rec32, aux.rec64, out.ab, aux.gstart,
                              aux.box, True, timer=self.timer, pool=self.pool,
                              live_masks=self._masks, mask_vpl=self._mask_vpl)
        import torch.distributed as dist
        self._mark("allreduce")
        red = self._reduce_buffer(gsum, out)
        dist.all_reduce(red, group=self.group)
        self._unpack_reduced(red, gsum, out)
        if skip_nonfinite and not math.isfinite(out.loss()):
            self._mark(None)           # the global loss is known only now: no update
            return
        self._mark("update")
        _adam_launch(f, state, lrs, beta1, beta2, eps, None, None, gsum, opts.precision_code,
                     self.pool)
    else:
        pdt = opts.torch_dtype
        partials = _alloc(self.pool, "partials", (max(idx.pair_count, 1), 12), pdt, f.device)
        self._mark("backward")
        _lib.check(lib.gsv_backward(
            f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
            aux.rec32.data_ptr(), _lib.ptr(aux.rec64),
            idx.starts.data_ptr(), idx.gids.data_ptr(), aux.gstart.data_ptr(), aux.box.data_ptr(),
            _lib.make_grid(self.grid), _lib.make_bricks(self.grid, idx.brick_dims, idx.slab),
            float(opts.cutoff_sigma), opts.precision_code, out.ab.data_ptr(),
            _lib.ptr(self._masks), int(self._mask_vpl), partials.data_ptr(),
            _lib.stream_ptr()), "backward")
        self._mark("update")
        _adam_launch(f, state, lrs, beta1, beta2, eps, partials, aux.gstart, None,
                     opts.precision_code, self.pool)
    self._mark(None)


TrainStep.update = _update_method


# ------------------------------------------------------------ graph-replayed step
_GRAPH_HEADROOM = 1.15       # pair capacity over the pair count seen at capture
# Renderer graphs: less room -- the sort runs over the whole capacity, and a
# render's field moves less between calls than a fit step's (an overflow
# still re-captures with 1.5x)
_RENDER_HEADROOM = 1.05
_RESULT_SLOTS = 4            # pinned result slots (at most 2 steps are in flight)
_BC_CHUNK = 16384            # bias-correction table length per capture
_CHG_CAP = 8192              # changed Gaussians tracked per step (incremental binning)
_OPS_CAP = 16384             # list edits per step (kOpsCap of gsv_bin.cu)


def _bias_corrections(beta1: float, beta2: float, t0: int, count: int) -> torch.Tensor:
    """[1 - beta1^t, 1 - beta2^t] for t = 1 .. t0 + count, Python float pow like
    the reference's step_optimizer (optimize.py:141-142) -- bit-identical."""
    vals = []
    for t in range(1, t0 + count + 1):
        vals.append(1.0 - beta1 ** t)
        vals.append(1.0 - beta2 ** t)
    return torch.tensor(vals, dtype=torch.float64)


class _StepGraph:
    """Buffers and the captured CUDA graph(s) of one fused fit() iteration.

    The graph holds the whole iteration -- the scan of the pair counts, the
    lists (incremental binning: last step's lists edited for the Gaussians
    whose boxes changed, gsv_bin_incremental; or a capacity-mode full build),
    the pair count never read by the host, forward with the fused loss and
    live masks, loss sum, gate, masked backward, the one-pass tail with the
    step counter and bias corrections read on the device, the next step's
    preprocess (with change tracking), and the step advance, whose kernel also
    writes the 16-byte {loss sum, flags} result into a pinned host ring -- so a
    replay costs one launch and one event wait, with no per-kernel host work
    and no copy node between replays.  Incremental binning captures two graphs
    that alternate the two list buffers (``graphs``, replayed by parity).
    """

    def __init__(self, key, cap: int, t_max: int):
        self.key = key
        self.cap = cap
        self.t_max = t_max           # largest state.t the bias table covers
        self.t_synced = -1
        self.prep_version = -1
        self.graph = None
        self.bufs: dict = {}
        self.launches = 0            # replays so far (ring slot = launches % _RESULT_SLOTS)
        self.graphs: list = []       # incremental binning: [even replays, odd replays]

    def lists(self):
        """(starts, gids) of the last replay (the capture's lists before any)."""
        b = self.bufs
        if not b.get("incr") or self.launches == 0:
            return b["starts"], b["gids"]
        return _list_buffers(b, (self.launches - 1) % 2)[1]


def _graph_key(self, f: GaussianField, state, lrs: dict, beta1, beta2, eps):
    groups = ("positions", "log_scales", "rotations", "raw_amplitude", "raw_relax")
    return (f.count, f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
            f.raw_amplitude.data_ptr(), f.raw_relax.data_ptr(), int(f.amplitude_enabled),
            int(f.relax_enabled), tuple(state.m[g].data_ptr() for g in groups),
            tuple(state.v[g].data_ptr() for g in groups), self.target.data_ptr(),
            (lambda t: None if t is None else t.data_ptr())(getattr(self, "_target_src", None)),
            tuple(float(lrs[g]) for g in groups), float(beta1), float(beta2), float(eps))


def _graph_supported(self) -> bool:
    if self.sharded:
        # the all_reduce is captured too: NCCL collectives are graph-capturable
        import torch.distributed as dist
        try:
            if dist.get_backend(self.group) != "nccl":
                return False
        except (RuntimeError, ValueError):
            return False
        if os.environ.get("GSV_NO_SHARD_GRAPH"):
            return False
    bd = self.brick_dims
    return (self.opts.precision == "f32"
            and (tuple(bd) == (8, 8, 4) or _masks_fit(bd, _resolve_vpl(bd)))
            and not os.environ.get("GSV_NO_GRAPH") and not os.environ.get("GSV_NO_LIVE_MASKS")
            and not os.environ.get("GSV_TAIL_SPLIT"))


def _graph_body(self, f: GaussianField, g: _StepGraph, parity: int = 0) -> None:
    """The launch sequence captured into the graph (also run once, dry, to
    warm every kernel up before capture).  With incremental binning two
    graphs are captured that alternate the list buffers: parity 0 edits
    (starts, gids) into (starts_out, gids_out), parity 1 the other way."""
    import ctypes
    lib = _lib.lib()
    b = g.bufs
    s = _lib.stream_ptr()
    grid, opts, n = self.grid, self.opts, f.count
    gr, br = _lib.make_grid(grid), b["bricks"]
    cap = g.cap
    # the bound host target (set_target_source): its H2D copy runs on a
    # branch of the graph that overlaps binning and joins before the forward
    src = getattr(self, "_target_src", None)
    join = None
    if src is not None:
        cur = torch.cuda.current_stream()
        side = b.setdefault("h2d_stream", torch.cuda.Stream(device=self.target.device))
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            self.target.copy_(src, non_blocking=True)
        join = side
    # rec32 / counts / box for this step were written by the previous replay's
    # tail (or by _graph_preprocess): binning starts at the scan
    ws = b["ws"]
    _lib.check(lib.gsv_bin_scan(b["counts"].data_ptr(), n, b["gstart"].data_ptr(),
                                ws.data_ptr(), ws.numel(), s), "bin_scan")
    if b["incr"]:
        # last step's lists edited for the Gaussians whose boxes changed
        # (recorded by the previous step's preprocess pass)
        src, dst = _list_buffers(b, parity)
        _lib.check(lib.gsv_bin_incremental(
            b["counts"].data_ptr(), b["box"].data_ptr(), b["gstart"].data_ptr(), n, cap, br,
            b["chg_count"].data_ptr(),
            b["chg_gid"].data_ptr(), b["chg_old"].data_ptr(), b["chg_oldcnt"].data_ptr(),
            _CHG_CAP, src[0].data_ptr(), src[1].data_ptr(), dst[0].data_ptr(),
            dst[1].data_ptr(), b["ops"].data_ptr(), b["nops"].data_ptr(),
            b["lens"].data_ptr(), b["dry"].data_ptr(), b["overflow"].data_ptr(), 0,
            ws.data_ptr(), ws.numel(), s), "bin_incremental")
        # the kernels read the edited lists (starts zeroed on overflow)
        lst, lgids = dst
    else:
        k = b["keys"]
        _lib.check(lib.gsv_bin_fill_capacity(
            b["counts"].data_ptr(), b["box"].data_ptr(), b["gstart"].data_ptr(), n, cap, br,
            k[0].data_ptr(), k[1].data_ptr(), k[2].data_ptr(), b["gids"].data_ptr(),
            b["starts"].data_ptr(), b["dry"].data_ptr(), b["overflow"].data_ptr(),
            ws.data_ptr(), ws.numel(), s), "bin_fill_capacity")
        lst, lgids = b["starts"], b["gids"]
    nvox = grid.num_voxels
    # a target arriving over PCIe: the forward runs without the fused loss and
    # the copy joins before the loss pass (bit-identical partials), so the
    # H2D overlaps binning and the whole forward
    split = join is not None and b["fwd_vpl"] in (16, 8) and tuple(self.brick_dims) == (8, 8, 4)
    if join is not None and not split:
        torch.cuda.current_stream().wait_stream(join)
    tdt = int(self.target.dtype == torch.float64)
    _lib.check(lib.gsv_forward(
        f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
        b["rec32"].data_ptr(), None, lst.data_ptr(), lgids.data_ptr(), gr, br,
        float(opts.cutoff_sigma), float(opts.epsilon_w), 0, b["S"].data_ptr(),
        b["W"].data_ptr(), b["I"].data_ptr(), None if split else self.target.data_ptr(),
        tdt, self.loss_kind, float(nvox), b["ab"].data_ptr(), b["loss_part"].data_ptr(),
        b["masks"].data_ptr(), b["fwd_vpl"], s), "forward")
    if split:
        torch.cuda.current_stream().wait_stream(join)
        _lib.check(lib.gsv_loss_bricks(
            gr, br, float(opts.epsilon_w), b["W"].data_ptr(), b["I"].data_ptr(),
            self.target.data_ptr(), tdt, self.loss_kind, float(nvox), b["fwd_vpl"],
            b["ab"].data_ptr(), b["loss_part"].data_ptr(), s), "loss_bricks")
    _lib.check(lib.gsv_sum(b["loss_part"].data_ptr(), b["nb"], b["loss_sum"].data_ptr(), s),
               "sum")
    if not self.sharded:
        _lib.check(lib.gsv_step_gate(b["loss_sum"].data_ptr(), b["overflow"].data_ptr(),
                                     b["gate"].data_ptr(), b["result"].data_ptr(), s),
                   "step_gate")
    _lib.check(lib.gsv_backward(
        f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
        b["rec32"].data_ptr(), None, lst.data_ptr(), lgids.data_ptr(),
        b["gstart"].data_ptr(), b["box"].data_ptr(), gr, br, float(opts.cutoff_sigma), 0,
        b["ab"].data_ptr(), b["masks"].data_ptr(), b["vpl"], b["partials"].data_ptr(), s),
        "backward")
    gsum = None
    hooks = getattr(self, "halo_hooks", None)
    if hooks is not None:
        # owner-computes + halo exchange (halo.py): merge, the halo rows'
        # partials to their owners, a 2-value all_reduce of {loss, overflow}
        # for the gate; the parameter exchange and the reach check follow the
        # update below
        _lib.check(lib.gsv_merge(b["partials"].data_ptr(), b["gstart"].data_ptr(), n, 0,
                                 b["gsum"].data_ptr(), s), "merge")
        hooks.exchange_partials(b["gsum"])
        hooks.reduce_loss(b["loss_sum"], b["overflow"], b["gloss"], b["govf"])
        _lib.check(lib.gsv_step_gate(b["gloss"].data_ptr(), b["govf"].data_ptr(),
                                     b["gate"].data_ptr(), b["result"].data_ptr(), s),
                   "step_gate")
        gsum = b["gsum"]
    elif self.sharded:
        # merge this slab's pair partials per Gaussian, then the step's one
        # collective: partials + loss + overflow flag in a single all_reduce;
        # the gate then sees the global loss and any rank's overflow
        import torch.distributed as dist
        _lib.check(lib.gsv_merge(b["partials"].data_ptr(), b["gstart"].data_ptr(), n, 0,
                                 b["gsum"].data_ptr(), s), "merge")
        _lib.check(lib.gsv_shard_pack(b["gsum"].data_ptr(), n, b["loss_sum"].data_ptr(),
                                      b["overflow"].data_ptr(), b["red"].data_ptr(), s),
                   "shard_pack")
        dist.all_reduce(b["red"], group=self.group)
        _lib.check(lib.gsv_shard_unpack(b["red"].data_ptr(), n, b["gsum"].data_ptr(),
                                        b["gloss"].data_ptr(), b["govf"].data_ptr(), s),
                   "shard_unpack")
        _lib.check(lib.gsv_step_gate(b["gloss"].data_ptr(), b["govf"].data_ptr(),
                                     b["gate"].data_ptr(), b["result"].data_ptr(), s),
                   "step_gate")
        gsum = b["gsum"]
    # next-step records: the TMA tail + a separate preprocess pass (measured
    # 17 us/step faster at config 3 than the tail with records fused in,
    # which GSV_GRAPH_FUSED_PREP=1 selects)
    split_prep = os.environ.get("GSV_GRAPH_FUSED_PREP") != "1"
    _lib.check(lib.gsv_fused_update_device(
        None if gsum is not None else b["partials"].data_ptr(),
        None if gsum is not None else b["gstart"].data_ptr(), _lib.ptr(gsum), n,
        f.positions.data_ptr(),
        f.log_scales.data_ptr(), f.rotations.data_ptr(), f.raw_amplitude.data_ptr(),
        f.raw_relax.data_ptr(), b["mv"], int(f.amplitude_enabled), int(f.relax_enabled),
        ctypes.byref(b["hp"]), b["bc"].data_ptr(), b["t"].data_ptr(), b["gate"].data_ptr(), gr,
        br, float(opts.cutoff_sigma), None if split_prep else b["rec32"].data_ptr(),
        b["counts"].data_ptr(), b["box"].data_ptr(), s), "fused_update_device")
    if hooks is not None:
        # owners' updated rows to the ranks holding them as halo (a gated step
        # sends unchanged rows), then the reach check into the result flags
        hooks.exchange_params(f)
        hooks.reach_check(f, b["result"])
    if split_prep:
        # the next step's records from a separate pass over the updated field
        # (a gated step leaves the field, and so its records, unchanged)
        _graph_preprocess(self, f, b)
    # the step's result goes straight into the pinned ring (no D2H copy node
    # between consecutive replays)
    _lib.check(lib.gsv_step_advance_publish(
        b["t"].data_ptr(), b["gate"].data_ptr(), b["result"].data_ptr(),
        b["result_host"].data_ptr(), b["rcount"].data_ptr(), _RESULT_SLOTS, s),
        "step_advance_publish")


def _list_buffers(b: dict, parity: int):
    """((starts, gids) read, (starts, gids) written) of an incremental replay."""
    a, o = (b["starts"], b["gids"]), (b["starts_out"], b["gids_out"])
    return (a, o) if parity == 0 else (o, a)


def _graph_preprocess(self, f: GaussianField, b: dict) -> None:
    """gsv_preprocess into the graph's buffers: before the first replay, and
    whenever the field was changed outside the graph (version mismatch)."""
    lib = _lib.lib()
    if b.get("track"):
        # incremental binning: also record the Gaussians whose boxes change
        _lib.check(lib.gsv_preprocess_track(
            f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
            f.raw_amplitude.data_ptr(), f.raw_relax.data_ptr(), f.count, int(f.relax_enabled),
            float(self.opts.cutoff_sigma), _lib.make_grid(self.grid), b["bricks"],
            b["rec32"].data_ptr(), b["counts"].data_ptr(), b["box"].data_ptr(),
            b["chg_count"].data_ptr(), b["chg_gid"].data_ptr(), b["chg_old"].data_ptr(),
            b["chg_oldcnt"].data_ptr(), _CHG_CAP, _lib.stream_ptr()), "preprocess_track")
        return
    _lib.check(lib.gsv_preprocess(
        f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
        f.raw_amplitude.data_ptr(), f.raw_relax.data_ptr(), f.count, int(f.relax_enabled),
        float(self.opts.cutoff_sigma), _lib.make_grid(self.grid), b["bricks"],
        b["rec32"].data_ptr(), None, b["counts"].data_ptr(), b["box"].data_ptr(),
        _lib.stream_ptr()), "preprocess")


def _graph_capture(self, f: GaussianField, state, lrs: dict, beta1, beta2, eps, key,
                   min_cap: int = 0) -> _StepGraph:
    import ctypes
    lib = _lib.lib()
    self.graph_captures = getattr(self, "graph_captures", 0) + 1     # diagnostics
    dev = f.device
    grid, opts, n = self.grid, self.opts, f.count
    bricks = _lib.make_bricks(grid, self.brick_dims, self.slab)
    nb = bricks.b1 - bricks.b0
    gp = _lib.BufferPool(dev)        # private: replays need fixed addresses
    b = {"bricks": bricks, "nb": max(nb, 1),
         "rec32": gp.get("rec32", (n, 16), torch.float32),
         "counts": gp.get("counts", (n,), torch.int32),
         "box": gp.get("box", (n, 4), torch.int32),
         "gstart": gp.get("gstart", (n + 1,), torch.int64)}
    # records for the first replay, and the exact pair count -- read once per
    # capture, never per step
    _graph_preprocess(self, f, b)
    nbytes = ctypes.c_size_t(0)
    _lib.check(lib.gsv_bin_workspace(n, 1, nb, ctypes.byref(nbytes)), "bin_workspace")
    ws0 = _lib.workspace(nbytes.value, dev, "bin")
    _lib.check(lib.gsv_bin_scan(b["counts"].data_ptr(), n, b["gstart"].data_ptr(),
                                ws0.data_ptr(), ws0.numel(), _lib.stream_ptr()), "bin_scan")
    pairs = int(b["gstart"][-1].item())
    cap = max(int(pairs * _GRAPH_HEADROOM) + 4096, min_cap, 1)
    g = _StepGraph(key, cap, state.t + _BC_CHUNK - 1)
    g.bufs = b
    nbytes = ctypes.c_size_t(0)
    _lib.check(lib.gsv_bin_workspace(n, cap, nb, ctypes.byref(nbytes)), "bin_workspace")
    wsb = nbytes.value
    # incremental binning (any slab; sharded and halo steps too), with the
    # next-step records from the separate preprocess pass
    # (GSV_BIN_INCREMENTAL=0 rebuilds the lists every step)
    b["incr"] = (os.environ.get("GSV_BIN_INCREMENTAL", "1") == "1"
                 and os.environ.get("GSV_GRAPH_FUSED_PREP") != "1")
    if b["incr"]:
        _lib.check(lib.gsv_bin_incremental_workspace(nb, ctypes.byref(nbytes)),
                   "bin_incremental_workspace")
        wsb = max(wsb, nbytes.value)
        b["chg_count"] = gp.get("chg_count", (1,), torch.int32)
        b["chg_gid"] = gp.get("chg_gid", (_CHG_CAP,), torch.int32)
        b["chg_old"] = gp.get("chg_old", (_CHG_CAP, 4), torch.int32)
        b["chg_oldcnt"] = gp.get("chg_oldcnt", (_CHG_CAP,), torch.int32)
        b["starts_out"] = gp.get("starts_out", (nb + 1,), torch.int64)
        b["gids_out"] = gp.get("gids_out", (cap,), torch.int32)
        b["ops"] = gp.get("ops", (2 * _OPS_CAP,), torch.int64)
        b["nops"] = gp.get("nops", (1,), torch.int32, zeroed=True)
        b["lens"] = gp.get("lens", (8 * (nb + 1),), torch.int32, zeroed=True)
        b["nops"].zero_()
        b["lens"].zero_()
    b["ws"] = gp.get("ws", (wsb,), torch.uint8)
    b["keys"] = gp.get("keys", (3, cap), torch.int32)
    b["gids"] = gp.get("gids", (cap,), torch.int32)
    b["starts"] = gp.get("starts", (nb + 1,), torch.int64)
    nvox = grid.num_voxels
    for name in ("S", "W", "I"):               # voxels outside a slab stay zero
        b[name] = gp.get(name, (nvox,), torch.float32, zeroed=self.slab is not None)
    b["ab"] = gp.get("ab", (nvox, 2), torch.float32)
    # zeroed: an empty slab (b0 == b1) never writes its loss partial, and the
    # loss sum still reads entry 0
    b["loss_part"] = gp.get("loss_part", (max(nb, 1),), torch.float64, zeroed=True)
    b["loss_sum"] = gp.get("loss_sum", (1,), torch.float64)
    b["masks"] = gp.get("masks", (cap, 4, 2), torch.int32)
    b["partials"] = gp.get("partials", (cap, 12), torch.float32)
    b["dry"] = gp.get("dry", (1,), torch.int32)
    b["overflow"] = gp.get("overflow", (1,), torch.int32)
    b["gate"] = gp.get("gate", (1,), torch.int32)
    b["result"] = gp.get("result", (2,), torch.float64)
    # results go into a ring of pinned slots (written by the graph's last
    # kernel), so a step in flight never overwrites the one being read
    b["result_host"] = torch.zeros((_RESULT_SLOTS, 2), dtype=torch.float64).pin_memory()
    b["rcount"] = gp.get("rcount", (1,), torch.int64)
    if self.sharded:
        b["gsum"] = gp.get("gsum", (n, 12), torch.float64)
        b["red"] = gp.get("red", (n, 12), torch.float32)
        b["gloss"] = gp.get("gloss", (1,), torch.float64)
        b["govf"] = gp.get("govf", (1,), torch.int32)
    b["t"] = gp.get("t", (1,), torch.int64)
    b["bc"] = _bias_corrections(beta1, beta2, state.t, _BC_CHUNK).to(dev)
    # the forward kernel (and so the mask layout) for this capture, from the
    # pair density seen at capture (raster._use_grouped)
    reach = n if self.slab is None else int(torch.count_nonzero(b["counts"]).item())
    b["vpl"] = _train_mask_vpl(self.brick_dims, pairs, reach)
    b["fwd_vpl"] = _forward_vpl_arg(self.brick_dims, pairs, reach)
    hp = _lib.GsvAdamHparams()
    for i, name in enumerate(("positions", "log_scales", "rotations", "raw_amplitude",
                              "raw_relax")):
        hp.lr[i] = float(lrs[name])
    hp.b1, hp.b2, hp.eps, hp.bc1, hp.bc2 = beta1, beta2, eps, 0.0, 0.0
    b["hp"] = hp
    groups = ("positions", "log_scales", "rotations", "raw_amplitude", "raw_relax")
    b["mv"] = (ctypes.c_void_p * 10)(*([state.m[x].data_ptr() for x in groups] +
                                       [state.v[x].data_ptr() for x in groups]))
    if b["incr"]:
        # the first lists in full (from the records of _graph_preprocess above);
        # from here on the preprocess pass tracks box changes
        k = b["keys"]
        b["dry"].zero_()
        _lib.check(lib.gsv_bin_fill_capacity(
            b["counts"].data_ptr(), b["box"].data_ptr(), b["gstart"].data_ptr(), n, cap,
            bricks, k[0].data_ptr(), k[1].data_ptr(), k[2].data_ptr(), b["gids"].data_ptr(),
            b["starts"].data_ptr(), b["dry"].data_ptr(), b["overflow"].data_ptr(),
            b["ws"].data_ptr(), b["ws"].numel(), _lib.stream_ptr()), "bin_fill_capacity")
        # lists that did not fit make the first replay report an overflow
        # (more changes than tracked), which re-captures with more room
        b["chg_count"].fill_(0 if pairs <= cap else _CHG_CAP + 1)
        b["track"] = True
    # dry run (every kernel once, empty lists, no update), then capture
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(side):
        b["dry"].fill_(1)
        _graph_body(self, f, g)
        b["dry"].zero_()
    torch.cuda.current_stream(dev).wait_stream(side)
    torch.cuda.synchronize(dev)
    g.graphs = []
    for parity in range(2 if b["incr"] else 1):
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side, capture_error_mode="thread_local"):
            _graph_body(self, f, g, parity)
        g.graphs.append(graph)
    g.graph = g.graphs[0]
    g.prep_version = f.version
    b["t"].fill_(int(state.t))
    g.t_synced = state.t
    b["rcount"].zero_()            # ring slot of replay k = k % _RESULT_SLOTS
    g.launches = 0
    return g


class StepHandle:
    """One launched fit() iteration.  ``loss()`` waits for it, commits its
    bookkeeping (step count, field version) and returns the mean loss; a step
    that hit the pair capacity is re-run there.  Steps are committed in launch
    order: a step whose loss is non-finite or that overflowed applied nothing,
    so the step queued behind it sees the same field and is gated the same
    way (the device gate makes the one-step-ahead pipeline safe)."""

    def __init__(self, step, f, state, lrs, hyper, g=None, slot=None, event=None,
                 value=None):
        self._step, self._f, self._state, self._lrs, self._hyper = step, f, state, lrs, hyper
        self._g, self._slot, self._event = g, slot, event
        self._value = value

    def loss(self) -> float:
        if self._value is not None:
            return self._value
        step, f, state, g = self._step, self._f, self._state, self._g
        if step._pending and step._pending[0] is not self:
            step._pending[0].loss()              # commit in launch order
        self._event.synchronize()
        step._pending.remove(self)
        row = g.bufs["result_host"][self._slot]
        loss_sum, flags = float(row[0]), int(row[1])
        if flags & 1:
            # pair capacity overflow (on any rank, when sharded): nothing was
            # applied, by this step or by those queued behind it.  Drain them,
            # re-capture with more room (every rank: the capture's collectives
            # must match across ranks; more room where this rank overflowed),
            # then run this step and the drained ones again, in launch order.
            drained = []
            while step._pending:
                p = step._pending.pop(0)
                p._event.synchronize()
                drained.append(p)
            if step._graph is g:
                b = g.bufs
                if step.sharded:
                    local = bool(int(b["overflow"].item()))
                elif b.get("incr"):
                    # incremental binning also overflows on too many edits:
                    # more room only if the pairs did not fit
                    local = int(b["gstart"][-1].item()) > g.cap
                else:
                    local = True
                step._graph = None
                step._graph = _graph_capture(step, f, state, self._lrs, *self._hyper, g.key,
                                             min_cap=int(g.cap * 1.5) if local else g.cap)
            self._value = _step_launch(step, f, state, self._lrs, *self._hyper).loss()
            for p in drained:
                p._value = _step_launch(step, p._f, p._state, p._lrs, *p._hyper).loss()
            return self._value
        loss = loss_sum / step.grid.num_voxels
        if flags & 4:                            # a Gaussian left its planned reach
            step._replan_needed = True           # (halo.py re-plans before the next step)
        if not flags & 2:                        # applied (finite loss)
            state.t += 1
            g.t_synced = state.t
            f.bump_version()
            f.bump_version()
            g.prep_version = f.version           # the replay's tail wrote the new records
        self._value = loss
        return loss


def _step_launch(self, f: GaussianField, state, lrs: dict, beta1: float = 0.9,
                 beta2: float = 0.999, eps: float = 1e-8) -> StepHandle:
    """Enqueue one whole fit() iteration (see _step_method) and return its
    handle without waiting.  Graph path only asynchronous; elsewhere the step
    runs to completion and the handle is already resolved."""
    hyper = (beta1, beta2, eps)
    if not _graph_supported(self) or (self.sharded and f.count < 2):
        out = self.forward(f)
        if self.sharded:
            # the global loss rides the step's one all_reduce, inside update():
            # it is checked there, before Adam
            self.update(f, out, state, lrs, beta1, beta2, eps, skip_nonfinite=True)
            return StepHandle(self, f, state, lrs, hyper, value=out.loss())
        loss = out.loss()
        if math.isfinite(loss):
            self.update(f, out, state, lrs, beta1, beta2, eps)
        return StepHandle(self, f, state, lrs, hyper, value=loss)
    pending = self.__dict__.setdefault("_pending", [])
    # the result ring has _RESULT_SLOTS pinned slots: commit the oldest step
    # before a new replay could overwrite a slot whose result is unread
    while len(pending) >= _RESULT_SLOTS - 1:
        pending[0].loss()
    key = _graph_key(self, f, state, lrs, beta1, beta2, eps)
    g = getattr(self, "_graph", None)
    # every queued step may still advance t on the device: the replay being
    # launched runs at t <= state.t + len(pending) + 1, which the bias table
    # must cover (t_max is the largest pre-step t it covers)
    if g is None or g.key != key or state.t + len(pending) > g.t_max:
        while pending:                           # captures start from committed state
            pending[0].loss()
        self._graph = None
        _nvtx_push("gsv.step.capture")
        g = self._graph = _graph_capture(self, f, state, lrs, beta1, beta2, eps, key)
        _nvtx_pop()
    b = g.bufs
    if not pending:
        # the field / step count were changed outside the graph
        if g.t_synced != state.t:
            b["t"].fill_(int(state.t))
            g.t_synced = state.t
        if g.prep_version != f.version:
            _graph_preprocess(self, f, b)
            g.prep_version = f.version
    _nvtx_push("gsv.step.replay")
    g.graphs[g.launches % len(g.graphs)].replay()   # incremental: alternate list buffers
    _nvtx_pop()
    slot = g.launches % _RESULT_SLOTS
    g.launches += 1
    ev = torch.cuda.Event()
    ev.record(torch.cuda.current_stream(f.device))
    h = StepHandle(self, f, state, lrs, hyper, g=g, slot=slot, event=ev)
    pending.append(h)
    return h


def _step_method(self, f: GaussianField, state, lrs: dict, beta1: float = 0.9,
                 beta2: float = 0.999, eps: float = 1e-8) -> float:
    """One whole fit() iteration (optimize.py:177-197): render + loss, then --
    only if the loss is finite, as the reference raises before updating --
    backward, chain rule, Adam and renormalisation.  Returns the mean loss
    (a Python float: the iteration's one device->host read).

    Replays a captured CUDA graph (f32; single GPU, or sharded over an NCCL
    group with the step's one all_reduce captured too): no host work per
    kernel, no pair-count read.  The graph is (re)captured when the field /
    optimizer buffers, target, hyper-parameters or pair capacity change.
    Elsewhere (gloo groups, f64) it runs forward() + update() eagerly.
    ``step_async`` is the same iteration without the wait (one step can be
    queued behind another; see StepHandle).
    """
    return _step_launch(self, f, state, lrs, beta1, beta2, eps).loss()


TrainStep.step = _step_method
TrainStep.step_async = _step_launch


class Renderer:
    """Repeated renders of fields at one grid with reusable buffers: the
    render path of the reference (build_brick_index + forward, cli.py:231-233)
    without per-call allocations.  Returned tensors are views valid until the
    next call.

    f32 renders replay a captured CUDA graph (preprocess -> scan -> capacity
    binning -> forward): no pair-count read and no per-kernel host work; the
    only host read is the overflow flag, and an overflow re-captures with more
    room.  The graph is re-captured when the field's buffers change."""

    def __init__(self, grid, opts: RenderOptions = RenderOptions(), brick_dims=(8, 8, 4),
                 slab=None, device=None):
        self.grid = grid
        self.opts = opts
        self.brick_dims = tuple(brick_dims)
        self.slab = slab
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self.pool = _lib.BufferPool(dev)
        self.last_index = None
        self._graph = None

    def pair_count(self) -> int:
        """Pairs of the last render (one device read)."""
        if self.last_index is not None:
            return self.last_index.pair_count
        return int(self._graph.bufs["gstart"][-1].item())

    def __call__(self, f: GaussianField) -> RenderCache:
        if self.opts.precision != "f32" or os.environ.get("GSV_NO_GRAPH"):
            return self._eager(f)
        key = (f.count, f.positions.data_ptr(), f.log_scales.data_ptr(),
               f.rotations.data_ptr(), f.raw_amplitude.data_ptr(), f.raw_relax.data_ptr(),
               int(f.relax_enabled))
        g = self._graph
        if g is None or g.key != key:
            self._graph = None
            g = self._graph = self._capture(f, key)
        b = g.bufs
        _nvtx_push("gsv.render.replay")
        g.graph.replay()
        _nvtx_pop()
        b["ovf_host"].copy_(b["overflow"], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        ev.synchronize()
        if int(b["ovf_host"][0]):
            self._graph = None
            self._graph = self._capture(f, key, min_cap=int(g.cap * 1.5))
            return self(f)
        self.last_index = None
        return RenderCache(self.grid, b["S"], b["W"], b["I"], f.version)

    def _eager(self, f: GaussianField) -> RenderCache:
        idx = build_brick_index(f, self.grid, self.opts, self.brick_dims, slab=self.slab,
                                pool=self.pool)
        n = self.grid.num_voxels
        dt = self.opts.torch_dtype
        z = self.slab is not None          # voxels outside a slab stay zero
        S = self.pool.get("S", (n,), dt, zeroed=z)
        W = self.pool.get("W", (n,), dt, zeroed=z)
        I = self.pool.get("I", (n,), dt, zeroed=z)
        _forward_into(f, self.grid, idx, self.opts, idx._aux.rec32, idx._aux.rec64, S, W, I)
        self.last_index = idx
        return RenderCache(self.grid, S, W, I, f.version)

    def _body(self, f: GaussianField, g) -> None:
        lib = _lib.lib()
        b, s, n = g.bufs, _lib.stream_ptr(), f.count
        gr, br, opts = _lib.make_grid(self.grid), b["bricks"], self.opts
        _lib.check(lib.gsv_preprocess(
            f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
            f.raw_amplitude.data_ptr(), f.raw_relax.data_ptr(), n, int(f.relax_enabled),
            float(opts.cutoff_sigma), gr, br, b["rec32"].data_ptr(), None,
            b["counts"].data_ptr(), b["box"].data_ptr(), s), "preprocess")
        ws, k = b["ws"], b["keys"]
        _lib.check(lib.gsv_bin_scan(b["counts"].data_ptr(), n, b["gstart"].data_ptr(),
                                    ws.data_ptr(), ws.numel(), s), "bin_scan")
        _lib.check(lib.gsv_bin_fill_capacity(
            b["counts"].data_ptr(), b["box"].data_ptr(), b["gstart"].data_ptr(), n, g.cap, br,
            k[0].data_ptr(), k[1].data_ptr(), k[2].data_ptr(), b["gids"].data_ptr(),
            b["starts"].data_ptr(), b["dry"].data_ptr(), b["overflow"].data_ptr(),
            ws.data_ptr(), ws.numel(), s), "bin_fill_capacity")
        _lib.check(lib.gsv_forward(
            f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
            b["rec32"].data_ptr(), None, b["starts"].data_ptr(), b["gids"].data_ptr(), gr, br,
            float(opts.cutoff_sigma), float(opts.epsilon_w), 0, b["S"].data_ptr(),
            b["W"].data_ptr(), b["I"].data_ptr(), None, 0, 0, float(self.grid.num_voxels), None,
            None, None, _forward_vpl_arg(self.brick_dims, b["pairs"], b["active"], masks=False), s),
            "forward")

    def _capture(self, f: GaussianField, key, min_cap: int = 0):
        import ctypes
        lib = _lib.lib()
        dev, n = self.device, f.count
        bricks = _lib.make_bricks(self.grid, self.brick_dims, self.slab)
        nb = bricks.b1 - bricks.b0
        gp = _lib.BufferPool(dev)
        b = {"bricks": bricks,
             "rec32": gp.get("rec32", (n, 16), torch.float32),
             "counts": gp.get("counts", (n,), torch.int32),
             "box": gp.get("box", (n, 4), torch.int32),
             "gstart": gp.get("gstart", (n + 1,), torch.int64)}
        _lib.check(lib.gsv_preprocess(
            f.positions.data_ptr(), f.log_scales.data_ptr(), f.rotations.data_ptr(),
            f.raw_amplitude.data_ptr(), f.raw_relax.data_ptr(), n, int(f.relax_enabled),
            float(self.opts.cutoff_sigma), _lib.make_grid(self.grid), bricks,
            b["rec32"].data_ptr(), None, b["counts"].data_ptr(), b["box"].data_ptr(),
            _lib.stream_ptr()), "preprocess")
        gst = _scan(b["counts"], nb, self.pool)
        pairs = int(gst[-1].item())
        # Gaussians that reach the bricks (as raster._reaching): N for the
        # whole grid, counted for a slab
        active = n if self.slab is None else int(torch.count_nonzero(b["counts"]).item())
        cap = max(int(pairs * _RENDER_HEADROOM) + 4096, min_cap, 1)
        nbytes = ctypes.c_size_t(0)
        _lib.check(lib.gsv_bin_workspace(n, cap, nb, ctypes.byref(nbytes)), "bin_workspace")
        nv = self.grid.num_voxels
        b["pairs"] = pairs                   # with b["active"], picks the forward's tiling
        b["active"] = active
        b.update({"ws": gp.get("ws", (nbytes.value,), torch.uint8),
                  "keys": gp.get("keys", (3, cap), torch.int32),
                  "gids": gp.get("gids", (cap,), torch.int32),
                  "starts": gp.get("starts", (nb + 1,), torch.int64),
                  "S": gp.get("S", (nv,), torch.float32, zeroed=self.slab is not None),
                  "W": gp.get("W", (nv,), torch.float32, zeroed=self.slab is not None),
                  "I": gp.get("I", (nv,), torch.float32, zeroed=self.slab is not None),
                  "dry": gp.get("dry", (1,), torch.int32),
                  "overflow": gp.get("overflow", (1,), torch.int32),
                  "ovf_host": torch.zeros(1, dtype=torch.int32).pin_memory()})
        g = _StepGraph(key, cap, 0)
        g.bufs = b
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            b["dry"].fill_(1)
            self._body(f, g)
            b["dry"].zero_()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side, capture_error_mode="thread_local"):
            self._body(f, g)
        g.graph = graph
        return g
