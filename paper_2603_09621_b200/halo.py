"""Multi-GPU train step with owner-computes and halo exchange.

The all_reduce design (TrainStep with a process group) keeps every parameter
replicated: each rank preprocesses all N Gaussians, all_reduces an (N, 12)
buffer and runs Adam on all N -- an O(N) floor per rank that caps strong
scaling.  Here each rank holds only the Gaussians its slab
needs, and the only O(N) work left is the occasional re-plan:

  plan (at attach, and whenever a Gaussian may leave its planned reach):
    owner(g)      the rank whose slab holds the brick of g's centre voxel;
    reach(g)      the ranks whose brick-id ranges meet the brick-id interval
                  of g's 3-sigma box widened by `margin` voxels -- a
                  contiguous rank interval [r_lo, r_hi];
    local(r)      {g : r in reach(g)} u owned(r), ascending gid.  The rank
                  runs the ordinary slab step on this compact field: ascending
                  local ids are ascending gids, so its brick lists are the
                  global slab lists renamed, and its slab render is
                  bit-identical to the single-GPU render.
  step on rank r:
    1. bin / forward (+ fused loss) / masked backward on the slab, per-
       Gaussian merge of the pair partials (f64);
    2. partial exchange: the merged rows of the halo Gaussians (owned by p)
       go to p, which adds the rows it receives, peer by peer in rank order
       (a fixed association: deterministic for a given rank count);
    3. one small all_reduce: the global loss and the gate flags;
    4. chain rule + Adam + renormalisation on the local field (rows of halo
       Gaussians are overwritten next);
    5. parameter exchange: owners send the updated rows of their Gaussians
       that lie in other ranks' local sets;
    6. reach check: every owned Gaussian's new box must stay inside its
       planned reach; if any does not, every rank re-plans before the next
       step (the margin makes that rare: Adam moves a Gaussian by about its
       learning rate per step, ~1e-3 voxel for positions).
  Communication per step is O(halo) both ways (all_to_all_single with
  fixed splits), compute O(N/k + halo).  Adam moments live only with the
  owner; `gather()` assembles the full field and moments on every rank.

Correctness does not depend on the margin: the reach check guarantees that
every Gaussian reaching a slab is in that rank's local set at every step.
"""

from __future__ import annotations

import math
import os

import torch

from .field import PARAM_NAMES, GaussianField
from .optimize import AdamState
from .render import RenderOptions
from .volume import Volume

_ROWW = 12            # f64 words per exchanged row: 11 partials (+1 free) or 12 parameters


# ----------------------------------------------------------------- plan
def _rotation(q: torch.Tensor) -> torch.Tensor:
    """R of the stored quaternion, verbatim (field.py:141-154)."""
    w, x, y, z = q.unbind(1)
    return torch.stack([
        1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
        2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
        2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1).view(-1, 3, 3)


def _slab_of(ids: torch.Tensor, b0s: torch.Tensor) -> torch.Tensor:
    """Rank whose brick-id range [b0, b1) holds each id (slabs contiguous, in
    rank order; an empty slab shares its b0 with the next one)."""
    return torch.searchsorted(b0s, ids, right=True) - 1


def reach_consts(grid, brick_dims, slabs, device):
    """The device constants reach_and_owner needs (built once: a CUDA-graph
    capture may not create tensors from host data)."""
    return {"dims": torch.tensor(grid.dims, dtype=torch.float64, device=device),
            "org": torch.tensor(grid.origin, dtype=torch.float64, device=device),
            "sp": torch.tensor(grid.spacing, dtype=torch.float64, device=device),
            "bd": torch.tensor(brick_dims, dtype=torch.int64, device=device),
            "bg": [-(-d // b) for d, b in zip(grid.dims, brick_dims)],
            "b0s": torch.tensor([s[0] for s in slabs], dtype=torch.int64, device=device)}


def reach_and_owner(positions, log_scales, rotations, grid, brick_dims, slabs,
                    cutoff_sigma: float = 3.0, margin: float = 0.0, consts=None):
    """(owner, r_lo, r_hi) per Gaussian, int64 tensors on the inputs' device.

    The box is binning's conservative 3-sigma box (raster.py:173-198) widened
    by `margin` voxels; r_lo > r_hi when it misses the grid.  The owner's
    slab holds the brick of the centre voxel (clamped into the grid), so a
    Gaussian inside the grid is always in its owner's reach."""
    c = consts if consts is not None else reach_consts(grid, brick_dims, slabs,
                                                       positions.device)
    dims, org, sp, bd, bg, b0s = c["dims"], c["org"], c["sp"], c["bd"], c["bg"], c["b0s"]
    R = _rotation(rotations)
    var = torch.exp(2.0 * log_scales)
    sig = torch.einsum("nkm,nm->nk", R * R, var)
    half = cutoff_sigma * torch.sqrt(sig)
    glo = (positions - half - org) / sp - margin
    ghi = (positions + half - org) / sp + margin
    inside = ((ghi >= -0.5) & (glo <= dims - 0.5)).all(dim=1)
    hi_lim = (dims - 1).to(torch.int64)
    vlo = torch.minimum(torch.clamp(torch.ceil(glo - 0.5), min=0).to(torch.int64), hi_lim)
    vhi = torch.minimum(torch.clamp(torch.floor(ghi + 0.5), min=0).to(torch.int64), hi_lim)
    blo, bhi = vlo // bd, vhi // bd
    idmin = blo[:, 0] + bg[0] * (blo[:, 1] + bg[1] * blo[:, 2])
    idmax = bhi[:, 0] + bg[0] * (bhi[:, 1] + bg[1] * bhi[:, 2])
    r_lo = _slab_of(idmin, b0s)
    r_hi = _slab_of(idmax, b0s)
    r_lo = torch.where(inside, r_lo, torch.ones_like(r_lo))
    r_hi = torch.where(inside, r_hi, torch.zeros_like(r_hi))
    cv = torch.minimum(torch.clamp(torch.round((positions - org) / sp), min=0).to(torch.int64),
                       hi_lim) // bd
    owner = _slab_of(cv[:, 0] + bg[0] * (cv[:, 1] + bg[1] * cv[:, 2]), b0s)
    return owner, r_lo, r_hi


class HaloPlan:
    """One rank's view of a plan: its local gids and the exchange lists.

    local_gids   ascending gids of local(r)
    owned        bool over local ids: owner == rank
    to_owner[p]  local ids of Gaussians owned by p (p != rank), ascending:
                 their partial rows go to p; their parameters come from p
    from_peer[p] local ids of owned Gaussians in p's local set, ascending:
                 p's partial rows for them are added here; their updated
                 parameters go to p
    Rank r's to_owner[p] and rank p's from_peer[r] list the same gids in the
    same order, so fixed all_to_all splits line the rows up.
    """

    def __init__(self, owner, r_lo, r_hi, rank: int, world: int):
        self.rank, self.world = rank, world
        ar = torch.arange(owner.shape[0], device=owner.device)
        in_reach = (r_lo <= rank) & (rank <= r_hi)
        local = in_reach | (owner == rank)
        self.local_gids = ar[local]
        lo, hi, own = r_lo[local], r_hi[local], owner[local]
        self.owned = own == rank
        self.r_lo, self.r_hi = lo, hi
        la = torch.arange(self.local_gids.shape[0], device=owner.device)
        self.to_owner = [la[own == p] if p != rank else la[:0] for p in range(world)]
        self.from_peer = [la[self.owned & (lo <= p) & (p <= hi)] if p != rank else la[:0]
                          for p in range(world)]

    @property
    def n_local(self) -> int:
        return int(self.local_gids.shape[0])

    def halo_counts(self):
        return ([int(t.shape[0]) for t in self.to_owner],
                [int(t.shape[0]) for t in self.from_peer])


# ------------------------------------------------------------ exchange
def _a2a_rows(dist, group, send_lists, recv_counts, rows_of):
    """all_to_all_single of f64 rows: send rows_of(idx) for each peer's list,
    receive recv_counts[p] rows from each peer; returns per-peer views."""
    send = torch.cat([rows_of(idx) for idx in send_lists], 0) if send_lists else None
    dev = send.device
    out = torch.empty((sum(recv_counts), _ROWW), dtype=torch.float64, device=dev)
    in_splits = [int(t.shape[0]) * _ROWW for t in send_lists]
    out_splits = [c * _ROWW for c in recv_counts]
    if dev.type == "cuda" and _backend(dist, group) == "gloo":
        # gloo moves CPU tensors (test path: ranks sharing one GPU)
        out_h = torch.empty(out.numel(), dtype=torch.float64)
        dist.all_to_all_single(out_h, send.reshape(-1).cpu(), out_splits, in_splits, group=group)
        out.copy_(out_h.view_as(out))
    else:
        dist.all_to_all_single(out.view(-1), send.reshape(-1), out_splits, in_splits,
                               group=group)
    views, o = [], 0
    for c in recv_counts:
        views.append(out[o:o + c])
        o += c
    return views


def _backend(dist, group) -> str:
    try:
        return dist.get_backend(group)
    except (RuntimeError, ValueError):
        return "gloo"


def _pack_params(f: GaussianField, idx: torch.Tensor) -> torch.Tensor:
    return torch.cat([f.positions[idx], f.log_scales[idx], f.rotations[idx],
                      f.raw_amplitude[idx, None], f.raw_relax[idx, None]], 1)


def _unpack_params(f: GaussianField, idx: torch.Tensor, rows: torch.Tensor) -> None:
    f.positions.index_copy_(0, idx, rows[:, 0:3].contiguous())
    f.log_scales.index_copy_(0, idx, rows[:, 3:6].contiguous())
    f.rotations.index_copy_(0, idx, rows[:, 6:10].contiguous())
    f.raw_amplitude.index_copy_(0, idx, rows[:, 10].contiguous())
    f.raw_relax.index_copy_(0, idx, rows[:, 11].contiguous())


class _Resolved:
    """A finished step's handle (eager mode), like train.StepHandle."""

    def __init__(self, v):
        self.v = v

    def loss(self):
        return self.v


# ------------------------------------------------- graph-capturable hooks
class _HaloHooks:
    """The halo step's exchanges as hooks of TrainStep's captured graph
    (train._graph_body): fixed plan, fixed buffers and splits, NCCL
    collectives -- nothing reads the host, so one replay holds a whole step."""

    def __init__(self, hs: "HaloTrainStep"):
        p, dev = hs.plan, hs.f.device
        self.dist, self.group = hs.dist, hs.group
        self.world = hs.world
        self.to_owner, self.from_peer = p.to_owner, p.from_peer
        self.n_to = [int(t.shape[0]) for t in p.to_owner]
        self.n_from = [int(t.shape[0]) for t in p.from_peer]
        self.cat_to = torch.cat(p.to_owner)
        self.cat_from = torch.cat(p.from_peer)
        z = lambda k: torch.zeros((max(k, 1), _ROWW), dtype=torch.float64, device=dev)  # noqa
        self.part_send, self.part_recv = z(sum(self.n_to)), z(sum(self.n_from))
        self.prm_send, self.prm_recv = z(sum(self.n_from)), z(sum(self.n_to))
        self.red2 = torch.zeros(2, dtype=torch.float64, device=dev)
        self.oi = torch.nonzero(p.owned).view(-1)
        self.plan_lo, self.plan_hi = p.r_lo[self.oi], p.r_hi[self.oi]
        self.consts = reach_consts(hs.target.grid, hs.bd, hs.slabs, dev)
        self.grid, self.bd, self.slabs = hs.target.grid, hs.bd, hs.slabs
        self.cut, self.check_margin = hs.opts.cutoff_sigma, hs.check_margin

    def _a2a(self, recv, send, n_recv, n_send):
        ns, nr = sum(n_send), sum(n_recv)
        self.dist.all_to_all_single(recv[:nr].view(-1), send[:ns].view(-1),
                                    [c * _ROWW for c in n_recv], [c * _ROWW for c in n_send],
                                    group=self.group)

    def exchange_partials(self, gsum):
        ns = sum(self.n_to)
        if ns:
            torch.index_select(gsum, 0, self.cat_to, out=self.part_send[:ns])
        self._a2a(self.part_recv, self.part_send, self.n_from, self.n_to)
        o = 0
        for q in range(self.world):
            c = self.n_from[q]
            if c:
                gsum.index_add_(0, self.from_peer[q], self.part_recv[o:o + c])
            o += c

    def reduce_loss(self, loss_sum, overflow, gloss, govf):
        self.red2[0:1].copy_(loss_sum[0:1])
        self.red2[1:2].copy_(overflow[0:1].to(torch.float64))
        self.dist.all_reduce(self.red2, group=self.group)
        gloss.copy_(self.red2[0:1])
        govf.copy_((self.red2[1:2] > 0).to(torch.int32))

    def exchange_params(self, f):
        ns = sum(self.n_from)
        if ns:
            self.prm_send[:ns].copy_(_pack_params(f, self.cat_from))
        self._a2a(self.prm_recv, self.prm_send, self.n_to, self.n_from)
        o = 0
        for q in range(self.world):
            c = self.n_to[q]
            if c:
                _unpack_params(f, self.to_owner[q], self.prm_recv[o:o + c])
            o += c

    def reach_check(self, f, result):
        oi = self.oi
        _, lo, hi = reach_and_owner(f.positions[oi], f.log_scales[oi], f.rotations[oi],
                                    self.grid, self.bd, self.slabs, self.cut, self.check_margin,
                                    consts=self.consts)
        bad = (lo <= hi) & ((lo < self.plan_lo) | (hi > self.plan_hi))
        result[1:2] += 4.0 * bad.any().to(torch.float64).view(1)


# ------------------------------------------------------------- the step
class HaloTrainStep:
    """fit()'s iteration sharded over ranks with owner-computes + halo
    exchange (module docstring).  Eager; works over NCCL and, for tests, gloo.

    step = HaloTrainStep(lr_volume, slabs, rank, group)
    step.attach(field, state)        # full field on every rank (replicated)
    loss = step.step(lrs)            # one fit() iteration, global mean loss
    f, st = step.gather()            # full field and moments, every rank
    """

    def __init__(self, target: Volume, slabs, rank: int, group, opts=RenderOptions(),
                 brick_dims=(8, 8, 4), loss: str = "l1", margin: float = 1.0,
                 check_margin: float = 1e-3):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.target, self.slabs, self.rank = target, list(slabs), rank
        self.world = len(self.slabs)
        self.opts, self.bd, self.loss_kind, self.margin = opts, tuple(brick_dims), loss, margin
        # the reach check's widening: a hair above the binning's own rounding
        # (the plan's f64 torch box and the binning's numpy-order box agree
        # to an ulp); larger values re-plan earlier (tests force re-plans).
        # Graph mode queues one step ahead, so it checks against half the
        # margin: the queued step stays inside the plan.
        self.check_margin = check_margin
        if self.graph_mode:
            self.check_margin = max(check_margin, 0.5 * margin)
        self.replans = 0
        self.last_halo = None

    # -- plan / re-plan from a full replicated field
    def attach(self, f: GaussianField, state: AdamState) -> None:
        from .train import TrainStep
        own, lo, hi = reach_and_owner(f.positions, f.log_scales, f.rotations, self.target.grid,
                                      self.bd, self.slabs, self.opts.cutoff_sigma, self.margin)
        self.plan = p = HaloPlan(own, lo, hi, self.rank, self.world)
        g = p.local_gids
        self.f = GaussianField(*[getattr(f, n)[g] for n in PARAM_NAMES],
                               amplitude_enabled=f.amplitude_enabled,
                               relax_enabled=f.relax_enabled, device=f.device)
        self.state = AdamState(state.t, {k: v[g].contiguous() for k, v in state.m.items()},
                               {k: v[g].contiguous() for k, v in state.v.items()})
        self.n_global = f.count
        self.amp_en, self.rel_en = f.amplitude_enabled, f.relax_enabled
        if self.graph_mode:
            # the whole iteration as one CUDA-graph replay: TrainStep's
            # sharded graph with the halo exchanges as its collective hooks
            self.inner = TrainStep(self.target, self.opts, self.bd, self.loss_kind,
                                   slab=self.slabs[self.rank], process_group=self.group,
                                   world_size=self.world)
            self.inner.halo_hooks = _HaloHooks(self)
        else:
            self.inner = TrainStep(self.target, self.opts, self.bd, self.loss_kind,
                                   slab=self.slabs[self.rank])
        self.replans += 1
        self.last_halo = p.halo_counts()

    @property
    def graph_mode(self) -> bool:
        """NCCL (collectives capturable), the f32 engine, graphs not disabled."""
        return (_backend(self.dist, self.group) == "nccl" and self.opts.precision == "f32"
                and not os.environ.get("GSV_NO_GRAPH")
                and not os.environ.get("GSV_NO_SHARD_GRAPH"))

    def _replan(self) -> None:
        if self.graph_mode:
            while self.inner.__dict__.get("_pending"):
                self.inner._pending[0].loss()
        f, st = self.gather()
        self.attach(f, st)

    def step_async(self, lrs: dict, beta1: float = 0.9, beta2: float = 0.999,
                   eps: float = 1e-8):
        """Graph mode: enqueue one replay (one step may be queued behind another,
        as fit() runs; a flagged reach violation re-plans before the next
        launch -- the check's half-margin hysteresis keeps the queued step
        valid).  Eager mode: the step runs to completion."""
        if not self.graph_mode:
            return _Resolved(self.step(lrs, beta1, beta2, eps))
        if self.inner.__dict__.get("_replan_needed"):
            self._replan()
        return self.inner.step_async(self.f, self.state, lrs, beta1, beta2, eps)

    # -- one iteration
    def step(self, lrs: dict, beta1: float = 0.9, beta2: float = 0.999,
             eps: float = 1e-8) -> float:
        if self.graph_mode:
            loss = self.step_async(lrs, beta1, beta2, eps).loss()
            if self.inner.__dict__.get("_replan_needed"):
                self._replan()
            return loss
        return self._step_eager(lrs, beta1, beta2, eps)

    def _step_eager(self, lrs: dict, beta1: float = 0.9, beta2: float = 0.999,
                    eps: float = 1e-8) -> float:
        from .raster import _pair_partials
        from .train import _adam_launch
        dist, group, p, f = self.dist, self.group, self.plan, self.f
        ts = self.inner
        out = ts.forward(f)
        aux = out.idx._aux
        gsum = _pair_partials(f, self.target.grid, out.idx, self.opts, aux.rec32, aux.rec64,
                              out.ab, aux.gstart, aux.box, True, pool=ts.pool,
                              live_masks=ts._masks, mask_vpl=ts._mask_vpl)
        # 2. halo partials -> owners; owners add, peer by peer in rank order
        recv_counts = [int(t.shape[0]) for t in p.from_peer]
        got = _a2a_rows(dist, group, p.to_owner, recv_counts, lambda idx: gsum[idx])
        for q in range(self.world):
            if recv_counts[q]:
                gsum.index_add_(0, p.from_peer[q], got[q])
        # 3. global loss (slab voxels are disjoint) and gate
        red = torch.stack([out.loss_sum[0], torch.zeros_like(out.loss_sum[0])])
        dist.all_reduce(red, group=group)
        loss = float(red[0].item()) / self.target.grid.num_voxels
        if not math.isfinite(loss):
            return loss                      # the reference raises before updating
        # 4. chain rule + Adam + renorm on the local rows
        _adam_launch(f, self.state, lrs, beta1, beta2, eps, None, None, gsum,
                     self.opts.precision_code, ts.pool)
        # 5. owners' updated parameters -> the ranks holding them as halo
        recv_counts = [int(t.shape[0]) for t in p.to_owner]
        got = _a2a_rows(dist, group, p.from_peer, recv_counts,
                        lambda idx: _pack_params(f, idx))
        for q in range(self.world):
            if recv_counts[q]:
                _unpack_params(f, p.to_owner[q], got[q])
        f.bump_version()
        # 6. reach check on owned Gaussians: the new box (widened by
        # check_margin) must stay inside the planned reach (widened by margin)
        oi = torch.nonzero(p.owned).view(-1)
        _, lo, hi = reach_and_owner(f.positions[oi], f.log_scales[oi], f.rotations[oi],
                                    self.target.grid, self.bd, self.slabs,
                                    self.opts.cutoff_sigma, self.check_margin)
        inside = lo <= hi
        bad = inside & ((lo < p.r_lo[oi]) | (hi > p.r_hi[oi]))
        flag = torch.tensor([float(bool(bad.any()))], dtype=torch.float64, device=f.device)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=group)
        if float(flag.item()) > 0:
            self._replan()
        return loss

    # -- assemble the full field and moments on every rank
    def gather(self):
        dist, group, p, f = self.dist, self.group, self.plan, self.f
        oi = torch.nonzero(p.owned).view(-1)
        gids = p.local_gids[oi]
        rows = torch.cat([_pack_params(f, oi)] +
                         [torch.cat([self.state.m[n][oi].reshape(len(oi), -1)
                                     for n in PARAM_NAMES], 1),
                          torch.cat([self.state.v[n][oi].reshape(len(oi), -1)
                                     for n in PARAM_NAMES], 1)], 1)   # 12 + 12 + 12
        cnt = torch.tensor([len(oi)], dtype=torch.int64, device=f.device)
        counts = [torch.zeros_like(cnt) for _ in range(self.world)]
        self._all_gather(counts, cnt)
        mx = int(max(int(c.item()) for c in counts))
        pad = torch.zeros((mx, 37), dtype=torch.float64, device=f.device)
        pad[:len(oi), 0] = gids.to(torch.float64)
        pad[:len(oi), 1:] = rows
        bufs = [torch.zeros_like(pad) for _ in range(self.world)]
        self._all_gather(bufs, pad)
        n = self.n_global
        full = torch.empty((n, 36), dtype=torch.float64, device=f.device)
        for c, b in zip(counts, bufs):
            k = int(c.item())
            full[b[:k, 0].to(torch.int64)] = b[:k, 1:]
        parts = torch.split(full[:, :12], [3, 3, 4, 1, 1], 1)
        fg = GaussianField(parts[0], parts[1], parts[2], parts[3].reshape(-1),
                           parts[4].reshape(-1), amplitude_enabled=self.amp_en,
                           relax_enabled=self.rel_en, device=f.device)
        widths = {"positions": 3, "log_scales": 3, "rotations": 4, "raw_amplitude": 1,
                  "raw_relax": 1}
        m, v, o = {}, {}, 12
        for name in PARAM_NAMES:
            w = widths[name]
            shp = (n, w) if w > 1 else (n,)
            m[name] = full[:, o:o + w].reshape(shp).contiguous()
            v[name] = full[:, o + 12:o + 12 + w].reshape(shp).contiguous()
            o += w
        return fg, AdamState(self.state.t, m, v)

    def _all_gather(self, outs, t):
        if t.device.type == "cuda" and _backend(self.dist, self.group) == "gloo":
            oh = [torch.empty_like(t, device="cpu") for _ in outs]
            self.dist.all_gather(oh, t.cpu(), group=self.group)
            for o, h in zip(outs, oh):
                o.copy_(h)
        else:
            self.dist.all_gather(outs, t, group=self.group)
