"""Multi-GPU sharding of the partition algorithms.

One process per GPU (``torchrun`` / ``bench.py --gpus N``), ``torch.distributed``
for the plumbing: NCCL on GPUs (gloo with CPU tensors in the tests).  Every
rank draws the plan bit-exactly from the seed; each rank holds ONLY the input
rows its share needs (``*_shard(...).local_rows``, in that order), so the
host->device traffic of N ranks adds up to about one copy of the input.

The step stays on the device: per-rank kernels, then one all-gather of small
fixed-size record tensors (per-piece fit figures, statuses and per-segment
column sums), a plan-order sort and fold of those records for the final
re-centring, and one shift pass.  Nothing is read on the host until
``finish()``, which decodes the gathered records identically on every rank
(so every rank raises the same exception for a failing piece — no rank can
be left waiting in a collective), and ``gather_points`` assembles the n x r
configuration on rank 0 with one NCCL gather.

* divide-and-conquer (algorithms.py:128-172): every rank solves the anchor
  (subset 1) and its contiguous share of subsets 2..p and aligns them locally
  (the anchor is known everywhere, so nothing is broadcast).
* fast (algorithms.py:285-348): the root's level-1 subtrees are dealt to ranks
  in contiguous blocks; every rank also solves the root's alignment set (raw
  rows of every child's samples — computed redundantly) and aligns its
  children onto their slices of it.
* interpolation (algorithms.py:245-274): rank 0 solves the landmark set and
  the Gower context and broadcasts them as one device vector; every rank
  streams a contiguous block of rows (fixed 65 536-row blocks).

The re-centring mean is a fold of per-segment sums in plan order (subsets,
level-1 children, row blocks), and every segment is summed by one rank, so
results are bitwise identical for every world size.  The per-rank compute is
behind a small backend interface: ``GpuBackend`` (libmdsx kernels, the
product); the CPU tests drive the same code with an oracle-backed backend in
``tests/``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .errors import InvalidInputError, NumericalError
from .params import AlgorithmParams
from .plans import (DcPlan, FastPlan, flatten_fast_shard, flatten_subsets, interpolation_sample,
                    plan_device_cache, plan_divide_conquer, plan_fast)
from .results import MdsConfiguration

SUM_BLOCK = 65536      # canonical row block of the interpolation re-centring sums
_SENTINEL = 2.0 ** 62  # record id of padding rows (sorts after every real id)
_STATUS = np.dtype([("code", np.int32), ("index", np.int32), ("value", np.float64)])


def shard(count: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split of range(count): [lo, hi) for `rank`."""
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def decode_status(t) -> np.ndarray:
    """(k, 2) float64 status records (16-byte mdsx_piece_status) -> structured."""
    raw = np.ascontiguousarray(t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else t,
                               dtype=np.float64)
    return raw.view(np.uint8).reshape(-1, 16).copy().view(_STATUS).reshape(-1)


# ------------------------------------------------------------------ collectives
class Comm:
    """Tensor collectives over a torch.distributed group (device tensors with
    NCCL, CPU tensors with gloo)."""

    def __init__(self, group=None, device=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device if device is not None else torch.device("cpu")
        self.nccl = dist.get_backend(group) == "nccl"

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """[world * t.shape[0], ...]: every rank's equally shaped tensor, rank order."""
        if self.world == 1:
            return t
        out = torch.empty((self.world * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype,
                          device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=self.group)
        return out

    def broadcast_(self, t: torch.Tensor, src: int = 0) -> torch.Tensor:
        if self.world > 1:
            dist.broadcast(t, src=src, group=self.group)
        return t

    def gather(self, t: torch.Tensor, dst: int = 0):
        """Equally shaped tensors of every rank -> [world, ...] on `dst`, None elsewhere."""
        if self.world == 1:
            return t[None]
        if self.rank == dst:
            parts = [torch.empty_like(t) for _ in range(self.world)]
            dist.gather(t.contiguous(), gather_list=parts, dst=dst, group=self.group)
            return torch.stack(parts)
        dist.gather(t.contiguous(), dst=dst, group=self.group)
        return None

    def sum_(self, t: torch.Tensor) -> torch.Tensor:
        """In-place sum over the ranks (exact for terms with disjoint supports)."""
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def max_int(self, v: int) -> int:
        if self.world == 1:
            return int(v)
        t = torch.tensor([v], dtype=torch.int64, device=self.device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        return int(t.item())


def _pad_rows(t: torch.Tensor, rows: int, fill: float = 0.0) -> torch.Tensor:
    if t.shape[0] == rows:
        return t
    pad = torch.full((rows - t.shape[0],) + tuple(t.shape[1:]), fill, dtype=t.dtype,
                     device=t.device)
    return torch.cat([t, pad])


def _gather_records(comm: Comm, recs: torch.Tensor, kmax: int, count: int) -> torch.Tensor:
    """All-gather per-rank record rows (column 0 = global id), drop padding
    and return the `count` real records sorted by id (on the device)."""
    allr = comm.all_gather(_pad_rows(recs, kmax, _SENTINEL))
    order = torch.argsort(allr[:, 0], stable=True)
    return allr.index_select(0, order[:count])


def _fold_mean(sums: torch.Tensor, n: int) -> torch.Tensor:
    """Column sums folded in record order (the same tensor shape on every
    world size -> the same arithmetic), divided by n."""
    return torch.cumsum(sums, dim=0)[-1] / n


@dataclass
class ShardResult:
    """One rank's share: `out` rows [report_lo, report_hi) are this rank's
    rows of the configuration; finish() fills the fit figures."""

    out: torch.Tensor
    report_lo: int
    report_hi: int
    finish_fn: object
    estimates: np.ndarray | None = None
    gof_g1: float | None = None
    gof_g2: float | None = None
    rows_fn: object = None          # rank k -> global row ids of its reported rows

    def finish(self) -> "ShardResult":
        if self.estimates is None:
            self.estimates, self.gof_g1, self.gof_g2 = self.finish_fn()
        return self


def gather_points(res: ShardResult, n: int, comm: Comm, to_host: bool = True):
    """Assemble the full n x r configuration on rank 0 (None elsewhere):
    one gather of every rank's reported rows (padded to the largest share),
    one device scatter into input row order."""
    res.finish()
    r = res.out.shape[1]
    mine = res.out[res.report_lo:res.report_hi]
    cap = comm.max_int(mine.shape[0])
    parts = comm.gather(_pad_rows(mine, cap))
    if comm.rank != 0:
        return None
    rows, vals = [], []
    for k in range(comm.world):
        idx = res.rows_fn(k)
        rows.append(idx)
        vals.append(parts[k, :len(idx)])
    idx_t = torch.from_numpy(np.ascontiguousarray(np.concatenate(rows), dtype=np.int64)).to(
        res.out.device)
    out = torch.empty((n, r), dtype=res.out.dtype, device=res.out.device)
    out.index_copy_(0, idx_t, torch.cat(vals))
    if not to_host:
        return out
    from . import _device as D
    return D.to_host(out) if out.is_cuda else out.numpy()


# ================================================================= D&C
@dataclass
class DcShard:
    """Rank `rank`'s share of a D&C plan.  Local matrix rows: the anchor subset
    (connecting rows first), then the own rows of every owned subset."""

    pieces: np.ndarray        # global subset ids, anchor (0) first
    local_rows: np.ndarray    # global row id of each local matrix row
    row_idx: np.ndarray       # flattened per-subset local row lists
    piece_off: np.ndarray
    own_off: np.ndarray       # own-row segments of the subsets in local order
    report_lo: int            # first local row this rank reports (anchor: rank 0 only)


def _shard_cached(plan, key, make):
    """Shard layouts are pure functions of (plan, world, rank): memoised on the
    plan's cache (dropped with the plan)."""
    try:
        cache = plan_device_cache(plan)
    except (AttributeError, TypeError):
        cache = None
    if cache is None:
        return make()
    if key not in cache:
        cache[key] = make()
    return cache[key]


def dc_shard(plan: DcPlan, world: int, rank: int) -> DcShard:
    return _shard_cached(plan, ("dc_shard", world, rank), lambda: _dc_shard(plan, world, rank))


def _dc_shard(plan: DcPlan, world: int, rank: int) -> DcShard:
    P, c = plan.p, plan.c
    lo, hi = shard(P - 1, world, rank)
    mine = np.arange(1 + lo, 1 + hi, dtype=np.int64)
    anchor = np.asarray(plan.subsets[0], dtype=np.int64)
    l0 = len(anchor)
    own = [np.asarray(plan.subsets[j][c:], dtype=np.int64) for j in mine]
    sizes = np.array([l0] + [len(o) for o in own], dtype=np.int64)
    own_off = np.zeros(len(sizes) + 1, dtype=np.int64)
    np.cumsum(sizes, out=own_off[1:])
    local_rows = np.concatenate([anchor] + own) if own else anchor.copy()
    conn = np.arange(c, dtype=np.int64)
    lists = [np.arange(l0, dtype=np.int64)] + [
        np.concatenate([conn, np.arange(own_off[i + 1], own_off[i + 2], dtype=np.int64)])
        for i in range(len(own))]
    row_idx, piece_off = flatten_subsets(lists)
    return DcShard(np.concatenate([[0], mine]), local_rows, row_idx, piece_off, own_off,
                   0 if rank == 0 else l0)


class ShardedDivide:
    """divide_and_conquer_mds over comm.world ranks.  `x_local` holds the rows
    ``dc_shard(plan, world, rank).local_rows`` in that order."""

    def __init__(self, backend, x_local, plan: DcPlan, r: int, comm: Comm):
        self.be, self.x, self.plan, self.r, self.comm = backend, x_local, plan, r, comm
        self.sh = sh = dc_shard(plan, comm.world, comm.rank)
        if x_local.shape[0] != len(sh.local_rows):
            raise ValueError(f"rank {comm.rank}: local matrix has {x_local.shape[0]} rows, "
                             f"the shard needs {len(sh.local_rows)}")
        dev = backend.device
        self.dev = dev
        up = _shard_cached(plan, ("dc_dev", comm.world, comm.rank, str(dev)),
                           lambda: (backend.index(sh.row_idx), backend.index(sh.own_off)))
        self.row_idx, self.own_off = up
        npc = len(sh.pieces)
        self.out = torch.empty((len(sh.local_rows), r), dtype=torch.float64, device=dev)
        self.est = torch.empty((npc, r), dtype=torch.float64, device=dev)
        self.gof = torch.empty((npc, 2), dtype=torch.float64, device=dev)
        self.status = torch.zeros((npc, 2), dtype=torch.float64, device=dev)
        self.sums = torch.empty((npc, r), dtype=torch.float64, device=dev)
        self.ids = torch.tensor(sh.pieces, dtype=torch.float64, device=dev)[:, None]
        self.first = 0 if comm.rank == 0 else 1          # the anchor's record: rank 0 only
        self.kmax = 1 + shard(plan.p - 1, comm.world, 0)[1]
        self.recs = None

    def _gather_sorted(self, rows: torch.Tensor) -> torch.Tensor:
        """This rank's per-subset rows (local subset order, the anchor's first)
        -> every subset's row in global subset order, the anchor's from rank
        0: one all-gather into a padded buffer and a cached selection (the
        layout is fixed by the plan and the world size)."""
        rows = rows[self.first:]
        comm = self.comm
        if comm.world == 1:
            return rows
        key = ("dc_sel", comm.world, rows.shape[1], str(rows.device))
        cache = _shard_cached(self.plan, key, lambda: {})
        if "sel" not in cache:
            pos = []
            for k in range(comm.world):
                s = dc_shard(self.plan, comm.world, k)
                ids = np.asarray(s.pieces[0 if k == 0 else 1:], dtype=np.int64)
                pos.append(np.stack([ids, k * self.kmax + np.arange(len(ids))], axis=1))
            pos = np.concatenate(pos)
            cache["sel"] = torch.from_numpy(pos[np.argsort(pos[:, 0], kind="stable"), 1].copy()).to(
                rows.device)
            cache["buf"] = torch.zeros((self.kmax, rows.shape[1]), dtype=rows.dtype, device=rows.device)
        buf = cache["buf"]
        buf[:rows.shape[0]].copy_(rows)
        return comm.all_gather(buf).index_select(0, cache["sel"])

    def _gather_contrib(self, local: torch.Tensor) -> torch.Tensor:
        """Every rank's subset contributions in global subset order."""
        return self._gather_sorted(local)

    def launch(self) -> ShardResult:
        be, sh, r = self.be, self.sh, self.r
        if getattr(be, "dc_run_sharded", None) is not None and be.dc_run_sharded(
                self.x, self.row_idx, sh.piece_off, self.plan.c, r, self.out, self.est, self.gof,
                self.status, self.plan.n, self.plan.p, self._gather_contrib):
            # re-centred on the device inside the call: the mean of every
            # subset's contribution in global order (no sums pass, no shift)
            self.recs = self._gather_sorted(
                torch.cat([self.ids, self.gof, self.est, self.sums.zero_(), self.status], dim=1))
            return ShardResult(self.out, sh.report_lo, len(sh.local_rows), self.finish,
                               rows_fn=self.rows_of)
        be.dc_run(self.x, self.row_idx, sh.piece_off, self.plan.c, r, self.out, self.est,
                  self.gof, self.status)
        be.range_sums(self.out, self.own_off, len(sh.pieces), self.sums)
        # record: [subset id, g1, g2, est(r), sums(r), status(2)]
        recs = torch.cat([self.ids, self.gof, self.est, self.sums, self.status], dim=1)[self.first:]
        self.recs = _gather_records(self.comm, recs, self.kmax, self.plan.p)
        mean = _fold_mean(self.recs[:, 3 + r:3 + 2 * r], self.plan.n)
        be.shift_rows(self.out, mean)
        return ShardResult(self.out, sh.report_lo, len(sh.local_rows), self.finish,
                           rows_fn=self.rows_of)

    def rows_of(self, k: int) -> np.ndarray:
        s = dc_shard(self.plan, self.comm.world, k)
        return s.local_rows[s.report_lo:]

    def finish(self):
        """Host decode of the gathered records (identical on every rank)."""
        from .primitives import raise_piece_status
        r, plan = self.r, self.plan
        recs = self.recs.cpu().numpy()
        st = decode_status(recs[:, 3 + 2 * r:])
        if np.any(st["code"] == 3):
            raise InvalidInputError("data contains non-finite values")
        bad = np.flatnonzero(st["code"] != 0)
        if bad.size:                                      # first failing subset in plan order
            raise_piece_status(st[bad[0]], r, f"subset {bad[0] + 1}")
        sizes = np.fromiter((len(q) for q in plan.subsets), dtype=np.float64, count=plan.p)
        weights = sizes.copy()
        weights[1:] -= plan.c                             # algorithms.py:158-166
        g1 = float(np.dot(weights, recs[:, 1]) / plan.n)
        g2 = float(np.dot(weights, recs[:, 2]) / plan.n)
        per = recs[:, 3:3 + r] * (sizes / weights)[:, None]
        return per.mean(axis=0), g1, g2


# ================================================================= interpolation
@dataclass
class InterpShard:
    lo: int
    hi: int                   # global rows [lo, hi) of this rank
    b_lo: int
    b_hi: int                 # canonical sum blocks [b_lo, b_hi)
    land_pos: np.ndarray      # local positions of the landmarks inside [lo, hi)
    land_sel: np.ndarray      # ... and their index in the sample

    @property
    def local_rows(self) -> np.ndarray:
        return np.arange(self.lo, self.hi, dtype=np.int64)


def interp_shard(n: int, sample: np.ndarray, world: int, rank: int) -> InterpShard:
    blocks = (n + SUM_BLOCK - 1) // SUM_BLOCK
    b_lo, b_hi = shard(blocks, world, rank)
    lo, hi = b_lo * SUM_BLOCK, min(n, b_hi * SUM_BLOCK)
    sel = np.flatnonzero((sample >= lo) & (sample < hi)).astype(np.int64)
    return InterpShard(lo, hi, b_lo, b_hi, (sample[sel] - lo).astype(np.int64), sel)


class ShardedInterpolation:
    """interpolation_mds over comm.world ranks.  `x_local` holds rows
    [lo, hi) of ``interp_shard``; rank 0 also gets the landmark rows
    `x_landmarks` (sample order)."""

    def __init__(self, backend, x_local, n: int, sample: np.ndarray, r: int, comm: Comm,
                 x_landmarks=None):
        self.be, self.x, self.n, self.r, self.comm = backend, x_local, n, r, comm
        self.sample = np.asarray(sample, dtype=np.int64)
        self.l = l = len(self.sample)
        self.sh = sh = interp_shard(n, self.sample, comm.world, comm.rank)
        if x_local.shape[0] != sh.hi - sh.lo:
            raise ValueError(f"rank {comm.rank}: local matrix has {x_local.shape[0]} rows, "
                             f"the shard needs {sh.hi - sh.lo}")
        if comm.rank == 0 and x_landmarks is None:
            raise ValueError("rank 0 needs the landmark rows")
        self.xl = x_landmarks
        dev = self.dev = backend.device
        p = x_local.shape[1]
        self.head_len = backend.head_len(l, p, r)
        self.head = torch.zeros(self.head_len, dtype=torch.float64, device=dev)
        self.out = torch.empty((sh.hi - sh.lo, r), dtype=torch.float64, device=dev)
        self.land_pos = backend.index(sh.land_pos)
        self.land_sel = backend.index(sh.land_sel)
        nb = sh.b_hi - sh.b_lo
        bounds = np.minimum(sh.hi, np.arange(sh.b_lo, sh.b_hi + 1, dtype=np.int64) * SUM_BLOCK) - sh.lo
        self.bounds = backend.index(bounds)
        self.nb = nb
        self.blocks = (n + SUM_BLOCK - 1) // SUM_BLOCK
        self.kmax = shard(self.blocks, comm.world, 0)[1]
        self.recs = None
        # tile route: the Gower pass writes per-tile column sums (tile_rows rows;
        # rank row ranges start on SUM_BLOCK, a multiple of the tile), the
        # landmark overwrite a per-landmark correction; both are gathered in row /
        # sample order and folded identically on every rank
        self.tr = backend.tile_rows(x_local, r) if hasattr(backend, "tile_rows") else 0
        if self.tr and SUM_BLOCK % self.tr == 0:
            nt = (sh.hi - sh.lo + self.tr - 1) // self.tr
            counts = [(s.hi - s.lo + self.tr - 1) // self.tr
                      for s in (interp_shard(n, self.sample, comm.world, k) for k in range(comm.world))]
            self.ntiles, self.ktile = nt, max(counts)
            self.ntiles_total = sum(counts)
            self.tbuf = torch.zeros((self.ktile + 1, r), dtype=torch.float64, device=dev)
            self.corr = torch.zeros((l, r), dtype=torch.float64, device=dev)
            if comm.world > 1:
                sel = np.concatenate([k * (self.ktile + 1) + 1 + np.arange(c, dtype=np.int64)
                                      for k, c in enumerate(counts)])
                self.tsel = backend.index(sel)
            self.flags = None
        else:
            self.tr = 0
            self.sums = torch.empty((nb, r), dtype=torch.float64, device=dev)
            self.ids = torch.arange(sh.b_lo, sh.b_hi, dtype=torch.float64, device=dev)[:, None]
            self.nf = torch.zeros((nb, 1), dtype=torch.float64, device=dev)

    def launch(self) -> ShardResult:
        be, sh, r, l = self.be, self.sh, self.r, self.l
        if self.comm.rank == 0:
            be.landmark_head(self.xl, r, self.head)
        self.comm.broadcast_(self.head, 0)
        base = self.head[-l * r:].view(l, r)
        if self.tr:
            flag = be.gower_tiles(self.head, l, r, self.x, self.out, self.tbuf[1:1 + self.ntiles])
            be.landmark_overwrite(base, self.land_sel, self.land_pos, self.out, self.corr)
            self.tbuf[0, 0] = flag
            if self.comm.world == 1:
                tiles, self.flags = self.tbuf[1:1 + self.ntiles], self.tbuf[:1, 0]
            else:
                allt = self.comm.all_gather(self.tbuf)
                tiles = allt.index_select(0, self.tsel)
                self.flags = allt[::self.ktile + 1, 0]
                self.comm.sum_(self.corr)
            be.interp_recenter(tiles, self.corr, self.n, self.out)
            return ShardResult(self.out, 0, sh.hi - sh.lo, self.finish, rows_fn=self.rows_of)
        flag = be.gower_rows(self.head, l, r, self.x, self.out)
        if len(sh.land_sel):
            be.scatter_rows(base.index_select(0, self.land_sel), self.land_pos, self.out)
        be.range_sums(self.out, self.bounds, self.nb, self.sums)
        if self.nb:
            self.nf[0, 0] = flag
        recs = torch.cat([self.ids, self.sums, self.nf], dim=1)
        self.recs = _gather_records(self.comm, recs, self.kmax, self.blocks)
        self.flags = self.recs[:, 1 + r]
        be.shift_rows(self.out, _fold_mean(self.recs[:, 1:1 + r], self.n))
        return ShardResult(self.out, 0, sh.hi - sh.lo, self.finish, rows_fn=self.rows_of)

    def rows_of(self, k: int) -> np.ndarray:
        s = interp_shard(self.n, self.sample, self.comm.world, k)
        return np.arange(s.lo, s.hi, dtype=np.int64)

    def finish(self):
        from .primitives import raise_piece_status
        r = self.r
        head = self.head[:self.be.HEAD_FIXED + r].cpu().numpy()
        g1, g2, est = float(head[0]), float(head[1]), head[2:2 + r]
        st = decode_status(head[2 + r:4 + r])[0]
        flag, cond = int(head[4 + r]), float(head[5 + r])
        if int(st["code"]) == 3 or self.flags.abs().sum().item() > 0:
            raise InvalidInputError("data contains non-finite values")
        raise_piece_status(st, r, "sample subset")
        if flag == 1:
            raise NumericalError(f"base covariance is ill-conditioned (condition estimate "
                                 f"{cond:.3e}); the requested dimension exceeds the usable rank")
        if flag == 2:
            raise NumericalError("base covariance is not positive definite")
        return est.copy(), g1, g2


# ================================================================= fast
@dataclass
class FastShard:
    lo: int
    hi: int                   # level-1 children [lo, hi) of the root
    flat: object              # plans.FastFlat with piece rows remapped to local rows
    flat_global: object       # ... as flattened (global row ids)
    local_rows: np.ndarray    # owned subtree rows (DFS order), then extra alignment rows
    n_own: int                # rows of the owned subtrees (reported)
    leaf_base: int            # global DFS index of the first owned leaf
    eval_base: int            # global evaluation position of the first owned piece
    child_off: np.ndarray     # owned children's row ranges in local order


def _subtree_counts(node) -> tuple[int, int]:
    """(leaves, pieces) of a subtree: every leaf and every internal node's
    alignment set is one classical-MDS piece."""
    if node.is_leaf:
        return 1, 1
    lv, pc = 0, 1
    for ch in node.children:
        a, b = _subtree_counts(ch)
        lv += a
        pc += b
    return lv, pc


def fast_shard(plan: FastPlan, world: int, rank: int, counts=None) -> FastShard:
    return _shard_cached(plan, ("fast_shard", world, rank),
                         lambda: _fast_shard(plan, world, rank, counts))


def _fast_shard(plan: FastPlan, world: int, rank: int, counts=None) -> FastShard:
    kids = plan.root.children
    lo, hi = shard(len(kids), world, rank)
    flat = flatten_fast_shard(plan, lo, hi)
    order = flat.order
    need = np.unique(flat.piece_rows)
    pos = np.full(plan.n, -1, dtype=np.int64)
    pos[order] = np.arange(len(order), dtype=np.int64)
    extra = need[pos[need] < 0]
    local_rows = np.concatenate([order, extra])
    pos[extra] = len(order) + np.arange(len(extra), dtype=np.int64)
    from dataclasses import replace
    flat_l = replace(flat, piece_rows=pos[flat.piece_rows], order=np.arange(len(order), dtype=np.int64))
    flat_l._dev_cache = {}                  # device uploads of this shard (algorithms.FastRun)
    counts = counts if counts is not None else [_subtree_counts(ch) for ch in kids]
    leaf_base = int(sum(c[0] for c in counts[:lo]))
    eval_base = int(sum(c[1] for c in counts[:lo]))
    child_off = np.concatenate([[0], np.cumsum([kids[i].size for i in range(lo, hi)])]).astype(np.int64)
    return FastShard(lo, hi, flat_l, flat, local_rows, len(order), leaf_base, eval_base, child_off)


class ShardedFast:
    """fast_mds over comm.world ranks.  `x_local` holds the rows
    ``fast_shard(plan, world, rank).local_rows`` in that order."""

    def __init__(self, backend, x_local, plan: FastPlan, r: int, comm: Comm):
        if plan.root.is_leaf:
            raise ValueError("a single-leaf fast plan is classical MDS (no sharding)")
        self.be, self.x, self.plan, self.r, self.comm = backend, x_local, plan, r, comm
        self.counts = [_subtree_counts(ch) for ch in plan.root.children]
        self.sh = sh = fast_shard(plan, comm.world, comm.rank, self.counts)
        if x_local.shape[0] != len(sh.local_rows):
            raise ValueError(f"rank {comm.rank}: local matrix has {x_local.shape[0]} rows, "
                             f"the shard needs {len(sh.local_rows)}")
        dev = self.dev = backend.device
        self.run = backend.fast_prepare(x_local, plan, sh.flat, r)
        nk = sh.hi - sh.lo
        self.child_off = backend.index(sh.child_off)
        self.sums = torch.empty((nk, r), dtype=torch.float64, device=dev)
        self.child_ids = torch.arange(sh.lo, sh.hi, dtype=torch.float64, device=dev)[:, None]
        flat = sh.flat
        root_pid = len(flat.piece_off) - 2
        ev = [pid for pid in flat.eval_order if pid != root_pid]
        self.root_pid = root_pid
        # piece records in global evaluation order (root alignment set: rank 0, last)
        ev_ids = np.arange(sh.eval_base, sh.eval_base + len(ev), dtype=np.float64)
        total_pieces = int(sum(c[1] for c in self.counts))
        self.total_pieces = total_pieces + 1
        leaf_of = np.full(len(flat.piece_off) - 1, -1.0)
        leaf_of[:flat.n_leaves] = sh.leaf_base + np.arange(flat.n_leaves)
        sel = list(ev)
        ids = list(ev_ids)
        if comm.rank == 0:
            sel.append(root_pid)
            ids.append(float(total_pieces))
        self.piece_sel = backend.index(np.asarray(sel, dtype=np.int64))
        self.piece_ids = torch.tensor(np.stack([ids, leaf_of[sel]], axis=1), dtype=torch.float64,
                                      device=dev)
        kmax_c = comm.max_int(nk)
        self.kmax_c = kmax_c
        self.kmax_p = comm.max_int(len(sel))
        self.recs_c = self.recs_p = None
        self.n_leaves_total = int(sum(c[0] for c in self.counts))

    def _layout(self):
        """Cached all-gather selections (fixed by the plan and the world size):
        piece records in global evaluation order, leaf contributions in global
        leaf order."""
        comm = self.comm
        key = ("fast_sel", comm.world, str(self.dev))

        def make():
            ppos, lpos = [], []
            kp = kl = 0
            shards = [fast_shard(self.plan, comm.world, k, self.counts) for k in range(comm.world)]
            for s_ in shards:
                kl = max(kl, s_.flat.n_leaves)
                kp = max(kp, len(s_.flat.eval_order) - 1 + (1 if s_ is shards[0] else 0))
            for k, s_ in enumerate(shards):
                nev = len(s_.flat.eval_order) - 1
                ppos.append(np.stack([s_.eval_base + np.arange(nev), k * kp + np.arange(nev)], axis=1))
                if k == 0:                      # the root alignment set: last
                    ppos.append(np.array([[self.total_pieces - 1, nev]]))
                lpos.append(k * kl + np.arange(s_.flat.n_leaves))
            ppos = np.concatenate(ppos)
            psel = ppos[np.argsort(ppos[:, 0], kind="stable"), 1]
            return dict(kp=kp, kl=kl, psel=self.be.index(psel),
                        lsel=self.be.index(np.concatenate(lpos)))
        return _shard_cached(self.plan, key, make)

    def _gather(self, rows: torch.Tensor, kmax: int, sel) -> torch.Tensor:
        if self.comm.world == 1:
            return rows
        buf = torch.zeros((kmax,) + tuple(rows.shape[1:]), dtype=rows.dtype, device=rows.device)
        buf[:rows.shape[0]].copy_(rows)
        return self.comm.all_gather(buf).index_select(0, sel)

    def launch(self) -> ShardResult:
        be, sh, r = self.be, self.sh, self.r
        fused = getattr(be, "fast_run_sharded", None)
        if fused is not None:
            lay = self._layout()
            res = fused(self.run, self.plan.n, self.n_leaves_total,
                        lambda local: self._gather(local, lay["kl"], lay["lsel"]))
            if res is not None:
                # re-centred inside the call (leaf contributions gathered in
                # global leaf order): no sums pass, no shift
                pts, est, gof, status = res
                s = self.piece_sel
                recs_p = torch.cat([self.piece_ids, gof.index_select(0, s), est.index_select(0, s),
                                    status.index_select(0, s)], dim=1)
                self.recs_p = self._gather(recs_p, lay["kp"], lay["psel"])
                return ShardResult(pts[:sh.n_own], 0, sh.n_own, self.finish, rows_fn=self.rows_of)
        pts, est, gof, status = be.fast_run(self.run)
        out = pts[:sh.n_own]
        be.range_sums(out, self.child_off, sh.hi - sh.lo, self.sums)
        recs_c = torch.cat([self.child_ids, self.sums], dim=1)
        self.recs_c = _gather_records(self.comm, recs_c, self.kmax_c, len(self.plan.root.children))
        # piece records: [eval position, global leaf index (-1: alignment set), g1, g2, est, status]
        s = self.piece_sel
        recs_p = torch.cat([self.piece_ids, gof.index_select(0, s), est.index_select(0, s),
                            status.index_select(0, s)], dim=1)
        self.recs_p = _gather_records(self.comm, recs_p, self.kmax_p, self.total_pieces)
        be.shift_rows(out, _fold_mean(self.recs_c[:, 1:1 + r], self.plan.n))
        return ShardResult(out, 0, sh.n_own, self.finish, rows_fn=self.rows_of)

    def rows_of(self, k: int) -> np.ndarray:
        kids = self.plan.root.children
        lo, hi = shard(len(kids), self.comm.world, k)
        return (np.concatenate([ch.indices for ch in kids[lo:hi]]) if hi > lo
                else np.empty(0, dtype=np.int64))

    def _label(self, pos: int) -> str:
        """Label of the piece at global evaluation position `pos` (error path)."""
        if pos == self.total_pieces - 1:
            return "root alignment set"
        for k in range(self.comm.world):
            sh = fast_shard(self.plan, self.comm.world, k, self.counts)
            root_pid = len(sh.flat.piece_off) - 2
            ev = [pid for pid in sh.flat.eval_order if pid != root_pid]
            if sh.eval_base <= pos < sh.eval_base + len(ev):
                return sh.flat.labels[ev[pos - sh.eval_base]]
        return f"piece {pos + 1}"

    def finish(self):
        from .primitives import raise_piece_status
        r = self.r
        recs = self.recs_p.cpu().numpy()
        st = decode_status(recs[:, 4 + r:])
        if np.any(st["code"] == 3):
            raise InvalidInputError("data contains non-finite values")
        bad = np.flatnonzero(st["code"] != 0)
        if bad.size:                                  # first failure in evaluation order
            raise_piece_status(st[bad[0]], r, self._label(int(recs[bad[0], 0])))
        leaves = recs[recs[:, 1] >= 0]
        leaves = leaves[np.argsort(leaves[:, 1], kind="stable")]
        from .algorithms import fast_aggregate
        from .plans import flatten_fast_cached
        g1, g2, e = fast_aggregate(self.plan, flatten_fast_cached(self.plan), leaves[:, 2:4],
                                   leaves[:, 4:4 + r])                 # algorithms.py:289-320
        return e, float(g1), float(g2)


# ================================================================= GPU backend
class GpuBackend:
    """Per-rank compute through the C-ABI on the rank's GPU."""

    HEAD_FIXED = 6            # [g1, g2] + est(r) + [status(2), flag, cond] -> 2 + r + 4

    def __init__(self, device):
        from . import _device as D
        self.D = D
        self.device = torch.device(device)

    def index(self, a: np.ndarray) -> torch.Tensor:
        return self.D.index_tensor(np.asarray(a, dtype=np.int64), self.device)

    def _h(self):
        return self.D.handle(self.device), self.D.stream_ptr(self.device)

    def dc_run(self, x, row_idx, piece_off, c, r, out, est, gof, status) -> None:
        h, sp = self._h()
        off = np.ascontiguousarray(piece_off, dtype=np.int64)
        h.call("mdsx_divide_conquer_ex", x.data_ptr(), self.D.dtype_code(x), x.shape[1],
               x.shape[0], x.shape[1], row_idx.data_ptr(), off.ctypes.data, len(off) - 1, c, r,
               out.data_ptr(), est.data_ptr(), gof.data_ptr(), status.data_ptr(), 1, sp)

    def dc_run_sharded(self, x, row_idx, piece_off, c, r, out, est, gof, status, n_total,
                       np_total, gather) -> bool:
        """mdsx_divide_conquer_sharded: the rank's subsets solved and written
        re-centred, the contributions gathered by `gather` (device tensors,
        current stream) from inside the call.  False when the fused output
        route does not apply (the caller re-centres with segment sums)."""
        from ._lib import GATHER_FN
        from .errors import MdsError
        h, sp = self._h()
        off = np.ascontiguousarray(piece_off, dtype=np.int64)
        npl = len(off) - 1
        local = torch.empty((npl, r), dtype=torch.float64, device=self.device)
        glob = torch.empty((np_total, r), dtype=torch.float64, device=self.device)
        failure = []

        def cb(_ctx, _stream):
            try:
                glob.copy_(gather(local))
                return 0
            except Exception as exc:           # reported after the call returns
                failure.append(exc)
                return 1
        fn = GATHER_FN(cb)
        try:
            h.call("mdsx_divide_conquer_sharded", x.data_ptr(), self.D.dtype_code(x), x.shape[1],
                   x.shape[0], x.shape[1], row_idx.data_ptr(), off.ctypes.data, npl, c, r,
                   out.data_ptr(), est.data_ptr(), gof.data_ptr(), status.data_ptr(), n_total,
                   np_total, local.data_ptr(), glob.data_ptr(), fn, None, sp)
        except Exception as exc:
            if failure:
                raise failure[0] from exc
            if type(exc) is MdsError:             # MDSX_UNSUPPORTED: no fused output route
                return False
            raise
        return True

    def range_sums(self, out, off_dev, nseg, sums) -> None:
        if nseg == 0:
            return
        h, sp = self._h()
        h.call("mdsx_segment_colsums", out.data_ptr(), None, off_dev.data_ptr(), nseg,
               out.shape[1], sums.data_ptr(), sp)

    def shift_rows(self, out, mean) -> None:
        if out.shape[0] == 0:
            return
        h, sp = self._h()
        mean = mean.contiguous()
        h.call("mdsx_shift_rows", out.data_ptr(), None, out.shape[0], out.shape[1],
               mean.data_ptr(), sp)

    def scatter_rows(self, src, idx, out) -> None:
        h, sp = self._h()
        src = src.contiguous()
        h.call("mdsx_scatter_rows", src.data_ptr(), idx.data_ptr(), idx.numel(), out.shape[1],
               out.data_ptr(), sp)

    # interpolation -------------------------------------------------------
    def head_len(self, l: int, p: int, r: int) -> int:
        h = self.D.handle(self.device)
        return 2 + r + 4 + int(h.lib.mdsx_gower_context_size(l, p, r)) + l * r

    def landmark_head(self, xl, r: int, head) -> None:
        """head = [g1, g2, est(r), status(2), flag, cond, context, landmark
        configuration] of the landmark rows `xl` (classical MDS + Gower context)."""
        from .primitives import classical_pieces
        D = self.D
        l, p = xl.shape
        idx = self._iota(l)
        pts, est, gof, st = classical_pieces(xl, idx, np.array([0, l], np.int64), r)
        h, sp = self._h()
        size = int(h.lib.mdsx_gower_context_size(l, p, r))
        c0 = 2 + r + 4
        flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        h.call("mdsx_gower_context", xl.data_ptr(), D.dtype_code(xl), p, p, idx.data_ptr(), l,
               pts.data_ptr(), r, head[c0:c0 + size].data_ptr(), head[5 + r:6 + r].data_ptr(),
               flag.data_ptr(), sp)
        head[0:2] = gof[0]
        head[2:2 + r] = est[0]
        head[2 + r:4 + r] = st[0]
        head[4 + r] = flag[0].to(torch.float64)
        head[c0 + size:] = pts.reshape(-1)

    def _iota(self, l: int) -> torch.Tensor:
        key = ("iota", l)
        cache = self.__dict__.setdefault("_cache", {})
        if key not in cache:
            cache[key] = torch.arange(l, dtype=torch.int64, device=self.device)
        return cache[key]

    def gower_rows(self, head, l: int, r: int, x, out) -> torch.Tensor:
        """Gower coordinates of every row of x into out; returns the
        non-finite flag (device scalar, float64)."""
        D = self.D
        h, sp = self._h()
        p = x.shape[1]
        nf = torch.zeros(1, dtype=torch.int32, device=self.device)
        if x.shape[0]:
            h.call("mdsx_gower_interpolate", head[2 + r + 4:].data_ptr(), l, p, r, x.data_ptr(),
                   D.dtype_code(x), p, x.shape[0], out.data_ptr(), r, nf.data_ptr(), 1, sp)
        return nf[0].to(torch.float64)

    def tile_rows(self, x, r: int) -> int:
        """Rows per Gower tile of the tile route (0: the shape takes the row route)."""
        if x.dim() != 2 or not x.is_contiguous() or x.data_ptr() % 16:
            return 0
        h = self.D.handle(self.device)
        return int(h.lib.mdsx_gower_tile_rows(h.ptr, self.D.dtype_code(x), x.shape[1], r))

    def gower_tiles(self, head, l: int, r: int, x, out, tsum) -> torch.Tensor:
        """Gower coordinates of x into out and the per-tile column sums into
        tsum; returns the non-finite flag (device scalar, float64)."""
        h, sp = self._h()
        nf = torch.zeros(1, dtype=torch.int32, device=self.device)
        h.call("mdsx_gower_tiles", head[2 + r + 4:].data_ptr(), l, x.shape[1], r, x.data_ptr(),
               self.D.dtype_code(x), x.shape[0], out.data_ptr(), tsum.data_ptr(), nf.data_ptr(),
               1, sp)
        return nf[0].to(torch.float64)

    def landmark_overwrite(self, base, sel, pos, out, corr) -> None:
        h, sp = self._h()
        base = base.contiguous()
        h.call("mdsx_landmark_overwrite", base.data_ptr(), base.shape[0], base.shape[1],
               sel.data_ptr(), pos.data_ptr(), pos.numel(), out.data_ptr(), corr.data_ptr(), sp)

    def interp_recenter(self, tiles, corr, n: int, out) -> None:
        h, sp = self._h()
        tiles = tiles.contiguous()
        h.call("mdsx_interp_recenter", tiles.data_ptr(), tiles.shape[0], corr.data_ptr(),
               corr.shape[0], corr.shape[1], n, out.data_ptr(), out.shape[0], sp)

    # fast ----------------------------------------------------------------
    def fast_prepare(self, x, plan, flat, r):
        from .algorithms import FastRun
        return FastRun(x, plan, r, flat=flat, local=True)

    def fast_run(self, run):
        run.launch()
        return run.pts, run.est, run.gof, run.status

    def fast_run_sharded(self, run, n_total: int, nleaves_total: int, gather):
        """mdsx_fast_mds_sharded: the rank's subtrees solved and written
        re-centred, the leaf contributions gathered by `gather` from inside
        the call.  None when the one-call route does not apply."""
        if run.route is None:
            return None
        from ._lib import GATHER_FN
        x, r = run.compact(), run.r
        h, sp = self._h()
        nl = run.flat.n_leaves
        bufs = run.__dict__.setdefault("_shard_bufs", {})
        if bufs.get("n") != nleaves_total:
            bufs.update(n=nleaves_total,
                        local=torch.empty((nl, r), dtype=torch.float64, device=self.device),
                        glob=torch.empty((nleaves_total, r), dtype=torch.float64, device=self.device))
        local, glob = bufs["local"], bufs["glob"]
        failure = []

        def cb(_ctx, _stream):
            try:
                glob.copy_(gather(local))
                return 0
            except Exception as exc:           # reported after the call returns
                failure.append(exc)
                return 1
        fn = GATHER_FN(cb)
        try:
            h.call("mdsx_fast_mds_sharded", x.data_ptr(), self.D.dtype_code(x), x.shape[1],
                   x.shape[1], run._route_ref, r, run.out.shape[0], run.out.data_ptr(),
                   run.est.data_ptr(), run.gof.data_ptr(), run.status.data_ptr(), n_total,
                   nleaves_total, local.data_ptr(), glob.data_ptr(), fn, None, sp)
        except Exception as exc:
            if failure:
                raise failure[0] from exc
            raise
        return run.pts, run.est, run.gof, run.status


# ================================================================= entry points
def sharded_divide_and_conquer(backend, x_local, n: int, params: AlgorithmParams, comm: Comm,
                               plan: DcPlan | None = None) -> ShardResult:
    """divide_and_conquer_mds (algorithms.py:128-172) over comm.world ranks;
    returns this rank's finished share (fit figures filled)."""
    prm = params.resolved("divide")
    plan = plan if plan is not None else plan_divide_conquer(n, prm.l, prm.c, prm.seed)
    return ShardedDivide(backend, x_local, plan, prm.r, comm).launch().finish()


def sharded_interpolation(backend, x_local, n: int, params: AlgorithmParams, comm: Comm,
                          sample: np.ndarray | None = None, x_landmarks=None) -> ShardResult:
    prm = params.resolved("interpolate")
    sample = sample if sample is not None else interpolation_sample(n, prm.l, prm.seed)
    return ShardedInterpolation(backend, x_local, n, sample, prm.r, comm,
                                x_landmarks).launch().finish()


def sharded_fast(backend, x_local, n: int, params: AlgorithmParams, comm: Comm,
                 plan: FastPlan | None = None) -> ShardResult:
    prm = params.resolved("fast")
    plan = plan if plan is not None else plan_fast(n, prm.l, prm.s, prm.seed)
    return ShardedFast(backend, x_local, plan, prm.r, comm).launch().finish()


def local_rows(algo: str, plan, n: int, world: int, rank: int) -> np.ndarray:
    """Global row ids of the local matrix rank `rank` needs, in order."""
    if algo == "divide":
        return dc_shard(plan, world, rank).local_rows
    if algo == "fast":
        return fast_shard(plan, world, rank).local_rows
    return interp_shard(n, np.asarray(plan, dtype=np.int64), world, rank).local_rows


def to_configuration(res: ShardResult, points) -> MdsConfiguration:
    res.finish()
    return MdsConfiguration(points, res.estimates, res.gof_g1, res.gof_g2)
