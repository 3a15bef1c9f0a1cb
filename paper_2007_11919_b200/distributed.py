"""Multi-GPU sharding of the partition algorithms.

One process per GPU (``torchrun``), ``torch.distributed`` for the plumbing
(NCCL on GPUs; gloo in the CPU tests).  Every rank holds the input (replicated
once, outside any timed region) and the plan (drawn bit-exactly on every rank
from the same seed), so the only exchanges are small:

* divide-and-conquer: every rank solves the anchor piece (subset 1) itself and
  its contiguous share of subsets 2..p, aligns them locally (the anchor is
  known everywhere — no broadcast needed), and writes their rows of the n x r
  output.  Per-subset column sums of the owned rows and per-subset fit figures
  are all-gathered and combined in plan order, so the re-centring shift and
  G1/G2/estimates are identical on every rank and independent of the number
  of ranks.
* fast: the root's level-1 subtrees are dealt to ranks (contiguous blocks);
  every rank solves its subtrees completely (leaves, alignment sets, internal
  alignments) and the root's alignment set (samples of ALL children, raw
  rows — computed redundantly, no broadcast needed), aligns its children onto
  their slices of it, and writes their rows.  Per-child column sums and fit
  figures are all-gathered and combined in child order (the reference's
  recursion, algorithms.py:314-320).
* interpolation: rank 0 computes the landmark MDS and Gower context and
  broadcasts it (the north star's "computed once and broadcast"); each rank
  streams a contiguous block of rows; per-block column sums are all-gathered
  (fixed 65 536-row blocks, plan order) for the re-centring.

The per-rank compute is behind a small backend interface: ``GpuBackend``
(libmdsx kernels, the product) and, for the CPU tests only, an oracle-backed
backend in ``tests/``.  ``gather_points`` assembles the full n x r result on
rank 0 (outside the timed region in bench.py).
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .params import AlgorithmParams
from .plans import (DcPlan, FastPlan, flatten_fast_shard, flatten_subsets, interpolation_sample,
                    plan_divide_conquer, plan_fast)

SUM_BLOCK = 65536      # canonical row block of the interpolation re-centring sums


def shard(count: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split of range(count): [lo, hi) for `rank`."""
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class ShardResult:
    """One rank's share of a sharded run.  `rows` (global row indices, input
    order) and `local` (their positions in `out`) may be given as arrays or
    as (lo, hi) ranges, materialised only when asked for (gather time)."""

    def __init__(self, rows, out, local, estimates, gof_g1, gof_g2, backend=None):
        self._rows, self._local = rows, local
        self.out = out
        self.estimates = estimates
        self.gof_g1, self.gof_g2 = gof_g1, gof_g2
        self.backend = backend

    @staticmethod
    def _arr(v):
        if isinstance(v, tuple):
            return np.arange(v[0], v[1], dtype=np.int64)
        return v() if callable(v) else v

    @property
    def rows(self) -> np.ndarray:
        return self._arr(self._rows)

    @property
    def local(self) -> np.ndarray:
        return self._arr(self._local)

    def points(self) -> np.ndarray:
        """(len(rows), r) float64 on the host."""
        if isinstance(self._local, tuple) and self._local[0] == 0 and \
                self._local[1] == self.out.shape[0]:
            return self.backend.take_all(self.out)
        return self.backend.take(self.out, self.local)


class Comm:
    """Collectives used by the sharded algorithms (a torch.distributed group)."""

    def __init__(self, group=None, device=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device if device is not None else torch.device("cpu")

    def allgather(self, arr: np.ndarray) -> list:
        """All-gather equally shaped float64 arrays -> list in rank order."""
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(self.device)
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.group)
        return [o.cpu().numpy() for o in out]

    def allgather_ragged(self, arr: np.ndarray) -> list:
        """All-gather float64 arrays of different leading sizes (padded)."""
        arr = np.ascontiguousarray(arr, dtype=np.float64)
        n = np.array([arr.shape[0]], dtype=np.float64)
        sizes = [int(s[0]) for s in self.allgather(n)]
        width = int(np.prod(arr.shape[1:])) if arr.ndim > 1 else 1
        pad = np.zeros((max(sizes), width))
        pad[:arr.shape[0]] = arr.reshape(arr.shape[0], width)
        parts = self.allgather(pad)
        return [p[:s].reshape((s,) + arr.shape[1:]) for p, s in zip(parts, sizes)]

    def broadcast(self, arr: np.ndarray, src: int = 0) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).to(self.device)
        dist.broadcast(t, src=src, group=self.group)
        return t.cpu().numpy()


# ------------------------------------------------------------------ GPU backend
class GpuBackend:
    """Per-rank compute on the rank's GPU through the C-ABI."""

    def __init__(self, x: torch.Tensor, reuse: bool = False):
        """reuse=True: keep the per-plan setup (flattened sub-plans, uploaded
        index arrays, result buffers) across calls with the same plan, as the
        single-GPU runners do (results of a call are overwritten by the next)."""
        from . import _device as D
        self.D = D
        self.x = x
        self.dev = x.device
        self.reuse = reuse
        self._cache = {}

    def dc_subplan(self, subsets: list, c: int, r: int, key=None):
        """D&C of a sub-plan (anchor first) without re-centring -> (out_dev, est, gof, status)."""
        D, x = self.D, self.x
        ck = ("dc", key, c, r)
        if self.reuse and key is not None and ck in self._cache:
            ridx, off, out, est, gof, st, own = self._cache[ck]
            self._own = own                 # every owned row is rewritten: no clearing pass
            return self._run_dc(ridx, off, c, r, out, est, gof, st)
        rows, off = flatten_subsets(subsets)
        ridx = D.index_tensor(rows, self.dev)
        npc = len(subsets)
        out = torch.zeros((x.shape[0], r), dtype=torch.float64, device=self.dev)
        est = D.empty((npc, r), self.dev)
        gof = D.empty((npc, 2), self.dev)
        st = D.status_tensor(npc, self.dev)
        # rows each subset contributes (anchor: all; others: own rows) as device
        # index segments carved from the uploaded plan indices (no second upload)
        keep = np.ones(int(off[-1]), dtype=bool)
        for j in range(1, npc):
            keep[off[j]:off[j] + c] = False
        own = ridx[torch.from_numpy(keep).to(self.dev)]
        sizes = np.diff(off) - np.r_[0, np.full(npc - 1, c)]
        own_off = np.zeros(npc + 1, dtype=np.int64)
        np.cumsum(sizes, out=own_off[1:])
        self._own = (own, own_off,
                     torch.from_numpy(np.ascontiguousarray(own_off)).to(self.dev))
        if self.reuse and key is not None:
            self._cache[ck] = (ridx, off, out, est, gof, st, self._own)
        return self._run_dc(ridx, off, c, r, out, est, gof, st)

    def _run_dc(self, ridx, off, c, r, out, est, gof, st):
        D, x = self.D, self.x
        npc = len(off) - 1
        D.handle(self.dev).call(
            "mdsx_divide_conquer_ex", x.data_ptr(), D.dtype_code(x), x.shape[1], x.shape[0],
            x.shape[1], ridx.data_ptr(), off.ctypes.data, npc, c, r, out.data_ptr(),
            est.data_ptr(), gof.data_ptr(), st.data_ptr(), 1, D.stream_ptr(self.dev))
        return out, est.cpu().numpy(), gof.cpu().numpy(), D.decode_status(st)

    def own_segment_sums(self, out, r: int) -> np.ndarray:
        """Column sums of each dc_subplan subset's own rows (fixed order)."""
        own, own_off, own_off_dev = self._own
        return self._segsums(out, own.data_ptr(), own_off, r, own_off_dev)

    def shift_own(self, out, mean: np.ndarray) -> None:
        own = self._own[0]
        self._shift(out, own.data_ptr(), own.numel(), mean)

    def range_sums(self, out, offsets: np.ndarray, r: int) -> np.ndarray:
        """Column sums of the contiguous row ranges [offsets[j], offsets[j+1]) of out."""
        return self._segsums(out, None, offsets, r)

    def shift_all(self, out, mean: np.ndarray) -> None:
        self._shift(out, None, out.shape[0], mean)

    def _segsums(self, out, idx_ptr, offsets, r, doff=None):
        D = self.D
        nseg = len(offsets) - 1
        sums = D.empty((max(nseg, 1), r), self.dev)
        if nseg > 0:
            if doff is None:
                doff = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).to(self.dev)
            D.handle(self.dev).call("mdsx_segment_colsums", out.data_ptr(), idx_ptr,
                                    doff.data_ptr(), nseg, r, sums.data_ptr(),
                                    D.stream_ptr(self.dev))
        return sums.cpu().numpy()[:nseg]

    def _shift(self, out, idx_ptr, n, mean):
        D = self.D
        m = torch.from_numpy(np.ascontiguousarray(mean, dtype=np.float64)).to(self.dev)
        D.handle(self.dev).call("mdsx_shift_rows", out.data_ptr(), idx_ptr, n, out.shape[1],
                                m.data_ptr(), D.stream_ptr(self.dev))

    def fast_subtrees(self, plan: FastPlan, lo: int, hi: int, r: int, key=None):
        """One rank's share of fast MDS (plans.flatten_fast_shard), aligned,
        not re-centred -> (out_dev (rows in flat.order), flat, est, gof, status)."""
        from .algorithms import FastRun
        D = self.D
        ck = ("fast", key, lo, hi, r)
        run = self._cache.get(ck) if self.reuse and key is not None else None
        if run is None:
            flat = flatten_fast_shard(plan, lo, hi)
            run = FastRun(self.x, plan, r, flat=flat, local=True)
            if self.reuse and key is not None:
                self._cache[ck] = run
        flat = run.flat
        run.launch()
        out = run.pts[:len(flat.order)]
        return out, flat, run.est.cpu().numpy(), run.gof.cpu().numpy(), D.decode_status(run.status)

    def segment_sums(self, out, segments: list, r: int) -> np.ndarray:
        D = self.D
        rows, off = flatten_subsets(segments)
        ridx = D.index_tensor(rows, self.dev)
        doff = D.index_tensor(off, self.dev)
        sums = D.empty((len(segments), r), self.dev)
        D.handle(self.dev).call("mdsx_segment_colsums", out.data_ptr(), ridx.data_ptr(),
                                doff.data_ptr(), len(segments), r, sums.data_ptr(),
                                D.stream_ptr(self.dev))
        return sums.cpu().numpy()

    def shift(self, out, rows: np.ndarray, mean: np.ndarray) -> None:
        D = self.D
        ridx = D.index_tensor(rows, self.dev)
        m = torch.from_numpy(np.ascontiguousarray(mean)).to(self.dev)
        D.handle(self.dev).call("mdsx_shift_rows", out.data_ptr(), ridx.data_ptr(), len(rows),
                                out.shape[1], m.data_ptr(), D.stream_ptr(self.dev))

    def take(self, out, rows: np.ndarray) -> np.ndarray:
        return out[self.D.index_tensor(rows, self.dev)].cpu().numpy()

    def take_all(self, out) -> np.ndarray:
        return self.D.to_host(out)

    def place(self, out, local: np.ndarray, values: np.ndarray) -> None:
        """out[local[i]] = values[i] (mdsx_scatter_rows)."""
        if len(local) == 0:
            return
        D = self.D
        src = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64)).to(self.dev)
        D.handle(self.dev).call("mdsx_scatter_rows", src.data_ptr(),
                                D.index_tensor(local, self.dev).data_ptr(), len(local),
                                out.shape[1], out.data_ptr(), D.stream_ptr(self.dev))

    # interpolation pieces -------------------------------------------------
    def landmark_context(self, sample: np.ndarray, r: int):
        """Classical MDS of the sample + Gower context, flattened for broadcast."""
        from .primitives import classical_pieces, raise_piece_status
        D, x = self.D, self.x
        idx = D.index_tensor(sample, self.dev)
        pts, est, gof, st = classical_pieces(x, idx, np.array([0, len(sample)], np.int64), r)
        raise_piece_status(D.decode_status(st)[0], r, "sample subset")
        h = D.handle(self.dev)
        l, p = len(sample), x.shape[1]
        size = int(h.lib.mdsx_gower_context_size(l, p, r))
        ctx = D.empty((size,), self.dev)
        cond = D.empty((1,), self.dev)
        flag = torch.zeros(1, dtype=torch.int32, device=self.dev)
        h.call("mdsx_gower_context", x.data_ptr(), D.dtype_code(x), p, p, idx.data_ptr(), l,
               pts.data_ptr(), r, ctx.data_ptr(), cond.data_ptr(), flag.data_ptr(),
               D.stream_ptr(self.dev))
        if int(flag.item()):
            from .errors import NumericalError
            raise NumericalError("base covariance is ill-conditioned or not positive definite")
        g = gof.cpu().numpy()[0]
        return (np.concatenate([ctx.cpu().numpy(), pts.cpu().numpy().ravel()]),
                est.cpu().numpy()[0], float(g[0]), float(g[1]))

    def _cached_index(self, key, arr: np.ndarray):
        ck = ("idx", key)
        if ck not in self._cache:
            self._cache[ck] = self.D.index_tensor(arr, self.dev)
        return self._cache[ck]

    def landmark_context_dev(self, sample: np.ndarray, r: int):
        """landmark_context kept on the device: (head, check) with head =
        [g1, g2, est(r), context, landmark configuration] as one device vector
        (broadcast as is) and check() raising the deferred failures."""
        from .primitives import classical_pieces, raise_piece_status
        D, x = self.D, self.x
        idx = self._cached_index(("sample", id(sample)), sample)
        pts, est, gof, st = classical_pieces(x, idx, np.array([0, len(sample)], np.int64), r)
        h = D.handle(self.dev)
        l, p = len(sample), x.shape[1]
        size = int(h.lib.mdsx_gower_context_size(l, p, r))
        head = D.empty((2 + r + size + l * r,), self.dev)
        cond = D.empty((1,), self.dev)
        flag = torch.zeros(1, dtype=torch.int32, device=self.dev)
        h.call("mdsx_gower_context", x.data_ptr(), D.dtype_code(x), p, p, idx.data_ptr(), l,
               pts.data_ptr(), r, head[2 + r:].data_ptr(), cond.data_ptr(), flag.data_ptr(),
               D.stream_ptr(self.dev))
        head[0:2] = gof[0]
        head[2:2 + r] = est[0]
        head[2 + r + size:] = pts.reshape(-1)

        def check():
            raise_piece_status(D.decode_status(st)[0], r, "sample subset")
            if int(flag.item()):
                from .errors import NumericalError
                raise NumericalError("base covariance is ill-conditioned or not positive definite")
        return head, check

    def gower_rows_dev(self, head, l: int, r: int, lo: int, hi: int):
        D, x = self.D, self.x
        p = x.shape[1]
        h = D.handle(self.dev)
        rows = x[lo:hi]
        out = D.empty((hi - lo, r), self.dev)
        nf = torch.zeros(1, dtype=torch.int32, device=self.dev)
        h.call("mdsx_gower_interpolate", head[2 + r:].data_ptr(), l, p, r, rows.data_ptr(),
               D.dtype_code(x), p, hi - lo, out.data_ptr(), r, nf.data_ptr(),
               D.stream_ptr(self.dev))
        return out

    def place_dev(self, out, key, local: np.ndarray, values_dev) -> None:
        """out[local[i]] = values_dev[i] with the index upload cached under key."""
        if len(local) == 0:
            return
        D = self.D
        li = self._cached_index(key, local)
        D.handle(self.dev).call("mdsx_scatter_rows", values_dev.data_ptr(), li.data_ptr(),
                                len(local), out.shape[1], out.data_ptr(), D.stream_ptr(self.dev))

    def gower_rows(self, packed: np.ndarray, l: int, r: int, lo: int, hi: int):
        D, x = self.D, self.x
        p = x.shape[1]
        h = D.handle(self.dev)
        size = int(h.lib.mdsx_gower_context_size(l, p, r))
        ctx = torch.from_numpy(np.ascontiguousarray(packed[:size])).to(self.dev)
        rows = x[lo:hi]
        out = D.empty((hi - lo, r), self.dev)
        nf = torch.zeros(1, dtype=torch.int32, device=self.dev)
        h.call("mdsx_gower_interpolate", ctx.data_ptr(), l, p, r, rows.data_ptr(),
               D.dtype_code(x), p, hi - lo, out.data_ptr(), r, nf.data_ptr(),
               D.stream_ptr(self.dev))
        return out


# ------------------------------------------------------------------ algorithms
def fold_rows(rows: np.ndarray, r: int) -> np.ndarray:
    """Left fold (((0 + s_0) + s_1) + ...) of the rows in the given order: a
    sequential running sum, identical on every rank and for every world size
    (np.add.reduce would pair them up instead)."""
    if len(rows) == 0:
        return np.zeros(r)
    return np.cumsum(np.asarray(rows, dtype=np.float64), axis=0)[-1]


def sharded_divide_and_conquer(backend, n: int, params: AlgorithmParams, comm: Comm,
                               plan: DcPlan | None = None) -> ShardResult:
    """divide_and_conquer_mds (algorithms.py:128-172) over comm.world ranks."""
    prm = params.resolved("divide")
    plan = plan if plan is not None else plan_divide_conquer(n, prm.l, prm.c, prm.seed)
    P, c, r = plan.p, prm.c, prm.r
    lo, hi = shard(P - 1, comm.world, comm.rank)
    mine = list(range(1 + lo, 1 + hi))                    # owned subsets besides the anchor
    out, est, gof, st = backend.dc_subplan([plan.subsets[0]] + [plan.subsets[j] for j in mine], c, r,
                                           key=(id(plan), lo, hi))
    from .primitives import raise_piece_status
    if np.any(st["code"] == 3):
        from .errors import InvalidInputError
        raise InvalidInputError("data contains non-finite values")
    labels = [0] + mine
    bad = np.flatnonzero(st["code"] != 0)
    if bad.size:                                          # first failing subset in plan order
        raise_piece_status(st[bad[0]], r, f"subset {labels[bad[0]] + 1}")
    # rows each subset contributes (anchor: all its rows; others: own rows)
    own = [plan.subsets[0]] + [plan.subsets[j][c:] for j in mine]
    sums = backend.own_segment_sums(out, r)              # (1 + len(mine), r)
    # plan-order all-gather of per-subset sums and fit figures
    width = 3 + 2 * r                                    # [j, g1, g2, est(r), sums(r)]
    recs = np.zeros((len(mine), width))
    recs[:, 0] = mine
    recs[:, 1:3] = gof[1:1 + len(mine)]
    recs[:, 3:3 + r] = est[1:1 + len(mine)]
    recs[:, 3 + r:3 + 2 * r] = sums[1:1 + len(mine)]
    allrecs = np.concatenate(comm.allgather_ragged(recs)) if comm.world > 1 else recs
    allrecs = allrecs[np.argsort(allrecs[:, 0], kind="stable")]
    seg_sums = np.vstack([sums[0:1], allrecs[:, 3 + r:3 + 2 * r]])
    total = fold_rows(seg_sums, r)                        # plan order
    mean = total / n
    backend.shift_own(out, mean)
    sizes = np.fromiter((len(q) for q in plan.subsets), dtype=np.float64, count=P)
    weights = sizes.copy()
    weights[1:] -= c                                      # algorithms.py:158-166
    g1s = np.concatenate([gof[0:1, 0], allrecs[:, 1]])
    g2s = np.concatenate([gof[0:1, 1], allrecs[:, 2]])
    ests = np.vstack([est[0:1], allrecs[:, 3:3 + r]])
    g1 = float(np.dot(weights, g1s) / n)
    g2 = float(np.dot(weights, g2s) / n)
    per = ests * (sizes / weights)[:, None]
    # the anchor's rows belong to rank 0; index lists built only when gathered
    parts = own if comm.rank == 0 else own[1:]
    rows = (lambda: np.concatenate(parts)) if parts else np.empty(0, np.int64)
    return ShardResult(rows, out, rows, per.mean(axis=0), g1, g2, backend)


def sharded_fast(backend, n: int, params: AlgorithmParams, comm: Comm,
                 plan: FastPlan | None = None) -> ShardResult:
    """fast_mds (algorithms.py:285-348) over comm.world ranks."""
    from .errors import InvalidInputError
    from .primitives import raise_piece_status
    prm = params.resolved("fast")
    r = prm.r
    plan = plan if plan is not None else plan_fast(n, prm.l, prm.s, prm.seed)
    if plan.root.is_leaf:                                 # n <= l: classical MDS (algorithms.py:337-338)
        out, est, gof, st = backend.dc_subplan([plan.root.indices], 1, r)
        raise_piece_status(st[0], r, "leaf 1")
        rows = plan.root.indices if comm.rank == 0 else np.empty(0, np.int64)
        return ShardResult(rows, out, rows, est[0], float(gof[0, 0]), float(gof[0, 1]), backend)
    kids = plan.root.children
    lo, hi = shard(len(kids), comm.world, comm.rank)
    out, flat, est, gof, st = backend.fast_subtrees(plan, lo, hi, r, key=id(plan))
    # failures: a consistent decision on every rank (all raise, no rank hangs)
    root_pid = len(flat.piece_off) - 2                    # the root alignment set, evaluated last
    ev = np.asarray(flat.eval_order, dtype=np.int64)
    bad = np.flatnonzero((ev != root_pid) & (st["code"][ev] != 0))
    first = int(bad[0]) if bad.size else -1
    flags = np.array([float(np.any(st["code"] == 3)), float(first >= 0)])
    allflags = np.vstack(comm.allgather(flags)) if comm.world > 1 else flags[None]
    if allflags[:, 0].any():
        raise InvalidInputError("data contains non-finite values")
    if allflags[:, 1].any():
        culprit = int(np.flatnonzero(allflags[:, 1])[0])
        if culprit == comm.rank:
            pid = flat.eval_order[first]
            raise_piece_status(st[pid], r, flat.labels[pid])
        raise RuntimeError(f"fast MDS failed on rank {culprit}")
    raise_piece_status(st[root_pid], r, flat.labels[root_pid])
    # per-child aggregates of the owned subtrees (algorithms.py:289-320); a node
    # whose children are all leaves is reduced with array ops over its leaf range
    leaf = [0]

    def agg(node):
        if node.is_leaf:
            j = leaf[0]
            leaf[0] += 1
            return gof[j, 0], gof[j, 1], est[j], node.size
        kids_ = node.children
        if all(ch.is_leaf for ch in kids_):
            j0 = leaf[0]
            leaf[0] += len(kids_)
            sizes = np.array([ch.size for ch in kids_], dtype=np.float64)
            tot = sizes.sum()
            return (float(np.dot(sizes, gof[j0:leaf[0], 0]) / tot),
                    float(np.dot(sizes, gof[j0:leaf[0], 1]) / tot),
                    est[j0:leaf[0]].mean(axis=0), int(tot))
        fits = [agg(ch) for ch in kids_]
        sizes = np.array([f[3] for f in fits], dtype=np.float64)
        tot = sizes.sum()
        return (float(np.dot(sizes, [f[0] for f in fits]) / tot),
                float(np.dot(sizes, [f[1] for f in fits]) / tot),
                np.stack([f[2] for f in fits]).mean(axis=0), int(tot))

    mine = kids[lo:hi]
    shape = _fast_shape(plan, mine, backend)
    if shape is not None:                                 # two-level subtrees: array ops only
        owner, lsize = shape
        starts_l = np.searchsorted(owner, np.arange(len(mine) + 1))
        g1c, g2c = np.ascontiguousarray(gof[:, 0]), np.ascontiguousarray(gof[:, 1])
        fits = [(float(np.dot(lsize[a:b], g1c[a:b]) / lsize[a:b].sum()),
                 float(np.dot(lsize[a:b], g2c[a:b]) / lsize[a:b].sum()),
                 est[a:b].mean(axis=0), int(lsize[a:b].sum()))
                for a, b in zip(starts_l[:-1], starts_l[1:])]
    else:
        fits = [agg(ch) for ch in mine]
    starts = np.cumsum([0] + [ch.size for ch in mine]).astype(np.int64)
    sums = backend.range_sums(out, starts, r)
    width = 4 + 2 * r                                     # [i, g1, g2, size, est(r), sums(r)]
    recs = np.zeros((len(mine), width))
    if fits:
        recs[:, 0] = np.arange(lo, lo + len(mine))
        recs[:, 1] = [f[0] for f in fits]
        recs[:, 2] = [f[1] for f in fits]
        recs[:, 3] = [f[3] for f in fits]
        recs[:, 4:4 + r] = np.stack([f[2] for f in fits])
        recs[:, 4 + r:] = sums[:len(mine)]
    allrecs = np.concatenate(comm.allgather_ragged(recs)) if comm.world > 1 else recs
    allrecs = allrecs[np.argsort(allrecs[:, 0], kind="stable")]
    sizes = allrecs[:, 3]
    tot = sizes.sum()
    g1 = float(np.dot(sizes, allrecs[:, 1]) / tot)
    g2 = float(np.dot(sizes, allrecs[:, 2]) / tot)
    estimates = allrecs[:, 4:4 + r].mean(axis=0)
    total = fold_rows(allrecs[:, 4 + r:], r)              # child order
    backend.shift_all(out, total / n)
    return ShardResult(flat.order, out, (0, len(flat.order)), estimates, g1, g2, backend)


def _fast_shape(plan, mine, backend):
    """For subtrees whose children are all leaves (the BASELINE fast plans):
    (child index of every leaf in DFS order, leaf sizes), cached per plan on
    the backend; None for deeper trees."""
    cache = getattr(backend, "_fast_shape_cache", None)
    if cache is None:
        cache = backend._fast_shape_cache = {}
    key = (id(plan), id(mine[0]) if mine else 0, len(mine))
    if key not in cache:
        if not mine or not all(not ch.is_leaf and all(g.is_leaf for g in ch.children)
                               for ch in mine):
            cache[key] = None
        else:
            owner = np.concatenate([np.full(len(ch.children), t, np.int64)
                                    for t, ch in enumerate(mine)])
            lsize = np.array([g.size for ch in mine for g in ch.children], dtype=np.float64)
            cache[key] = (owner, lsize)
    return cache[key]


def sharded_interpolation(backend, n: int, params: AlgorithmParams, comm: Comm,
                          sample: np.ndarray | None = None) -> ShardResult:
    """interpolation_mds (algorithms.py:245-274) over comm.world ranks."""
    prm = params.resolved("interpolate")
    r, l = prm.r, prm.l
    sample = sample if sample is not None else interpolation_sample(n, l, prm.seed)
    l = len(sample)
    blocks = (n + SUM_BLOCK - 1) // SUM_BLOCK
    b_lo, b_hi = shard(blocks, comm.world, comm.rank)
    lo, hi = b_lo * SUM_BLOCK, min(n, b_hi * SUM_BLOCK)
    in_shard = (sample >= lo) & (sample < hi)
    if hasattr(backend, "landmark_context_dev"):
        # device-resident: the context is computed on rank 0 and broadcast as a
        # device vector (no host round trip inside the step)
        check = None
        if comm.rank == 0:
            head_dev, check = backend.landmark_context_dev(sample, r)
        else:
            size = backend_context_len(backend, l, r) + 2 + r
            head_dev = torch.zeros(size, dtype=torch.float64, device=backend.dev)
        if comm.world > 1:
            dist.broadcast(head_dev, src=0, group=comm.group)
        out = backend.gower_rows_dev(head_dev, l, r, lo, hi)
        base_dev = head_dev[-l * r:].reshape(l, r)
        if in_shard.all():
            vals = base_dev
        else:
            sel = backend._cached_index(("insel", id(sample), lo, hi), np.flatnonzero(in_shard))
            vals = base_dev.index_select(0, sel)
        backend.place_dev(out, ("local", id(sample), lo, hi), (sample[in_shard] - lo).astype(np.int64),
                          vals)
        if check is not None:
            check()
        head_small = head_dev[:2 + r].cpu().numpy()
        g1, g2, est = float(head_small[0]), float(head_small[1]), head_small[2:2 + r]
    else:
        if comm.rank == 0:
            packed, est, g1, g2 = backend.landmark_context(sample, r)
            head = np.concatenate([[g1, g2], est, packed])
        else:
            size = backend_context_len(backend, l, r) + 2 + r
            head = np.zeros(size)
        head = comm.broadcast(head, src=0) if comm.world > 1 else head
        g1, g2, est, packed = float(head[0]), float(head[1]), head[2:2 + r], head[2 + r:]
        base = packed[-l * r:].reshape(l, r)
        out = backend.gower_rows(packed, l, r, lo, hi)        # (hi - lo) x r, shard-local rows
        # landmark rows inside the shard take the classical configuration
        backend.place(out, (sample[in_shard] - lo).astype(np.int64), base[in_shard])
    bounds = np.minimum(hi, np.arange(b_lo, b_hi + 1, dtype=np.int64) * SUM_BLOCK) - lo
    sums = backend.range_sums(out, bounds, r)
    recs = np.hstack([np.arange(b_lo, b_hi, dtype=np.float64)[:, None], sums])
    allrecs = np.concatenate(comm.allgather_ragged(recs)) if comm.world > 1 else recs
    allrecs = allrecs[np.argsort(allrecs[:, 0], kind="stable")]
    total = fold_rows(allrecs[:, 1:], r)                  # canonical block order
    backend.shift_all(out, total / n)
    return ShardResult((lo, hi), out, (0, hi - lo), est, g1, g2, backend)


def backend_context_len(backend, l: int, r: int) -> int:
    return backend.context_len(l, r) if hasattr(backend, "context_len") else \
        _gpu_context_len(backend, l, r)


def _gpu_context_len(backend, l: int, r: int) -> int:
    h = backend.D.handle(backend.dev)
    return int(h.lib.mdsx_gower_context_size(l, backend.x.shape[1], r)) + l * r


def gather_points(res: ShardResult, n: int, r: int, comm: Comm) -> np.ndarray | None:
    """Assemble the full n x r configuration on rank 0 (None elsewhere)."""
    block = np.hstack([res.rows[:, None].astype(np.float64), res.points()])
    parts = comm.allgather_ragged(block) if comm.world > 1 else [block]
    if comm.rank != 0:
        return None
    out = np.empty((n, r))
    for part in parts:
        out[part[:, 0].astype(np.int64)] = part[:, 1:]
    return out
