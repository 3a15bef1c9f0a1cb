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

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .params import AlgorithmParams
from .plans import DcPlan, flatten_subsets, interpolation_sample, plan_divide_conquer

SUM_BLOCK = 65536      # canonical row block of the interpolation re-centring sums


def shard(count: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split of range(count): [lo, hi) for `rank`."""
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


@dataclass
class ShardResult:
    rows: np.ndarray            # global row indices this rank owns (input order)
    out: object                 # backend buffer holding those rows (device tensor on GPU)
    local: np.ndarray           # positions of `rows` inside `out`
    estimates: np.ndarray
    gof_g1: float
    gof_g2: float
    backend: object = None

    def points(self) -> np.ndarray:
        """(len(rows), r) float64 on the host."""
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

    def __init__(self, x: torch.Tensor):
        from . import _device as D
        self.D = D
        self.x = x
        self.dev = x.device

    def dc_subplan(self, subsets: list, c: int, r: int):
        """D&C of a sub-plan (anchor first) without re-centring -> (out_dev, est, gof, status)."""
        D, x = self.D, self.x
        rows, off = flatten_subsets(subsets)
        ridx = D.index_tensor(rows, self.dev)
        npc = len(subsets)
        out = torch.zeros((x.shape[0], r), dtype=torch.float64, device=self.dev)
        est = D.empty((npc, r), self.dev)
        gof = D.empty((npc, 2), self.dev)
        st = D.status_tensor(npc, self.dev)
        D.handle(self.dev).call(
            "mdsx_divide_conquer_ex", x.data_ptr(), D.dtype_code(x), x.shape[1], x.shape[0],
            x.shape[1], ridx.data_ptr(), off.ctypes.data, npc, c, r, out.data_ptr(),
            est.data_ptr(), gof.data_ptr(), st.data_ptr(), 1, D.stream_ptr(self.dev))
        return out, est.cpu().numpy(), gof.cpu().numpy(), D.decode_status(st)

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
def sharded_divide_and_conquer(backend, n: int, params: AlgorithmParams, comm: Comm,
                               plan: DcPlan | None = None) -> ShardResult:
    """divide_and_conquer_mds (algorithms.py:128-172) over comm.world ranks."""
    prm = params.resolved("divide")
    plan = plan if plan is not None else plan_divide_conquer(n, prm.l, prm.c, prm.seed)
    P, c, r = plan.p, prm.c, prm.r
    lo, hi = shard(P - 1, comm.world, comm.rank)
    mine = list(range(1 + lo, 1 + hi))                    # owned subsets besides the anchor
    out, est, gof, st = backend.dc_subplan([plan.subsets[0]] + [plan.subsets[j] for j in mine], c, r)
    from .primitives import raise_piece_status
    if np.any(st["code"] == 3):
        from .errors import InvalidInputError
        raise InvalidInputError("data contains non-finite values")
    labels = [0] + mine
    for rec, j in zip(st, labels):
        raise_piece_status(rec, r, f"subset {j + 1}")
    # rows each subset contributes (anchor: all its rows; others: own rows)
    own = [plan.subsets[0]] + [plan.subsets[j][c:] for j in mine]
    sums = backend.segment_sums(out, own, r)             # (1 + len(mine), r)
    # plan-order all-gather of per-subset sums and fit figures
    width = 3 + 2 * r                                    # [j, g1, g2, est(r), sums(r)]
    recs = np.zeros((len(mine), width))
    for t, j in enumerate(mine):
        recs[t, 0] = j
        recs[t, 1:3] = gof[1 + t]
        recs[t, 3:3 + r] = est[1 + t]
        recs[t, 3 + r:3 + 2 * r] = sums[1 + t]
    allrecs = np.concatenate(comm.allgather_ragged(recs)) if comm.world > 1 else recs
    allrecs = allrecs[np.argsort(allrecs[:, 0], kind="stable")]
    seg_sums = np.vstack([sums[0:1], allrecs[:, 3 + r:3 + 2 * r]])
    total = np.zeros(r)
    for row in seg_sums:                                  # plan order
        total = total + row
    mean = total / n
    rows = np.concatenate(own)
    backend.shift(out, rows, mean)
    sizes = np.array([len(q) for q in plan.subsets], dtype=np.float64)
    weights = sizes.copy()
    weights[1:] -= c                                      # algorithms.py:158-166
    g1s = np.concatenate([gof[0:1, 0], allrecs[:, 1]])
    g2s = np.concatenate([gof[0:1, 1], allrecs[:, 2]])
    ests = np.vstack([est[0:1], allrecs[:, 3:3 + r]])
    g1 = float(np.dot(weights, g1s) / n)
    g2 = float(np.dot(weights, g2s) / n)
    per = np.stack([ests[j] * (sizes[j] / weights[j]) for j in range(P)])
    if comm.rank != 0:                                    # the anchor's rows belong to rank 0
        rows = np.concatenate(own[1:]) if len(own) > 1 else np.empty(0, np.int64)
    return ShardResult(rows, out, rows, per.mean(axis=0), g1, g2, backend)


def sharded_interpolation(backend, n: int, params: AlgorithmParams, comm: Comm,
                          sample: np.ndarray | None = None) -> ShardResult:
    """interpolation_mds (algorithms.py:245-274) over comm.world ranks."""
    prm = params.resolved("interpolate")
    r, l = prm.r, prm.l
    sample = sample if sample is not None else interpolation_sample(n, l, prm.seed)
    l = len(sample)
    if comm.rank == 0:
        packed, est, g1, g2 = backend.landmark_context(sample, r)
        head = np.concatenate([[g1, g2], est, packed])
    else:
        size = backend_context_len(backend, l, r) + 2 + r
        head = np.zeros(size)
    head = comm.broadcast(head, src=0) if comm.world > 1 else head
    g1, g2, est, packed = float(head[0]), float(head[1]), head[2:2 + r], head[2 + r:]
    base = packed[-l * r:].reshape(l, r)
    blocks = (n + SUM_BLOCK - 1) // SUM_BLOCK
    b_lo, b_hi = shard(blocks, comm.world, comm.rank)
    lo, hi = b_lo * SUM_BLOCK, min(n, b_hi * SUM_BLOCK)
    out = backend.gower_rows(packed, l, r, lo, hi)        # (hi - lo) x r, shard-local rows
    # landmark rows inside the shard take the classical configuration
    in_shard = (sample >= lo) & (sample < hi)
    backend.place(out, (sample[in_shard] - lo).astype(np.int64), base[in_shard])
    local = np.arange(hi - lo, dtype=np.int64)
    segs = [local[s * SUM_BLOCK - lo:min(hi, (s + 1) * SUM_BLOCK) - lo] for s in range(b_lo, b_hi)]
    sums = backend.segment_sums(out, segs, r) if segs else np.zeros((0, r))
    recs = np.hstack([np.arange(b_lo, b_hi, dtype=np.float64)[:, None], sums])
    allrecs = np.concatenate(comm.allgather_ragged(recs)) if comm.world > 1 else recs
    allrecs = allrecs[np.argsort(allrecs[:, 0], kind="stable")]
    total = np.zeros(r)
    for row in allrecs[:, 1:]:                            # canonical block order
        total = total + row
    backend.shift(out, local, total / n)
    return ShardResult(np.arange(lo, hi, dtype=np.int64), out, local, est, g1, g2, backend)


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
