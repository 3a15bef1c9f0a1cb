"""The three partition-based MDS algorithms on the GPU — drop-in for
``interpolation_mds``, ``divide_and_conquer_mds``, ``fast_mds`` and
``run_algorithm`` (algorithms.py:128-363): same names, positional arguments,
defaults, results and exceptions.  Extra keyword-only arguments:

  device=        CUDA device (default: current)
  plan=          explicit plan (DcPlan / InterpPlan / FastPlan) instead of
                 drawing one from params.seed
  return_device= keep ``points`` as a CUDA tensor (no D2H copy)
  threads=       accepted and ignored (results never depend on it)

Each algorithm is split into prepare (plan flattening, H2D of indices),
launch (pure device work, no host sync — what bench.py times) and finish
(one small D2H read of statuses/fit figures, error mapping, host-side
aggregation of per-piece G1/G2/estimates in plan order).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from .errors import InvalidInputError, NumericalError, ParamError
from .params import ALGORITHM_NAMES, AlgorithmParams
from .plans import (DcPlan, FastPlan, InterpPlan, flatten_fast_cached, flatten_subsets,
                    flatten_subsets_cached, plan_device_cache, route_cached,
                    interpolation_sample, plan_divide_conquer, plan_fast)
from .primitives import classical_mds_from_data, raise_piece_status
from .results import MdsConfiguration


def _cached_upload(plan, dev, name, make):
    """Device copy of a plan's index arrays, made once per (plan, device) when
    the plan is cached by identity (plans.plan_device_cache); `plan` may also
    be a dict to cache into (a shard's flattened plan)."""
    cache = plan if isinstance(plan, dict) else (
        plan_device_cache(plan) if plan is not None else None)
    if cache is None:
        return make()
    key = (str(dev), name)
    if key not in cache:
        cache[key] = make()
    return cache[key]


def _finish_points(points: torch.Tensor, return_device: bool):
    return points if return_device else D.to_host(points)


# ====================================================================== D&C
class DivideRun:
    """divide_and_conquer_mds (algorithms.py:128-172) with an explicit plan."""

    def __init__(self, x: torch.Tensor, plan: DcPlan, r: int, c: int):
        self.x, self.plan, self.r, self.c = x, plan, r, c
        self.dev = x.device
        self.compact = D.ColumnCompactor(x)
        rows, off = flatten_subsets_cached(plan)
        self.row_idx = _cached_upload(plan, self.dev, "rows", lambda: D.index_tensor(rows, self.dev))
        self.piece_off = off
        n, npc = plan.n, plan.p
        self.out = D.empty((n, r), self.dev)
        self.est = D.empty((npc, r), self.dev)
        self.gof = D.empty((npc, 2), self.dev)
        self.status = D.status_tensor(npc, self.dev)

    def launch(self) -> None:
        x = self.compact()
        D.handle(self.dev).call(
            "mdsx_divide_conquer", x.data_ptr(), D.dtype_code(x), x.shape[1], x.shape[0],
            x.shape[1], self.row_idx.data_ptr(), self.piece_off.ctypes.data, self.plan.p, self.c,
            self.r, self.out.data_ptr(), self.est.data_ptr(), self.gof.data_ptr(),
            self.status.data_ptr(), D.stream_ptr(self.dev))

    def finish(self, return_device: bool = False) -> MdsConfiguration:
        st = D.decode_status(self.status)
        if np.any(st["code"] == 3):
            raise InvalidInputError("data contains non-finite values")
        bad = np.flatnonzero(st["code"] != 0)
        if bad.size:                                      # first failing subset in plan order
            raise_piece_status(st[bad[0]], self.r, f"subset {bad[0] + 1}")
        gof = self.gof.cpu().numpy()
        est = self.est.cpu().numpy()
        n, c = self.plan.n, self.c
        sizes = np.diff(self.piece_off).astype(np.float64)
        weights = sizes.copy()
        weights[1:] -= c                                  # algorithms.py:158-166
        g1 = float(np.dot(weights, gof[:, 0]) / n)
        g2 = float(np.dot(weights, gof[:, 1]) / n)
        per = est * (sizes / weights)[:, None]
        return MdsConfiguration(_finish_points(self.out, return_device), per.mean(axis=0), g1, g2)


def divide_and_conquer_mds(data, params: AlgorithmParams, *, threads=None, device=None,
                           plan: DcPlan | None = None, return_device: bool = False):
    dev = D.require_device(device)
    x = D.to_device_matrix(data, dev)
    prm = params.resolved("divide")
    n = x.shape[0]
    if n <= prm.l:
        return classical_mds_from_data(x, prm.r, device=dev, return_device=return_device)
    plan = plan if plan is not None else plan_divide_conquer(n, prm.l, prm.c, prm.seed)
    run = DivideRun(x, plan, prm.r, prm.c)
    run.launch()
    return run.finish(return_device)


# ============================================================ interpolation
class InterpolationRun:
    """interpolation_mds (algorithms.py:245-274) given the landmark sample."""

    def __init__(self, x: torch.Tensor, sample: np.ndarray, r: int):
        self.x, self.r = x, r
        self.dev = x.device
        self.compact = D.ColumnCompactor(x)
        self.sample = D.index_tensor(sample, self.dev)
        self.l = len(sample)
        self.out = D.empty((x.shape[0], r), self.dev)
        self.est = D.empty((1, r), self.dev)
        self.gof = D.empty((1, 2), self.dev)
        self.status = D.status_tensor(1, self.dev)
        self.cond = D.empty((1,), self.dev)
        self.flags = torch.zeros(2, dtype=torch.int32, device=self.dev)

    def launch(self) -> None:
        x = self.compact()
        D.handle(self.dev).call(
            "mdsx_interpolation", x.data_ptr(), D.dtype_code(x), x.shape[1], x.shape[0],
            x.shape[1], self.sample.data_ptr(), self.l, self.r, self.out.data_ptr(),
            self.est.data_ptr(), self.gof.data_ptr(), self.status.data_ptr(),
            self.cond.data_ptr(), self.flags.data_ptr(), D.stream_ptr(self.dev))

    def finish(self, return_device: bool = False) -> MdsConfiguration:
        flags = self.flags.cpu().numpy()
        st = D.decode_status(self.status)[0]
        if int(st["code"]) == 3 or flags[1]:
            raise InvalidInputError("data contains non-finite values")
        raise_piece_status(st, self.r, "sample subset")
        if flags[0] == 1:
            raise NumericalError(f"base covariance is ill-conditioned (condition estimate "
                                 f"{float(self.cond.item()):.3e}); the requested dimension "
                                 "exceeds the usable rank")
        if flags[0] == 2:
            raise NumericalError("base covariance is not positive definite")
        g = self.gof.cpu().numpy()[0]
        return MdsConfiguration(_finish_points(self.out, return_device),
                                self.est.cpu().numpy()[0], float(g[0]), float(g[1]))


def interpolation_mds(data, params: AlgorithmParams, *, threads=None, device=None,
                      plan: InterpPlan | None = None, return_device: bool = False):
    dev = D.require_device(device)
    x = D.to_device_matrix(data, dev)
    prm = params.resolved("interpolate")
    n = x.shape[0]
    if n <= prm.l:
        return classical_mds_from_data(x, prm.r, device=dev, return_device=return_device)
    sample = plan.subsets[0] if plan is not None else interpolation_sample(n, prm.l, prm.seed)
    run = InterpolationRun(x, sample, prm.r)
    run.launch()
    return run.finish(return_device)


# ==================================================================== fast
class FastRun:
    """fast_mds (algorithms.py:285-348) as three device waves: one batched
    classical-MDS launch over every leaf and alignment set, then per depth
    (deepest first) one batched Procrustes fit + one batched in-place apply,
    then scatter to input order and re-centre."""

    def __init__(self, x: torch.Tensor, plan: FastPlan, r: int, flat=None, local: bool = False):
        """`flat` (plans.flatten_fast_shard) + `local`: run one rank's share of
        sharded fast MDS — no scatter to input order, no re-centring; the
        rank's rows stay in `pts[:len(flat.order)]` (distributed.py)."""
        self.x, self.plan, self.r, self.local = x, plan, r, local
        self.dev = dev = x.device
        self.compact = D.ColumnCompactor(x)
        own_flat = flat is None
        flat = self.flat = flat if flat is not None else flatten_fast_cached(plan)
        # the caller's flat may carry its own upload cache (distributed.fast_shard)
        cplan = plan if own_flat else getattr(flat, "_dev_cache", None)
        self.piece_rows = _cached_upload(cplan, dev, "piece_rows",
                                         lambda: D.index_tensor(flat.piece_rows, dev))
        self._cplan = cplan
        npc = len(flat.piece_off) - 1
        self.est = D.empty((npc, r), dev)
        self.gof = D.empty((npc, 2), dev)
        self.status = D.status_tensor(npc, dev)
        self.route = None
        if _fast_route_ok(x, flat, r):
            self._setup_route(flat, plan, r, dev, local)
            return
        self.order = D.index_tensor(flat.order, dev)
        self.levels = []
        for lv in flat.levels:
            nj = len(lv.start)
            self.levels.append(dict(
                tgt=D.index_tensor(lv.tgt_rows, dev), src=D.index_tensor(lv.src_rows, dev),
                job_off=np.ascontiguousarray(lv.job_off), start=D.index_tensor(lv.start, dev),
                length=D.index_tensor(lv.length, dev), max_len=int(lv.length.max()), nj=nj,
                rot=D.empty((nj, r, r), dev), trans=D.empty((nj, r), dev),
                loss=D.empty((nj,), dev), deg=torch.empty(nj, dtype=torch.int32, device=dev)))
        total = int(flat.piece_off[-1])
        self.pts = D.empty((total, r), dev)
        self.out = None if local else D.empty((plan.n, r), dev)
        # the shallowest level's jobs tile rows 0..n of the working buffer
        # contiguously: its apply, the scatter and the re-centring run as one
        # pass (mdsx_fast_finish)
        self.finish_off = None
        if not local and flat.levels:
            top = flat.levels[-1]
            st_, ln_ = np.asarray(top.start, np.int64), np.asarray(top.length, np.int64)
            off = np.concatenate([st_, [st_[-1] + ln_[-1]]]) if len(st_) else None
            if (off is not None and off[0] == 0 and off[-1] == plan.n
                    and np.array_equal(off[1:-1], st_[:-1] + ln_[:-1])):
                self.finish_off = np.ascontiguousarray(off)

    def _setup_route(self, flat, plan, r, dev, local):
        """mdsx_fast_mds (one call: no leaf point matrices, fused output
        pass) for plans with form-0 leaves (k_dcout.cu)."""
        import ctypes as C

        from ._lib import FastPlanC
        rt = route_cached(flat)
        nl = flat.n_leaves
        leaf_total = int(flat.piece_off[nl])
        def i32(a):
            return torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(dev)

        keep = _cached_upload(self._cplan, dev, "route", lambda: {
            "piece_off": np.ascontiguousarray(flat.piece_off, dtype=np.int64),
            "level_njobs": np.ascontiguousarray(rt.level_njobs, dtype=np.int32),
            "job_off": np.ascontiguousarray(rt.job_off, dtype=np.int64),
            "trk_row": D.index_tensor(rt.trk_row, dev), "trk_leaf": i32(rt.trk_leaf),
            "job_src": D.index_tensor(rt.job_src, dev), "job_tgt": D.index_tensor(rt.job_tgt, dev),
            "trk_job": i32(rt.trk_job), "leaf_job": i32(rt.leaf_job)})
        keep = self._keep = dict(keep)          # holds every device array the plan struct points to
        if local:
            keep["out_idx"] = torch.arange(leaf_total, dtype=torch.int64, device=dev)
            self.out = D.empty((leaf_total, r), dev)
            self.pts = self.out               # the rank's rows in DFS order (distributed.py)
        else:
            keep["out_idx"] = self.piece_rows[:leaf_total]
            self.out = D.empty((plan.n, r), dev)
        ptr = lambda a: a.ctypes.data if isinstance(a, np.ndarray) else a.data_ptr()  # noqa: E731
        self.route = FastPlanC(
            len(flat.piece_off) - 1, nl, len(rt.level_njobs), ptr(keep["piece_off"]),
            self.piece_rows.data_ptr(), keep["out_idx"].data_ptr(), len(rt.trk_row),
            ptr(keep["trk_row"]), ptr(keep["trk_leaf"]), ptr(keep["level_njobs"]),
            ptr(keep["job_off"]), ptr(keep["job_src"]), ptr(keep["job_tgt"]),
            ptr(keep["trk_job"]), ptr(keep["leaf_job"]))
        self._route_ref = C.byref(self.route)

    def launch(self) -> None:
        x, r, dev = self.compact(), self.r, self.dev
        h, sp = D.handle(dev), D.stream_ptr(dev)
        if self.route is not None:
            h.call("mdsx_fast_mds", x.data_ptr(), D.dtype_code(x), x.shape[1], x.shape[1],
                   self._route_ref, r, self.out.shape[0], 0 if self.local else 1,
                   self.out.data_ptr(), self.est.data_ptr(), self.gof.data_ptr(),
                   self.status.data_ptr(), sp)
            return
        npc = len(self.flat.piece_off) - 1
        h.call("mdsx_classical_pieces", x.data_ptr(), D.dtype_code(x), x.shape[1], x.shape[1],
               self.piece_rows.data_ptr(), self.flat.piece_off.ctypes.data, npc, r,
               self.pts.data_ptr(), self.est.data_ptr(), self.gof.data_ptr(),
               self.status.data_ptr(), sp)
        P = self.pts.data_ptr()
        for li, lv in enumerate(self.levels):
            h.call("mdsx_procrustes_fit", P, lv["tgt"].data_ptr(), P, lv["src"].data_ptr(),
                   lv["job_off"].ctypes.data, lv["nj"], r, lv["rot"].data_ptr(),
                   lv["trans"].data_ptr(), lv["loss"].data_ptr(), lv["deg"].data_ptr(), sp)
            if li == len(self.levels) - 1 and self.finish_off is not None:
                break                       # applied by mdsx_fast_finish below
            h.call("mdsx_procrustes_apply", P, r, lv["start"].data_ptr(), lv["length"].data_ptr(),
                   lv["nj"], lv["max_len"], lv["rot"].data_ptr(), lv["trans"].data_ptr(), sp)
        if self.local:
            return
        if self.finish_off is not None:
            lv = self.levels[-1]
            h.call("mdsx_fast_finish", P, r, self.finish_off.ctypes.data, lv["nj"],
                   lv["rot"].data_ptr(), lv["trans"].data_ptr(), self.order.data_ptr(),
                   self.plan.n, self.out.data_ptr(), sp)
            return
        h.call("mdsx_scatter_rows", P, self.order.data_ptr(), self.plan.n, r,
               self.out.data_ptr(), sp)
        h.call("mdsx_recenter", self.out.data_ptr(), self.plan.n, r, sp)

    def finish(self, return_device: bool = False) -> MdsConfiguration:
        st = D.decode_status(self.status)
        if np.any(st["code"] == 3):
            raise InvalidInputError("data contains non-finite values")
        ev = np.asarray(self.flat.eval_order, dtype=np.int64)
        bad = np.flatnonzero(st["code"][ev] != 0)
        if bad.size:                                   # first failure in evaluation order
            pid = int(ev[bad[0]])
            raise_piece_status(st[pid], self.r, self.flat.labels[pid])
        gof = self.gof.cpu().numpy()
        est = self.est.cpu().numpy()
        g1, g2, e = fast_aggregate(self.plan, self.flat, gof, est)
        return MdsConfiguration(_finish_points(self.out, return_device), e, float(g1), float(g2))


def fast_aggregate(plan: FastPlan, flat, gof: np.ndarray, est: np.ndarray):
    """The recursive fit aggregation of algorithms.py:289-320 (G1/G2
    size-weighted over children, estimates the plain mean of the children's),
    evaluated level by level with array operations over a program cached on
    the flattened plan: internal nodes grouped by height, children
    contiguous per parent."""
    prog = getattr(flat, "_agg", None)
    if prog is None:
        prog = flat._agg = _fast_agg_program(plan, flat.n_leaves)
    nl = flat.n_leaves
    sizes, groups = prog
    n_nodes = len(sizes)
    g1 = np.zeros(n_nodes)
    g2 = np.zeros(n_nodes)
    es = np.zeros((n_nodes, est.shape[1]))
    g1[:nl], g2[:nl], es[:nl] = gof[:nl, 0], gof[:nl, 1], est[:nl]
    for parents, children, starts in groups:
        w = sizes[children]
        g1[parents] = np.add.reduceat(w * g1[children], starts) / sizes[parents]
        g2[parents] = np.add.reduceat(w * g2[children], starts) / sizes[parents]
        cnt = np.diff(np.append(starts, len(children)))
        es[parents] = np.add.reduceat(es[children], starts, axis=0) / cnt[:, None]
    root = n_nodes - 1
    return g1[root], g2[root], es[root]


def _fast_agg_program(plan: FastPlan, nl: int):
    """(node sizes, [(parents, children, segment starts) per height]) with
    leaves 0..nl-1 in DFS order and internal nodes numbered in post-order
    (the root last)."""
    sizes, kids_of, height = [], {}, {}
    leaf = [0]
    internal = []

    def walk(node):
        if node.is_leaf:
            i = leaf[0]
            leaf[0] += 1
            return i, 0
        res = [walk(ch) for ch in node.children]
        internal.append((node.size, [c for c, _ in res], 1 + max(h for _, h in res)))
        return -len(internal), internal[-1][2]        # provisional id (negative)

    walk(plan.root)
    leaf_sizes = [lv.size for lv in plan.leaves()] if hasattr(plan, "leaves") else []
    n_int = len(internal)
    sizes = np.zeros(nl + n_int)
    sizes[:nl] = leaf_sizes[:nl] if leaf_sizes else 0.0

    def gid(c):
        return c if c >= 0 else nl + (-c - 1)
    by_h: dict = {}
    for k, (sz, ch, h) in enumerate(internal):
        sizes[nl + k] = sz
        by_h.setdefault(h, []).append((nl + k, [gid(c) for c in ch]))
    groups = []
    for h in sorted(by_h):
        parents = np.array([p for p, _ in by_h[h]], dtype=np.int64)
        children = np.concatenate([np.asarray(c, np.int64) for _, c in by_h[h]])
        starts = np.cumsum([0] + [len(c) for _, c in by_h[h]])[:-1].astype(np.int64)
        groups.append((parents, children, starts))
    return sizes, groups


def _fast_route_ok(x: torch.Tensor, flat, r: int) -> bool:
    """mdsx_fast_mds handles plans whose leaves all have more rows than
    features, with p <= 128, r <= 16 and 16-byte aligned rows."""
    import os
    p = x.shape[1]
    if os.environ.get("MDSX_FAST_PIECES") or not flat.levels:
        return False
    if not (p <= 128 and r <= 16 and (p * x.element_size()) % 16 == 0 and x.data_ptr() % 16 == 0
            and x.is_contiguous()):
        return False
    sizes = np.diff(np.asarray(flat.piece_off[:flat.n_leaves + 1]))
    return bool(np.all(sizes > p))


def fast_mds(data, params: AlgorithmParams, *, threads=None, device=None,
             plan: FastPlan | None = None, return_device: bool = False):
    dev = D.require_device(device)
    x = D.to_device_matrix(data, dev)
    prm = params.resolved("fast")
    n = x.shape[0]
    if n <= prm.l:
        return classical_mds_from_data(x, prm.r, device=dev, return_device=return_device)
    plan = plan if plan is not None else plan_fast(n, prm.l, prm.s, prm.seed)
    run = FastRun(x, plan, prm.r)
    run.launch()
    return run.finish(return_device)


def run_algorithm(name: str, data, params: AlgorithmParams, *, threads=None, **kw):
    """algorithms.py:351-363."""
    if name == "classical":
        return classical_mds_from_data(data, params.r, **kw)
    if name == "divide":
        return divide_and_conquer_mds(data, params, threads=threads, **kw)
    if name == "interpolate":
        return interpolation_mds(data, params, threads=threads, **kw)
    if name == "fast":
        return fast_mds(data, params, threads=threads, **kw)
    raise ParamError(f"unknown algorithm {name!r}; expected one of {ALGORITHM_NAMES}")
