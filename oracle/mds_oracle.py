"""CPU ORACLE — test infrastructure only, never the product path.

A numpy restatement of the reference ``scalemds`` hot path (interpolation,
divide-and-conquer and fast MDS plus the dense primitives under them), used
as the checker for the CUDA path in ``paper_2007_11919_b200``.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module.

Parity pin: the golden fixtures under ``tests/golden/`` were produced by
importing the reference package itself (``tests/golden/make_golden.py``);
``tests/test_oracle.py`` checks this restatement against them (plans
bit-exact, arrays to round-off).  Every function cites the reference
file:line it restates (paths relative to ``/root/reference/pkg/src/scalemds``).

The arithmetic lives in numpy/scipy (OpenBLAS dgemm, LAPACK dsyevd/dgesdd/
dpotrf) exactly as in the reference; this file only fixes the order of calls.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import cho_factor, cho_solve

EXACT_SIZE_GUARD = 20_000          # linalg.py:21
EIGENVALUE_ZERO_TOL = 1e-8         # linalg.py:25
DEGENERATE_SV_RATIO = 1e-12        # procrustes.py:20
COVARIANCE_CONDITION_LIMIT = 1e12  # algorithms.py:45


class OracleError(Exception):
    """Raised with ``kind`` naming the reference exception class."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


# ---------------------------------------------------------------- rng / data
def generator(seed: int, *path: int) -> np.random.Generator:
    """rng.py:14-17 — PCG64 keyed by SeedSequence(entropy=seed, spawn_key=path)."""
    return np.random.Generator(np.random.PCG64(
        np.random.SeedSequence(entropy=seed, spawn_key=tuple(path))))


def box_muller(gen: np.random.Generator, rows: int, cols: int) -> np.ndarray:
    """rng.py:26-41 — normals from two uniform streams, cos half then sin half."""
    total = rows * cols
    half = (total + 1) // 2
    u = gen.random(half)
    v = gen.random(half)
    rad = np.sqrt(-2.0 * np.log1p(-u))
    ang = (2.0 * np.pi) * v
    return np.concatenate([rad * np.cos(ang), rad * np.sin(ang)])[:total].reshape(rows, cols)


def scenario(n: int, k: int, h: int, seed: int = 0, rep: int = 0,
             dominant_sd: float = 15.0 ** 0.5) -> np.ndarray:
    """simulation.py:68-80 — first h columns scaled by sqrt(15)."""
    x = box_muller(generator(seed, rep), n, k)
    x[:, :h] *= dominant_sd
    return x


# ---------------------------------------------------------------- primitives
def as_data(x, name="data") -> np.ndarray:
    """linalg.py:28-38."""
    a = np.asarray(x, dtype=np.float64)
    if a.ndim != 2:
        raise OracleError("InvalidInputError", f"{name} must be 2-dimensional")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise OracleError("InvalidInputError", f"{name} must be non-empty")
    if not np.isfinite(a).all():
        raise OracleError("InvalidInputError", f"{name} contains non-finite values")
    return a


def sqdist_self(x, guard: int = EXACT_SIZE_GUARD) -> np.ndarray:
    """linalg.py:61-82 — Gram trick, symmetrise, clamp, zero diagonal."""
    a = as_data(x)
    if a.shape[0] > guard:
        raise OracleError("ParamError", "exceeds the exact-size guard")
    nrm = np.einsum("ij,ij->i", a, a)
    d = nrm[:, None] + nrm[None, :] - 2.0 * (a @ a.T)
    d = 0.5 * (d + d.T)
    np.maximum(d, 0.0, out=d)
    np.fill_diagonal(d, 0.0)
    return d


def sqdist_cross(a, b) -> np.ndarray:
    """linalg.py:85-104 — no symmetrisation, clamp at zero."""
    a = as_data(a, "a")
    b = as_data(b, "b")
    if a.shape[1] != b.shape[1]:
        raise OracleError("ShapeError", "column mismatch")
    d = a @ b.T
    d *= -2.0
    d += np.einsum("ij,ij->i", a, a)[:, None]
    d += np.einsum("ij,ij->i", b, b)[None, :]
    np.maximum(d, 0.0, out=d)
    return d


def check_delta(delta) -> np.ndarray:
    """linalg.py:41-58."""
    d = np.asarray(delta, dtype=np.float64)
    if d.ndim != 2 or d.shape[0] != d.shape[1] or d.shape[0] < 1:
        raise OracleError("InvalidInputError", "delta must be square")
    if not np.isfinite(d).all():
        raise OracleError("InvalidInputError", "delta contains non-finite values")
    tol = 1e-9 * max(float(np.abs(d).max()), 1.0)
    if float(np.abs(d - d.T).max()) > tol:
        raise OracleError("InvalidInputError", "delta is not symmetric")
    if float(np.abs(np.diagonal(d)).max(initial=0.0)) > tol:
        raise OracleError("InvalidInputError", "delta has a nonzero diagonal")
    if float(d.min()) < -tol:
        raise OracleError("InvalidInputError", "delta has negative entries")
    return d


def center_delta(delta) -> np.ndarray:
    """linalg.py:107-121 — scalar double-centering with one row-mean vector."""
    d = check_delta(delta)
    mu = d.mean(axis=1)
    q = -0.5 * (d - mu[:, None] - mu[None, :] + mu.mean())
    return 0.5 * (q + q.T)


def sign_fix(v: np.ndarray) -> np.ndarray:
    """linalg.py:139-146 — largest-|.| entry positive, lowest index on ties."""
    if v.shape[1] == 0:
        return v
    lead = np.argmax(np.abs(v), axis=0)
    s = np.sign(v[lead, np.arange(v.shape[1])])
    s[s == 0] = 1.0
    return v * s


def eigh_desc(q):
    """linalg.py:149-169 — full dsyevd, stable descending order, signs, rank."""
    a = np.asarray(q, dtype=np.float64)
    w, v = np.linalg.eigh(a)
    order = np.argsort(-w, kind="stable")
    w = w[order]
    v = sign_fix(v[:, order])
    scale = float(np.abs(w).max(initial=0.0))
    rank = int(np.count_nonzero(w > EIGENVALUE_ZERO_TOL * scale)) if scale > 0 else 0
    return w, v, rank


def svd_signed(m):
    """linalg.py:186-205 — thin SVD, sign rule applied to left/right in pairs."""
    u, s, vt = np.linalg.svd(np.asarray(m, dtype=np.float64), full_matrices=False)
    lead = np.argmax(np.abs(u), axis=0)
    sg = np.sign(u[lead, np.arange(u.shape[1])])
    sg[sg == 0] = 1.0
    return u * sg, s, vt.T * sg


# ---------------------------------------------------------------- classical MDS
@dataclass
class Embedding:
    """classical.py:27-47 — points, variance-scale eigenvalues, G1, G2."""
    points: np.ndarray
    estimates: np.ndarray
    g1: float
    g2: float


def gof(values: np.ndarray, r: int):
    """classical.py:59-85."""
    ev = np.asarray(values, dtype=np.float64)
    absolute = float(np.abs(ev).sum())
    if absolute == 0.0:
        raise OracleError("DegenerateRankError", "all eigenvalues are zero")
    kept = float(ev[:r].sum())
    return kept / absolute, kept / float(np.maximum(ev, 0.0).sum())


def mds_from_delta(delta, r: int, guard: int = EXACT_SIZE_GUARD) -> Embedding:
    """classical.py:88-150 — trivial-mode removal, zero snap, V_r sqrt(lambda_r)."""
    d = np.asarray(delta, dtype=np.float64)
    n = d.shape[0] if d.ndim == 2 else 0
    if not 1 <= r <= n - 1:
        raise OracleError("ParamError", f"r must satisfy 1 <= r <= n-1, got r={r}, n={n}")
    if n > guard:
        raise OracleError("ParamError", "exceeds the exact-size guard")
    w, v, _ = eigh_desc(center_delta(check_delta(d)))
    trivial = int(np.argmax(np.abs(v.T @ np.ones(n))))
    keep = np.arange(n) != trivial
    w = w[keep].copy()
    v = v[:, keep]
    w[np.abs(w) <= EIGENVALUE_ZERO_TOL * float(np.abs(w).max(initial=0.0))] = 0.0
    bad = np.nonzero(w[:r] <= 0.0)[0]
    if bad.size:
        raise OracleError("DegenerateRankError",
                          f"eigenvalue {bad[0] + 1} of {r} is not positive "
                          f"({w[bad[0]]:.3e}); reduce r")
    g1, g2 = gof(w, r)
    return Embedding(v[:, :r] * np.sqrt(w[:r]), w[:r] / n, g1, g2)


def mds_from_data(x, r: int, guard: int = EXACT_SIZE_GUARD) -> Embedding:
    """classical.py:153-160."""
    a = np.asarray(x, dtype=np.float64)
    n = a.shape[0] if a.ndim == 2 else 0
    if not 1 <= r <= n - 1:
        raise OracleError("ParamError", f"r must satisfy 1 <= r <= n-1, got r={r}, n={n}")
    return mds_from_delta(sqdist_self(a, guard), r, guard)


def _labelled(rows, r, label) -> Embedding:
    """algorithms.py:115-119 — DegenerateRank relabelled with the piece name."""
    try:
        return mds_from_data(rows, r)
    except OracleError as e:
        if e.kind == "DegenerateRankError":
            raise OracleError(e.kind, f"{label}: {e}") from e
        raise


# ---------------------------------------------------------------- Procrustes
@dataclass
class Transform:
    """procrustes.py:23-36."""
    rotation: np.ndarray
    translation: np.ndarray
    loss: float
    degenerate: bool


def procrustes_fit(target, source) -> Transform:
    """procrustes.py:46-78 — T = Omega Gamma^T from the centred cross-product."""
    t = np.asarray(target, dtype=np.float64)
    s = np.asarray(source, dtype=np.float64)
    if t.ndim != 2 or t.shape != s.shape or t.shape[0] < 2 or t.shape[1] < 1:
        raise OracleError("ShapeError", "bad Procrustes shapes")
    left, sv, right = svd_signed((t - t.mean(axis=0)).T @ (s - s.mean(axis=0)))
    top = sv[0] if sv.size else 0.0
    degenerate = bool(sv.size == 0 or sv[-1] <= DEGENERATE_SV_RATIO * top)
    rot = right @ left.T
    shift = (t - s @ rot).mean(axis=0)
    res = t - s @ rot - shift
    return Transform(rot, shift, float(np.sum(res * res)), degenerate)


def procrustes_apply(points, tr: Transform) -> np.ndarray:
    """procrustes.py:99-105."""
    return np.asarray(points, dtype=np.float64) @ tr.rotation + tr.translation


# ---------------------------------------------------------------- plans
def _resolve(algorithm: str, r: int, l, c, s):
    """algorithms.py:67-101 — defaults l=400 (divide) / 1000, c = s = 2r."""
    if r < 1:
        raise OracleError("ParamError", f"r must be >= 1, got {r}")
    if l is None:
        l = 400 if algorithm == "divide" else 1000
    if l > EXACT_SIZE_GUARD:
        raise OracleError("ParamError", "exceeds the exact-size guard")
    if algorithm == "divide":
        c = 2 * r if c is None else c
        if c < r or l <= c:
            raise OracleError("ParamError", "bad c")
    elif algorithm == "interpolate":
        if l < 2:
            raise OracleError("ParamError", "bad l")
    elif algorithm == "fast":
        s = 2 * r if s is None else s
        if s < r or s < 2 or l < 2 * s:
            raise OracleError("ParamError", "bad s")
    else:
        raise OracleError("ParamError", f"unknown algorithm {algorithm!r}")
    return l, c, s


def plan_divide(n: int, l: int, c: int, seed: int):
    """partition.py:184-214 -> (connecting, subsets)."""
    if n <= l:
        return np.empty(0, np.int64), [np.arange(n, dtype=np.int64)]
    g = generator(seed)
    conn = np.sort(g.choice(n, size=c, replace=False)).astype(np.int64)
    order = g.permutation(np.setdiff1d(np.arange(n, dtype=np.int64), conn))
    step = l - c
    parts = [order[i:i + step] for i in range(0, order.size, step)]
    if len(parts) > 1 and parts[-1].size < c + 1:
        tail = parts.pop()
        parts[-1] = np.concatenate([parts[-1], tail])
    return conn, [np.concatenate([conn, np.sort(q)]) for q in parts]


def plan_interp(n: int, l: int, seed: int):
    """partition.py:217-232 -> list of index arrays (sample first)."""
    if n <= l:
        return [np.arange(n, dtype=np.int64)]
    g = generator(seed)
    sample = np.sort(g.choice(n, size=l, replace=False)).astype(np.int64)
    order = g.permutation(np.setdiff1d(np.arange(n, dtype=np.int64), sample))
    return [sample] + [np.sort(order[i:i + l]) for i in range(0, order.size, l)]


@dataclass
class Node:
    """partition.py:89-112."""
    indices: np.ndarray
    children: list = field(default_factory=list)
    positions: np.ndarray | None = None


def plan_fast_tree(n: int, l: int, s: int, seed: int) -> Node:
    """partition.py:244-274 — shuffle, array_split into l//s, sample min(s,size)."""
    parts = l // s

    def grow(idx, path):
        if idx.size <= l:
            return Node(np.sort(idx))
        g = generator(seed, *path)
        chunks = np.array_split(g.permutation(idx), parts)
        pos = [np.sort(g.choice(ch.size, size=min(s, ch.size), replace=False)) for ch in chunks]
        kids = []
        for i, ch in enumerate(chunks):
            kid = grow(ch, path + (i,))
            kid.positions = pos[i]
            kids.append(kid)
        return Node(np.concatenate([k.indices for k in kids]), kids)

    return grow(np.arange(n, dtype=np.int64), ())


# ---------------------------------------------------------------- algorithms
def _pmap(fn, items, threads):
    """algorithms.py:104-112 — ordered map, optional thread pool."""
    items = list(items)
    if threads is None:
        threads = min(len(items), os.cpu_count() or 1)
    if threads <= 1 or len(items) <= 1:
        return [fn(it) for it in items]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(fn, items))


def divide_conquer(data, r, l=None, c=None, seed=0, threads=None, plan=None) -> Embedding:
    """algorithms.py:128-172."""
    x = as_data(data)
    l, c, _ = _resolve("divide", r, l, c, None)
    n = x.shape[0]
    if n <= l:
        return mds_from_data(x, r)
    subsets = plan if plan is not None else plan_divide(n, l, c, seed)[1]
    embs = _pmap(lambda j: _labelled(x[subsets[j]], r, f"subset {j + 1}"),
                 range(len(subsets)), threads)
    out = np.empty((n, r))
    out[subsets[0]] = embs[0].points
    anchor = embs[0].points[:c]
    for j in range(1, len(subsets)):
        tr = procrustes_fit(anchor, embs[j].points[:c])
        out[subsets[j][c:]] = procrustes_apply(embs[j].points[c:], tr)
    size = np.array([q.size for q in subsets], dtype=np.float64)
    w = size.copy()
    w[1:] -= c
    g1 = float(np.dot(w, [e.g1 for e in embs]) / n)
    g2 = float(np.dot(w, [e.g2 for e in embs]) / n)
    est = np.stack([e.estimates * (sz / wt) for e, sz, wt in zip(embs, size, w)]).mean(axis=0)
    return Embedding(out - out.mean(axis=0), est, g1, g2)


@dataclass
class GowerCtx:
    """algorithms.py:175-190."""
    base_config: np.ndarray
    q_diag: np.ndarray
    covariance: np.ndarray
    base_rows: np.ndarray


def gower_ctx(base_rows, base_config) -> GowerCtx:
    """algorithms.py:193-217."""
    rows = as_data(base_rows, "base_rows")
    cfg = np.asarray(base_config, dtype=np.float64)
    if cfg.ndim != 2 or cfg.shape[0] != rows.shape[0]:
        raise OracleError("ShapeError", "base_config must have one row per base row")
    qd = np.ascontiguousarray(np.diagonal(center_delta(sqdist_self(rows))))
    if float(qd.min()) < -1e-9 * max(float(np.abs(qd).max(initial=0.0)), 1.0):
        raise OracleError("NumericalError", "inner-product diagonal negative")
    cc = cfg - cfg.mean(axis=0)
    cov = cc.T @ cc / rows.shape[0]
    ev = np.linalg.eigvalsh(cov)
    cond = np.inf if ev[0] <= 0.0 else ev[-1] / ev[0]
    if cond > COVARIANCE_CONDITION_LIMIT:
        raise OracleError("NumericalError", f"base covariance is ill-conditioned "
                                            f"(condition estimate {cond:.3e})")
    return GowerCtx(cfg, qd, cov, rows)


def gower_project(ctx: GowerCtx, rows) -> np.ndarray:
    """algorithms.py:220-242 — (1q' - A2) X1 S^-1 / (2l) via Cholesky."""
    y = as_data(rows, "new_rows")
    if y.shape[1] != ctx.base_rows.shape[1]:
        raise OracleError("ShapeError", "column mismatch")
    a2 = sqdist_cross(y, ctx.base_rows)
    np.subtract(ctx.q_diag[None, :], a2, out=a2)
    proj = a2 @ ctx.base_config / (2.0 * ctx.base_rows.shape[0])
    fac = cho_factor(ctx.covariance, lower=True, check_finite=False)
    return np.ascontiguousarray(cho_solve(fac, proj.T, check_finite=False).T)


def interpolation(data, r, l=None, seed=0, threads=None, plan=None) -> Embedding:
    """algorithms.py:245-274."""
    x = as_data(data)
    l, _, _ = _resolve("interpolate", r, l, None, None)
    n = x.shape[0]
    if n <= l:
        return mds_from_data(x, r)
    subsets = plan if plan is not None else plan_interp(n, l, seed)
    base = _labelled(x[subsets[0]], r, "sample subset")
    ctx = gower_ctx(x[subsets[0]], base.points)
    blocks = _pmap(lambda idx: gower_project(ctx, x[idx]), subsets[1:], threads)
    out = np.empty((n, r))
    out[subsets[0]] = base.points
    for idx, blk in zip(subsets[1:], blocks):
        out[idx] = blk
    return Embedding(out - out.mean(axis=0), base.estimates, base.g1, base.g2)


def _fast_node(node: Node, x, r, threads, label):
    """algorithms.py:285-320 -> (points in node.indices order, (g1, g2, est, size))."""
    if not node.children:
        e = _labelled(x[node.indices], r, label or "leaf 1")
        return e.points, (e.g1, e.g2, e.estimates, node.indices.size)
    solved = _pmap(lambda it: _fast_node(it[1], x, r, 1,
                                         f"{label}.{it[0] + 1}" if label else f"branch {it[0] + 1}"),
                   enumerate(node.children), threads)
    samp = np.concatenate([k.indices[k.positions] for k in node.children])
    align = _labelled(x[samp], r, f"{label or 'root'} alignment set")
    blocks, off = [], 0
    for kid, (pts, _) in zip(node.children, solved):
        cnt = kid.positions.size
        tr = procrustes_fit(align.points[off:off + cnt], pts[kid.positions])
        off += cnt
        blocks.append(procrustes_apply(pts, tr))
    fits = [f for _, f in solved]
    size = np.array([f[3] for f in fits], dtype=np.float64)
    tot = size.sum()
    g1 = float(np.dot(size, [f[0] for f in fits]) / tot)
    g2 = float(np.dot(size, [f[1] for f in fits]) / tot)
    est = np.stack([f[2] for f in fits]).mean(axis=0)
    return np.vstack(blocks), (g1, g2, est, int(tot))


def fast(data, r, l=None, s=None, seed=0, threads=None, plan=None) -> Embedding:
    """algorithms.py:323-348."""
    x = as_data(data)
    l, _, s = _resolve("fast", r, l, None, s)
    n = x.shape[0]
    if n <= l:
        return mds_from_data(x, r)
    root = plan if plan is not None else plan_fast_tree(n, l, s, seed)
    blk, (g1, g2, est, _) = _fast_node(root, x, r, threads, "")
    out = np.empty((n, r))
    out[root.indices] = blk
    return Embedding(out - out.mean(axis=0), est, g1, g2)


def run(name: str, data, r: int, l=None, c=None, s=None, seed=0, threads=None) -> Embedding:
    """algorithms.py:351-363."""
    if name == "classical":
        return mds_from_data(data, r)
    if name == "divide":
        return divide_conquer(data, r, l, c, seed, threads)
    if name == "interpolate":
        return interpolation(data, r, l, seed, threads)
    if name == "fast":
        return fast(data, r, l, s, seed, threads)
    raise OracleError("ParamError", f"unknown algorithm {name!r}")
