"""Function-level seams of the hot path, GPU-backed (same names, arguments,
results and error behaviour as the reference):

    euclidean_distance_matrix   linalg.py:61-82
    cross_squared_distances     linalg.py:85-104
    double_center               linalg.py:107-121
    classical_mds               classical.py:109-150
    classical_mds_from_data     classical.py:153-160
    goodness_of_fit/gof_breakdown classical.py:59-85 (host arithmetic on a spectrum)
    fit_procrustes / apply_procrustes   procrustes.py:53-105
    gower_context / gower_interpolate   algorithms.py:193-242

Every numeric result is computed by libmdsx kernels; numpy only converts.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _lib
from .errors import (DegenerateRankError, InvalidInputError, NumericalError, ParamError,
                     ShapeError)
from .params import EIGENVALUE_ZERO_TOL, EXACT_SIZE_GUARD
from .results import GofBreakdown, GowerContext, MdsConfiguration, ProcrustesTransform

JACOBI_KMAX = 112        # mdsx_common.cuh MDSX_JACOBI_KMAX: largest in-kernel full spectrum


# ---------------------------------------------------------------- distances
def euclidean_distance_matrix(data, *, exact_guard: int = EXACT_SIZE_GUARD, device=None):
    dev = D.require_device(device)
    x = D.to_device_matrix(data, dev)
    n, p = x.shape
    if n > exact_guard:
        raise ParamError(f"n={n} exceeds the exact-size guard ({exact_guard}); "
                         "use one of the partition-based algorithms instead")
    out = D.empty((n, n), dev)
    h = D.handle(dev)
    h.call("mdsx_sqdist_self", x.data_ptr(), D.dtype_code(x), p, n, p, out.data_ptr(), n,
           D.stream_ptr(dev))
    _check_finite_matrix(x, "data")
    return out.cpu().numpy()


def cross_squared_distances(a, b, *, device=None):
    dev = D.require_device(device)
    xa = D.to_device_matrix(a, dev, "a")
    xb = D.to_device_matrix(b, dev, "b")
    if xa.shape[1] != xb.shape[1]:
        raise ShapeError(f"column mismatch: a has {xa.shape[1]} columns, b has {xb.shape[1]}")
    if xa.dtype != xb.dtype:
        xa, xb = xa.double(), xb.double()
    _check_finite_matrix(xa, "a")
    _check_finite_matrix(xb, "b")
    ma, mb, p = xa.shape[0], xb.shape[0], xa.shape[1]
    out = D.empty((ma, mb), dev)
    D.handle(dev).call("mdsx_sqdist_cross", xa.data_ptr(), p, ma, xb.data_ptr(), p, mb,
                       D.dtype_code(xa), p, out.data_ptr(), mb, D.stream_ptr(dev))
    return out.cpu().numpy()


def _check_finite_matrix(x: torch.Tensor, name: str) -> None:
    if not bool(torch.isfinite(x).all()):
        raise InvalidInputError(f"{name} contains non-finite values")


_DELTA_MSG = [(1, "contains non-finite values"), (2, "is not symmetric"),
              (4, "has a nonzero diagonal"), (8, "has negative entries")]


def _validate_delta(d: torch.Tensor, name: str = "delta") -> None:
    """linalg.py:41-58, checked by mdsx_delta_check."""
    if d.dim() != 2 or d.shape[0] != d.shape[1]:
        raise InvalidInputError(f"{name} must be square, got shape {tuple(d.shape)}")
    if d.shape[0] < 1:
        raise InvalidInputError(f"{name} must be non-empty")
    dev = d.device
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    D.handle(dev).call("mdsx_delta_check", d.data_ptr(), d.shape[0], flags.data_ptr(),
                       D.stream_ptr(dev))
    f = int(flags.item())
    for bit, msg in _DELTA_MSG:
        if f & bit:
            raise InvalidInputError(f"{name} {msg}")


def _delta_tensor(delta, dev) -> torch.Tensor:
    if isinstance(delta, torch.Tensor):
        return delta.to(dev, torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(delta, dtype=np.float64))).to(dev)


def double_center(delta, *, device=None):
    dev = D.require_device(device)
    d = _delta_tensor(delta, dev)
    _validate_delta(d)
    m = d.shape[0]
    q = D.empty((m, m), dev)
    D.handle(dev).call("mdsx_double_center", d.data_ptr(), m, q.data_ptr(), D.stream_ptr(dev))
    return q.cpu().numpy()


# ---------------------------------------------------------------- fit ratios
def gof_breakdown(eigenvalues, r: int) -> GofBreakdown:
    """classical.py:59-72 (bookkeeping on an already-computed spectrum)."""
    ev = np.asarray(eigenvalues, dtype=np.float64)
    if ev.ndim != 1 or ev.size == 0:
        raise ParamError("eigenvalues must be a non-empty 1-D sequence")
    if np.any(np.diff(ev) > 0):
        raise ParamError("eigenvalues must be sorted in descending order")
    if not 1 <= r <= ev.size:
        raise ParamError(f"r must satisfy 1 <= r <= {ev.size}, got {r}")
    return GofBreakdown(float(ev[:r].sum()), float(np.maximum(ev, 0.0).sum()),
                        float(np.abs(ev).sum()))


def goodness_of_fit(eigenvalues, r: int) -> tuple[float, float]:
    """classical.py:75-85."""
    parts = gof_breakdown(eigenvalues, r)
    if parts.absolute_sum == 0.0:
        raise DegenerateRankError("all eigenvalues are zero; fit ratios undefined")
    return parts.retained_sum / parts.absolute_sum, parts.retained_sum / parts.positive_sum


# ---------------------------------------------------------------- classical MDS
def raise_piece_status(st, r: int, label: str | None = None) -> None:
    """Map one mdsx_piece_status onto the reference's exceptions/messages."""
    code = int(st["code"])
    if code == _lib.OK:
        return
    prefix = f"{label}: " if label else ""
    if code == _lib.DEGENERATE:
        idx = int(st["index"])
        if idx == 0:
            raise DegenerateRankError(prefix + "all eigenvalues are zero; fit ratios undefined")
        raise DegenerateRankError(prefix + f"eigenvalue {idx} of {r} is not positive "
                                           f"({float(st['value']):.3e}); reduce r")
    if code == _lib.INVALID:
        raise InvalidInputError("data contains non-finite values")
    if code == _lib.NUMERICAL:
        raise NumericalError(prefix + "eigendecomposition failed: Jacobi sweeps did not converge")
    raise _lib.status_error(code, prefix + f"piece failed with status {code}")


def _check_r(r: int, n: int) -> None:
    if not 1 <= r <= n - 1:
        raise ParamError(f"r must satisfy 1 <= r <= n-1, got r={r}, n={n}")


def classical_pieces(x: torch.Tensor, row_idx: torch.Tensor, piece_off: np.ndarray, r: int):
    """Batched classical MDS of plan pieces -> (points, estimates, gof, status) on device."""
    dev = x.device
    npieces = len(piece_off) - 1
    total = int(piece_off[-1] - piece_off[0])
    pts = D.empty((total, r), dev)
    est = D.empty((npieces, r), dev)
    gof = D.empty((npieces, 2), dev)
    st = D.status_tensor(npieces, dev)
    off = np.ascontiguousarray(piece_off, dtype=np.int64)
    D.handle(dev).call("mdsx_classical_pieces", x.data_ptr(), D.dtype_code(x), x.shape[1],
                       x.shape[1], row_idx.data_ptr(), off.ctypes.data, npieces, r,
                       pts.data_ptr(), est.data_ptr(), gof.data_ptr(), st.data_ptr(),
                       D.stream_ptr(dev))
    return pts, est, gof, st


def classical_mds_from_data(data, r: int, *, exact_guard: int = EXACT_SIZE_GUARD, device=None,
                            return_device: bool = False) -> MdsConfiguration:
    dev = D.require_device(device)
    x = D.to_device_matrix(data, dev)
    n = x.shape[0]
    _check_r(r, n)
    if n > exact_guard:
        raise ParamError(f"n={n} exceeds the exact-size guard ({exact_guard}); "
                         "use one of the partition-based algorithms instead")
    idx = torch.arange(n, dtype=torch.int64, device=dev)
    pts, est, gof, st = classical_pieces(x, idx, np.array([0, n], dtype=np.int64), r)
    raise_piece_status(D.decode_status(st)[0], r)
    g = gof.cpu().numpy()[0]
    return MdsConfiguration(pts if return_device else D.to_host(pts),
                            est.cpu().numpy()[0], float(g[0]), float(g[1]))


def classical_mds(delta, r: int, *, exact_guard: int = EXACT_SIZE_GUARD, device=None) -> MdsConfiguration:
    dev = D.require_device(device)
    arr = np.asarray(delta, dtype=np.float64) if not isinstance(delta, torch.Tensor) else delta
    n = arr.shape[0] if arr.ndim == 2 else 0
    _check_r(r, n)
    if n > exact_guard:
        raise ParamError(f"n={n} exceeds the exact-size guard ({exact_guard}); "
                         "use one of the partition-based algorithms instead")
    d = _delta_tensor(arr, dev)
    _validate_delta(d)
    spectrum = None
    if n > JACOBI_KMAX:
        # beyond the in-kernel full-spectrum solver: the top-r pairs come from
        # the block-Krylov kernels below; the full spectrum that G1/G2 and the
        # DegenerateRank rule need (classical.py:88-150) from the device
        # tridiagonalisation + bisection (mdsx_sym_eigvals)
        q = D.empty((n, n), dev)
        w = D.empty((n,), dev)
        h = D.handle(dev)
        h.call("mdsx_double_center", d.data_ptr(), n, q.data_ptr(), D.stream_ptr(dev))
        h.call("mdsx_sym_eigvals", q.data_ptr(), n, w.data_ptr(), D.stream_ptr(dev))
        ev = w.cpu().numpy()[::-1].copy()
        del q, w
        ev = np.delete(ev, int(np.argmin(np.abs(ev))))          # the structural zero (Q 1 = 0)
        ev[np.abs(ev) <= EIGENVALUE_ZERO_TOL * float(np.abs(ev).max(initial=0.0))] = 0.0
        bad = np.nonzero(ev[:r] <= 0.0)[0]
        if bad.size:
            raise DegenerateRankError(f"eigenvalue {bad[0] + 1} of {r} is not positive "
                                      f"({ev[bad[0]]:.3e}); reduce r")
        spectrum = ev
    pts = D.empty((n, r), dev)
    est = D.empty((1, r), dev)
    gof = D.empty((1, 2), dev)
    st = D.status_tensor(1, dev)
    D.handle(dev).call("mdsx_classical_delta", d.data_ptr(), n, r, pts.data_ptr(), est.data_ptr(),
                       gof.data_ptr(), st.data_ptr(), D.stream_ptr(dev))
    rec = D.decode_status(st)[0]
    if spectrum is not None:
        if int(rec["code"]) != _lib.DEGENERATE:                # the host spectrum decided that
            raise_piece_status(rec, r)
        g1, g2 = goodness_of_fit(spectrum, r)
        return MdsConfiguration(pts.cpu().numpy(), est.cpu().numpy()[0], g1, g2)
    raise_piece_status(rec, r)
    g = gof.cpu().numpy()[0]
    return MdsConfiguration(pts.cpu().numpy(), est.cpu().numpy()[0], float(g[0]), float(g[1]))


# ---------------------------------------------------------------- Procrustes
def _config(x, name: str) -> np.ndarray:
    arr = np.asarray(x, dtype=np.float64)
    if arr.ndim != 2:
        raise ShapeError(f"{name} must be 2-dimensional, got ndim={arr.ndim}")
    return arr


def fit_procrustes(target, source, *, device=None) -> ProcrustesTransform:
    dev = D.require_device(device)
    t = _config(target, "target")
    s = _config(source, "source")
    if t.shape != s.shape:
        raise ShapeError(f"shape mismatch: target {t.shape} vs source {s.shape}")
    n, r = t.shape
    if n < 2 or r < 1:
        raise ShapeError(f"need at least 2 rows and 1 column, got {t.shape}")
    tt = torch.from_numpy(np.ascontiguousarray(t)).to(dev)
    ss = torch.from_numpy(np.ascontiguousarray(s)).to(dev)
    rows = torch.arange(n, dtype=torch.int64, device=dev)
    rot = D.empty((1, r, r), dev)
    tr = D.empty((1, r), dev)
    loss = D.empty((1,), dev)
    deg = torch.empty(1, dtype=torch.int32, device=dev)
    off = np.array([0, n], dtype=np.int64)
    D.handle(dev).call("mdsx_procrustes_fit", tt.data_ptr(), rows.data_ptr(), ss.data_ptr(),
                       rows.data_ptr(), off.ctypes.data, 1, r, rot.data_ptr(), tr.data_ptr(),
                       loss.data_ptr(), deg.data_ptr(), D.stream_ptr(dev))
    return ProcrustesTransform(rotation=rot.cpu().numpy()[0], translation=tr.cpu().numpy()[0],
                               loss=float(loss.item()), degenerate=bool(deg.item()))


def apply_procrustes(points, transform: ProcrustesTransform, *, device=None) -> np.ndarray:
    dev = D.require_device(device)
    arr = _config(points, "points")
    r = transform.rotation.shape[0]
    if arr.shape[1] != r:
        raise ShapeError(f"points have {arr.shape[1]} columns, transform expects {r}")
    buf = torch.from_numpy(np.array(arr, dtype=np.float64, order="C")).to(dev)
    rot = torch.from_numpy(np.ascontiguousarray(transform.rotation, dtype=np.float64)).to(dev)
    tr = torch.from_numpy(np.ascontiguousarray(transform.translation, dtype=np.float64)).to(dev)
    n = arr.shape[0]
    start = torch.zeros(1, dtype=torch.int64, device=dev)
    length = torch.full((1,), n, dtype=torch.int64, device=dev)
    D.handle(dev).call("mdsx_procrustes_apply", buf.data_ptr(), r, start.data_ptr(),
                       length.data_ptr(), 1, n, rot.data_ptr(), tr.data_ptr(), D.stream_ptr(dev))
    return buf.cpu().numpy()


# ---------------------------------------------------------------- Gower
def gower_context(base_rows, base_config, *, device=None) -> GowerContext:
    dev = D.require_device(device)
    rows = D.to_device_matrix(base_rows, dev, "base_rows")
    cfg = np.asarray(base_config.cpu() if isinstance(base_config, torch.Tensor) else base_config,
                     dtype=np.float64)
    l, p = rows.shape
    if cfg.ndim != 2 or cfg.shape[0] != l:
        raise ShapeError(f"base_config must have one row per base row, got {cfg.shape} "
                         f"for {l} rows")
    _check_finite_matrix(rows, "base_rows")
    r = cfg.shape[1]
    x1 = torch.from_numpy(np.ascontiguousarray(cfg)).to(dev)
    h = D.handle(dev)
    size = int(h.lib.mdsx_gower_context_size(l, p, r))
    ctx = D.empty((size,), dev)
    cond = D.empty((1,), dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    h.call("mdsx_gower_context", rows.data_ptr(), D.dtype_code(rows), p, p, None, l, x1.data_ptr(),
           r, ctx.data_ptr(), cond.data_ptr(), flag.data_ptr(), D.stream_ptr(dev))
    f = int(flag.item())
    if f == 1:
        raise NumericalError(f"base covariance is ill-conditioned (condition estimate "
                             f"{float(cond.item()):.3e}); the requested dimension exceeds the "
                             "usable rank")
    host = ctx.cpu().numpy()
    cov = host[p + p * r + r: p + p * r + r + r * r].reshape(r, r).copy()
    q = host[p + p * r + r + r * r:].copy()
    base_np = rows.cpu().numpy().astype(np.float64, copy=False)
    return GowerContext(base_config=cfg, q_diag=q, covariance=cov, base_rows=base_np,
                        device_ctx=ctx, device_flag=f)


def gower_interpolate(ctx: GowerContext, new_rows, *, device=None) -> np.ndarray:
    dev = ctx.device_ctx.device if ctx.device_ctx is not None else D.require_device(device)
    y = D.to_device_matrix(new_rows, dev, "new_rows")
    p = ctx.base_rows.shape[1]
    if y.shape[1] != p:
        raise ShapeError(f"column mismatch: new rows have {y.shape[1]} columns, base has {p}")
    if ctx.device_flag == 2:
        raise NumericalError("base covariance is not positive definite")
    if ctx.device_ctx is None:
        ctx = gower_context(ctx.base_rows, ctx.base_config, device=dev)
    m, r = y.shape[0], ctx.base_config.shape[1]
    out = D.empty((m, r), dev)
    nf = torch.zeros(1, dtype=torch.int32, device=dev)
    D.handle(dev).call("mdsx_gower_interpolate", ctx.device_ctx.data_ptr(), ctx.l, p, r,
                       y.data_ptr(), D.dtype_code(y), p, m, out.data_ptr(), r, nf.data_ptr(),
                       0, D.stream_ptr(dev))
    if int(nf.item()):
        raise InvalidInputError("new_rows contains non-finite values")
    return out.cpu().numpy()
