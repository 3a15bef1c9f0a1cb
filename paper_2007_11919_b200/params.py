"""Algorithm parameters and package constants (drop-in for the reference's
``AlgorithmParams``, ``algorithms.py:50-101``, and ``linalg.py:21,25``)."""

from __future__ import annotations

from dataclasses import dataclass, replace

from .errors import ParamError

EXACT_SIZE_GUARD = 20_000            # linalg.py:21 — largest dense piece
EIGENVALUE_ZERO_TOL = 1e-8           # linalg.py:25 — relative zero snap
DEGENERATE_SV_RATIO = 1e-12          # procrustes.py:20
COVARIANCE_CONDITION_LIMIT = 1e12    # algorithms.py:45
DEFAULT_L_DIVIDE = 400               # algorithms.py:39
DEFAULT_L = 1000                     # algorithms.py:40
ALGORITHM_NAMES = ("classical", "divide", "interpolate", "fast")   # algorithms.py:47


@dataclass(frozen=True)
class AlgorithmParams:
    """``r`` target dimension, ``l`` largest classical-MDS piece, ``c``
    connecting rows (divide), ``s`` sampling rows per part (fast), ``seed``.
    ``None`` fields take per-algorithm defaults on :meth:`resolved`."""

    r: int
    l: int | None = None
    c: int | None = None
    s: int | None = None
    seed: int = 0

    def resolved(self, algorithm: str) -> "AlgorithmParams":
        """Defaults + validation for one algorithm (algorithms.py:67-101)."""
        if self.r < 1:
            raise ParamError(f"r must be >= 1, got {self.r}")
        if algorithm == "classical":
            return self
        if algorithm not in ("divide", "interpolate", "fast"):
            raise ParamError(f"unknown algorithm {algorithm!r}")
        l = self.l
        if l is None:
            l = DEFAULT_L_DIVIDE if algorithm == "divide" else DEFAULT_L
        if l > EXACT_SIZE_GUARD:
            raise ParamError(f"l={l} exceeds the exact-size guard ({EXACT_SIZE_GUARD})")
        c, s = self.c, self.s
        if algorithm == "divide":
            if c is None:
                c = 2 * self.r
            if c < self.r:
                raise ParamError(f"c must be >= r, got c={c}, r={self.r}")
            if l <= c:
                raise ParamError(f"l must exceed c, got l={l}, c={c}")
        elif algorithm == "interpolate":
            if l < 2:
                raise ParamError(f"l must be >= 2, got l={l}")
        else:
            if s is None:
                s = 2 * self.r
            if s < self.r:
                raise ParamError(f"s must be >= r, got s={s}, r={self.r}")
            if s < 2:
                raise ParamError("s must be >= 2: alignment needs two sampling rows")
            if l < 2 * s:
                raise ParamError(f"l must be >= 2*s, got l={l}, s={s}")
        return replace(self, l=l, c=c, s=s)
