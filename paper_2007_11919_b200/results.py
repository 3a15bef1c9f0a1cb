"""Result types of the drop-in API (same fields as the reference)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class MdsConfiguration:
    """classical.py:27-47 — n x r embedding plus fit figures.

    ``points`` is a numpy float64 array (or a CUDA tensor when the caller asked
    for ``return_device=True``); ``eigenvalue_estimates`` are on the variance
    scale (lambda / rows in the decomposition)."""

    points: object
    eigenvalue_estimates: np.ndarray
    gof_g1: float
    gof_g2: float

    @property
    def dimension(self) -> int:
        return self.points.shape[1]

    @property
    def n_rows(self) -> int:
        return self.points.shape[0]


@dataclass(frozen=True)
class GofBreakdown:
    """classical.py:50-56."""

    retained_sum: float
    positive_sum: float
    absolute_sum: float


@dataclass(frozen=True)
class ProcrustesTransform:
    """procrustes.py:23-36 — orthogonal map + translation, residual, flag."""

    rotation: np.ndarray
    translation: np.ndarray
    loss: float
    degenerate: bool = False


@dataclass(frozen=True)
class EigenSystem:
    """linalg.py:124-136."""

    eigenvalues: np.ndarray
    eigenvectors: np.ndarray
    rank_used: int


@dataclass(frozen=True)
class GowerContext:
    """algorithms.py:175-190 — plus the packed device context
    [mean | M | v | S | q] the interpolation kernel consumes."""

    base_config: np.ndarray
    q_diag: np.ndarray
    covariance: np.ndarray
    base_rows: np.ndarray
    device_ctx: object = None
    device_flag: int = 0

    @property
    def l(self) -> int:
        return self.base_rows.shape[0]
