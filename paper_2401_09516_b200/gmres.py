"""Solver configuration and report (kryrec/gmres.py:26-56) and the GMRES(m)
baseline, which is the k = 0 path of the device GCRO-DR engine
(gmres.py:193-267; gcrodr.py:326-330)."""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["SolverConfig", "SolveReport", "gmres_solve"]


@dataclass(frozen=True)
class SolverConfig:
    """Restart length m, tolerance, operator-application cap, recycle size k."""

    m: int = 50
    tol: float = 1e-8
    max_iter: int = 10000
    k: int = 10

    def __post_init__(self):
        if self.m < 2:
            raise ValueError("m must be >= 2")
        if not self.tol > 0:
            raise ValueError("tol must be positive")
        if self.max_iter < 1:
            raise ValueError("max_iter must be >= 1")
        if not 0 <= self.k < self.m:
            raise ValueError("k must satisfy 0 <= k < m")


@dataclass
class SolveReport:
    """Outcome of one linear solve (gmres.py:46-56) plus device timing."""

    x: np.ndarray
    iterations: int
    residual_history: np.ndarray
    true_relative_residual: float
    converged: bool
    wall_time: float
    diagnostics: dict = field(default_factory=dict)
    device_ms: float = 0.0
    x_device: object = None


def gmres_solve(A, b, x0=None, M=None, cfg: SolverConfig | None = None,
                collect_diagnostics: bool = False) -> SolveReport:
    """Restarted GMRES(m) on the GPU: GCRO-DR with k = 0 (no recycling)."""
    from dataclasses import replace

    from .gcrodr import gcrodr_solve

    cfg = cfg or SolverConfig()
    rep, _ = gcrodr_solve(A, b, x0=x0, M=M, cfg=replace(cfg, k=0),
                          collect_diagnostics=collect_diagnostics)
    rep.diagnostics.pop("gmres_fallback", None)
    rep.diagnostics.pop("deflated_steps", None)
    rep.diagnostics.pop("recycle_k", None)
    return rep
