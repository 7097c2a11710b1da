"""Left preconditioners on the hot path: none and Jacobi.

Mirrors ``kryrec.precond`` (precond.py:24-77, :251-312) for the two kinds the
benchmark configurations use. The Jacobi diagonal is applied inside the CUDA
kernels as an IEEE division (v / diag), the reference's arithmetic. The
triangular kinds (bjacobi, sor, ilu0, icc0) are out of this round's scope
 and raise NotImplementedError.
"""

from __future__ import annotations

import numpy as np

from .sparse import CsrMatrix

KINDS = ("none", "jacobi", "bjacobi", "sor", "ilu0", "icc0")
SUPPORTED = ("none", "jacobi")


class ZeroPivotError(ValueError):
    """Factorization hit a zero pivot (precond.py:24-31)."""

    def __init__(self, kind: str, row: int, value: float = 0.0):
        self.kind = kind
        self.row = int(row)
        self.value = float(value)
        super().__init__(f"{kind}: zero pivot at row {self.row} (value {value:g})")


class Preconditioner:
    kind = "none"

    def __init__(self, n: int):
        self.n = int(n)

    def apply(self, v):
        raise NotImplementedError

    def __repr__(self):
        return f"{type(self).__name__}(n={self.n})"


class IdentityPreconditioner(Preconditioner):
    kind = "none"

    def apply(self, v):
        return np.array(v, dtype=np.float64, copy=True)


class JacobiPreconditioner(Preconditioner):
    kind = "jacobi"

    def __init__(self, diag):
        super().__init__(len(diag))
        self.diag = np.asarray(diag, dtype=np.float64)
        self._dev = {}

    def apply(self, v):
        v = np.asarray(v, dtype=np.float64)
        return v / (self.diag if v.ndim == 1 else self.diag[:, None])

    def device_diag(self, device="cuda"):
        import torch

        key = str(device)
        if key not in self._dev:
            self._dev[key] = torch.from_numpy(self.diag).to(device)
        return self._dev[key]


def build_preconditioner(A, kind: str, *, sor_omega: float = 1.0,
                         bjacobi_block: int = 64) -> Preconditioner:
    """precond.py:251-312 restricted to none | jacobi."""
    A = CsrMatrix.of(A)
    if A.n_rows != A.n_cols:
        raise ValueError(f"preconditioner needs a square matrix, got {A.shape}")
    kind = kind.lower()
    if kind == "none":
        return IdentityPreconditioner(A.n_rows)
    if kind == "jacobi":
        diag = A.diagonal()
        zero = np.flatnonzero(diag == 0.0)
        if len(zero):
            raise ZeroPivotError("jacobi", zero[0])
        return JacobiPreconditioner(diag)
    if kind in KINDS:
        raise NotImplementedError(
            f"preconditioner {kind!r} is outside the B200 hot path (supported: {SUPPORTED})")
    raise ValueError(f"unknown preconditioner kind {kind!r}; expected one of {KINDS}")
