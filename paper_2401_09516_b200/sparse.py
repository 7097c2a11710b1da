"""CSR container (host) and its device-resident form.

``CsrMatrix`` mirrors ``kryrec.sparse.CsrMatrix`` (sparse.py:16-112): same
constructor, invariants, error messages and read-only arrays (int64 indices,
float64 values). Its validation is vectorised instead of the reference's
per-row Python loop (sparse.py:52-55). ``DeviceCsr`` is the GPU form the
kernels consume: int32 row pointers / column indices, fp64 values, optional
Jacobi diagonal, uploaded once per system.
"""

from __future__ import annotations

import ctypes
import os
from typing import Sequence

import numpy as np

from . import _lib

__all__ = ["CsrMatrix", "DeviceCsr", "spmv", "dot", "norm2", "axpy", "as_vector", "eye"]


class CsrMatrix:
    """Sparse real matrix in compressed-sparse-row form (reference-compatible)."""

    __slots__ = ("n_rows", "n_cols", "row_ptr", "col_idx", "values", "_scipy")

    def __init__(self, n_rows, n_cols, row_ptr, col_idx, values, *, validate: bool = True):
        n_rows = int(n_rows)
        n_cols = int(n_cols)
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        col_idx = np.ascontiguousarray(col_idx, dtype=np.int64)
        values = np.ascontiguousarray(values, dtype=np.float64)
        if n_rows < 0 or n_cols < 0:
            raise ValueError("matrix dimensions must be nonnegative")
        if row_ptr.shape != (n_rows + 1,):
            raise ValueError(f"row_ptr has length {row_ptr.shape[0]}, expected {n_rows + 1}")
        if row_ptr[0] != 0 or row_ptr[-1] != len(values):
            raise ValueError("row_ptr must start at 0 and end at nnz")
        if validate:
            if np.any(np.diff(row_ptr) < 0):
                raise ValueError("row_ptr must be nondecreasing")
            if col_idx.shape != values.shape:
                raise ValueError("col_idx and values must have equal length")
            if len(col_idx) and (col_idx.min() < 0 or col_idx.max() >= n_cols):
                raise ValueError("column index out of range")
            if len(col_idx) > 1:
                # strictly increasing within each row: check consecutive pairs
                # that do not straddle a row boundary
                bad = np.diff(col_idx) <= 0
                starts = row_ptr[1:-1]
                starts = starts[(starts > 0) & (starts < len(col_idx))]
                bad[starts - 1] = False
                if np.any(bad):
                    pos = int(np.argmax(bad))
                    row = int(np.searchsorted(row_ptr, pos, side="right") - 1)
                    raise ValueError(f"row {row}: column indices not strictly increasing")
            if not np.all(np.isfinite(values)):
                raise ValueError("matrix values must be finite")
        elif col_idx.shape != values.shape:
            raise ValueError("col_idx and values must have equal length")
        for arr in (row_ptr, col_idx, values):
            arr.flags.writeable = False
        self.n_rows = n_rows
        self.n_cols = n_cols
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.values = values
        self._scipy = None

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    @property
    def nnz(self):
        return len(self.values)

    def to_scipy(self):
        import scipy.sparse as _sp

        if self._scipy is None:
            self._scipy = _sp.csr_matrix((self.values, self.col_idx, self.row_ptr),
                                         shape=(self.n_rows, self.n_cols))
        return self._scipy

    @classmethod
    def from_scipy(cls, mat) -> "CsrMatrix":
        import scipy.sparse as _sp

        csr = _sp.csr_matrix(mat)
        csr.sort_indices()
        return cls(csr.shape[0], csr.shape[1], csr.indptr, csr.indices, csr.data)

    @classmethod
    def of(cls, A) -> "CsrMatrix":
        """Adopt any object with n_rows/n_cols/row_ptr/col_idx/values (e.g. kryrec's)."""
        if isinstance(A, cls):
            return A
        return cls(A.n_rows, A.n_cols, A.row_ptr, A.col_idx, A.values, validate=False)

    def diagonal(self) -> np.ndarray:
        rows = np.repeat(np.arange(self.n_rows), np.diff(self.row_ptr))
        d = np.zeros(min(self.n_rows, self.n_cols))
        on = rows == self.col_idx
        d[rows[on]] = self.values[on]
        return d

    def to_dense(self) -> np.ndarray:
        return self.to_scipy().toarray()

    def __repr__(self):
        return f"CsrMatrix(shape={self.shape}, nnz={self.nnz})"


def stencil_offsets(row_ptr, col_idx):
    """Diagonal offsets (sx, sxy) of a 5-/7-point stencil matrix in natural
    ordering, read off row 0's upper entries (columns 1, sx[, sxy]), or None.
    Only a guess: skr_stencil_build verifies every row on the device."""
    if len(row_ptr) < 2:
        return None
    e = int(row_ptr[1])
    cols = np.asarray(col_idx[:e]).astype(np.int64)
    up = cols[cols > 0]
    if len(up) == 2 and up[0] == 1 and up[1] >= 2:
        return int(up[1]), 0
    if len(up) == 3 and up[0] == 1 and up[1] >= 2 and up[2] > up[1]:
        return int(up[1]), int(up[2])
    return None


def stencil_enabled() -> bool:
    """The stencil form is used unless SKR_NO_STENCIL=1 (A/B runs, tests)."""
    return os.environ.get("SKR_NO_STENCIL", "0") in ("", "0")


class DeviceCsr:
    """Device-resident CSR (int32 indices, fp64 values) + optional Jacobi
    diagonal + optional stencil form (skr_stencil_build; the kernels use it
    only if the device check found the matrix to be a symmetric 7-diagonal
    one, with bit-identical results)."""

    def __init__(self, n, row_ptr, col_idx, values, diag=None, keep=None, stencil=None,
                 precond=None):
        self.n = int(n)
        self.row_ptr = row_ptr
        self.col_idx = col_idx
        self.values = values
        self.diag = diag
        self._keep = keep
        self.stencil = stencil  # (device buffer, sx, sxy) or None
        # general preconditioner: an object with .buffer (device bytes built by
        # skr_precond_build; it keeps the pattern it was built on alive) or None
        self.precond = precond
        buf, sx, sxy = stencil if stencil is not None else (None, 0, 0)
        self.c = _lib.SkrCsr(self.n, int(values.numel()), row_ptr.data_ptr(),
                             col_idx.data_ptr(), values.data_ptr(),
                             diag.data_ptr() if diag is not None else None,
                             buf.data_ptr() if buf is not None else None, int(sx), int(sxy),
                             precond.buffer.data_ptr() if precond is not None else None,
                             _lib.PC_KINDS.get(getattr(precond, "kind", ""), 0))

    def stencil_active(self) -> bool:
        """True when the device check accepted the stencil form (syncs)."""
        if self.stencil is None:
            return False
        return int(self.stencil[0][:4].view(__import__("torch").int32).item()) == 1

    def build_stencil(self, offsets, stream=None):
        """Build (and verify on the device) the stencil form for `offsets`."""
        import torch

        sx, sxy = offsets
        L = _lib.load()
        nbytes = int(L.skr_stencil_bytes(self.n, sx, sxy))
        if nbytes == 0:
            return self
        buf = torch.empty(nbytes, dtype=torch.uint8, device=self.values.device)
        probe = _lib.SkrCsr(self.n, int(self.values.numel()), self.row_ptr.data_ptr(),
                            self.col_idx.data_ptr(), self.values.data_ptr(), None, None, 0, 0,
                            None, 0)
        _lib.check(L.skr_stencil_build(ctypes.byref(probe), sx, sxy, buf.data_ptr(), nbytes,
                                       _lib.stream_handle(stream)), "skr_stencil_build")
        return DeviceCsr(self.n, self.row_ptr, self.col_idx, self.values, self.diag, self._keep,
                         (buf, sx, sxy), self.precond)

    @property
    def nnz(self) -> int:
        return int(self.values.numel())

    @classmethod
    def from_host(cls, A, jacobi: bool = False, device=None, stream=None, non_blocking=False,
                  check_pivot: bool = True):
        """Upload a CsrMatrix-like (numpy or torch CPU arrays).

        ``jacobi``: also keep the Jacobi diagonal; a zero pivot raises
        ``ZeroPivotError`` (precond.py:153-158) here, which synchronises the
        stream. ``check_pivot=False`` defers that check to
        ``raise_if_zero_pivot()`` (one synchronisation for a whole batch)."""
        import torch

        dev = torch.device(device) if device is not None else torch.device("cuda")
        if A.n_rows != A.n_cols:
            raise ValueError("gcrodr needs a square matrix")
        n = int(A.n_rows)
        if n >= 2**31 - 1 or len(A.values) >= 2**31 - 1:
            raise ValueError("matrix too large for int32 device indices")

        def _t(a, dt):
            if isinstance(a, torch.Tensor):
                return a.to(device=dev, dtype=dt, non_blocking=non_blocking)
            arr = np.asarray(a)
            if dt == torch.int32 and arr.dtype != np.int32:
                arr = arr.astype(np.int32)
            return torch.from_numpy(np.ascontiguousarray(arr)).to(dev, non_blocking=non_blocking)

        ctx = torch.cuda.stream(stream) if stream is not None else _nullctx()
        with ctx:
            rp = _t(A.row_ptr, torch.int32)
            ci = _t(A.col_idx, torch.int32)
            vals = _t(A.values, torch.float64)
            dA = cls(n, rp, ci, vals, None)
            off = stencil_offsets(A.row_ptr, A.col_idx) if stencil_enabled() else None
            if off is not None:
                dA = dA.build_stencil(off, stream=stream)
            if jacobi:
                # the stencil build writes every row's diagonal entry into D
                # (0 where a row has none), whether or not the form qualified
                diag = (dA.stencil[0][64:64 + 8 * n].view(torch.float64)
                        if dA.stencil is not None else _device_diagonal(n, rp, ci, vals))
                dA = dA.with_diag(diag)
                dA._pivot_flag = (diag == 0).any()
                if check_pivot:
                    dA.raise_if_zero_pivot()
        return dA

    def raise_if_zero_pivot(self):
        """ZeroPivotError for a zero Jacobi pivot (deferred check of from_host)."""
        flag = getattr(self, "_pivot_flag", None)
        if flag is not None and bool(flag):
            import torch

            from .precond import ZeroPivotError

            zero = int(torch.nonzero(self.diag == 0)[0].item())
            raise ZeroPivotError("jacobi", zero)

    def with_diag(self, diag):
        return DeviceCsr(self.n, self.row_ptr, self.col_idx, self.values, diag, self._keep,
                         self.stencil, self.precond)

    def with_precond(self, precond):
        """The same matrix with a general preconditioner (precond.DevicePreconditioner
        or None) attached; it replaces the Jacobi diagonal in every kernel."""
        if precond is not None and precond.n != self.n:
            raise ValueError(f"preconditioner size {precond.n} does not match {self.n} rows")
        return DeviceCsr(self.n, self.row_ptr, self.col_idx, self.values,
                         None if precond is not None else self.diag, self._keep, self.stencil,
                         precond)


class _nullctx:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def _device_diagonal(n, rp, ci, vals):
    import torch

    counts = (rp[1:] - rp[:-1]).to(torch.int64)
    rows = torch.repeat_interleave(torch.arange(n, device=vals.device), counts)
    on = rows == ci.to(torch.int64)
    d = torch.zeros(n, dtype=torch.float64, device=vals.device)
    d[rows[on]] = vals[on]
    return d


def spmv(A, x):
    """y = A x on the GPU (sparse.py:155-160). Bit-exact with scipy csr_matvec."""
    import torch

    _lib.require_cuda()
    L = _lib.load()
    dA = A if isinstance(A, DeviceCsr) else DeviceCsr.from_host(CsrMatrix.of(A))
    host = not isinstance(x, torch.Tensor)
    xt = torch.as_tensor(np.asarray(x, dtype=np.float64) if host else x, dtype=torch.float64)
    if xt.shape != (dA.n,):
        raise ValueError(f"vector length {tuple(xt.shape)} does not match {dA.n} columns")
    xt = xt.to("cuda").contiguous()
    y = torch.empty_like(xt)
    _lib.check(L.skr_spmv(ctypes.byref(dA.c), xt.data_ptr(), y.data_ptr(), 0,
                          _lib.stream_handle()), "skr_spmv")
    return y.cpu().numpy() if host else y


def dot(x, y) -> float:
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise ValueError(f"length mismatch: {x.shape} vs {y.shape}")
    return float(np.dot(x, y))


def norm2(x) -> float:
    return float(np.linalg.norm(np.asarray(x, dtype=np.float64)))


def axpy(alpha: float, x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if x.shape != y.shape:
        raise ValueError(f"length mismatch: {x.shape} vs {y.shape}")
    return y + alpha * x


def as_vector(values: Sequence[float]) -> np.ndarray:
    v = np.ascontiguousarray(values, dtype=np.float64)
    if v.ndim != 1:
        raise ValueError("expected a 1-D vector")
    if not np.all(np.isfinite(v)):
        raise ValueError("vector entries must be finite")
    return v


def eye(n: int) -> CsrMatrix:
    idx = np.arange(n, dtype=np.int64)
    return CsrMatrix(n, n, np.arange(n + 1, dtype=np.int64), idx, np.ones(n))
