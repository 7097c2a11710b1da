"""Left preconditioners: none, Jacobi, block Jacobi, SOR, ILU(0), IC(0).

Mirrors ``kryrec.precond`` (precond.py:24-312): the same class names, ``kind``
strings, constructor errors (``ZeroPivotError``, ``ValueError``) and the
``apply(v)`` = "solve M z = v" contract. The Jacobi diagonal is applied inside
the CUDA kernels as an IEEE division (v / diag), the reference's arithmetic.
The other kinds are analysed and factored on the device (``skr_precond_build``,
csrc/precond.cu): dependency levels of the triangular sweeps, the ILU(0) /
IC(0) factor on A's own pattern in the reference's operation order (the factor
values are bit-identical to the reference's), ``M = D / omega + L`` for SOR, a
dense LU with partial pivoting per diagonal block for block Jacobi. Their
``apply`` (standalone and inside ``gcrodr_solve`` / ``gmres_solve``) is a
level-scheduled sparse triangular sweep on the GPU; the reference applies the
same factors through SuperLU, so applies agree to rounding, not bitwise.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .sparse import CsrMatrix, DeviceCsr

KINDS = ("none", "jacobi", "bjacobi", "sor", "ilu0", "icc0")
SUPPORTED = KINDS
DEVICE_KINDS = ("bjacobi", "sor", "ilu0", "icc0")
BJACOBI_MAX_BLOCK = 256


class ZeroPivotError(ValueError):
    """Factorization hit a zero (or, for IC, nonpositive) pivot (precond.py:24-31)."""

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


class DevicePreconditioner(Preconditioner):
    """A factorization living on the GPU (SOR, ILU(0), IC(0), block Jacobi).

    ``matrix`` is the ``DeviceCsr`` it was built from (its pattern arrays are
    referenced by the factor and kept alive here); ``buffer`` the device bytes
    written by ``skr_precond_build``."""

    def __init__(self, matrix: DeviceCsr, buffer, layout):
        super().__init__(matrix.n)
        self.matrix = matrix
        self.buffer = buffer
        self._layout = layout  # (kind id, n, nnz, block)

    def apply(self, v):
        """Solve M z = v on the GPU. A vector (n,) or a block of columns (n, m);
        numpy in -> numpy out, CUDA tensor in -> CUDA tensor out."""
        import torch

        host = not isinstance(v, torch.Tensor)
        vt = torch.as_tensor(np.asarray(v, dtype=np.float64) if host else v,
                             dtype=torch.float64)
        if vt.ndim not in (1, 2) or vt.shape[0] != self.n:
            raise ValueError(f"expected {self.n} rows, got shape {tuple(vt.shape)}")
        cols = 1 if vt.ndim == 1 else int(vt.shape[1])
        # column-major block on the device (leading dimension n)
        work = vt.to("cuda").reshape(self.n, cols).t().contiguous()
        L = _lib.load()
        _lib.check(L.skr_precond_apply(self.buffer.data_ptr(), work.data_ptr(), work.data_ptr(),
                                       cols, self.n, self.n, _lib.stream_handle()),
                   "skr_precond_apply")
        out = work.t().reshape(vt.shape)
        return out.cpu().numpy() if host else out.contiguous()

    # -- the factor as host CSR triangles (the reference keeps these as attributes)
    def _factor_values(self) -> np.ndarray:
        import torch

        kind, n, nnz, _ = self._layout
        off = 256 * ((_HEADER_BYTES + 255) // 256)
        return self.buffer[off:off + 8 * nnz].view(torch.float64).cpu().numpy()

    def _triangle(self, which: str, unit_diag: bool = False) -> CsrMatrix:
        rp = self.matrix.row_ptr.cpu().numpy().astype(np.int64)
        ci = self.matrix.col_idx.cpu().numpy().astype(np.int64)
        fv = self._factor_values()
        rows = np.repeat(np.arange(self.n), np.diff(rp))
        if which == "lower":
            keep = ci <= rows if not unit_diag else ci < rows
        else:
            keep = ci >= rows
        r, c, v = rows[keep], ci[keep], fv[keep]
        if unit_diag:
            r = np.concatenate([r, np.arange(self.n)])
            c = np.concatenate([c, np.arange(self.n)])
            v = np.concatenate([v, np.ones(self.n)])
        order = np.lexsort((c, r))
        r, c, v = r[order], c[order], v[order]
        ptr = np.zeros(self.n + 1, dtype=np.int64)
        np.add.at(ptr, r + 1, 1)
        return CsrMatrix(self.n, self.n, np.cumsum(ptr), c, v, validate=False)


_HEADER_BYTES = 1024  # >= sizeof(PcHeader); the factor values start at the next 256-byte line


class BlockJacobiPreconditioner(DevicePreconditioner):
    kind = "bjacobi"

    def __init__(self, matrix, buffer, layout, block_size: int):
        super().__init__(matrix, buffer, layout)
        self.block_size = int(block_size)


class SorPreconditioner(DevicePreconditioner):
    """Forward SOR sweep: M = D/omega + L with L the strict lower part of A."""

    kind = "sor"

    def __init__(self, matrix, buffer, layout, omega: float):
        super().__init__(matrix, buffer, layout)
        self.omega = float(omega)


class Ilu0Preconditioner(DevicePreconditioner):
    """No-fill incomplete LU; factor pattern is a subset of A's pattern."""

    kind = "ilu0"

    @property
    def lower(self) -> CsrMatrix:  # unit lower triangular (diagonal stored as 1)
        return self._triangle("lower", unit_diag=True)

    @property
    def upper(self) -> CsrMatrix:
        return self._triangle("upper")


class Icc0Preconditioner(DevicePreconditioner):
    """No-fill incomplete Cholesky, M = sign * L L^T (sign = -1 when A had an
    all-negative diagonal: the factorization then runs on -A)."""

    kind = "icc0"

    def __init__(self, matrix, buffer, layout, sign: float):
        super().__init__(matrix, buffer, layout)
        self.sign = float(sign)

    @property
    def lower(self) -> CsrMatrix:
        return self._triangle("lower")


def build_device_preconditioner(dA: DeviceCsr, kind: str, *, sor_omega: float = 1.0,
                                bjacobi_block: int = 64, stream=None,
                                check: bool = True) -> DevicePreconditioner:
    """precond.py:251-312 for the device kinds, from a device-resident matrix.

    ``check=False`` skips the host read of the build status (no stream
    synchronisation; a failed factorization then shows up as a non-converged
    solve instead of ``ZeroPivotError``)."""
    import torch

    _lib.require_cuda()
    kind = kind.lower()
    if kind not in DEVICE_KINDS:
        raise ValueError(f"unknown device preconditioner kind {kind!r}")
    kid = _lib.PC_KINDS[kind]
    omega, bs = float(sor_omega), int(bjacobi_block)
    if kind == "bjacobi":
        if bs < 1:
            raise ValueError("bjacobi block size must be >= 1")
        if bs > BJACOBI_MAX_BLOCK:
            raise _lib.SkrExtensionError(
                f"bjacobi block size {bs} exceeds the compiled limit {BJACOBI_MAX_BLOCK}")
    if kind == "sor" and not 0.0 < omega < 2.0:
        raise ValueError(f"SOR omega must lie in (0, 2), got {omega}")
    L = _lib.load()
    nbytes = int(L.skr_precond_bytes(kid, dA.n, dA.nnz, bs))
    if nbytes == 0 or nbytes < _HEADER_BYTES:
        raise _lib.SkrExtensionError("skr_precond_bytes rejected the configuration")
    buf = torch.empty(nbytes, dtype=torch.uint8, device=dA.values.device)
    info = (ctypes.c_int32 * 2)(0, 0)
    val = ctypes.c_double(0.0)
    plain = _lib.SkrCsr(dA.n, dA.nnz, dA.row_ptr.data_ptr(), dA.col_idx.data_ptr(),
                        dA.values.data_ptr(), None, None, 0, 0, None, 0)
    _lib.check(L.skr_precond_build(ctypes.byref(plain), kid, omega, bs, buf.data_ptr(), nbytes,
                                   info if check else None,
                                   ctypes.byref(val) if check else None,
                                   _lib.stream_handle(stream)), "skr_precond_build")
    if check:
        if info[0] == 1:
            raise ZeroPivotError(kind, info[1], val.value)
        if info[0] == 2:
            raise ValueError("icc0 requires a symmetric matrix (pattern and values)")
    layout = (kid, dA.n, dA.nnz, bs)
    if kind == "bjacobi":
        return BlockJacobiPreconditioner(dA, buf, layout, bs)
    if kind == "sor":
        return SorPreconditioner(dA, buf, layout, omega)
    if kind == "ilu0":
        return Ilu0Preconditioner(dA, buf, layout)
    # the sign the device chose: -1 iff every diagonal entry is negative
    diag_neg = bool((_diag_of(dA) < 0).all()) if check else False
    return Icc0Preconditioner(dA, buf, layout, -1.0 if diag_neg else 1.0)


def _diag_of(dA: DeviceCsr):
    from .sparse import _device_diagonal

    return dA.diag if dA.diag is not None else _device_diagonal(dA.n, dA.row_ptr, dA.col_idx,
                                                                dA.values)


def build_preconditioner(A, kind: str, *, sor_omega: float = 1.0,
                         bjacobi_block: int = 64) -> Preconditioner:
    """Factor A for the requested preconditioner kind (precond.py:251-312).

    ``kind`` is one of ``none | jacobi | bjacobi | sor | ilu0 | icc0``. ``A`` is
    a host ``CsrMatrix`` (uploaded here) or a ``DeviceCsr``."""
    dev = A if isinstance(A, DeviceCsr) else None
    if dev is None:
        A = CsrMatrix.of(A)
        if A.n_rows != A.n_cols:
            raise ValueError(f"preconditioner needs a square matrix, got {A.shape}")
    kind = kind.lower()
    n = dev.n if dev is not None else A.n_rows
    if kind == "none":
        return IdentityPreconditioner(n)
    if kind == "jacobi":
        diag = _diag_of(dev).cpu().numpy() if dev is not None else A.diagonal()
        zero = np.flatnonzero(diag == 0.0)
        if len(zero):
            raise ZeroPivotError("jacobi", zero[0])
        return JacobiPreconditioner(diag)
    if kind in DEVICE_KINDS:
        if kind == "bjacobi" and int(bjacobi_block) < 1:
            raise ValueError("bjacobi block size must be >= 1")
        if kind == "sor" and not 0.0 < float(sor_omega) < 2.0:
            raise ValueError(f"SOR omega must lie in (0, 2), got {float(sor_omega)}")
        _lib.require_cuda()  # the factorization lives on the device: no CPU fallback
        if dev is None:
            dev = DeviceCsr.from_host(A)
        return build_device_preconditioner(dev, kind, sor_omega=sor_omega,
                                           bjacobi_block=bjacobi_block)
    raise ValueError(f"unknown preconditioner kind {kind!r}; expected one of {KINDS}")
