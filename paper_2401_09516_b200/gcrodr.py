"""GCRO-DR with a recycle space carried between systems -- device engine.

Drop-in for ``kryrec.gcrodr`` (gcrodr.py:37-44 RecycleSpace, :295-496
gcrodr_solve, :173-240 harmonic Ritz). The whole solve -- refresh of the
incoming recycle basis, restart cycles, recycle updates, explicit residuals
-- runs in libskr.so on the GPU (``skr_gcrodr_solve``); this module uploads
inputs, owns the device workspace and maps the C report back to the
reference's ``SolveReport`` and warnings.
"""

from __future__ import annotations

import ctypes
import time
import warnings
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .gmres import SolveReport, SolverConfig
from .precond import (DEVICE_KINDS, DevicePreconditioner, JacobiPreconditioner, Preconditioner,
                      build_device_preconditioner)
from .sparse import CsrMatrix, DeviceCsr

__all__ = ["RecycleSpace", "GcroDrEngine", "gcrodr_solve", "harmonic_ritz_first_cycle",
           "harmonic_ritz_subsequent", "engine_for"]


@dataclass(frozen=True)
class RecycleSpace:
    """Recycle pair op @ U = C (gcrodr.py:37-44). U, C: (n, k) torch CUDA
    tensors (column-major storage) or numpy arrays."""

    U: object
    C: object
    k: int
    source_id: Optional[object] = None

    def numpy(self) -> "RecycleSpace":
        def _np(a):
            return a.detach().cpu().numpy() if hasattr(a, "detach") else np.asarray(a)

        return RecycleSpace(_np(self.U), _np(self.C), self.k, self.source_id)


def _colmajor_device(U, n):
    """(n, k) -> (tensor, ld) with column-major device storage."""
    import torch

    if isinstance(U, torch.Tensor):
        t = U.to(device="cuda", dtype=torch.float64)
        if t.dim() != 2 or t.shape[0] != n:
            raise ValueError("recycle basis shape does not match the matrix")
        if t.stride(0) == 1 and t.stride(1) >= n:
            return t, t.stride(1)
        tt = t.t().contiguous()  # (k, n) row-major == (n, k) column-major
        return tt.t(), n
    a = np.asarray(U, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != n:
        raise ValueError("recycle basis shape does not match the matrix")
    tt = torch.from_numpy(np.ascontiguousarray(a.T)).to("cuda")
    return tt.t(), n


class GcroDrEngine:
    """Device workspace + solve loop for systems of size n under one config."""

    def __init__(self, n: int, cfg: SolverConfig, device=None):
        import torch

        self.L = _lib.load()
        self.n = int(n)
        self.cfg = cfg
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        nbytes = self.L.skr_gcrodr_workspace_bytes(self.n, cfg.m, cfg.k, cfg.max_iter)
        if nbytes == 0:
            raise ValueError(f"unsupported configuration for the device engine: {cfg}")
        self.ws = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        self.nbytes = int(nbytes)
        self.hist = np.zeros(cfg.max_iter + 2 * (cfg.k + 1) + 8)
        self.checks = np.zeros(2 * (cfg.max_iter + 2 * (cfg.k + 1) + 8))
        self.c_cfg = _lib.SkrConfig(cfg.m, cfg.k, cfg.max_iter, 0, cfg.tol)

    # -- raw solve -----------------------------------------------------------
    def solve(self, dA: DeviceCsr, b, x, x0=None, U_in=None, ldu=0, k_in=0, stream=None,
              want_history=True):
        rep = _lib.SkrReport()
        hp = self.hist.ctypes.data if want_history else None
        cp = self.checks.ctypes.data if want_history else None
        cap = len(self.hist) if want_history else 0
        st = self.L.skr_gcrodr_solve(
            ctypes.byref(dA.c), b.data_ptr(), x0.data_ptr() if x0 is not None else None,
            x.data_ptr(), ctypes.byref(self.c_cfg),
            U_in if isinstance(U_in, int) else (U_in.data_ptr() if U_in is not None else None),
            int(ldu), int(k_in), self.ws.data_ptr(), self.nbytes, ctypes.byref(rep), hp, cap,
            cp, cap, _lib.stream_handle(stream))
        _lib.check(st, "skr_gcrodr_solve")
        return rep

    def recycle_views(self):
        """(U, C, k, ld): torch views of the recycle pair left in the workspace."""
        import torch

        Up = ctypes.c_void_p()
        Cp = ctypes.c_void_p()
        k = ctypes.c_int32()
        ld = ctypes.c_int32()
        _lib.check(self.L.skr_gcrodr_recycle_view(self.ws.data_ptr(), self.nbytes, self.n,
                                                  self.cfg.m, self.cfg.k, ctypes.byref(Up),
                                                  ctypes.byref(Cp), ctypes.byref(k),
                                                  ctypes.byref(ld)), "recycle_view")
        k = k.value
        ld = ld.value
        w64 = self.ws.view(torch.float64)
        base = self.ws.data_ptr()

        def view(ptr):
            off = (ptr - base) // 8
            return w64[off: off + k * ld].view(k, ld)[:, : self.n].t()

        if k == 0:
            e = torch.zeros((self.n, 0), dtype=torch.float64, device=self.device)
            return e, e, 0, ld
        return view(Up.value), view(Cp.value), k, ld

    def u_block_ptr(self):
        return self.ws.data_ptr() + self._u_offset()

    def u_ptr_ld(self):
        """(device pointer of the U block, its leading dimension): fixed for the
        workspace, so chains read them once (no device read per system)."""
        if getattr(self, "_u_ptr_ld", None) is None:
            _, _, _, ld = self.recycle_views()
            self._u_ptr_ld = (self.u_block_ptr(), ld)
        return self._u_ptr_ld

    def _u_offset(self):
        Up = ctypes.c_void_p()
        Cp = ctypes.c_void_p()
        k = ctypes.c_int32()
        ld = ctypes.c_int32()
        _lib.check(self.L.skr_gcrodr_recycle_view(self.ws.data_ptr(), self.nbytes, self.n,
                                                  self.cfg.m, self.cfg.k, ctypes.byref(Up),
                                                  ctypes.byref(Cp), ctypes.byref(k),
                                                  ctypes.byref(ld)), "recycle_view")
        return Up.value - self.ws.data_ptr()


_ENGINES: dict = {}


def engine_for(n: int, cfg: SolverConfig, device=None, slot: int = 0,
               grid_ctas: int = 0) -> GcroDrEngine:
    """Cached engine (device workspace) per (device, n, m, k, max_iter, slot);
    concurrent chains use distinct slots and a ``grid_ctas`` share of the GPU
    (0 = the whole GPU; skr_config.grid_ctas)."""
    import torch

    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    key = (str(dev), int(n), cfg.m, cfg.k, cfg.max_iter, int(slot))
    eng = _ENGINES.get(key)
    if eng is None:
        if len(_ENGINES) > 16:
            _ENGINES.clear()
        eng = GcroDrEngine(n, cfg, dev)
        _ENGINES[key] = eng
    eng.c_cfg = _lib.SkrConfig(cfg.m, cfg.k, cfg.max_iter, int(grid_ctas), cfg.tol)
    eng.cfg = cfg
    return eng


_WARN_TEXT = {
    _lib.WARN_RANK_DROP: "dropped rank-deficient recycle columns",
    _lib.WARN_REFRESH_RANK: "recycle refresh dropped columns (rank loss)",
    _lib.WARN_SINGULAR_H: "singular Hessenberg: harmonic Ritz via generalized eigenproblem",
    _lib.WARN_SINGULAR_CROSS: "singular cross-Gram matrix: harmonic Ritz via pseudoinverse",
}


def _emit_warnings(bits: int):
    for bit, text in _WARN_TEXT.items():
        if bits & bit:
            warnings.warn(text, stacklevel=3)


def _to_device_vec(v, n, name):
    import torch

    if isinstance(v, torch.Tensor):
        t = v.to(device="cuda", dtype=torch.float64)
    else:
        a = np.asarray(v, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a)).to("cuda")
    if tuple(t.shape) != (n,):
        raise ValueError(f"{name} length mismatch")
    return t.contiguous()


def gcrodr_solve(A, b, x0=None, M: Optional[Preconditioner] = None,
                 cfg: Optional[SolverConfig] = None, recycle_in: Optional[RecycleSpace] = None,
                 system_id=None, collect_diagnostics: bool = False, *, return_device: bool = False,
                 stream=None):
    """Solve A x = b with GCRO-DR on the GPU (gcrodr.py:295-496).

    Returns ``(SolveReport, RecycleSpace)``. ``A`` may be a host CSR
    (this package's or kryrec's ``CsrMatrix``) or a ``DeviceCsr``; ``M`` is
    None or any preconditioner of ``build_preconditioner`` (none, jacobi,
    bjacobi, sor, ilu0, icc0). The recycle pair
    comes back as CUDA tensors and can be passed straight to the next call.
    """
    import torch

    cfg = cfg or SolverConfig()
    t0 = time.perf_counter()
    _lib.require_cuda()
    kind = getattr(M, "kind", "none") if M is not None else "none"
    jacobi = isinstance(M, JacobiPreconditioner) or kind == "jacobi"
    general = M if isinstance(M, DevicePreconditioner) else None
    # a preconditioner object of the reference itself (kryrec.precond.*): its
    # kind and parameters are taken over, the factorization is redone on the
    # device from A (the matrix the reference built it from)
    foreign = general is None and kind in DEVICE_KINDS
    if M is not None and not jacobi and general is None and not foreign and kind != "none":
        raise ValueError(f"unknown preconditioner kind {kind!r}")

    def jacobi_diag(host_diag):
        if isinstance(M, JacobiPreconditioner):
            return M.device_diag()
        d = getattr(M, "diag", None)
        return torch.from_numpy(np.ascontiguousarray(d if d is not None else host_diag(),
                                                     dtype=np.float64)).to("cuda")

    if isinstance(A, DeviceCsr):
        dA = A
        if general is None and dA.precond is not None:
            dA = dA.with_precond(None)
        if jacobi and dA.diag is None:
            dA = dA.with_diag(jacobi_diag(lambda: _device_diag_host(dA)))
        if not jacobi and dA.diag is not None:
            dA = dA.with_diag(None)
    else:
        host = CsrMatrix.of(A)
        if host.n_rows != host.n_cols:
            raise ValueError("gcrodr needs a square matrix")
        dA = DeviceCsr.from_host(host, jacobi=False, stream=stream)
        if jacobi:
            dA = dA.with_diag(jacobi_diag(host.diagonal))
    if foreign:
        general = build_device_preconditioner(
            dA, kind, sor_omega=float(getattr(M, "omega", 1.0)),
            bjacobi_block=int(getattr(M, "block_size", 64)), stream=stream)
    if general is not None:
        dA = dA.with_precond(general)
    n = dA.n
    bt = _to_device_vec(b, n, "right-hand side")
    x0t = _to_device_vec(x0, n, "x0") if x0 is not None else None
    eng = engine_for(n, cfg)
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    U_ptr, ldu, k_in = None, 0, 0
    if cfg.k > 0 and recycle_in is not None and recycle_in.k > 0:
        Ud, ldu = _colmajor_device(recycle_in.U, n)
        U_ptr, k_in = Ud, int(Ud.shape[1])
    refreshed = None
    if collect_diagnostics and k_in > 0:
        # the refreshed pair itself (gcrodr.py:364, diagnostics["refreshed_space"]):
        # the same solve stopped after the refresh (max_iter = k_in: the
        # refresh counts k_in iterations, gcrodr.py:363)
        keep = eng.c_cfg.max_iter
        eng.c_cfg.max_iter = k_in
        try:
            rep0 = eng.solve(dA, bt, x, x0t, U_ptr, ldu, k_in, stream=stream, want_history=False)
        finally:
            eng.c_cfg.max_iter = keep
        Ur, Cr, kr, _ = eng.recycle_views()
        refreshed = (RecycleSpace(_own_colmajor(Ur), _own_colmajor(Cr), kr, system_id)
                     if not rep0.zero_rhs else None)
    eng.c_cfg.flags = _lib.COLLECT_DIAGNOSTICS if collect_diagnostics else 0
    try:
        rep = eng.solve(dA, bt, x, x0t, U_ptr, ldu, k_in, stream=stream)
    finally:
        eng.c_cfg.flags = 0
    _emit_warnings(rep.warn_bits)
    hist = eng.hist[: rep.hist_len].copy()
    checks = [(float(eng.checks[2 * i]), float(eng.checks[2 * i + 1]))
              for i in range(rep.n_checks)]
    diag = {"restart_checks": checks, "deflated_steps": int(rep.deflated_steps),
            "recycle_k": int(rep.k_out)}
    if cfg.k == 0:
        diag["gmres_fallback"] = True
        diag["deflated_steps"] = 0
        out_space = RecycleSpace(torch.zeros((n, 0), dtype=torch.float64, device="cuda"),
                                 torch.zeros((n, 0), dtype=torch.float64, device="cuda"), 0,
                                 system_id)
    elif rep.zero_rhs:
        out_space = recycle_in or RecycleSpace(
            torch.zeros((n, 0), dtype=torch.float64, device="cuda"),
            torch.zeros((n, 0), dtype=torch.float64, device="cuda"), 0, system_id)
    else:
        U, C, k, _ = eng.recycle_views()
        if k == 0:
            diag["gmres_fallback"] = True
        # an independent copy (column-major): the RecycleSpace value must not
        # alias the engine workspace, which the next solve overwrites (with
        # ld == n a transposed .contiguous() would be a view)
        out_space = RecycleSpace(_own_colmajor(U) if k else U, _own_colmajor(C) if k else C, k,
                                 system_id)
    if collect_diagnostics:
        # gcrodr.py:372-376, :461-467, :484-485
        cap = cfg.max_iter + 2
        rec = np.zeros(4 * cap)
        nd = eng.L.skr_gcrodr_diagnostics(eng.ws.data_ptr(), eng.nbytes, n, cfg.m, cfg.k,
                                          cfg.max_iter, rec.ctypes.data, cap)
        if nd < 0:
            _lib.check(-nd, "skr_gcrodr_diagnostics")
        diag["cycles"] = [{"stage": "refresh" if rec[4 * i] == 0 else "cycle",
                           "k": int(rec[4 * i + 1]), "au_c": float(rec[4 * i + 2]),
                           "orth": float(rec[4 * i + 3])} for i in range(min(nd, cap))]
        diag["refreshed_space"] = refreshed
        if out_space.k > 0:
            diag["recycle_residuals"] = _recycle_residuals(dA, out_space)
    if rep.status_bits:
        diag["dense_status_bits"] = int(rep.status_bits)
    report = SolveReport(
        x=x if return_device else x.cpu().numpy(),
        iterations=int(rep.iterations),
        residual_history=hist,
        true_relative_residual=float(rep.true_relative_residual),
        converged=bool(rep.converged),
        wall_time=time.perf_counter() - t0,
        diagnostics=diag,
        device_ms=float(rep.device_ms),
        x_device=x,
    )
    return report, out_space


def _device_diag_host(dA):
    from .sparse import _device_diagonal

    return _device_diagonal(dA.n, dA.row_ptr, dA.col_idx, dA.values).cpu().numpy()


def _own_colmajor(X):
    """Column-major copy of an (n, k) device view."""
    import torch

    out = torch.empty((X.shape[1], X.shape[0]), dtype=X.dtype, device=X.device)
    out.copy_(X.t())
    return out.t()


def _recycle_residuals(dA: DeviceCsr, space: RecycleSpace):
    """(||op U - C||_F, ||C^T C - I||_F) (gcrodr.py:116-123), on the device."""
    import torch

    L = _lib.load()
    U, C = space.U, space.C
    opU = torch.empty_like(C.contiguous())
    for q in range(space.k):
        u = U[:, q].contiguous()
        y = torch.empty_like(u)
        _lib.check(L.skr_spmv(ctypes.byref(dA.c), u.data_ptr(), y.data_ptr(), 1,
                              _lib.stream_handle()), "skr_spmv")
        opU[:, q] = y
    rel = float(torch.linalg.norm(opU - C))
    orth = float(torch.linalg.norm(C.T @ C - torch.eye(space.k, dtype=C.dtype, device=C.device)))
    return rel, orth


def harmonic_ritz_first_cycle(H_m, h_sub: float, k: int):
    """gcrodr.py:173-206 on the device (single-CTA dense kernel). Returns P (numpy)."""
    import torch

    H = np.asarray(H_m, dtype=np.float64)
    m = H.shape[0]
    if H.shape != (m, m) or m == 0:
        raise ValueError("H_m must be square and nonempty")
    _lib.require_cuda()
    L = _lib.load()
    Hb = np.zeros((m + 1, m))
    Hb[:m] = H
    Hb[m, m - 1] = h_sub
    Hd = torch.from_numpy(np.asfortranarray(Hb).T.copy()).to("cuda")  # column-major
    P = torch.zeros((m + 2, m), dtype=torch.float64, device="cuda")
    nc = (ctypes.c_int32 * 2)()
    _lib.check(L.skr_dense_hr_first(Hd.data_ptr(), m + 1, m, int(k), P.data_ptr(), m,
                                    nc, _lib.stream_handle()), "hr_first")
    r = nc[0]
    _emit_warnings(nc[1] & (_lib.WARN_SINGULAR_H | _lib.WARN_SINGULAR_CROSS))
    if r < 0:
        raise np.linalg.LinAlgError(f"device harmonic Ritz failed (status {-r})")
    flat = P.cpu().numpy().ravel()[: m * r]
    return flat.reshape(r, m).T.copy()


def harmonic_ritz_subsequent(G, W_r_V, k: int):
    """gcrodr.py:209-240 on the device. Returns P (numpy)."""
    import torch

    G = np.asarray(G, dtype=np.float64)
    mm = G.shape[1]
    if G.shape[0] != mm + 1:
        raise ValueError("G must have shape (m+1) x m")
    X = np.asarray(W_r_V, dtype=np.float64)
    if X.shape != (mm, mm):
        raise ValueError("cross-Gram block must be m x m")
    _lib.require_cuda()
    L = _lib.load()
    Gd = torch.from_numpy(np.ascontiguousarray(G.T)).to("cuda")
    Xd = torch.from_numpy(np.ascontiguousarray(X.T)).to("cuda")
    P = torch.zeros((mm + 2, mm), dtype=torch.float64, device="cuda")
    nc = (ctypes.c_int32 * 2)()
    _lib.check(L.skr_dense_hr_next(Gd.data_ptr(), mm + 1, Xd.data_ptr(), mm, mm, int(k),
                                   P.data_ptr(), mm, nc, _lib.stream_handle()),
               "hr_next")
    r = nc[0]
    _emit_warnings(nc[1] & (_lib.WARN_SINGULAR_H | _lib.WARN_SINGULAR_CROSS))
    if r < 0:
        raise np.linalg.LinAlgError(f"device harmonic Ritz failed (status {-r})")
    flat = P.cpu().numpy().ravel()[: mm * r]
    return flat.reshape(r, mm).T.copy()
