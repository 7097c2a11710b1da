"""CPU oracle for the SKR hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU reference. The product (``paper_2401_09516_b200``) never calls
it; its solver runs on the CUDA extension or fails.

This is a numpy/scipy restatement of the reference package ``kryrec`` v0.1.0
(``/root/reference/pkg/src/kryrec``), written to perform the same floating
point operations in the same order, so that on the same inputs it reproduces
the reference bit for bit (pinned by ``tests/test_oracle_golden.py`` against
fixtures generated from the real reference by ``tests/golden/make_golden.py``).
The arithmetic itself lives in scipy sparsetools (CSR matvec), OpenBLAS and
LAPACK (dgeqp3, dgeev, dggev, dgelsd, dtrtrs, dgesdd, dgesv) exactly as in the
reference (numpy 2.3.5, scipy 1.18.1, scipy-openblas 0.3.30 in this image).

Citations are ``file:line`` into ``/root/reference/pkg/src/kryrec``.
"""

from __future__ import annotations

import time
import warnings
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

RANK_RTOL = 1e-12  # gcrodr.py:33
PAIR_IMAG_RTOL = 1e-12  # gcrodr.py:34
BREAKDOWN_RTOL = 1e-14  # gmres.py:22
REORTH_RTOL = 1e-8  # gmres.py:23


# --------------------------------------------------------------------------
# sort (sorting.py:45-80)
# --------------------------------------------------------------------------
def greedy_order(flat: np.ndarray) -> list[int]:
    """Greedy nearest-neighbour chain from row 0 (sorting.py:55-69, :72-80).

    Distances are ``np.linalg.norm(axis=1)`` of the row differences (numpy
    pairwise summation, zero start); the first minimum over the unvisited rows
    in ascending index order wins.
    """
    flat = np.asarray(flat, dtype=np.float64)
    n = flat.shape[0]
    if n == 0:
        raise ValueError("empty parameter batch")
    visited = np.zeros(n, dtype=bool)
    visited[0] = True
    chain = [0]
    for _ in range(n - 1):
        cand = np.flatnonzero(~visited)
        d = np.linalg.norm(flat[cand] - flat[chain[-1]], axis=1)
        nxt = int(cand[int(np.argmin(d))])
        visited[nxt] = True
        chain.append(nxt)
    return chain


def grouped_order(flat: np.ndarray, group_size: int) -> list[int]:
    """Greedy sort within coarse groups (sorting.py:83-111).

    Rows are bucketed by their coordinate along the first principal direction
    (right singular vector of the centered batch, sign fixed so its largest-
    magnitude component is positive, sorting.py:99-104), stable-argsorted,
    cut into contiguous groups of ``group_size``; each group (ascending
    original indices) is greedy-chained from its smallest index
    (sorting.py:55-69) and the chains are concatenated (sorting.py:106-110).
    """
    if group_size < 2:
        raise ValueError("group_size must be >= 2")
    flat = np.asarray(flat, dtype=np.float64)
    n = flat.shape[0]
    if n <= group_size:
        return greedy_order(flat)
    centered = flat - flat.mean(axis=0)
    _, _, vt = np.linalg.svd(centered, full_matrices=False)
    direction = vt[0]
    lead = np.argmax(np.abs(direction))
    if direction[lead] < 0:
        direction = -direction
    key = centered @ direction
    by_key = np.argsort(key, kind="stable")
    order: list[int] = []
    for start in range(0, n, group_size):
        group = np.sort(by_key[start:start + group_size])
        sub = greedy_order(flat[group])
        order.extend(int(group[i]) for i in sub)
    return order


def greedy_order_prefix(flat: np.ndarray, npos: int) -> list[int]:
    """The first ``npos`` positions of greedy_order (the chain is sequential, so
    a prefix costs npos passes instead of n); same arithmetic."""
    flat = np.asarray(flat, dtype=np.float64)
    n = flat.shape[0]
    visited = np.zeros(n, dtype=bool)
    visited[0] = True
    chain = [0]
    while len(chain) < min(npos, n):
        cand = np.flatnonzero(~visited)
        d = np.linalg.norm(flat[cand] - flat[chain[-1]], axis=1)
        nxt = int(cand[int(np.argmin(d))])
        visited[nxt] = True
        chain.append(nxt)
    return chain


def greedy_order_from_d2(D2: np.ndarray) -> list[int]:
    """Greedy chain from a precomputed squared-distance matrix (sqrt, first
    minimum) -- checker for the sharded-gather plumbing."""
    D2 = np.asarray(D2, dtype=np.float64)
    n = D2.shape[0]
    visited = np.zeros(n, dtype=bool)
    visited[0] = True
    chain = [0]
    for _ in range(n - 1):
        cand = np.flatnonzero(~visited)
        nxt = int(cand[int(np.argmin(np.sqrt(D2[chain[-1], cand])))])
        visited[nxt] = True
        chain.append(nxt)
    return chain


def pairwise_sum(a: np.ndarray) -> float:
    """numpy's float64 pairwise summation (blocks of 128, 8 accumulators).

    Restates numpy's ``pairwise_sum_DOUBLE`` (the kernel behind
    ``np.add.reduce`` on a contiguous row, which ``np.linalg.norm(axis=1)``
    uses at ``sorting.py:65``), starting from 0.0.
    """
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    if n < 8:
        s = 0.0
        for v in a:
            s += float(v)
        return s
    if n <= 128:
        r = [float(v) for v in a[:8]]
        i = 8
        stop = n - (n % 8)
        while i < stop:
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            s += float(a[i])
            i += 1
        return s
    half = n // 2
    half -= half % 8
    return pairwise_sum(a[:half]) + pairwise_sum(a[half:])


def reference_distance(p: np.ndarray, q: np.ndarray) -> float:
    """sqrt(pairwise_sum((p-q)^2)) -- the reference's per-candidate distance."""
    d = np.asarray(p, np.float64) - np.asarray(q, np.float64)
    return float(np.sqrt(0.0 + pairwise_sum(d * d)))


# --------------------------------------------------------------------------
# operator (sparse.py:76-83, gmres.py:184-190, precond.py:59-77)
# --------------------------------------------------------------------------
class Operator:
    """op(v) = M^{-1}(A v) with M = I, diag(A) or a general preconditioner
    (``prec``: a ``GeneralPrec``); blocks act column-wise."""

    def __init__(self, row_ptr, col_idx, values, n, jacobi: bool, prec=None):
        self.n = int(n)
        self.S = sp.csr_matrix(
            (np.asarray(values, np.float64), np.asarray(col_idx, np.int64),
             np.asarray(row_ptr, np.int64)), shape=(self.n, self.n))
        self.diag = self.S.diagonal() if jacobi else None
        self.general = prec
        if self.diag is not None and np.any(self.diag == 0.0):
            raise ValueError("jacobi: zero pivot")  # precond.py:153-158

    def prec(self, v):
        v = np.asarray(v, dtype=np.float64)
        if self.general is not None:
            return self.general.apply(v)
        if self.diag is None:
            return np.array(v, dtype=np.float64, copy=True)
        return v / (self.diag if v.ndim == 1 else self.diag[:, None])

    def __call__(self, v):
        if self.diag is None and self.general is None:
            return self.S @ v
        return self.prec(self.S @ v)


# --------------------------------------------------------------------------
# general preconditioners (precond.py:80-145, :161-312)
# --------------------------------------------------------------------------
class ZeroPivot(ValueError):
    def __init__(self, kind, row, value=0.0):
        self.kind, self.row, self.value = kind, int(row), float(value)
        super().__init__(f"{kind}: zero pivot at row {self.row} (value {value:g})")


def ilu0_values(row_ptr, col_idx, values):
    """IKJ ILU(0) on A's own pattern (precond.py:170-216): the factor as values
    on the pattern (multipliers l_ik left of the diagonal, U from it on). The
    same scalar operations in the same order as the reference's loops."""
    ptr = np.asarray(row_ptr, np.int64)
    col = np.asarray(col_idx, np.int64)
    val = np.array(values, dtype=np.float64)
    n = len(ptr) - 1
    pos = [{int(c): q for q, c in enumerate(col[ptr[i]:ptr[i + 1]], start=int(ptr[i]))}
           for i in range(n)]
    dpos = np.empty(n, dtype=np.int64)
    for i in range(n):
        q = pos[i].get(i, -1)
        if q < 0 or val[q] == 0.0:
            raise ZeroPivot("ilu0", i)
        dpos[i] = q
    for i in range(n):
        lo, hi = int(ptr[i]), int(ptr[i + 1])
        for p in range(lo, hi):
            k = int(col[p])
            if k >= i:
                break
            pivot = val[dpos[k]]
            if pivot == 0.0:
                raise ZeroPivot("ilu0", k)
            lik = val[p] / pivot
            val[p] = lik
            rk = pos[k]
            for q in range(p + 1, hi):
                pk = rk.get(int(col[q]))
                if pk is not None:
                    val[q] -= lik * val[pk]
    for i in range(n):
        if val[dpos[i]] == 0.0:
            raise ZeroPivot("ilu0", i)
    return val, dpos


def icc0_values(row_ptr, col_idx, values, sign):
    """IC(0) of sign * A on the lower triangle of A's pattern
    (precond.py:219-248): L as values on the pattern positions j <= i."""
    ptr = np.asarray(row_ptr, np.int64)
    col = np.asarray(col_idx, np.int64)
    aval = np.asarray(values, np.float64)
    n = len(ptr) - 1
    rows = [dict() for _ in range(n)]
    out = np.zeros(len(aval))
    for i in range(n):
        li = rows[i]
        for p in range(int(ptr[i]), int(ptr[i + 1])):
            j = int(col[p])
            if j > i:
                break
            a_ij = sign * aval[p]
            if j < i:
                lj = rows[j]
                s = a_ij
                for k, lik in li.items():
                    ljk = lj.get(k)
                    if ljk is not None:
                        s -= lik * ljk
                li[j] = s / lj[j]
                out[p] = li[j]
            else:
                d = a_ij - sum(x * x for k, x in li.items() if k < i)
                if d <= 0.0:
                    raise ZeroPivot("icc0", i, d)
                li[i] = float(np.sqrt(d))
                out[p] = li[i]
    return out


class GeneralPrec:
    """solve M z = v for M of kind sor | ilu0 | icc0 | bjacobi
    (precond.py:80-145). The reference hands the triangular factors to
    non-pivoting SuperLU; here they are solved by scipy's substitution, which
    agrees with it to rounding (pinned at 1e-12 by tests/golden/precond.npz)."""

    def __init__(self, row_ptr, col_idx, values, n, kind, sor_omega=1.0, bjacobi_block=64):
        import scipy.sparse.linalg as spla

        self.kind = kind
        self.n = int(n)
        S = sp.csr_matrix((np.asarray(values, np.float64), np.asarray(col_idx, np.int64),
                           np.asarray(row_ptr, np.int64)), shape=(n, n))
        rows = np.repeat(np.arange(n), np.diff(np.asarray(row_ptr, np.int64)))
        col = np.asarray(col_idx, np.int64)
        tri = lambda M, lower: (lambda v: spla.spsolve_triangular(  # noqa: E731
            sp.csr_matrix(M), v, lower=lower))
        if kind == "sor":  # precond.py:285-292
            diag = S.diagonal()
            if np.any(diag == 0.0):
                raise ZeroPivot("sor", np.flatnonzero(diag == 0.0)[0])
            M = sp.tril(S, k=-1, format="csr") + sp.diags(diag / float(sor_omega), format="csr")
            self._steps = [tri(M, True)]
            self.scale = 1.0
        elif kind == "ilu0":  # precond.py:294-297
            fv, _ = ilu0_values(row_ptr, col_idx, values)
            self.factor = fv
            lo = col < rows
            Lm = sp.csr_matrix((fv[lo], (rows[lo], col[lo])), shape=(n, n)) + sp.identity(n)
            Um = sp.csr_matrix((fv[~lo], (rows[~lo], col[~lo])), shape=(n, n))
            self._steps = [tri(Lm, True), tri(Um, False)]
            self.scale = 1.0
        elif kind == "icc0":  # precond.py:299-306
            if abs(S - S.T).nnz != 0:
                raise ValueError("icc0 requires a symmetric matrix (pattern and values)")
            diag = S.diagonal()
            if np.any(diag == 0.0):
                raise ZeroPivot("icc0", np.flatnonzero(diag == 0.0)[0])
            self.scale = -1.0 if np.all(diag < 0.0) else 1.0
            fv = icc0_values(row_ptr, col_idx, values, self.scale)
            self.factor = fv
            lo = col <= rows
            Lm = sp.csr_matrix((fv[lo], (rows[lo], col[lo])), shape=(n, n))
            self._steps = [tri(Lm, True), tri(sp.csr_matrix(Lm.T), False)]
        elif kind == "bjacobi":  # precond.py:270-283
            bs = int(bjacobi_block)
            fac = []
            for start in range(0, n, bs):
                end = min(n, start + bs)
                lu, piv = sla.lu_factor(S[start:end, start:end].toarray(), check_finite=False)
                bad = np.flatnonzero(np.diag(lu) == 0.0)
                if len(bad):
                    raise ZeroPivot("bjacobi", start + bad[0])
                fac.append((start, end, lu, piv))

            def blocks(v):
                z = np.empty_like(v)
                for start, end, lu, piv in fac:
                    z[start:end] = sla.lu_solve((lu, piv), v[start:end])
                return z

            self._steps = [blocks]
            self.scale = 1.0
        else:
            raise ValueError(f"unknown preconditioner kind {kind!r}")

    def apply(self, v):
        z = np.asarray(v, dtype=np.float64)
        for f in self._steps:
            z = f(z)
        return self.scale * z if self.scale != 1.0 else z


# --------------------------------------------------------------------------
# dense helpers (gcrodr.py:56-240)
# --------------------------------------------------------------------------
def qrcp_rank(W, rtol=RANK_RTOL):
    """Pivoted economic QR truncated at numerical rank (gcrodr.py:56-67)."""
    Q, R, piv = sla.qr(W, mode="economic", pivoting=True, check_finite=False)
    d = np.abs(np.diag(R))
    if d.size == 0 or d[0] == 0.0:
        return Q[:, :0], R[:0, :0], piv[:0]
    r = int(np.sum(d >= rtol * d[0]))
    return Q[:, :r], R[:r, :r], piv[:r]


def _inv_upper(R):
    return sla.solve_triangular(R, np.eye(R.shape[0]), check_finite=False)


def refresh(U_in, op: Operator):
    """Re-anchor U against the new operator (gcrodr.py:80-113). -> (U, C)."""
    Y = np.asarray(U_in, dtype=np.float64)
    Yo, _, _ = qrcp_rank(Y)
    if Yo.shape[1] < Y.shape[1]:
        warnings.warn("dropped rank-deficient recycle columns", stacklevel=2)
    if Yo.shape[1] == 0:
        return None, None
    W = np.asarray(op(Yo), dtype=np.float64)
    Q, R, kept = qrcp_rank(W)
    if Q.shape[1] == 0:
        return None, None
    if Q.shape[1] < Yo.shape[1]:
        warnings.warn("recycle refresh rank loss", stacklevel=2)
    return Yo[:, kept] @ _inv_upper(R), Q


def select_basis(vals, vecs, k, max_cols=None):
    """Real basis of the k smallest-|theta| invariant subspace (gcrodr.py:126-170)."""
    vals = np.asarray(vals, dtype=complex)
    ok = np.isfinite(vals.real) & np.isfinite(vals.imag)
    mags = np.where(ok, np.abs(vals), np.inf)
    taken = np.zeros(vals.shape[0], dtype=bool)
    cols = []
    for i in np.argsort(mags, kind="stable"):
        if taken[i] or not ok[i]:
            continue
        if len(cols) >= k:
            break
        lam, v = vals[i], vecs[:, i]
        taken[i] = True
        if abs(lam.imag) > PAIR_IMAG_RTOL * max(abs(lam), 1.0):
            gap = np.abs(vals - np.conj(lam))
            gap[taken | ~ok] = np.inf
            j = int(np.argmin(gap))
            if np.isfinite(gap[j]):
                taken[j] = True
            cols += [np.real(v), np.imag(v)]
        else:
            cols.append(np.real(v))
    if not cols:
        raise np.linalg.LinAlgError("no finite eigenvalues to deflate with")
    P = np.column_stack(cols)
    if max_cols is not None and P.shape[1] > max_cols:
        P = P[:, :max_cols]
    return qrcp_rank(P)[0]


def hr_first(Hs, hsub, k):
    """First-cycle harmonic Ritz basis (gcrodr.py:173-206)."""
    H = np.asarray(Hs, dtype=np.float64)
    m = H.shape[0]
    if m == 0 or H.shape != (m, m):
        raise ValueError("H_m must be square and nonempty")
    k = min(k, m)
    em = np.zeros(m)
    em[-1] = 1.0
    sv = sla.svdvals(H)
    if sv[0] == 0.0 or sv[-1] < 1e-14 * sv[0]:
        warnings.warn("singular Hessenberg: generalized harmonic Ritz", stacklevel=2)
        vals, vecs = sla.eig(H.T @ H + (hsub * hsub) * np.outer(em, em), H.T,
                             check_finite=False)
    else:
        f = sla.solve(H.T, em, check_finite=False)
        Hm = H.copy()
        Hm[:, m - 1] += (hsub * hsub) * f
        vals, vecs = np.linalg.eig(Hm)
    return select_basis(vals, vecs, k, max_cols=m)


def hr_next(G, cross, k):
    """Subsequent-cycle harmonic Ritz basis (gcrodr.py:209-240)."""
    G = np.asarray(G, dtype=np.float64)
    mm = G.shape[1]
    if G.shape[0] != mm + 1:
        raise ValueError("G must have shape (m+1) x m")
    cross = np.asarray(cross, dtype=np.float64)
    if cross.shape != (mm, mm):
        raise ValueError("cross-Gram block must be m x m")
    k = min(k, mm)
    lhs = G.T @ G
    rhs = G[:mm, :].T @ cross
    sv = sla.svdvals(rhs)
    if sv[0] == 0.0 or sv[-1] < 1e-14 * sv[0]:
        warnings.warn("singular cross-Gram: pseudoinverse", stacklevel=2)
        vals, vecs = np.linalg.eig(np.linalg.pinv(rhs) @ lhs)
    else:
        vals, vecs = sla.eig(lhs, rhs, check_finite=False)
    return select_basis(vals, vecs, k, max_cols=mm)


# --------------------------------------------------------------------------
# Arnoldi pieces (gmres.py:69-88, :125-181; gcrodr.py:243-257)
# --------------------------------------------------------------------------
def mgs_into(V, ncols, w, h):
    """MGS of w against V[:, :ncols] with the conditional second sweep (gmres.py:69-88)."""
    w0 = float(np.linalg.norm(w))
    for i in range(ncols):
        c = float(np.dot(V[:, i], w))
        w -= c * V[:, i]
        h[i] += c
    if ncols and w0 > 0.0:
        if float(np.linalg.norm(V[:, :ncols].T @ w)) > REORTH_RTOL * w0:
            for i in range(ncols):
                c = float(np.dot(V[:, i], w))
                w -= c * V[:, i]
                h[i] += c
    return w0


def gmres_cycle(op, r0, beta, m, abs_tol, max_steps):
    """One GMRES(m) cycle with Givens least squares (gmres.py:125-181)."""
    n = r0.shape[0]
    steps = min(m, max_steps)
    V = np.zeros((n, steps + 1))
    H = np.zeros((steps + 1, steps))
    R = np.zeros((steps + 1, steps))
    cs = np.zeros(steps)
    sn = np.zeros(steps)
    g = np.zeros(steps + 1)
    g[0] = beta
    V[:, 0] = r0 / beta
    res = []
    brk = False
    j = 0
    while j < steps:
        w = np.asarray(op(V[:, j]), dtype=np.float64)
        w0 = mgs_into(V, j + 1, w, H[:, j])
        hn = float(np.linalg.norm(w))
        H[j + 1, j] = hn
        if hn < BREAKDOWN_RTOL * max(w0, np.finfo(float).tiny):
            brk = True
        else:
            V[:, j + 1] = w / hn
        col = R[:, j]
        col[: j + 2] = H[: j + 2, j]
        for i in range(j):
            t = cs[i] * col[i] + sn[i] * col[i + 1]
            col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
            col[i] = t
        den = float(np.hypot(col[j], col[j + 1]))
        if den == 0.0:
            cs[j], sn[j] = 1.0, 0.0
        else:
            cs[j], sn[j] = col[j] / den, col[j + 1] / den
        col[j] = den
        col[j + 1] = 0.0
        g[j + 1] = -sn[j] * g[j]
        g[j] = cs[j] * g[j]
        res.append(abs(g[j + 1]))
        j += 1
        if brk or res[-1] <= abs_tol:
            break
    y = sla.solve_triangular(R[:j, :j], g[:j], check_finite=False)
    return V[:, : j + 1], H[: j + 1, :j], j, res, y, brk


def deflated_step(op, C, V, H, B, j):
    """(I - C C^T) op Arnoldi step (gcrodr.py:243-257); returns breakdown."""
    w = np.asarray(op(V[:, j]), dtype=np.float64)
    if C.shape[1]:
        c = C.T @ w
        B[:, j] = c
        w -= C @ c
    w0 = mgs_into(V, j + 1, w, H[:, j])
    hn = float(np.linalg.norm(w))
    H[j + 1, j] = hn
    if hn < BREAKDOWN_RTOL * max(w0, np.finfo(float).tiny):
        return True
    V[:, j + 1] = w / hn
    return False


def first_cycle_pair(V, H, j, k):
    """(U, C) from a fresh GMRES factorisation (gcrodr.py:280-292)."""
    try:
        P = hr_first(H[:j, :j], float(H[j, j - 1]), min(k, j))
    except (np.linalg.LinAlgError, ValueError):
        return None, None
    Y = V[:, :j] @ P
    Q, R, kept = qrcp_rank(H @ P)
    if Q.shape[1] == 0:
        return None, None
    return Y[:, kept] @ _inv_upper(R), V @ Q


# --------------------------------------------------------------------------
# solver (gmres.py:26-56, gcrodr.py:295-496)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Cfg:
    m: int = 50
    tol: float = 1e-8
    max_iter: int = 10000
    k: int = 10


@dataclass
class Result:
    x: np.ndarray
    iterations: int
    history: np.ndarray
    true_rel: float
    converged: bool
    wall_time: float
    U: np.ndarray | None
    C: np.ndarray | None
    info: dict = field(default_factory=dict)


def recycle_residuals(U, C, op):
    """(||op U - C||_F, ||C^T C - I||_F) (gcrodr.py:116-123)."""
    if U is None or U.shape[1] == 0:
        return 0.0, 0.0
    opU = np.column_stack([op(U[:, q]) for q in range(U.shape[1])])
    return (float(np.linalg.norm(opU - C, "fro")),
            float(np.linalg.norm(C.T @ C - np.eye(C.shape[1]), "fro")))


def gcrodr(op: Operator, b, cfg: Cfg, U_in=None, x0=None, trace=None, deadline=None,
           collect_diagnostics=False) -> Result:
    """GCRO-DR solve with a carried recycle basis (gcrodr.py:295-496).

    ``U_in`` is the previous system's recycle U (its C is discarded by the
    refresh, gcrodr.py:361-366). Returns the new (U, C) in ``Result``.
    """
    t0 = time.perf_counter()
    n = op.n
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (n,):
        raise ValueError("right-hand side length mismatch")
    if cfg.k == 0:
        return gmres(op, b, cfg, x0=x0)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    S = op.S
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:  # gcrodr.py:337-346
        U_pass = None if U_in is None else np.asarray(U_in)
        return Result(np.zeros(n), 0, np.zeros(1), 0.0, True,
                      time.perf_counter() - t0, U_pass, None, {"zero_rhs": True})
    abs_tol = cfg.tol * float(np.linalg.norm(op.prec(b)))
    r = op.prec(b - S @ x) if np.any(x) else op.prec(b)
    rnorm = float(np.linalg.norm(r))
    hist = [rnorm]
    checks = []
    iters = 0
    U = C = None
    defl = 0
    cyc_diag = []
    refreshed = None
    if U_in is not None and np.asarray(U_in).shape[1] > 0:
        U, C = refresh(U_in, op)
        iters += np.asarray(U_in).shape[1]
        refreshed = (U, C)
        if collect_diagnostics:  # gcrodr.py:372-376
            rel, orth = recycle_residuals(U, C, op)
            cyc_diag.append({"stage": "refresh", "k": 0 if U is None else U.shape[1],
                             "au_c": rel, "orth": orth})
        if U is not None:
            a = C.T @ r
            x = x + U @ a
            r = r - C @ a
            rnorm = float(np.linalg.norm(r))
            hist.append(rnorm)
    conv = rnorm <= abs_tol
    while not conv and iters < cfg.max_iter:
        # bench samples only: stop at a cycle boundary once the deadline passed
        if deadline is not None and time.perf_counter() >= deadline:
            break
        if U is None:
            V, H, j, sres, y, brk = gmres_cycle(op, r, rnorm, cfg.m, abs_tol,
                                                 cfg.max_iter - iters)
            iters += j
            hist.extend(sres)
            x += V[:, :j] @ y
            r = op.prec(b - S @ x)
            rnorm = float(np.linalg.norm(r))
            checks.append((sres[-1], rnorm))
            conv = rnorm <= abs_tol
            U, C = first_cycle_pair(V, H, j, cfg.k)
            if brk and not conv:
                break
            continue
        kc = U.shape[1]
        nsteps = min(max(1, cfg.m - kc), cfg.max_iter - iters)
        un = np.linalg.norm(U, axis=0)
        un[un == 0.0] = 1.0
        dk = 1.0 / un
        Ut = U * dk
        cr = C.T @ r
        beta = rnorm
        if trace is not None:  # diagnostics: |C^T r| / beta at every cycle start
            trace.append((iters, beta, float(np.linalg.norm(cr)) / beta))
        V = np.zeros((n, nsteps + 1))
        H = np.zeros((nsteps + 1, nsteps))
        B = np.zeros((kc, nsteps))
        V[:, 0] = r / beta
        sres = []
        j = 0
        brk = False
        while j < nsteps:
            brk = deflated_step(op, C, V, H, B, j)
            iters += 1
            j += 1
            G = np.zeros((kc + j + 1, kc + j))
            G[:kc, :kc] = np.diag(dk)
            G[:kc, kc:] = B[:, :j]
            G[kc:, kc:] = H[: j + 1, :j]
            rhs = np.zeros(kc + j + 1)
            rhs[:kc] = cr
            rhs[kc] = beta
            y, *_ = np.linalg.lstsq(G, rhs, rcond=None)
            res = float(np.linalg.norm(rhs - G @ y))
            sres.append(res)
            if brk or res <= abs_tol:
                break
        defl += j
        x += Ut @ y[:kc] + V[:, :j] @ y[kc:]
        r = op.prec(b - S @ x)
        rnorm = float(np.linalg.norm(r))
        hist.extend(sres)
        checks.append((sres[-1], rnorm))
        conv = rnorm <= abs_tol
        mm = kc + j
        Vh = np.hstack([Ut, V[:, :j]])
        Wh = np.hstack([C, V[:, : j + 1]])
        try:
            P = hr_next(G, Wh[:, :mm].T @ Vh, cfg.k)
        except (np.linalg.LinAlgError, ValueError):
            P = None
        if P is not None:
            Q, R, kept = qrcp_rank(G @ P)
            if Q.shape[1] > 0:
                C = Wh @ Q
                U = (Vh @ P)[:, kept] @ _inv_upper(R)
        if collect_diagnostics:  # gcrodr.py:461-467
            rel, orth = recycle_residuals(U, C, op)
            cyc_diag.append({"stage": "cycle", "k": U.shape[1], "au_c": rel, "orth": orth})
        if brk and not conv:
            break
    true_rel = float(np.linalg.norm(b - S @ x)) / bnorm
    info = {"restart_checks": checks, "deflated_steps": defl,
            "recycle_k": 0 if U is None else U.shape[1]}
    if collect_diagnostics:
        info["cycles"] = cyc_diag
        info["refreshed_space"] = refreshed
    if U is None:
        info["gmres_fallback"] = True
    return Result(x, iters, np.asarray(hist), true_rel, conv,
                  time.perf_counter() - t0, U, C, info)


def gmres(op: Operator, b, cfg: Cfg, x0=None) -> Result:
    """Restarted GMRES(m) (gmres.py:193-267); the k = 0 path of gcrodr."""
    t0 = time.perf_counter()
    n = op.n
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    S = op.S
    bnorm = float(np.linalg.norm(b))
    if bnorm == 0.0:
        return Result(np.zeros(n), 0, np.zeros(1), 0.0, True,
                      time.perf_counter() - t0, None, None, {"gmres_fallback": True})
    abs_tol = cfg.tol * float(np.linalg.norm(op.prec(b)))
    r = op.prec(b - S @ x) if np.any(x) else op.prec(b)
    rnorm = float(np.linalg.norm(r))
    hist = [rnorm]
    checks = []
    iters = 0
    conv = rnorm <= abs_tol
    while not conv and iters < cfg.max_iter:
        V, H, j, sres, y, brk = gmres_cycle(op, r, rnorm, cfg.m, abs_tol,
                                             cfg.max_iter - iters)
        iters += j
        hist.extend(sres)
        x += V[:, :j] @ y
        r = op.prec(b - S @ x)
        rnorm = float(np.linalg.norm(r))
        checks.append((sres[-1], rnorm))
        conv = rnorm <= abs_tol
        if brk and not conv:
            break
    true_rel = float(np.linalg.norm(b - S @ x)) / bnorm
    return Result(x, iters, np.asarray(hist), true_rel, conv,
                  time.perf_counter() - t0, None, None,
                  {"restart_checks": checks, "gmres_fallback": True,
                   "deflated_steps": 0})


def chain(ops, rhss, order, cfg: Cfg, U_first=None):
    """The SKR loop of harness.py:233-260: solve in ``order``, carrying U."""
    out = {}
    U = U_first
    for idx in order:
        res = gcrodr(ops[idx], rhss[idx], cfg, U_in=U)
        out[idx] = res
        U = res.U
    return out
