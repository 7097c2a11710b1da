"""CPU tests of the device dense-kernel numerics (csrc/dense.h, recycle.h),
compiled for the host into libskr_hostdense.so, against LAPACK (numpy/scipy)
and the reference's golden harmonic-Ritz outputs."""

import ctypes
import os

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import skr_oracle as orc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PD = ctypes.POINTER(ctypes.c_double)
PI = ctypes.POINTER(ctypes.c_int)


@pytest.fixture(scope="module")
def H():
    from paper_2401_09516_b200 import _build

    path = _build.build_host(verbose=False)
    return ctypes.CDLL(path)


def dp(a):
    return a.ctypes.data_as(PD)


def ip(a):
    return a.ctypes.data_as(PI)


def span_dist(P, Q):
    P = np.linalg.qr(P)[0]
    Q = np.linalg.qr(Q)[0]
    if P.shape[1] != Q.shape[1]:
        return np.inf
    return float(np.linalg.norm(P - Q @ (Q.T @ P)))


@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 16, 33, 40, 61, 64])
def test_eigenvalues_vs_lapack(H, n):
    rng = np.random.default_rng(n)
    for trial in range(3):
        A = np.asfortranarray(rng.standard_normal((n, n)))
        if trial == 2:  # nearly-defective / clustered spectrum
            Q = np.linalg.qr(rng.standard_normal((n, n)))[0]
            A = np.asfortranarray(Q @ np.diag(np.round(rng.standard_normal(n), 1)) @ Q.T)
        wr, wi = np.zeros(n), np.zeros(n)
        assert H.skrh_eig(dp(A), n, n, dp(wr), dp(wi)) == 0
        ev = np.sort_complex(wr + 1j * wi)
        ref = np.sort_complex(np.linalg.eigvals(A))
        assert np.max(np.abs(ev - ref)) <= 1e-11 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("m,n", [(10, 4), (41, 11), (61, 21), (5, 9), (33, 33)])
def test_qrcp_vs_lapack(H, m, n):
    rng = np.random.default_rng(m * 100 + n)
    A = np.asfortranarray(rng.standard_normal((m, n)))
    Q = np.zeros((m, n), order="F")
    R = np.zeros((min(m, n), n), order="F")
    jp = np.zeros(n, dtype=np.int32)
    r = H.skrh_qrcp(dp(A), m, m, n, ctypes.c_double(1e-12), dp(Q), m, dp(R), min(m, n), ip(jp))
    Qr, Rr, pr = sla.qr(A, mode="economic", pivoting=True)
    assert r == min(m, n)
    assert list(jp) == list(pr)
    np.testing.assert_allclose(Q[:, :r] @ R[:r], A[:, jp], atol=1e-12)
    np.testing.assert_allclose(np.abs(np.diag(R)), np.abs(np.diag(Rr)), rtol=1e-12)


def test_qrcp_rank_detection(H):
    rng = np.random.default_rng(7)
    B = rng.standard_normal((30, 4))
    A = np.asfortranarray(np.concatenate([B, B[:, :2] * 2.0, B[:, :1] + 1e-14 * B[:, 1:2]], 1))
    m, n = A.shape
    Q = np.zeros((m, n), order="F")
    R = np.zeros((n, n), order="F")
    jp = np.zeros(n, dtype=np.int32)
    r = H.skrh_qrcp(dp(A), m, m, n, ctypes.c_double(1e-12), dp(Q), m, dp(R), n, ip(jp))
    ref = orc.qrcp_rank(A)[0].shape[1]
    assert r == ref == 4


def test_harmonic_ritz_golden(H):
    d = np.load(os.path.join(GOLD, "dense.npz"))
    w = ctypes.c_int(0)
    for t in range(6):
        Hm = np.asfortranarray(d[f"hf{t}_H"])
        n = Hm.shape[1]
        P = np.zeros((n, 16), order="F")
        r = H.skrh_hr_first(dp(Hm), n + 1, n, min(10, n), dp(P), n, ctypes.byref(w))
        assert r == d[f"hf{t}_P"].shape[1]
        assert span_dist(P[:, :r], d[f"hf{t}_P"]) < 1e-8
        G = np.asfortranarray(d[f"hs{t}_G"])
        X = np.asfortranarray(d[f"hs{t}_cross"])
        kk = int(d[f"hs{t}_k"])
        P = np.zeros((n, 24), order="F")
        r = H.skrh_hr_next(dp(G), n + 1, dp(X), n, n, kk, dp(P), n, ctypes.byref(w))
        assert r == d[f"hs{t}_P"].shape[1]
        cond = np.linalg.cond(G[:n].T @ X)  # eig(rhs^-1 lhs) error ~ cond(rhs) eps
        assert span_dist(P[:, :r], d[f"hs{t}_P"]) < 1e-8 + 1e-12 * cond


def test_pair_widening_rotation(H):
    """SPEC example: a rotation block's conjugate pair is never split."""
    th = 0.7
    A = np.zeros((3, 3), order="F")
    A[:2, :2] = [[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]]
    A[2, 2] = 5.0
    P = np.zeros((3, 3), order="F")
    wr, wi = np.zeros(3), np.zeros(3)
    nc = H.skrh_select(dp(A), 3, 3, 1, 3, dp(P), 3, dp(wr), dp(wi))
    assert nc == 2  # k = 1 widened to the pair
    assert span_dist(P[:, :2], np.eye(3)[:, :2]) < 1e-12


def _random_cycle(rng, kc, j):
    Hm = np.zeros((j + 1, j))
    Hm[: j + 1, :j] = np.triu(rng.standard_normal((j + 1, j)), -1)
    Hm[np.arange(1, j + 1), np.arange(j)] = np.abs(Hm[np.arange(1, j + 1), np.arange(j)]) + 0.3
    B = rng.standard_normal((kc, j)) * 0.1
    dk = rng.uniform(0.5, 3.0, kc)
    mm = kc + j
    Y = np.linalg.qr(rng.standard_normal((4 * mm, mm)))[0]
    cross = Y.T @ (Y + 1e-3 * rng.standard_normal(Y.shape))
    return Hm, B, dk, cross


@pytest.mark.parametrize("kc,j", [(4, 8), (10, 20), (11, 29), (20, 40)])
def test_recycle_next_matches_reference_algebra(H, kc, j):
    """coefU/coefC from the device program == the reference's U/C algebra
    (gcrodr.py:444-460) applied to coordinates."""
    rng = np.random.default_rng(kc * 1000 + j)
    Hm, B, dk, cross = _random_cycle(rng, kc, j)
    mm = kc + j
    LDC = 97
    cu = np.zeros((LDC, 32), order="F")
    cc = np.zeros((LDC, 32), order="F")
    w = ctypes.c_int(0)
    Hf = np.asfortranarray(Hm)
    Bf = np.asfortranarray(B)
    Xf = np.asfortranarray(cross)
    r = H.skrh_recycle_next(dp(Hf), j + 1, dp(Bf), kc, dp(dk), kc, j, dp(Xf), mm, kc, dp(cu), LDC,
                            dp(cc), LDC, ctypes.byref(w))
    G = np.zeros((mm + 1, mm))
    G[:kc, :kc] = np.diag(dk)
    G[:kc, kc:] = B
    G[kc:, kc:] = Hm
    P = orc.hr_next(G, cross, kc)
    Q, R, kept = orc.qrcp_rank(G @ P)
    assert r == Q.shape[1]
    # C coordinates (in What = [C | V]) : span equality
    assert span_dist(cc[: mm + 1, :r], Q) < 1e-7
    # U coordinates in Vhat = [U diag(dk) | V]: reference Z = P[:, kept] R^-1
    Zref = P[:, kept] @ np.linalg.inv(R)
    Zdev = cu[:mm, :r].copy()
    Zdev[:kc] /= dk[:, None]  # device folds dk into the U rows
    # same pair (op U = C) <=> same Z up to the same column transform as C
    T = np.linalg.lstsq(Q, cc[: mm + 1, :r], rcond=None)[0]
    np.testing.assert_allclose(Zref @ T, Zdev, atol=1e-7 * np.max(np.abs(Zdev)))


@pytest.mark.parametrize("j,k", [(5, 3), (20, 10), (30, 10), (40, 10)])
def test_recycle_first_matches_reference_algebra(H, j, k):
    rng = np.random.default_rng(j * 7 + k)
    Hm = np.triu(rng.standard_normal((j + 1, j)), -1)
    Hm[np.arange(1, j + 1), np.arange(j)] = np.abs(Hm[np.arange(1, j + 1), np.arange(j)]) + 0.3
    LDC = 97
    cu = np.zeros((LDC, 32), order="F")
    cc = np.zeros((LDC, 32), order="F")
    w = ctypes.c_int(0)
    Hf = np.asfortranarray(Hm)
    r = H.skrh_recycle_first(dp(Hf), j + 1, j, k, dp(cu), LDC, dp(cc), LDC, ctypes.byref(w))
    P = orc.hr_first(Hm[:j, :j], Hm[j, j - 1], min(k, j))
    Q, R, kept = orc.qrcp_rank(Hm @ P)
    assert r == Q.shape[1]
    assert span_dist(cc[: j + 1, :r], Q) < 1e-7
    Zref = P[:, kept] @ np.linalg.inv(R)
    T = np.linalg.lstsq(Q, cc[: j + 1, :r], rcond=None)[0]
    np.testing.assert_allclose(Zref @ T, cu[:j, :r], atol=1e-7 * np.max(np.abs(cu[:j, :r])))


def test_cholqr2_orthonormal_and_rank(H):
    rng = np.random.default_rng(11)
    n = 500
    X = rng.standard_normal((n, 6)) * np.array([1, 1e3, 1e-3, 5, 1, 1])
    X = np.concatenate([X, X[:, :1] * 3.0], axis=1)  # exactly dependent 7th column
    Xf = np.asfortranarray(X)
    Q = np.zeros((n, 7), order="F")
    kept = np.zeros(7, dtype=np.int32)
    r = H.skrh_cholqr2(dp(Xf), n, n, 7, dp(Q), n, ip(kept))
    Qr, _, pr = orc.qrcp_rank(X)
    assert r == Qr.shape[1] == 6
    np.testing.assert_allclose(Q[:, :r].T @ Q[:, :r], np.eye(r), atol=1e-13)
    assert span_dist(Q[:, :r], Qr) < 1e-10


def test_harmonic_ritz_first_singular_h_golden(H):
    """Singular / nearly singular Hessenberg (sigma_min < 1e-14 sigma_max):
    the reference's generalized fallback (gcrodr.py:189-203, QZ on
    (H^T H + h^2 e e^T, H^T)) against its own outputs; the device solves the
    inverse problem of A^-1 H^T and selects on theta = 1 / mu, with the
    reference's warning bit."""
    d = np.load(os.path.join(GOLD, "dense_singular.npz"))
    t = 0
    while f"s{t}_H" in d:
        Hs = d[f"s{t}_H"]
        m = Hs.shape[0]
        Hf = np.zeros((m + 1, m), order="F")
        Hf[:m] = Hs
        Hf[m, m - 1] = float(d[f"s{t}_h"])
        P = np.zeros((m, m), order="F")
        w = ctypes.c_int(0)
        r = H.skrh_hr_first(dp(Hf), m + 1, m, int(d[f"s{t}_k"]), dp(P), m, ctypes.byref(w))
        ref = d[f"s{t}_P"]
        assert w.value & 1, t  # W_SINGULAR_H
        assert r == ref.shape[1], (t, r, ref.shape)
        assert span_dist(P[:, :r], ref) < 1e-8, (t, span_dist(P[:, :r], ref))
        t += 1
    assert t == 4
