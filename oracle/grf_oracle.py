"""CPU restatement of the device field generator -- TEST INFRASTRUCTURE ONLY.

Only ``tests/`` may import this module, as the checker of ``csrc/grf.cu``
(``skr_grf_sample``, ``skr_philox_normals``, ``skr_philox_uniforms``). The
product never calls it.

The device generator is a seeded definition of its own (DESIGN.md §5,
"philox" inputs), not the reference's sampler: the reference's KL/SE samplers
(``kryrec/problems.py:97-162``, per-system seeding ``:488``) draw from numpy's
PCG64 and differ from BASELINE.json's configurations anyway. What is restated
here, independently of the CUDA code:

* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy
  as 1, 2, 3", SC'11): 10 rounds of two 32x32->64 multiplies (0xD2511F53,
  0xCD9E8D57) with Weyl key increments (0x9E3779B9, 0xBB67AE85); pinned by the
  published known-answer vectors (``tests/test_grf.py``);
* 53-bit uniforms and Box-Muller, in numpy's libm;
* the field through ``scipy.fft.idctn(type=2, norm="ortho")`` -- an FFT-based
  DCT, i.e. a different algorithm than the device's dense DCT-III GEMMs -- and
  the spectrum / coefficient laws of ``paper_2401_09516_b200/problems.py``.
Device and oracle agree to rounding (libm last bits, summation order), so the
tests compare with tolerances and the thresholded fields exactly.
"""

from __future__ import annotations

import numpy as np
import scipy.fft as _fft

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 over uint32 counter words; returns 4 uint32 arrays."""
    c = [np.asarray(v, dtype=np.uint64) & MASK for v in (c0, c1, c2, c3)]
    k0 = np.uint64(int(k0) & 0xFFFFFFFF)
    k1 = np.uint64(int(k1) & 0xFFFFFFFF)
    for _ in range(10):
        p0 = M0 * c[0]  # < 2^64: exact in uint64
        p1 = M1 * c[2]
        hi0, lo0 = p0 >> np.uint64(32), p0 & MASK
        hi1, lo1 = p1 >> np.uint64(32), p1 & MASK
        c = [hi1 ^ c[1] ^ k0, lo1, hi0 ^ c[3] ^ k1, lo0]
        k0 = (k0 + W0) & MASK
        k1 = (k1 + W1) & MASK
    return [v.astype(np.uint32) for v in c]


def _keys(seed: int, cid: int):
    return seed & 0xFFFFFFFF, ((seed >> 32) ^ cid) & 0xFFFFFFFF


def _u53(a, b, open0=False):
    hi = (a >> np.uint32(5)).astype(np.float64)
    lo = (b >> np.uint32(6)).astype(np.float64)
    v = hi * 67108864.0 + lo
    if open0:
        v = v + 1.0
    return v * (1.0 / 9007199254740992.0)


def normals(count: int, seed: int, cid: int, idx: int, stream: int) -> np.ndarray:
    """N(0,1) samples 0..count-1 of (system idx, stream): block p -> samples 2p, 2p+1."""
    npair = (count + 1) // 2
    p = np.arange(npair, dtype=np.uint64)
    k0, k1 = _keys(seed, cid)
    r = philox4x32_10(p & MASK, p >> np.uint64(32), np.full(npair, idx), np.full(npair, stream),
                      k0, k1)
    u1 = _u53(r[0], r[1], open0=True)
    u2 = _u53(r[2], r[3])
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = 6.283185307179586 * u2
    out = np.empty(2 * npair)
    out[0::2] = rad * np.cos(ang)
    out[1::2] = rad * np.sin(ang)
    return out[:count]


def uniforms(count: int, seed: int, cid: int, idx: int, stream: int) -> np.ndarray:
    npair = (count + 1) // 2
    p = np.arange(npair, dtype=np.uint64)
    k0, k1 = _keys(seed, cid)
    r = philox4x32_10(p, np.zeros(npair), np.full(npair, idx), np.full(npair, stream), k0, k1)
    out = np.empty(2 * npair)
    out[0::2] = _u53(r[0], r[1])
    out[1::2] = _u53(r[2], r[3])
    return out[:count]


def spectrum(shape: tuple, tau: float):
    """coef = 1 / (pi^2 |kappa|^2 + tau^2), coef_0 = 0, and the unit-variance norm."""
    lam = np.zeros(shape)
    for ax, n in enumerate(shape):
        kk = (np.pi * np.arange(n)) ** 2
        lam = lam + kk.reshape([-1 if a == ax else 1 for a in range(len(shape))])
    coef = 1.0 / (lam + tau * tau)
    coef.flat[0] = 0.0
    return coef, float(np.sqrt(np.sum(coef * coef) / coef.size))


def grf(dim: int, n: int, tau: float, seed: int, cid: int, idx: int) -> np.ndarray:
    shape = (n,) * dim
    coef, norm = spectrum(shape, tau)
    xi = normals(n ** dim, seed, cid, idx, 0).reshape(shape)
    return _fft.idctn(xi * coef, type=2, norm="ortho") / norm


def system_params(kind: str, dim: int, n: int, tau: float, scale: float, seed: int, cid: int,
                  idx: int) -> dict:
    """The device generator's fields for one system (problems.system_params laws)."""
    g = grf(dim, n, tau, seed, cid, idx)
    if kind == "darcy_binary":
        a = np.where(g > 0.0, 12.0, 3.0)
        return {"a": a, "g": g, "params": a.ravel()}
    if kind == "poisson_lognormal":
        a = np.exp(scale * g)
        return {"a": a, "g": g, "params": a.ravel()}
    if kind == "helmholtz":
        u = uniforms(1 + dim, seed, cid, idx, 1)
        k0 = 10.0 + 10.0 * u[0]
        center = 0.2 + 0.6 * u[1:1 + dim]
        kf = k0 * (1.0 + 0.3 * np.tanh(g))
        return {"kfield": kf, "k0": k0, "g": g, "center": center,
                "params": np.concatenate([[k0], g.ravel()])}
    raise ValueError(kind)
