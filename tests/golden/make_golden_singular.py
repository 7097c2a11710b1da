"""Golden harmonic-Ritz outputs of the REAL reference (kryrec) on singular and
near-singular Hessenberg matrices: the first-cycle fallback of
gcrodr.py:189-203 (sigma_min < 1e-14 sigma_max -> generalized problem
eig(H^T H + h^2 e e^T, H^T) with a warning). Run here:

    python tests/golden/make_golden_singular.py
"""
import os
import sys
import warnings

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np  # noqa: E402

import kryrec  # noqa: E402


def hess(rng, m):
    H = np.triu(rng.standard_normal((m, m)), -1)
    H[np.arange(1, m), np.arange(m - 1)] = np.abs(H[np.arange(1, m), np.arange(m - 1)]) + 0.3
    return H


def main():
    rng = np.random.default_rng(2401)
    out = {}
    cases = []
    # H singular with a null vector z, z_m != 0 (the last column a combination
    # of the others): the pencil (H^T H + h^2 e e^T, H^T) stays regular. (A
    # null vector with z_m = 0 -- e.g. a zero column -- makes the pencil
    # singular, det(lhs - s H^T) = 0 for every s, and QZ's output arbitrary.)
    for m, h, k, noise in ((12, 0.7, 4, 0.0), (20, 1.3, 10, 1e-16), (30, 0.2, 10, 0.0),
                           (40, 2.0, 10, 3e-17)):
        H = hess(rng, m)
        H[:, m - 1] = H[:, : m - 1] @ rng.standard_normal(m - 1)
        H[:, m - 1] += noise * rng.standard_normal(m)
        cases.append((H, h, k))
    for t, (H, h, k) in enumerate(cases):
        s = np.linalg.svd(H, compute_uv=False)
        with warnings.catch_warnings(record=True) as w:
            warnings.simplefilter("always")
            P = kryrec.harmonic_ritz_first_cycle(H, h, k)
        assert any("singular Hessenberg" in str(x.message) for x in w), t
        out[f"s{t}_H"] = H
        out[f"s{t}_h"] = np.array(h)
        out[f"s{t}_k"] = np.array(k)
        out[f"s{t}_P"] = P
        print(t, H.shape, "sigma ratio", s[-1] / s[0], "P", P.shape)
    np.savez_compressed(os.path.join(HERE, "dense_singular.npz"), **out)


if __name__ == "__main__":
    main()
