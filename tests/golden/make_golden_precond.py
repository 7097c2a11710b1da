"""Golden fixtures for the general preconditioners (SOR, ILU(0), IC(0), block
Jacobi; kryrec/precond.py:80-312) from the REAL reference:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_precond.py

Per (system, kind): the factor values, M.apply on a vector and a 3-column
block, and a 3-system GCRO-DR chain (iterations, x). Plus the reference's
failures: zero diagonal, IC(0) nonpositive pivot on an indefinite matrix,
IC(0) on a nonsymmetric matrix.
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import kryrec  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402

CASES = [  # tag, spec, systems of the chain, m, k
    ("darcy12", P.CONFIGS[0].reduced(n=12), (0, 1, 2), 12, 4),
    ("poisson16", P.CONFIGS[1].reduced(n=16), (3, 4, 5), 14, 5),
    ("darcy3d6", P.CONFIGS[3].reduced(n=6), (0, 1, 2), 10, 4),
]
KINDS = [("sor", dict(sor_omega=1.0)), ("sor12", dict(sor_omega=1.2)), ("ilu0", {}),
         ("icc0", {}), ("bjacobi", dict(bjacobi_block=20)), ("bjacobi64", dict(bjacobi_block=64))]


def kind_of(tag):
    return "sor" if tag.startswith("sor") else "bjacobi" if tag.startswith("bj") else tag


def main():
    out = {}
    rng = np.random.default_rng(2401)
    for tag, spec, idxs, m, k in CASES:
        sysl = []
        for i in idxs:
            rp, ci, v, b, _ = P.assemble(spec, i)
            sysl.append((kryrec.CsrMatrix(spec.N, spec.N, rp, ci, v), b))
        A0 = sysl[0][0]
        x = rng.standard_normal(spec.N)
        X = rng.standard_normal((spec.N, 3))
        out[f"{tag}_x"], out[f"{tag}_X"] = x, X
        out[f"{tag}_cfg"] = np.array([spec.cid, spec.n, m, k] + list(idxs))
        for ktag, kw in KINDS:
            kind = kind_of(ktag)
            M = kryrec.build_preconditioner(A0, kind, **kw)
            key = f"{tag}_{ktag}"
            out[f"{key}_ax"] = M.apply(x)
            out[f"{key}_aX"] = M.apply(X)
            if kind == "ilu0":
                out[f"{key}_lower"] = M.lower.values
                out[f"{key}_upper"] = M.upper.values
            if kind == "icc0":
                out[f"{key}_lower"] = M.lower.values
                out[f"{key}_sign"] = np.array(M.sign)
            cfg = kryrec.SolverConfig(m=m, tol=1e-8, max_iter=5000, k=k)
            rec, its, xs, conv = None, [], [], []
            for A, b in sysl:
                Mi = kryrec.build_preconditioner(A, kind, **kw)
                rep, rec = kryrec.gcrodr_solve(A, b, M=Mi, cfg=cfg, recycle_in=rec)
                its.append(rep.iterations)
                conv.append(rep.converged)
                xs.append(rep.x)
            out[f"{key}_iters"] = np.array(its)
            out[f"{key}_conv"] = np.array(conv)
            out[f"{key}_xs"] = np.stack(xs)
            # plain GMRES with the same preconditioner (gmres.py:193-267)
            g = kryrec.gmres_solve(sysl[0][0], sysl[0][1],
                                   M=kryrec.build_preconditioner(A0, kind, **kw), cfg=cfg)
            out[f"{key}_gmres_iters"] = np.array(g.iterations)
            print(key, its, conv, int(g.iterations), flush=True)
    # failures
    spec = P.CONFIGS[2].reduced(n=16)  # Helmholtz: indefinite
    rp, ci, v, b, _ = P.assemble(spec, 0)
    A = kryrec.CsrMatrix(spec.N, spec.N, rp, ci, v)
    try:
        kryrec.build_preconditioner(A, "icc0")
        out["helm_icc0_err"] = np.array([-1.0, 0.0])
    except kryrec.precond.ZeroPivotError as e:
        out["helm_icc0_err"] = np.array([e.row, e.value])
        print("helmholtz icc0:", e)
    out["helm_cfg"] = np.array([2, 16, 0])
    M = kryrec.build_preconditioner(A, "ilu0")
    xh = rng.standard_normal(spec.N)
    out["helm_x"] = xh
    out["helm_ilu0_ax"] = M.apply(xh)
    np.savez_compressed(os.path.join(HERE, "precond.npz"), **out)
    print("wrote precond.npz")


if __name__ == "__main__":
    main()
