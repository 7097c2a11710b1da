"""General preconditioners (SOR, ILU(0), IC(0), block Jacobi; SURVEY 8(f) row 4,
kryrec/precond.py:80-312) against fixtures from the real reference
(tests/golden/make_golden_precond.py -> precond.npz).

CPU: the oracle restatement reproduces the reference's factor values bit for
bit, its M.apply to 1e-12 and its GCRO-DR iteration counts exactly.
GPU (-m gpu): the device build gives bit-identical factor values, the
level-scheduled sweeps give the reference's M.apply to 1e-12, and chains solved
with each kind converge in the reference's iteration counts (+-1) to its x.
"""

import os

import numpy as np
import pytest

from oracle import skr_oracle as orc
from paper_2401_09516_b200 import problems as P

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "precond.npz"))
CASES = ["darcy12", "poisson16", "darcy3d6"]
KINDS = [("sor", dict(sor_omega=1.0)), ("sor12", dict(sor_omega=1.2)), ("ilu0", {}),
         ("icc0", {}), ("bjacobi", dict(bjacobi_block=20)), ("bjacobi64", dict(bjacobi_block=64))]


def kind_of(tag):
    return "sor" if tag.startswith("sor") else "bjacobi" if tag.startswith("bj") else tag


def case(tag):
    cfg = [int(v) for v in GOLD[f"{tag}_cfg"]]
    spec = P.CONFIGS[cfg[0]].reduced(n=cfg[1])
    return spec, cfg[2], cfg[3], cfg[4:]


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max())


# --------------------------------------------------------------------------- CPU: oracle pins
@pytest.mark.parametrize("tag", CASES)
@pytest.mark.parametrize("ktag,kw", KINDS)
def test_oracle_preconditioner_matches_reference(tag, ktag, kw):
    spec, m, k, idxs = case(tag)
    kind = kind_of(ktag)
    key = f"{tag}_{ktag}"
    rp, ci, v, b, _ = P.assemble(spec, idxs[0])
    G = orc.GeneralPrec(rp, ci, v, spec.N, kind, **kw)
    assert rel(G.apply(GOLD[f"{tag}_x"]), GOLD[f"{key}_ax"]) < 1e-12
    assert rel(G.apply(GOLD[f"{tag}_X"]), GOLD[f"{key}_aX"]) < 1e-12
    rows = np.repeat(np.arange(spec.N), np.diff(rp))
    if kind == "ilu0":
        assert np.array_equal(G.factor[ci >= rows], GOLD[f"{key}_upper"])
        lower = GOLD[f"{key}_lower"]  # unit diagonal stored as 1 (precond.py:195-198)
        cnt = np.bincount(rows[ci < rows], minlength=spec.N)
        dpos = np.cumsum(cnt + 1) - 1  # the diagonal closes every row of the reference's L
        strict = np.ones(len(lower), dtype=bool)
        strict[dpos] = False
        assert np.all(lower[dpos] == 1.0)
        assert np.array_equal(G.factor[ci < rows], lower[strict])
    if kind == "icc0":
        assert np.array_equal(G.factor[ci <= rows], GOLD[f"{key}_lower"])
        assert G.scale == float(GOLD[f"{key}_sign"])
    # the reference chain (harness.py:233-260) with this preconditioner
    U, its = None, []
    cfg = orc.Cfg(m=m, k=k, tol=1e-8, max_iter=5000)
    for p, i in enumerate(idxs):
        rp, ci, v, b, _ = P.assemble(spec, i)
        op = orc.Operator(rp, ci, v, spec.N, False,
                          prec=orc.GeneralPrec(rp, ci, v, spec.N, kind, **kw))
        r = orc.gcrodr(op, b, cfg, U_in=U)
        its.append(r.iterations)
        assert r.converged
        assert rel(r.x, GOLD[f"{key}_xs"][p]) < 1e-7
        U = r.U
    assert its == [int(t) for t in GOLD[f"{key}_iters"]]


def test_oracle_icc0_nonpositive_pivot():
    spec = P.CONFIGS[2].reduced(n=16)
    rp, ci, v, b, _ = P.assemble(spec, 0)
    with pytest.raises(orc.ZeroPivot) as e:
        orc.GeneralPrec(rp, ci, v, spec.N, "icc0")
    assert e.value.row == int(GOLD["helm_icc0_err"][0])
    assert e.value.value == float(GOLD["helm_icc0_err"][1])
    G = orc.GeneralPrec(rp, ci, v, spec.N, "ilu0")
    assert rel(G.apply(GOLD["helm_x"]), GOLD["helm_ilu0_ax"]) < 1e-11


def test_host_api_validation_without_gpu():
    import paper_2401_09516_b200 as skr

    A = skr.eye(4)
    with pytest.raises(ValueError):
        skr.build_preconditioner(A, "sor", sor_omega=2.0)
    with pytest.raises(ValueError):
        skr.build_preconditioner(A, "bjacobi", bjacobi_block=0)
    with pytest.raises(ValueError):
        skr.build_preconditioner(A, "ssor")


# --------------------------------------------------------------------------- GPU
def _skr():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2401_09516_b200 as skr

    return skr


@pytest.mark.gpu
@pytest.mark.parametrize("tag", CASES)
@pytest.mark.parametrize("ktag,kw", KINDS)
def test_gpu_preconditioner_matches_reference(tag, ktag, kw):
    skr = _skr()
    spec, m, k, idxs = case(tag)
    kind = kind_of(ktag)
    key = f"{tag}_{ktag}"
    rp, ci, v, b, _ = P.assemble(spec, idxs[0])
    A = skr.CsrMatrix(spec.N, spec.N, rp, ci, v)
    M = skr.build_preconditioner(A, kind, **kw)
    assert M.kind == kind and M.n == spec.N
    assert rel(M.apply(GOLD[f"{tag}_x"]), GOLD[f"{key}_ax"]) < 1e-12
    assert rel(M.apply(GOLD[f"{tag}_X"]), GOLD[f"{key}_aX"]) < 1e-12
    if kind == "ilu0":  # the factor itself is bit-identical to the reference's
        assert np.array_equal(M.upper.values, GOLD[f"{key}_upper"])
        assert np.array_equal(M.lower.values, GOLD[f"{key}_lower"])
    if kind == "icc0":
        assert np.array_equal(M.lower.values, GOLD[f"{key}_lower"])
        assert M.sign == float(GOLD[f"{key}_sign"])
    cfg = skr.SolverConfig(m=m, k=k, tol=1e-8, max_iter=5000)
    rec, its = None, []
    for p, i in enumerate(idxs):
        rp, ci, v, b, _ = P.assemble(spec, i)
        Ai = skr.CsrMatrix(spec.N, spec.N, rp, ci, v)
        Mi = skr.build_preconditioner(Ai, kind, **kw)
        rep, rec = skr.gcrodr_solve(Ai, b, M=Mi, cfg=cfg, recycle_in=rec)
        assert rep.converged and rep.true_relative_residual < 1e-6
        assert rel(rep.x, GOLD[f"{key}_xs"][p]) < 1e-6
        its.append(rep.iterations)
    ref = [int(t) for t in GOLD[f"{key}_iters"]]
    print(key, "gpu", its, "ref", ref)
    assert all(abs(a - r) <= 1 for a, r in zip(its, ref)), (its, ref)
    g = skr.gmres_solve(A, b=P.assemble(spec, idxs[0])[3], M=M, cfg=cfg)
    assert abs(g.iterations - int(GOLD[f"{key}_gmres_iters"])) <= 1


@pytest.mark.gpu
def test_gpu_preconditioner_failures_match_reference():
    skr = _skr()
    spec = P.CONFIGS[2].reduced(n=16)
    rp, ci, v, b, _ = P.assemble(spec, 0)
    A = skr.CsrMatrix(spec.N, spec.N, rp, ci, v)
    with pytest.raises(skr.ZeroPivotError) as e:
        skr.build_preconditioner(A, "icc0")
    assert e.value.kind == "icc0" and e.value.row == int(GOLD["helm_icc0_err"][0])
    assert e.value.value == float(GOLD["helm_icc0_err"][1])
    M = skr.build_preconditioner(A, "ilu0")
    assert rel(M.apply(GOLD["helm_x"]), GOLD["helm_ilu0_ax"]) < 1e-11
    # zero diagonal entry (precond.py:153-158): sor / ilu0 / icc0 raise at that row
    v2 = np.array(v)
    rows = np.repeat(np.arange(spec.N), np.diff(rp))
    v2[(rows == ci) & (rows == 37)] = 0.0
    A0 = skr.CsrMatrix(spec.N, spec.N, rp, ci, v2)
    for kind in ("sor", "ilu0", "icc0"):
        with pytest.raises(skr.ZeroPivotError) as e:
            skr.build_preconditioner(A0, kind)
        assert e.value.row == 37 and e.value.kind == kind
    # nonsymmetric values: IC(0) refuses (precond.py:303-304)
    v3 = np.array(v)
    v3[(rows == 5) & (ci == 6)] *= 2.0
    with pytest.raises(ValueError, match="symmetric"):
        skr.build_preconditioner(skr.CsrMatrix(spec.N, spec.N, rp, ci, v3), "icc0")
    with pytest.raises(skr._lib.SkrExtensionError):
        skr.build_preconditioner(A, "bjacobi", bjacobi_block=512)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["sor", "ilu0", "icc0", "bjacobi"])
def test_gpu_sequence_with_general_preconditioner(kind):
    """solve_sequence / solve_chains with a device-built preconditioner per
    system, on a grid large enough for several CTAs and wide levels; checked
    against the oracle chain (iterations within 5%, x to 1e-6)."""
    skr = _skr()
    spec = P.CONFIGS[3].reduced(n=20)  # 8,000 rows, 58 levels up to 300 rows wide
    ns = 3
    cfg = skr.SolverConfig(m=20, k=6, tol=1e-8, max_iter=3000)
    ocfg = orc.Cfg(m=20, k=6, tol=1e-8, max_iter=3000)
    systems, U, ref = [], None, []
    for i in range(ns):
        rp, ci, v, b, _ = P.assemble(spec, i)
        systems.append((skr.CsrMatrix(spec.N, spec.N, rp, ci, v), b))
        op = orc.Operator(rp, ci, v, spec.N, False, prec=orc.GeneralPrec(rp, ci, v, spec.N, kind))
        r = orc.gcrodr(op, b, ocfg, U_in=U)
        ref.append(r)
        U = r.U
    res = skr.solve_sequence(systems, list(range(ns)), cfg, kind)
    print(kind, "gpu", res.iterations, "oracle", [r.iterations for r in ref])
    for p in range(ns):
        assert res.converged[p]
        assert abs(res.iterations[p] - ref[p].iterations) <= max(1, 0.05 * ref[p].iterations)
        assert rel(res.x[p], ref[p].x) < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["sor", "ilu0", "bjacobi"])
def test_gpu_general_preconditioner_side_paths(kind):
    """x0 (the preconditioned initial residual, gcrodr.py:348-351), the
    diagnostics records (gcrodr.py:116-123, :372-376, :461-467), the CSR path
    without the stencil form, and the native multi-chain driver, all with a
    general preconditioner, against the oracle."""
    import torch

    skr = _skr()
    spec = P.CONFIGS[1].reduced(n=24)
    cfg = skr.SolverConfig(m=16, k=5, tol=1e-9, max_iter=3000)
    ocfg = orc.Cfg(m=16, k=5, tol=1e-9, max_iter=3000)
    rp, ci, v, b, _ = P.assemble(spec, 1)
    A = skr.CsrMatrix(spec.N, spec.N, rp, ci, v)
    M = skr.build_preconditioner(A, kind)
    op = orc.Operator(rp, ci, v, spec.N, False, prec=orc.GeneralPrec(rp, ci, v, spec.N, kind))
    # x0
    x0 = np.random.default_rng(3).standard_normal(spec.N)
    rep, sp0 = skr.gcrodr_solve(A, b, x0=x0, M=M, cfg=cfg)
    ref = orc.gcrodr(op, b, ocfg, x0=x0)
    assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
    assert rel(rep.x, ref.x) < 1e-7
    assert abs(rep.residual_history[0] - ref.history[0]) <= 1e-10 * ref.history[0]
    # diagnostics on a recycled solve
    rp1, ci1, v1, b1, _ = P.assemble(spec, 2)
    A1 = skr.CsrMatrix(spec.N, spec.N, rp1, ci1, v1)
    M1 = skr.build_preconditioner(A1, kind)
    op1 = orc.Operator(rp1, ci1, v1, spec.N, False,
                       prec=orc.GeneralPrec(rp1, ci1, v1, spec.N, kind))
    rep1, _ = skr.gcrodr_solve(A1, b1, M=M1, cfg=cfg, recycle_in=sp0, collect_diagnostics=True)
    ref1 = orc.gcrodr(op1, b1, ocfg, U_in=sp0.U.cpu().numpy(), collect_diagnostics=True)
    got, want = rep1.diagnostics["cycles"], ref1.info["cycles"]
    assert [(d["stage"], d["k"]) for d in got] == [(d["stage"], d["k"]) for d in want]
    for d, w in zip(got, want):
        assert d["au_c"] <= max(100 * w["au_c"], 1e-9), (d, w)
        assert d["orth"] <= max(100 * w["orth"], 1e-9), (d, w)
    assert abs(rep1.iterations - ref1.iterations) <= 1
    # CSR path (no stencil form): same iterations, same x to rounding
    os.environ["SKR_NO_STENCIL"] = "1"
    try:
        Mn = skr.build_preconditioner(A, kind)
        repn, _ = skr.gcrodr_solve(A, b, x0=x0, M=Mn, cfg=cfg)
    finally:
        del os.environ["SKR_NO_STENCIL"]
    assert repn.iterations == rep.iterations and rel(repn.x, rep.x) < 1e-12
    # native chains driver: two chains of two device-resident systems
    systems = []
    for i in range(4):
        dA, bd, _ = P.assemble_device(spec, i)
        systems.append((dA.with_diag(None), bd))
    torch.cuda.synchronize()
    res = skr.solve_chains(systems, list(range(4)), cfg, kind, [[0, 1], [2, 3]], keep_x="device")
    for c, chunk in enumerate(([0, 1], [2, 3])):
        U = None
        for p_, i in enumerate(chunk):
            rpi, cii, vi, bi, _ = P.assemble(spec, i)
            opi = orc.Operator(rpi, cii, vi, spec.N, False,
                               prec=orc.GeneralPrec(rpi, cii, vi, spec.N, kind))
            r = orc.gcrodr(opi, bi, ocfg, U_in=U)
            U = r.U
            assert res[c].converged[p_]
            assert abs(res[c].iterations[p_] - r.iterations) <= 1, (c, p_)
            assert rel(res[c].x[p_].cpu().numpy(), r.x) < 1e-6


def _random_system(n, density, seed, symmetric):
    """Diagonally dominant random sparse matrix (rows longer than the sweeps'
    slot-major prefix, irregular dependency levels, unsymmetric pattern)."""
    import scipy.sparse as sp

    rng = np.random.default_rng(seed)
    A = sp.random(n, n, density=density, random_state=rng, format="csr")
    A.data = rng.uniform(-1.0, 1.0, A.nnz)
    if symmetric:
        A = (A + A.T).tocsr()
    A = A + sp.diags(np.abs(A).sum(axis=1).A1 + 1.0)
    A = A.tocsr()
    A.sort_indices()
    return A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data.copy(), rng


@pytest.mark.parametrize("kind", ["sor", "ilu0", "icc0", "bjacobi"])
def test_oracle_general_csr_matches_reference_structure(kind):
    """CPU sanity of the fixture generator: the oracle solves the random system."""
    rp, ci, v, rng = _random_system(120, 0.08, 7, kind == "icc0")
    G = orc.GeneralPrec(rp, ci, v, 120, kind, bjacobi_block=32)
    x = rng.standard_normal(120)
    assert np.all(np.isfinite(G.apply(x)))


@pytest.mark.gpu
@pytest.mark.parametrize("n,density", [(1, 1.0), (7, 0.5), (300, 0.04), (900, 0.02)])
@pytest.mark.parametrize("kind", ["sor", "ilu0", "icc0", "bjacobi"])
def test_gpu_general_csr_preconditioners(kind, n, density):
    """Non-stencil matrices: long rows (beyond the slot-major prefix), irregular
    levels, tiny sizes; factor values bit-identical to the oracle's restatement
    of the reference loops, apply to 1e-12, GMRES / GCRO-DR iteration counts."""
    skr = _skr()
    rp, ci, v, rng = _random_system(n, density, 11 + n, kind == "icc0")
    A = skr.CsrMatrix(n, n, rp, ci, v)
    M = skr.build_preconditioner(A, kind, bjacobi_block=32)
    G = orc.GeneralPrec(rp, ci, v, n, kind, bjacobi_block=32)
    rows = np.repeat(np.arange(n), np.diff(rp))
    if kind == "ilu0":
        assert np.array_equal(M.upper.values, G.factor[ci >= rows])
    if kind == "icc0":
        assert np.array_equal(M.lower.values, G.factor[ci <= rows])
    x = rng.standard_normal(n)
    X = rng.standard_normal((n, 4))
    assert rel(M.apply(x), G.apply(x)) < 1e-12
    assert rel(M.apply(X), G.apply(X)) < 1e-12
    if n >= 7:
        b = rng.standard_normal(n)
        m = min(10, n - 1)
        cfg = skr.SolverConfig(m=m, k=min(3, m - 1), tol=1e-10, max_iter=500)
        rep, _ = skr.gcrodr_solve(A, b, M=M, cfg=cfg)
        ref = orc.gcrodr(orc.Operator(rp, ci, v, n, False, prec=G), b,
                         orc.Cfg(m=cfg.m, k=cfg.k, tol=1e-10, max_iter=500))
        assert rep.converged and abs(rep.iterations - ref.iterations) <= 1
        assert rel(rep.x, ref.x) < 1e-8


@pytest.mark.gpu
def test_gpu_accepts_reference_style_preconditioner_objects():
    """gcrodr_solve takes over kind / omega / block_size of a preconditioner
    object that is not this package's (the reference's classes expose the same
    attributes, precond.py:80-145) and factors on the device."""
    skr = _skr()
    spec, m, k, idxs = case("darcy12")
    rp, ci, v, b, _ = P.assemble(spec, idxs[0])
    A = skr.CsrMatrix(spec.N, spec.N, rp, ci, v)
    cfg = skr.SolverConfig(m=m, k=k, tol=1e-8, max_iter=5000)

    class Foreign:  # stands in for kryrec.precond.SorPreconditioner etc.
        def __init__(self, kind, **kw):
            self.kind = kind
            self.n = spec.N
            self.__dict__.update(kw)

    for ktag, obj in (("sor12", Foreign("sor", omega=1.2)), ("ilu0", Foreign("ilu0")),
                      ("bjacobi", Foreign("bjacobi", block_size=20)),
                      ("jac", Foreign("jacobi", diag=A.diagonal()))):
        rep, _ = skr.gcrodr_solve(A, b, M=obj, cfg=cfg)
        assert rep.converged
        if ktag != "jac":
            assert abs(rep.iterations - int(GOLD[f"darcy12_{ktag}_iters"][0])) <= 1
            assert rel(rep.x, GOLD[f"darcy12_{ktag}_xs"][0]) < 1e-6
        else:
            ref, _ = skr.gcrodr_solve(A, b, M=skr.build_preconditioner(A, "jacobi"), cfg=cfg)
            assert rep.iterations == ref.iterations
    with pytest.raises(ValueError):
        skr.gcrodr_solve(A, b, M=Foreign("ssor"), cfg=cfg)
