"""CPU checks of the C-ABI boundary and host logic (no compute without a GPU)."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "skr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(skr_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_2401_09516_b200 import _lib

    L = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), f"{s} declared in include/skr.h but not exported"
    assert set(_lib.EXPORTS) == set(syms)
    assert L.skr_version() == 101
    assert L.skr_status_string(0) == b"ok"


def test_report_struct_matches_header():
    """ctypes mirror of skr_report has the same fields, in order."""
    from paper_2401_09516_b200 import _lib

    src = open(os.path.join(ROOT, "include", "skr.h")).read()
    body = re.search(r"typedef struct skr_report \{(.*?)\} skr_report;", src, re.S).group(1)
    fields = re.findall(r"(?:int32_t|double)\s+([a-z_0-9]+);", body)
    assert fields == [f for f, _ in _lib.SkrReport._fields_]


def test_workspace_queries_host_only():
    from paper_2401_09516_b200 import _lib

    L = _lib.load()
    b1 = L.skr_gcrodr_workspace_bytes(65536, 40, 10, 10000)
    b3 = L.skr_gcrodr_workspace_bytes(2097152, 40, 20, 10000)
    assert b1 > 65536 * 8 * (2 * 11 + 41) and b3 > b1
    assert L.skr_gcrodr_workspace_bytes(100, 40, 40, 100) == 0  # k >= m
    assert L.skr_gcrodr_workspace_bytes(100, 64, 10, 100) == 0  # m + 1 > MMAX
    assert L.skr_sort_workspace_bytes(1024, 65536) >= 1024 * 1024 * 8
    assert L.skr_sort_workspace_bytes(0, 5) == 0


def test_no_gpu_fails_loudly():
    import torch

    import paper_2401_09516_b200 as skr

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    A = skr.eye(4)
    with pytest.raises(skr._lib.SkrExtensionError):
        skr.gcrodr_solve(A, np.ones(4))
    with pytest.raises(skr._lib.SkrExtensionError):
        skr.greedy_sort([skr.ParameterMatrix(np.ones(2))])
    with pytest.raises(skr._lib.SkrExtensionError):
        skr.spmv(A, np.ones(4))


def test_product_does_not_import_oracle():
    """The product package must not route through the CPU oracle."""
    pkg = os.path.join(ROOT, "paper_2401_09516_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            txt = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in re.sub(r"#.*", "", txt).replace('"""', ""), fn


def test_solver_config_and_csr_validation():
    import paper_2401_09516_b200 as skr

    with pytest.raises(ValueError):
        skr.SolverConfig(m=1)
    with pytest.raises(ValueError):
        skr.SolverConfig(k=50, m=50)
    with pytest.raises(ValueError):
        skr.SolverConfig(tol=0.0)
    cfg = skr.SolverConfig()
    assert (cfg.m, cfg.tol, cfg.max_iter, cfg.k) == (50, 1e-8, 10000, 10)
    with pytest.raises(ValueError, match="row_ptr"):
        skr.CsrMatrix(2, 2, [0, 1], [0], [1.0])
    with pytest.raises(ValueError, match="strictly increasing"):
        skr.CsrMatrix(2, 2, [0, 2, 2], [1, 0], [1.0, 2.0])
    with pytest.raises(ValueError, match="out of range"):
        skr.CsrMatrix(2, 2, [0, 1, 1], [2], [1.0])
    with pytest.raises(ValueError, match="finite"):
        skr.CsrMatrix(1, 1, [0, 1], [0], [np.nan])
    A = skr.CsrMatrix(3, 3, [0, 2, 3, 5], [0, 2, 1, 0, 2], [1.0, 2.0, 3.0, 4.0, 5.0])
    assert np.array_equal(A.diagonal(), [1.0, 3.0, 5.0])
    with pytest.raises(ValueError):
        skr.ParameterMatrix(np.array([np.inf]))
    with pytest.raises(skr.ZeroPivotError):
        skr.build_preconditioner(skr.CsrMatrix(2, 2, [0, 1, 2], [1, 0], [1.0, 1.0]), "jacobi")
    if not __import__("torch").cuda.is_available():
        # the factorization lives on the device: no CPU fallback
        with pytest.raises(skr._lib.SkrExtensionError):
            skr.build_preconditioner(skr.eye(2), "ilu0")
    with pytest.raises(ValueError):
        skr.build_preconditioner(skr.eye(2), "bogus")
    assert skr.build_preconditioner(skr.eye(3), "none").kind == "none"


def test_generators_match_reference_conventions():
    from paper_2401_09516_b200 import problems as P

    for cid, n in ((0, 16), (1, 16), (2, 16), (3, 8), (4, 16)):
        spec = P.CONFIGS[cid].reduced(n=n)
        rp, ci, v, b, prm = P.assemble(spec, 2)
        N = spec.N
        nnz = 5 * n * n - 4 * n if spec.dim == 2 else 7 * n ** 3 - 6 * n ** 2
        assert len(v) == nnz and rp[-1] == nnz
        import scipy.sparse as sp

        A = sp.csr_matrix((v, ci, rp), shape=(N, N))
        assert abs(A - A.T).max() == 0.0  # symmetric by construction
        d = A.diagonal()
        if spec.kind != "helmholtz":
            assert np.all(d < 0)  # negative-diagonal stencil
            if spec.kind == "darcy_binary":
                assert np.all(b < 0)  # b = -h^2 f with f = 1
            assert np.all(-d >= np.asarray(abs(A).sum(1)).ravel() + d - 1e-12)
        P2 = P.assemble(spec, 2)
        assert np.array_equal(P2[2], v) and np.array_equal(P2[4], prm)  # deterministic
    spec = P.CONFIGS[0]
    a = P.system_params(spec, 0)["a"]
    assert set(np.unique(a)) == {3.0, 12.0} and 0.2 < (a == 12).mean() < 0.8
    assert P.system_params(P.CONFIGS[2], 0)["params"].shape == (65537,)


def test_chain_grid_ctas_share():
    """Concurrent chains split the GPU: whole GPU for one chain, a share for
    several (never below 8 CTAs)."""
    from paper_2401_09516_b200.sequence import chain_grid_ctas

    assert chain_grid_ctas(1, sms=148) == 0
    assert chain_grid_ctas(8, sms=148) == 64
    assert chain_grid_ctas(4, sms=148) == 129
    assert chain_grid_ctas(200, sms=148) == 8


def test_skr_config_has_grid_ctas():
    from paper_2401_09516_b200 import _lib

    names = [f[0] for f in _lib.SkrConfig._fields_]
    assert names == ["m", "k", "max_iter", "grid_ctas", "tol", "flags"]
