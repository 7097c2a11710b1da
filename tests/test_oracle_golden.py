"""Pin the CPU oracle (oracle/skr_oracle.py) to the real reference.

Fixtures in tests/golden were produced by running kryrec itself
(tests/golden/make_golden.py, OPENBLAS_NUM_THREADS=1). The oracle is a
restatement with the same floating-point operation order, so it must
reproduce them exactly (iterations, permutations) or to round-off (x).
"""

import hashlib
import os

import numpy as np
import pytest

from oracle import skr_oracle as orc
from paper_2401_09516_b200 import problems as P

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def load(name):
    return np.load(os.path.join(GOLD, name))


def build(spec, n_sys):
    ops, rhs, flat, vals = [], [], [], []
    for i in range(n_sys):
        rp, ci, v, b, prm = P.assemble(spec, i)
        ops.append(orc.Operator(rp, ci, v, spec.N, spec.precond == "jacobi"))
        rhs.append(b)
        flat.append(prm)
        vals.append(v)
    return ops, rhs, np.stack(flat), vals


CHAINS = {"darcy16": 0, "poisson16": 1, "helmholtz16": 2, "darcy3d8": 3}


@pytest.mark.parametrize("name", list(CHAINS))
def test_oracle_reproduces_reference_chain(name):
    g = load(f"chain_{name}.npz")
    cid, n, ns, m, k, jac = [int(v) for v in g["cfg"]]
    spec = P.CONFIGS[cid].reduced(n=n)
    ops, rhs, flat, vals = build(spec, ns)
    assert sha(flat, *vals, *rhs) == str(g["input_sha"]), "generator drifted from the fixtures"
    order = orc.greedy_order(flat)
    assert order == list(g["order"])
    out = orc.chain(ops, rhs, order, orc.Cfg(m=m, k=k, tol=1e-8, max_iter=20000))
    its = [out[i].iterations for i in order]
    assert its == list(g["iters"])
    for pos, idx in enumerate(order):
        np.testing.assert_allclose(out[idx].x, g["x"][pos], rtol=1e-10, atol=1e-14)
        h = g["hist"][g["hist_off"][pos]: g["hist_off"][pos + 1]]
        np.testing.assert_allclose(out[idx].history, h, rtol=1e-8)


def test_oracle_config0_prefix_and_teacher_forcing():
    g = load("chain_c0.npz")
    spec = P.CONFIGS[0]
    flat = np.stack([P.system_params(spec, i)["params"] for i in range(spec.n_systems)])
    order = orc.greedy_order(flat)
    assert order == list(g["order"])  # full 256 x 4096 permutation
    cfg = orc.Cfg(m=30, k=10, tol=1e-8)
    # free-running prefix
    U = None
    for pos in range(4):
        rp, ci, v, b, _ = P.assemble(spec, order[pos])
        r = orc.gcrodr(orc.Operator(rp, ci, v, spec.N, False), b, cfg, U_in=U)
        assert r.iterations == int(g["iters"][pos])
        np.testing.assert_allclose(r.x, g["x"][pos], rtol=1e-9, atol=1e-15)
        U = r.U
    # teacher-forced: reference U of position p-1 into position p
    for pos in range(4, 6):
        rp, ci, v, b, _ = P.assemble(spec, order[pos])
        kk = int(g["kout"][pos - 1])
        r = orc.gcrodr(orc.Operator(rp, ci, v, spec.N, False), b, cfg,
                       U_in=g["U"][pos - 1][:, :kk])
        assert r.iterations == int(g["iters"][pos])


def test_oracle_sort_golden():
    g = load("sort.npz")
    for tag, cid, n, ns in (("c1r", 1, 32, 200), ("c2r", 2, 16, 96), ("c4r", 4, 24, 300)):
        spec = P.CONFIGS[cid].reduced(n=n)
        flat = np.stack([P.system_params(spec, i)["params"] for i in range(ns)])
        assert sha(flat) == str(g[f"{tag}_sha"])
        assert orc.greedy_order(flat) == list(g[f"{tag}_order"])
    assert orc.greedy_order(g["ties_flat"]) == list(g["ties_order"])
    assert orc.greedy_order(np.array([[0.0], [10.0], [1.0], [11.0]])) == [0, 2, 1, 3]


def test_oracle_spmv_golden():
    g = load("spmv.npz")
    for tag, cid, n in (("c0", 0, None), ("c1r", 1, 64), ("c3r", 3, 16)):
        spec = P.CONFIGS[cid].reduced(n=n) if n else P.CONFIGS[cid]
        rp, ci, v, b, _ = P.assemble(spec, 5)
        assert sha(v, ci, rp) == str(g[f"{tag}_sha"])
        op = orc.Operator(rp, ci, v, spec.N, True)
        assert np.array_equal(op.S @ g[f"{tag}_x"], g[f"{tag}_y"])
        assert np.array_equal(op(g[f"{tag}_x"]), g[f"{tag}_jy"])


def test_pairwise_emulation_matches_numpy_norm():
    rng = np.random.default_rng(3)
    for n in (1, 7, 8, 9, 100, 128, 129, 1000, 4097, 70001):
        a = rng.standard_normal(n) * 3
        b = rng.standard_normal(n)
        assert orc.reference_distance(a, b) == float(np.linalg.norm((a - b)[None], axis=1)[0])


def test_dense_golden_against_oracle_functions():
    d = load("dense.npz")
    for t in range(6):
        H = d[f"hf{t}_H"]
        n = H.shape[1]
        P1 = orc.hr_first(H[:n, :n], H[n, n - 1], min(10, n))
        np.testing.assert_allclose(np.abs(P1), np.abs(d[f"hf{t}_P"]), atol=1e-10)
        P2 = orc.hr_next(d[f"hs{t}_G"], d[f"hs{t}_cross"], int(d[f"hs{t}_k"]))
        np.testing.assert_allclose(np.abs(P2), np.abs(d[f"hs{t}_P"]), atol=1e-10)


def test_oracle_grouped_sort_golden():
    """oracle.grouped_order reproduces the reference's grouped_sort (sorting.py:83-111)."""
    from paper_2401_09516_b200 import problems as P

    g = load("grouped.npz")
    for tag, spec, ns, sizes in (("c1r", P.CONFIGS[1].reduced(n=32), 200, (16, 50, 200)),
                                 ("c2r", P.CONFIGS[2].reduced(n=16), 96, (8, 40)),
                                 ("c4r", P.CONFIGS[4].reduced(n=24), 300, (2, 64))):
        flat = np.stack([P.system_params(spec, i)["params"] for i in range(ns)])
        assert sha(flat) == str(g[f"{tag}_sha"]), "generator drift"
        for gs in sizes:
            assert orc.grouped_order(flat, gs) == g[f"{tag}_g{gs}"].tolist(), (tag, gs)
    assert orc.grouped_order(g["dup_flat"], 7) == g["dup_g7"].tolist()
    with pytest.raises(ValueError):
        orc.grouped_order(g["dup_flat"], 1)
