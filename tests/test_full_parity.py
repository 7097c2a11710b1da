"""Full-size parity at the BASELINE.json configurations (BASELINE.md
section 3): the GPU path against fixtures produced by the REAL reference
(kryrec, OPENBLAS_NUM_THREADS=1) with tests/golden/make_golden_full.py.

* the full greedy-sort permutations of C1 / C2 (1,024 systems each), bit-exact;
* free-running chains over the reference's own prefixes (C1: the first 16
  sorted systems; C2: the first 4 sorted; C3: systems 0..3; C4: system 0):
  every solution meets the reference criterion, x matches the reference's on
  a fixed subsample (every stride-th entry) to 1e-6 relative, and the
  iteration counts match: the cold-started first system within 5%, the chain
  mean within 5% (per-system counts of a free-running chain drift with
  rounding);
* teacher-forced (SKR_FULL_PARITY=1, minutes of CPU on the box): every
  position solved with the reference arithmetic's incoming recycle U, which
  the oracle recomputes on the box, each within 5% of the oracle's count.
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _skr():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2401_09516_b200 as skr

    return skr


def _fixture(tag):
    path = os.path.join(GOLD, f"full_{tag}.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (tests/golden/make_golden_full.py {tag})")
    return np.load(path)


def _spec(cid):
    from paper_2401_09516_b200 import problems as P

    return P.CONFIGS[cid]


@pytest.mark.parametrize("tag,cid", [("c1", 1), ("c2", 2)])
def test_full_sort_permutation_matches_reference(tag, cid):
    """greedy_sort over all 1,024 parameter vectors == kryrec.greedy_sort."""
    skr = _skr()
    from paper_2401_09516_b200 import problems as P

    g = _fixture(tag)
    if "order" not in g:
        pytest.skip("fixture has no sort")
    spec = _spec(cid)
    flat = np.stack([P.system_params(spec, i)["params"] for i in range(spec.n_systems)])
    order = skr.greedy_sort_device(torch.from_numpy(flat).cuda())
    assert order == [int(v) for v in g["order"]]


def _device_systems(spec, idxs):
    from paper_2401_09516_b200 import problems as P

    out = []
    for i in idxs:
        dA, b, _ = P.assemble_device(spec, int(i))
        out.append((dA, b))
    torch.cuda.synchronize()
    return out


def _criterion(dA, b, x):
    """||M^-1 (b - A x)|| / ||M^-1 b|| with cuSPARSE (torch), M = diag or I."""
    S = torch.sparse_csr_tensor(dA.row_ptr.long(), dA.col_idx.long(), dA.values,
                                size=(dA.n, dA.n))
    r = b - (S @ x.unsqueeze(1)).squeeze(1)
    d = dA.diag if dA.diag is not None else torch.ones_like(b)
    return float(torch.linalg.norm(r / d) / torch.linalg.norm(b / d))


@pytest.mark.parametrize("tag,cid", [("c1", 1), ("c2", 2), ("c3", 3), ("c4", 4)])
def test_full_prefix_chain_matches_reference(tag, cid):
    skr = _skr()
    g = _fixture(tag)
    spec = _spec(cid)
    idxs = [int(v) for v in g["idx"]][: len(g["iters"])]
    stride = int(g["stride"])
    systems = _device_systems(spec, idxs)
    cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=spec.max_iter)
    res = skr.solve_sequence(systems, list(range(len(idxs))), cfg, spec.precond,
                             keep_x="device")
    it_gpu = np.array(res.iterations, dtype=float)
    it_ref = np.asarray(g["iters"], dtype=float)
    print(tag, "gpu", it_gpu.astype(int).tolist(), "ref", it_ref.astype(int).tolist())
    for p, (dA, b) in enumerate(systems):
        assert res.converged[p] and bool(g["conv"][p]), p
        assert _criterion(dA, b, res.x[p]) <= 1.05 * spec.tol, p
        xs = res.x[p][::stride].cpu().numpy()
        err = np.linalg.norm(xs - g["x_sub"][p]) / np.linalg.norm(g["x_sub"][p])
        assert err < 1e-6, (p, err)
        xn = float(torch.linalg.norm(res.x[p]))
        assert abs(xn - g["xnorm"][p]) <= 1e-6 * g["xnorm"][p], (p, xn, g["xnorm"][p])
    # the first system is a cold start (no recycle space): same problem
    assert abs(it_gpu[0] - it_ref[0]) <= 0.05 * it_ref[0]
    assert abs(it_gpu.mean() - it_ref.mean()) <= 0.05 * it_ref.mean()


@pytest.mark.skipif(os.environ.get("SKR_FULL_PARITY") != "1",
                    reason="teacher-forced full-size parity: set SKR_FULL_PARITY=1 (minutes)")
@pytest.mark.parametrize("cid,npos", [(1, 16), (3, 2), (2, 2)])
def test_teacher_forced_full_size(cid, npos):
    """Each position p >= 1 of the reference's prefix solved on the GPU with the
    recycle U the reference arithmetic (oracle, pinned to kryrec by the
    goldens) produced at p - 1: iterations within 5% of the oracle's and x
    within 1e-6 of it, per system."""
    skr = _skr()
    from oracle import skr_oracle as orc
    from paper_2401_09516_b200 import problems as P

    tag = f"c{cid}"
    g = _fixture(tag)
    spec = _spec(cid)
    idxs = [int(v) for v in g["idx"]][:npos]
    ocfg = orc.Cfg(m=spec.m, tol=spec.tol, max_iter=spec.max_iter, k=spec.k)
    cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=spec.max_iter)
    U = None
    rows = []
    for p, i in enumerate(idxs):
        rp, ci, v, b, _ = P.assemble(spec, i)
        op = orc.Operator(rp, ci, v, spec.N, spec.precond == "jacobi")
        ref = orc.gcrodr(op, b, ocfg, U_in=U)
        A = skr.CsrMatrix(spec.N, spec.N, rp, ci, v, validate=False)
        M = skr.build_preconditioner(A, spec.precond)
        rin = None if U is None else skr.RecycleSpace(U, None, U.shape[1])
        rep, _ = skr.gcrodr_solve(A, b, M=M, cfg=cfg, recycle_in=rin)
        err = np.linalg.norm(rep.x - ref.x) / np.linalg.norm(ref.x)
        rows.append((p, i, rep.iterations, ref.iterations, err))
        print(f"{tag} pos {p} sys {i}: gpu {rep.iterations} oracle {ref.iterations} "
              f"(kryrec free chain {int(g['iters'][p])}) x err {err:.1e}", flush=True)
        assert rep.converged and ref.converged
        assert abs(rep.iterations - ref.iterations) <= 0.05 * ref.iterations, rows[-1]
        assert err < 1e-6, rows[-1]
        U = ref.U


def test_c0_full_chain_matches_reference():
    """C0 (the BASELINE CPU-runnable run): the whole 256-system chain in the
    reference's sorted order, free-running on the GPU, against kryrec's own
    chain (tests/golden/chain_c0.npz): the permutation bit-exact, every system
    converged, the chain-mean iteration count within 5% and the per-system
    deviations small (a free-running chain drifts with rounding)."""
    skr = _skr()
    from paper_2401_09516_b200 import problems as P

    g = np.load(os.path.join(GOLD, "chain_c0.npz"))
    spec = _spec(0)
    flat = np.stack([P.system_params(spec, i)["params"] for i in range(spec.n_systems)])
    order = skr.greedy_sort_device(torch.from_numpy(flat).cuda())
    assert order == [int(v) for v in g["order"]]
    systems = _device_systems(spec, range(spec.n_systems))
    cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=spec.max_iter)
    res = skr.solve_sequence(systems, order, cfg, spec.precond, keep_x="none")
    it_gpu = np.array(res.iterations, dtype=float)
    it_ref = np.asarray(g["iters"], dtype=float)
    dev = (it_gpu - it_ref) / it_ref
    hist = np.histogram(np.abs(dev), bins=[0, 0.01, 0.02, 0.05, 0.1, 1.0])[0]
    print("C0 chain mean gpu %.2f ref %.2f; |dev| histogram [0,1,2,5,10,100]%%: %s"
          % (it_gpu.mean(), it_ref.mean(), hist.tolist()))
    assert all(res.converged)
    # measured: mean 309.6 vs 308.2; |dev| <1%: 45, 1-2%: 38, 2-5%: 97,
    # 5-10%: 64, >10%: 12 systems (a free-running chain's per-system counts
    # drift with rounding; BASELINE.md section 3 checks them teacher-forced)
    assert abs(it_gpu.mean() - it_ref.mean()) <= 0.05 * it_ref.mean()
    assert np.median(np.abs(dev)) <= 0.05
