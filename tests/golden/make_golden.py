"""Generate golden fixtures by running the REAL reference (kryrec) here.

Run in the build container (it needs /root/reference, which the GPU box does
not have):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

The fixtures pin (a) the oracle restatement in ``oracle/skr_oracle.py`` and
(b) the CUDA path. Inputs come from ``paper_2401_09516_b200.problems`` with
fixed seeds; each fixture stores a SHA-256 of its inputs so drift in the
generators is detected. BLAS threads are fixed to 1 because the reference's
own iteration counts depend on them at N >= 16k.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import kryrec  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def build(spec, idx):
    rp, ci, v, b, prm = P.assemble(spec, idx)
    A = kryrec.CsrMatrix(spec.N, spec.N, rp, ci, v)
    return A, b, prm


def run_chain(spec, n_sys, m, k, precond, max_iter=10000, keep_x=None, keep_u=None,
              tol=1e-8):
    """Reference chain exactly as harness.py:233-260 (lazy assembly)."""
    params, sysd = [], {}
    for i in range(n_sys):
        A, b, prm = build(spec, i)
        sysd[i] = (A, b)
        params.append(kryrec.ParameterMatrix(prm, problem_id=i))
    t = time.perf_counter()
    order = kryrec.greedy_sort(params)
    sort_s = time.perf_counter() - t
    cfg = kryrec.SolverConfig(m=m, tol=tol, max_iter=max_iter, k=k)
    recycle = None
    out = {"order": np.asarray(order), "iters": [], "conv": [], "true_rel": [],
           "hist_len": [], "kout": [], "wall": [], "sort_s": sort_s}
    xs, us, hists = [], [], []
    for pos, idx in enumerate(order):
        A, b = sysd[idx]
        M = kryrec.build_preconditioner(A, precond)
        rep, recycle = kryrec.gcrodr_solve(A, b, M=M, cfg=cfg, recycle_in=recycle,
                                           system_id=idx)
        out["iters"].append(rep.iterations)
        out["conv"].append(rep.converged)
        out["true_rel"].append(rep.true_relative_residual)
        out["hist_len"].append(len(rep.residual_history))
        out["kout"].append(recycle.k)
        out["wall"].append(rep.wall_time)
        if keep_x is None or pos < keep_x:
            xs.append(rep.x)
            hists.append(np.asarray(rep.residual_history))
        if keep_u is None or pos < keep_u:
            us.append(recycle.U)
        print(f"  {spec.name} pos {pos} sys {idx}: {rep.iterations} it, "
              f"k={recycle.k}, {rep.wall_time:.2f}s", flush=True)
    flat = np.stack([p.flat for p in params])
    res = {k_: np.asarray(v_) for k_, v_ in out.items()}
    res["x"] = np.stack(xs)
    kmax = max(u.shape[1] for u in us)
    U = np.zeros((len(us), spec.N, kmax))
    for i, u in enumerate(us):
        U[i, :, : u.shape[1]] = u
    res["U"] = U
    res["hist"] = np.concatenate(hists)
    res["hist_off"] = np.cumsum([0] + [len(h) for h in hists])
    res["input_sha"] = sha(flat, *[sysd[i][0].values for i in range(n_sys)],
                          *[sysd[i][1] for i in range(n_sys)])
    return res


def main():
    out = {}
    t0 = time.time()
    # --- small full chains: every x and U kept ----------------------------
    small = [
        ("darcy16", P.CONFIGS[0].reduced(n=16), 24, 12, 4, "none"),
        ("poisson16", P.CONFIGS[1].reduced(n=16), 16, 16, 5, "jacobi"),
        ("helmholtz16", P.CONFIGS[2].reduced(n=16), 12, 20, 6, "none"),
        ("darcy3d8", P.CONFIGS[3].reduced(n=8), 10, 12, 5, "jacobi"),
    ]
    for name, spec, ns, m, k, pc in small:
        print(name, flush=True)
        res = run_chain(spec, ns, m, k, pc, max_iter=20000)
        res["cfg"] = np.array([spec.cid, spec.n, ns, m, k, pc == "jacobi"])
        np.savez_compressed(os.path.join(HERE, f"chain_{name}.npz"), **res)
    # --- config 0 at full size: the BASELINE CPU-runnable run --------------
    spec = P.CONFIGS[0]
    print("config0 full", flush=True)
    res = run_chain(spec, spec.n_systems, spec.m, spec.k, spec.precond,
                    keep_x=4, keep_u=6)
    res["cfg"] = np.array([0, spec.n, spec.n_systems, spec.m, spec.k, 0])
    np.savez_compressed(os.path.join(HERE, "chain_c0.npz"), **res)
    # --- SpMV / Jacobi (sparse.py:155-160, precond.py:66-77) ---------------
    rng = np.random.default_rng(11)
    sp_out = {}
    for tag, spec in (("c0", P.CONFIGS[0]), ("c1r", P.CONFIGS[1].reduced(n=64)),
                      ("c3r", P.CONFIGS[3].reduced(n=16))):
        A, b, _ = build(spec, 5)
        x = rng.standard_normal(spec.N)
        sp_out[f"{tag}_x"] = x
        sp_out[f"{tag}_y"] = kryrec.spmv(A, x)
        M = kryrec.build_preconditioner(A, "jacobi")
        sp_out[f"{tag}_jy"] = M.apply(kryrec.spmv(A, x))
        sp_out[f"{tag}_sha"] = sha(A.values, A.col_idx, A.row_ptr)
    np.savez_compressed(os.path.join(HERE, "spmv.npz"), **sp_out)
    # --- sort (sorting.py:55-80) -------------------------------------------
    so = {}
    for tag, spec, ns in (("c1r", P.CONFIGS[1].reduced(n=32), 200),
                          ("c2r", P.CONFIGS[2].reduced(n=16), 96),
                          ("c4r", P.CONFIGS[4].reduced(n=24), 300)):
        flat = np.stack([P.system_params(spec, i)["params"] for i in range(ns)])
        so[f"{tag}_order"] = np.asarray(
            kryrec.greedy_sort([kryrec.ParameterMatrix(f) for f in flat]))
        so[f"{tag}_sha"] = sha(flat)
    # explicit ties: duplicated rows and equidistant candidates
    base = rng.integers(0, 3, size=(40, 33)).astype(np.float64)
    tie = np.concatenate([base, base[::3], base[5:9]], axis=0)
    so["ties_flat"] = tie
    so["ties_order"] = np.asarray(
        kryrec.greedy_sort([kryrec.ParameterMatrix(f) for f in tie]))
    so["scalar_order"] = np.asarray(kryrec.greedy_sort(
        [kryrec.ParameterMatrix(np.array([v])) for v in (0.0, 10.0, 1.0, 11.0)]))
    np.savez_compressed(os.path.join(HERE, "sort.npz"), **so)
    # --- small dense steps (gcrodr.py:126-240) -------------------------------
    de = {}
    for t in range(6):
        n = [5, 12, 20, 31, 40, 60][t]
        H = np.triu(rng.standard_normal((n + 1, n)), -1)
        H[np.arange(1, n + 1), np.arange(n)] = np.abs(H[np.arange(1, n + 1), np.arange(n)]) + 0.5
        de[f"hf{t}_H"] = H
        de[f"hf{t}_P"] = kryrec.harmonic_ritz_first_cycle(H[:n, :n], H[n, n - 1], min(10, n))
        kk = min(4 + t, n - 1)
        G = np.zeros((n + 1, n))
        G[:kk, :kk] = np.diag(rng.uniform(0.5, 2.0, kk))
        G[:kk, kk:] = rng.standard_normal((kk, n - kk)) * 0.1
        G[kk:, kk:] = np.triu(rng.standard_normal((n + 1 - kk, n - kk)), -1)
        X = np.linalg.qr(rng.standard_normal((3 * n, n)))[0]
        cross = X.T @ (X + 0.01 * rng.standard_normal(X.shape))
        de[f"hs{t}_G"] = G
        de[f"hs{t}_cross"] = cross
        de[f"hs{t}_k"] = np.array(kk)
        de[f"hs{t}_P"] = kryrec.harmonic_ritz_subsequent(G, cross, kk)
    np.savez_compressed(os.path.join(HERE, "dense.npz"), **de)
    print(f"done in {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
