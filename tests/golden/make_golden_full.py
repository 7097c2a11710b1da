"""Full-size golden fixtures from the REAL reference (kryrec), BASELINE.md §3.

Run here (the GPU box has no /root/reference); one job per configuration:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_full.py c1
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_full.py c2
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_full.py c3
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_full.py c4

Writes ``tests/golden/full_<cfg>.npz``:

* C1 / C2: the permutation of the reference's ``greedy_sort`` over all 1,024
  parameter vectors (sorting.py:72-80), then the reference chain
  (harness.py:233-260) over the first sorted positions (C1 16, C2 4);
* C3 / C4: the reference chain over systems 0.. in index order (C3 4, C4 1):
  their full sorts (8.6 / 34 GB of parameters) are infeasible on the CPU, and
  solver parity does not depend on which neighbour comes first.

Per position: iterations, converged, true relative residual, residual-history
length, ||x|| and a fixed subsample of x (every ``stride``-th entry, <= 8,192
values), wall time. x itself (up to 16 MB per system) and the recycle U are not
stored; tests that teacher-force the GPU chain regenerate the reference's U
with the oracle on the GPU box (tests/test_full_parity.py).
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

PLAN = {  # cfg: (config id, sort all?, positions)
    "c1": (1, True, 16),
    "c2": (2, True, 4),
    "c3": (3, False, 4),
    "c4": (4, False, 1),
}


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def stride_of(n: int) -> int:
    s = 1
    while n // s > 8192:
        s *= 2
    return s


def main(tag: str):
    cid, do_sort, npos = PLAN[tag]
    spec = P.CONFIGS[cid]
    out = {"cfg": np.array([cid, spec.n, spec.n_systems, spec.m, spec.k,
                            spec.precond == "jacobi", spec.max_iter])}
    t0 = time.time()
    if do_sort:
        flat = np.stack([P.system_params(spec, i)["params"] for i in range(spec.n_systems)])
        out["params_sha"] = sha(flat)
        params = [kryrec.ParameterMatrix(f, problem_id=i) for i, f in enumerate(flat)]
        del flat
        t = time.perf_counter()
        order = kryrec.greedy_sort(params)
        out["sort_s"] = time.perf_counter() - t
        out["order"] = np.asarray(order)
        del params
        print(f"{tag}: sort {out['sort_s']:.0f}s, first {order[:npos]}", flush=True)
        idxs = list(order[:npos])
    else:
        idxs = list(range(npos))
    out["idx"] = np.asarray(idxs)
    stride = stride_of(spec.N)
    out["stride"] = np.array(stride)
    cfg = kryrec.SolverConfig(m=spec.m, tol=spec.tol, max_iter=spec.max_iter, k=spec.k)
    recycle = None
    rec = {k: [] for k in ("iters", "conv", "true_rel", "hist_len", "kout", "wall", "xnorm",
                           "x_sub", "hist_tail", "sys_sha")}
    for pos, idx in enumerate(idxs):
        rp, ci, v, b, _ = P.assemble(spec, idx)
        A = kryrec.CsrMatrix(spec.N, spec.N, rp, ci, v)
        M = kryrec.build_preconditioner(A, spec.precond)
        rep, recycle = kryrec.gcrodr_solve(A, b, M=M, cfg=cfg, recycle_in=recycle,
                                           system_id=idx)
        rec["iters"].append(rep.iterations)
        rec["conv"].append(rep.converged)
        rec["true_rel"].append(rep.true_relative_residual)
        rec["hist_len"].append(len(rep.residual_history))
        rec["kout"].append(recycle.k)
        rec["wall"].append(rep.wall_time)
        rec["xnorm"].append(float(np.linalg.norm(rep.x)))
        rec["x_sub"].append(np.asarray(rep.x)[::stride].copy())
        rec["hist_tail"].append(np.asarray(rep.residual_history)[-4:])
        rec["sys_sha"].append(sha(v, b))
        print(f"{tag} pos {pos} sys {idx}: {rep.iterations} it conv {rep.converged} "
              f"true_rel {rep.true_relative_residual:.3e} k={recycle.k} "
              f"{rep.wall_time:.1f}s", flush=True)
        # partial results survive an interrupted run
        res = dict(out)
        res.update({k: np.asarray(v_) for k, v_ in rec.items() if k not in ("x_sub", "hist_tail")})
        res["x_sub"] = np.stack(rec["x_sub"])
        res["hist_tail"] = np.stack(rec["hist_tail"])
        res["threads"] = np.array(int(os.environ.get("OPENBLAS_NUM_THREADS", "0")))
        np.savez_compressed(os.path.join(HERE, f"full_{tag}.npz"), **res)
    print(f"{tag} done in {time.time() - t0:.0f}s", flush=True)


if __name__ == "__main__":
    for t in sys.argv[1:]:
        main(t)
