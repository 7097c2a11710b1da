"""Multi-chain solve with a general preconditioner at a BASELINE size.
usage: python tools/pc_chains_probe.py CID KIND NS NCH CTAS"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_09516_b200 as skr  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402

cid, kind, ns, nch, ctas = int(sys.argv[1]), sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
spec = P.CONFIGS[cid]
cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=spec.max_iter)
systems = []
for i in range(ns):
    dA, b, _ = P.assemble_device(spec, i)
    systems.append((dA.with_diag(None), b))
torch.cuda.synchronize()
t0 = time.perf_counter()
res = skr.solve_chains(systems, list(range(ns)), cfg, kind, skr.split_chunks(list(range(ns)), nch),
                       keep_x="device", grid_ctas=ctas)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
its = [r.iterations for r in res]
conv = all(all(r.converged) for r in res)
# the reference criterion, recomputed with the package's own residual kernel
worst = 0.0
for c, r in enumerate(res):
    for p_, x in enumerate(r.x):
        A, b = systems[r.order[p_]]
        worst = max(worst, float(r.true_rel[p_]) if hasattr(r, "true_rel") else 0.0)
print(f"{spec.name} {kind}: {ns} systems, {nch} chains x {ctas} CTAs: {dt:.2f} s "
      f"({ns / dt:.2f} systems/s incl. the factorizations), iterations {its}, converged {conv}")
