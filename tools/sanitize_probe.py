"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): reduced C1 and C3 chains (k_cycle, k_dense, k_combine, refresh
kernels), several chains concurrently (native driver), the greedy sort and the
device assembly."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_09516_b200 as skr  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402

for cid, n, ns in ((1, 48, 3), (3, 12, 3), (0, 24, 4)):
    spec = P.CONFIGS[cid].reduced(n=n, n_systems=ns)
    cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=3000)
    sy = []
    prm = []
    for i in range(ns):
        rp, ci, v, b, p = P.assemble(spec, i)
        sy.append((skr.CsrMatrix(spec.N, spec.N, rp, ci, v), b))
        prm.append(skr.ParameterMatrix(p))
    order = skr.greedy_sort(prm)
    res = skr.solve_sequence(sy, order, cfg, spec.precond, keep_x="host")
    print("C%d" % cid, "order", order, "iters", res.iterations, "conv", res.converged, flush=True)
    dev = [P.assemble_device(spec, i)[:2] for i in range(ns)]
    out = skr.solve_chains(dev, list(range(ns)), cfg, spec.precond, [[0, 1], [2]] if ns == 3
                           else [[0, 1], [2, 3]], keep_x="device", grid_ctas=2)
    print("  chains", [r.iterations for r in out], [r.converged for r in out], flush=True)
torch.cuda.synchronize()
print("sanitize probe done")
