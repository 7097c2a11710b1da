"""Build / apply / solve timings of the general preconditioners at a BASELINE
size. usage: python tools/prof_precond.py CID [NSYS]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_09516_b200 as skr  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402

cid = int(sys.argv[1])
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = P.CONFIGS[cid]
cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=spec.max_iter)
systems = []
for i in range(ns):
    dA, b, _ = P.assemble_device(spec, i)
    systems.append((dA, b))
torch.cuda.synchronize()
v = torch.randn(spec.N, dtype=torch.float64, device="cuda")
for kind in ("jacobi", "sor", "ilu0", "icc0", "bjacobi"):
    if kind == "icc0" and cid == 2:
        continue
    line = f"{spec.name} {kind:8s}"
    if kind != "jacobi":
        t0 = time.perf_counter()
        M = skr.build_device_preconditioner(systems[0][0].with_diag(None), kind)
        torch.cuda.synchronize()
        t_build = time.perf_counter() - t0
        M.apply(v)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            M.apply(v)
        e1.record()
        torch.cuda.synchronize()
        line += f" build {1e3 * t_build:8.1f} ms  apply {e0.elapsed_time(e1) / 10:7.3f} ms"
    syss = [(A if kind == "jacobi" else A.with_diag(None), b) for A, b in systems]
    res = skr.solve_sequence(syss, list(range(ns)), cfg, kind, keep_x="none")
    line += f"  iterations {res.iterations} device_ms {[round(x, 1) for x in res.device_ms]} conv {res.converged}"
    print(line, flush=True)
