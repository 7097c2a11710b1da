"""Solve the first systems of a large config's chain (C3/C4 sizes) and report
k_cycle algorithmic bandwidth (SURVEY 8(d) bytes / CUDA-event time)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2401_09516_b200 as skr  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nsys = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = P.CONFIGS[cid]
cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=spec.max_iter)
t = time.time()
systems = []
for i in range(nsys):
    rp, ci, v, b, _ = P.assemble(spec, i)
    systems.append((skr.CsrMatrix(spec.N, spec.N, rp, ci, v, validate=False), b))
print(f"assembled {nsys} systems of N={spec.N} in {time.time() - t:.1f}s", flush=True)
res = skr.solve_sequence(systems, list(range(nsys)), cfg, spec.precond, keep_x="none")
_prof = np.zeros(32, dtype=np.int64)
skr._lib.load().skr_gcrodr_profile(res.chain.engine.ws.data_ptr(), res.chain.engine.nbytes, spec.N,
                                   cfg.m, cfg.k, _prof.ctypes.data)
print("k_cycle grid", int(_prof[30]), "rows/CTA", int(_prof[31]), flush=True)
peak = 6547.5
gbs = res.spmv_ortho_bytes / (res.cycle_kernel_ms / 1e3) / 1e9
out = {"config": cid, "N": spec.N, "iterations": res.iterations, "converged": res.converged,
       "device_ms": res.device_ms, "cycle_kernel_ms": res.cycle_kernel_ms,
       "dense_kernel_ms": res.dense_kernel_ms, "arnoldi_steps": res.arnoldi_steps,
       "us_per_step": 1000 * res.cycle_kernel_ms / res.arnoldi_steps,
       "spmv_ortho_GBps": gbs, "frac_of_measured_hbm": gbs / peak}
print(json.dumps(out))
