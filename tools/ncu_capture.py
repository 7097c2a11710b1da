"""Workload for ncu captures of k_cycle in a bench chain shape: solve system 0
of config CID (warm-up, recycle space), then system 1 inside the NVTX range
"capture" with the per-chain CTA count of the bench (chain_grid_ctas(chains)).
Prints the capture solve's algorithmic SpMV+ortho bytes and k_cycle launches
(SURVEY 8(d)), the denominators of the DRAM/algorithmic ratio.
usage: python tools/ncu_capture.py CID [CTAS_PER_CHAIN]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_09516_b200 as skr  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctas = int(sys.argv[2]) if len(sys.argv) > 2 else 37
spec = P.CONFIGS[cid]
cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=spec.max_iter)
systems = [P.assemble_device(spec, i)[:2] for i in range(2)]
torch.cuda.synchronize()
g = ctas
r0 = skr.solve_sequence(systems, [0], cfg, spec.precond, keep_x="none", grid_ctas=g)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("capture")
r1 = skr.solve_sequence(systems, [1], cfg, spec.precond, keep_x="none", grid_ctas=g,
                        chain=r0.chain)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(json.dumps({"config": cid, "grid_ctas": g, "iterations": r1.iterations,
                  "converged": r1.converged, "k_cycle_launches": r1.cycles[0],
                  "algorithmic_bytes": r1.spmv_ortho_bytes,
                  "cycle_kernel_ms": r1.cycle_kernel_ms}))
