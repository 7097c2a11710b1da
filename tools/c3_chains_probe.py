"""Probe: C3 systems through solve_chains (8 chains x 64 CTAs), per-system report."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_09516_b200 as skr  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 16
nch = int(sys.argv[3]) if len(sys.argv) > 3 else 8
spec = P.CONFIGS[cid]
cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=spec.max_iter)
systems = []
for i in range(ns):
    dA, b, _ = P.assemble_device(spec, i)
    systems.append((dA, b))
torch.cuda.synchronize()
chunks = skr.split_chunks(list(range(ns)), nch)
res = skr.solve_chains(systems, list(range(ns)), cfg, spec.precond, chunks, keep_x="none",
                       grid_ctas=int(os.environ.get("PROBE_CTAS", "0")) or skr.chain_grid_ctas(nch))
for ch, r in zip(chunks, res):
    print("chunk", ch, "iters", r.iterations, "conv", r.converged, "true_rel",
          [f"{v:.2e}" for v in r.true_rel], "warn", r.warn_bits, "v0proj", r.v0_projections)
