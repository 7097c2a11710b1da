"""GPU counterpart of tools/oracle_c2_chain.py: the same C2 chain, and the
last system cold. usage: python tools/c2_gpu_chain.py IDX [IDX ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_09516_b200 as skr  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402

spec = P.CONFIGS[2]
cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=spec.max_iter)
idx = [int(a) for a in sys.argv[1:]]
sy = [P.assemble_device(spec, i)[:2] for i in idx]
r = skr.solve_sequence(sy, list(range(len(idx))), cfg, "none", keep_x="none")
print("chain", idx, r.iterations, r.converged, [f"{t:.2e}" for t in r.true_rel])
r = skr.solve_sequence(sy, [len(idx) - 1], cfg, "none", keep_x="none")
print("cold", idx[-1], r.iterations, r.converged, [f"{t:.2e}" for t in r.true_rel])
