"""Oracle (reference arithmetic) chain on a few systems of a config, printing
|C^T r| / beta at every cycle start (the DCGS2 / V_0 analysis in DESIGN.md)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import skr_oracle as orc  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402

cid = int(sys.argv[1])
idxs = [int(v) for v in sys.argv[2].split(",")]
spec = P.CONFIGS[cid]
cfg = orc.Cfg(m=spec.m, tol=spec.tol, max_iter=spec.max_iter, k=spec.k)
U = None
for i in idxs:
    rp, ci, v, b, _ = P.assemble(spec, i)
    op = orc.Operator(rp, ci, v, spec.N, spec.precond == "jacobi")
    tr = []
    t0 = time.time()
    res = orc.gcrodr(op, b, cfg, U_in=U, trace=tr)
    U = res.U
    print(f"system {i}: iters {res.iterations} conv {res.converged} true_rel {res.true_rel:.3e} "
          f"({time.time() - t0:.0f} s)", flush=True)
    for it, beta, rat in tr:
        print(f"   it {it} beta {beta:.3e} cr/beta {rat:.3e}", flush=True)
