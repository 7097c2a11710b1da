import os, sys; sys.path.insert(0, '.')
import numpy as np
import paper_2401_09516_b200 as skr
from paper_2401_09516_b200 import problems as P
from oracle import skr_oracle as orc
spec = P.CONFIGS[1].reduced(n=32)
sy = []
for i in range(2):
    rp, ci, v, b, _ = P.assemble(spec, i)
    sy.append((skr.CsrMatrix(spec.N, spec.N, rp, ci, v), b))
cfg = skr.SolverConfig(m=20, k=6, tol=1e-10)
ocfg = orc.Cfg(m=20, tol=1e-10, k=6)
A0, b0 = sy[0]
M0 = skr.build_preconditioner(A0, "jacobi")
r0, s0 = skr.gcrodr_solve(A0, b0, M=M0, cfg=cfg, collect_diagnostics=True)
op0 = orc.Operator(A0.row_ptr, A0.col_idx, A0.values, spec.N, True)
f0 = orc.gcrodr(op0, b0, ocfg, collect_diagnostics=True)
print("iters", r0.iterations, f0.iterations)
for d, w in zip(r0.diagnostics["cycles"], f0.info["cycles"]):
    print(d["stage"], d["k"], w["k"], "au_c %.2e %.2e orth %.2e %.2e" % (d["au_c"], w["au_c"], d["orth"], w["orth"]))
print([ (round(a,12), round(b,12)) for a,b in r0.diagnostics["restart_checks"]][-3:])
