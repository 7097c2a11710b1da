import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2401_09516_b200 as skr
from paper_2401_09516_b200 import problems as P
spec = P.CONFIGS[1].reduced(n=32)
sy = []
for i in range(2):
    rp, ci, v, b, _ = P.assemble(spec, i)
    sy.append((skr.CsrMatrix(spec.N, spec.N, rp, ci, v), b))
cfg = skr.SolverConfig(m=20, k=6, tol=1e-10)
A0, b0 = sy[0]; A1, b1 = sy[1]
M0 = skr.build_preconditioner(A0, "jacobi"); M1 = skr.build_preconditioner(A1, "jacobi")
r0, s0 = skr.gcrodr_solve(A0, b0, M=M0, cfg=cfg)
for d in (False, True, False, True, False):
    r, _ = skr.gcrodr_solve(A1, b1, M=M1, cfg=cfg, recycle_in=s0, collect_diagnostics=d)
    print("diag", d, "iters", r.iterations, "cycles", len(r.diagnostics.get("cycles", [])), r.diagnostics["restart_checks"][:2])
