"""Oracle (reference arithmetic) chain over given C2 systems with max_iter
50,000: does the reference itself converge where the GPU chain times out?
usage: python tools/oracle_c2_chain.py IDX [IDX ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import skr_oracle as orc  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402

spec = P.CONFIGS[2]
U = None
for i in [int(a) for a in sys.argv[1:]]:
    rp, ci, v, b, prm = P.assemble(spec, i)
    op = orc.Operator(rp, ci, v, spec.N, False)
    t = time.time()
    r = orc.gcrodr(op, b, orc.Cfg(m=spec.m, tol=spec.tol, max_iter=spec.max_iter, k=spec.k),
                   U_in=U)
    U = r.U
    print("sys", i, "k0 %.2f" % prm[0], "iters", r.iterations, "conv", r.converged,
          "true_rel %.3e" % r.true_rel, "%.0fs" % (time.time() - t), flush=True)
