"""Per-phase k_cycle profile (CTA 0 clocks) of every chain in the bench's
multi-chain shape: solve_chains over NS systems of config CID with NCH chains
x CTAS CTAs, then print each chain's last-solve phase times.
usage: python tools/prof_chains.py CID NS NCH CTAS"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_09516_b200 as skr  # noqa: E402
from paper_2401_09516_b200 import _lib, problems as P  # noqa: E402

cid, ns, nch, ctas = (int(a) for a in sys.argv[1:5])
spec = P.CONFIGS[cid]
cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=spec.max_iter)
systems = [P.assemble_device(spec, i)[:2] for i in range(ns)]
torch.cuda.synchronize()
chunks = skr.split_chunks(list(range(ns)), nch)
res = skr.solve_chains(systems, list(range(ns)), cfg, spec.precond, chunks, keep_x="none",
                       grid_ctas=ctas)
L = _lib.load()
names = ["sweep1", "barrier(red)", "LS+control", "sweep2", "barrier2"]
tot = np.zeros(32)
for c, r in enumerate(res):
    eng = r.chain.engine
    prof = np.zeros(32, dtype=np.int64)
    L.skr_gcrodr_profile(eng.ws.data_ptr(), eng.nbytes, spec.N, cfg.m, cfg.k, prof.ctypes.data)
    tot += prof
    its = max(1, prof[22])
    print(f"chain {c}: iters {r.iterations} device_ms {[round(x, 1) for x in r.device_ms]} "
          f"cycle_ms {r.cycle_kernel_ms:.1f} dense_ms {r.dense_kernel_ms:.1f}")
its = max(1, tot[22])
ncyc = max(1, tot[9])
for i, nm in enumerate(names):
    print(f"  all chains {nm:13s} {tot[16 + i] / its / 1.9e3:8.2f} us/iteration")
for i, nm in ((7, "last sweep2+y"), (8, "x update+Gram"), (9, "barrier x"), (10, "resid"),
              (11, "barrier"), (5, "reduce tail"), (12, "START update"), (13, "START V0+sync")):
    idx = 16 + i if i != 5 else 21
    print(f"  all chains cycle end {nm:14s} {tot[idx] / ncyc / 1.9e3:8.2f} us/cycle")
print("  dense calls", int(tot[9]), "sweeps", int(tot[22]))
