"""Profile the per-cycle dense recycle kernel and the cycle kernel on C1 systems."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2401_09516_b200 as skr  # noqa: E402
from paper_2401_09516_b200 import _lib, problems as P  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
nsys = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = P.CONFIGS[cid]
cfg = skr.SolverConfig(m=spec.m, k=spec.k, tol=spec.tol, max_iter=spec.max_iter)
systems = []
for i in range(nsys):
    rp, ci, v, b, _ = P.assemble(spec, i)
    systems.append((skr.CsrMatrix(spec.N, spec.N, rp, ci, v), b))
res = skr.solve_sequence(systems, list(range(nsys)), cfg, spec.precond, keep_x="none",
                         grid_ctas=int(os.environ.get("SKR_PROF_CTAS", "0")))
eng = res.chain.engine
L = _lib.load()
prof = np.zeros(32, dtype=np.int64)
L.skr_gcrodr_profile(eng.ws.data_ptr(), eng.nbytes, spec.N, cfg.m, cfg.k, prof.ctypes.data)
calls = max(1, prof[9])
names = ["products", "LU", "solve+kappa", "eig(hess+QR)", "select+eigvec", "qrcp(P)", "GP tail"]
print("iterations", res.iterations, "device_ms", [round(x, 2) for x in res.device_ms])
print("cycle_ms", round(res.cycle_kernel_ms, 2), "dense_ms", round(res.dense_kernel_ms, 2),
      "steps", res.arnoldi_steps, "us/step", round(1000 * res.cycle_kernel_ms / res.arnoldi_steps, 2))
print("dense calls (last solve)", calls, "QR its/call", prof[7] / calls, "bulge/call", prof[8] / calls)
names[3] = "hqr"
for i, nm in enumerate(names):
    print(f"  {nm:14s} {prof[i] / calls / 1.9e3:9.1f} us/call (at 1.9 GHz)")
print(f"  {'hessenberg':14s} {prof[10] / calls / 1.9e3:9.1f} us/call")
for i, nm in enumerate(["hqr scan+shift", "hqr scalars", "hqr row mod", "hqr col+Z mod"]):
    print(f"  {nm:14s} {prof[11 + i] / calls / 1.9e3:9.1f} us/call  ({prof[11 + i] / max(1, prof[8]):.0f} cyc/bulge)")
its = max(1, prof[22])
for i, nm in enumerate(["sweep1", "barrier(red)", "LS+control", "sweep2", "barrier2"]):
    print(f"  cycle {nm:13s} {prof[16 + i] / its / 1.9e3:8.2f} us/iteration")
ncyc = max(1, prof[9])
for i, nm in ((7, "last sweep2+y"), (8, "x update"), (9, "barrier x"), (10, "resid+Gram"),
              (11, "barrier Gram"), (5, "reduce tail"), (12, "START update"), (13, "START V0+sync")):
    idx = 16 + i if i != 5 else 21
    print(f"  cycle end {nm:14s} {prof[idx] / ncyc / 1.9e3:8.2f} us/cycle")
