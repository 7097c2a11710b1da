"""Standalone apply time of the triangular preconditioners per dependency level.
usage: python tools/prof_pc_apply.py CID   (SKR_PC_GRID=G: CTAs of the apply kernel)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_09516_b200 as skr  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402

cid = int(sys.argv[1])
spec = P.CONFIGS[cid]
dA, b, _ = P.assemble_device(spec, 0)
v = torch.randn(spec.N, dtype=torch.float64, device="cuda")
for kind in ("sor", "ilu0"):
    M = skr.build_device_preconditioner(dA.with_diag(None), kind)
    M.apply(v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        M.apply(v)
    e1.record()
    torch.cuda.synchronize()
    print(f"{spec.name} {kind} grid {os.environ.get('SKR_PC_GRID', 'sms')}: apply "
          f"{e0.elapsed_time(e1) / 20:.3f} ms")
