"""Golden permutations of the reference's ``grouped_sort`` (sorting.py:83-111),
produced by running the REAL reference here (it needs /root/reference):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_grouped.py

Inputs are the seeded parameter batches of ``paper_2401_09516_b200.problems``
(continuous C1/C2 fields, binary C4 fields) plus a batch with duplicated rows.
"""

from __future__ import annotations

import hashlib
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import kryrec  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {}
    cases = (("c1r", P.CONFIGS[1].reduced(n=32), 200, (16, 50, 200)),
             ("c2r", P.CONFIGS[2].reduced(n=16), 96, (8, 40)),
             ("c4r", P.CONFIGS[4].reduced(n=24), 300, (2, 64)))
    for tag, spec, ns, sizes in cases:
        flat = np.stack([P.system_params(spec, i)["params"] for i in range(ns)])
        out[f"{tag}_sha"] = sha(flat)
        for gs in sizes:
            out[f"{tag}_g{gs}"] = np.asarray(
                kryrec.grouped_sort([kryrec.ParameterMatrix(f) for f in flat], gs))
    rng = np.random.default_rng(240109516)
    base = rng.standard_normal((30, 17))
    dup = np.concatenate([base, base[::4], base[3:6]], axis=0)
    out["dup_flat"] = dup
    out["dup_g7"] = np.asarray(kryrec.grouped_sort([kryrec.ParameterMatrix(f) for f in dup], 7))
    np.savez_compressed(os.path.join(HERE, "grouped.npz"), **out)
    print({k: v.shape for k, v in out.items() if hasattr(v, "shape")})


if __name__ == "__main__":
    main()
