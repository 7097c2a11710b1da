"""SHA-256 of every file the REAL reference's ``export_dataset``
(kryrec/harness.py:445-505) writes for a small seeded batch with fixed
solutions; tests/test_dataset.py checks this package's writer against them.
Needs /root/reference:  python tests/golden/make_golden_dataset.py
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import kryrec  # noqa: E402
from kryrec.harness import export_dataset  # noqa: E402
from kryrec.problems import LinearSystem  # noqa: E402
from paper_2401_09516_b200 import problems as P  # noqa: E402


class _Rep:
    def __init__(self, x, it, conv, rel, wt):
        self.x, self.iterations, self.converged = x, it, conv
        self.true_relative_residual, self.wall_time = rel, wt


def batch_and_reports():
    """Shared with the test: 3 reduced C1 systems + fixed pseudo-solutions."""
    spec = P.CONFIGS[1].reduced(n=6)
    out = []
    for i in range(3):
        rp, ci, v, b, prm = P.assemble(spec, i)
        out.append((rp, ci, v, b, prm))
    rng = np.random.default_rng(3)
    reps = [(rng.standard_normal(spec.N), 17 + i, i != 1, 1e-9 * (i + 1), 0.25 * i)
            for i in range(3)]
    return spec, out, reps


def main():
    spec, sys_, reps = batch_and_reports()
    batch = [LinearSystem(kryrec.CsrMatrix(spec.N, spec.N, rp, ci, v), b,
                          kryrec.ParameterMatrix(prm.reshape(spec.n, spec.n)),
                          (spec.n, spec.n), "poisson_lognormal", id=10 + i)
             for i, (rp, ci, v, b, prm) in enumerate(sys_)]
    reports = [_Rep(*r) for r in reps]
    reports[2] = None
    with tempfile.TemporaryDirectory() as d:
        export_dataset(batch, reports, d, order=[2, 0, 1], config=None)
        hashes = {f: hashlib.sha256(open(os.path.join(d, f), "rb").read()).hexdigest()
                  for f in sorted(os.listdir(d))}
    with open(os.path.join(HERE, "dataset_sha.json"), "w") as fh:
        json.dump(hashes, fh, indent=1, sort_keys=True)
    print(hashes)


if __name__ == "__main__":
    main()
