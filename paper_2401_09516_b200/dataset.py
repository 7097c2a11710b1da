"""Dataset export of a solved batch (the end product of SKR, PAPER step 6):
matrices, right-hand sides, solutions, parameters and a JSON manifest, in the
reference's formats (kryrec/harness.py:445-505 ``export_dataset``,
kryrec/io.py:17-59 Matrix Market + one-value-per-line vectors, %.17g so a
write/read round trip is bit-exact). Host-side IO: the solutions come back
from the device chains (``solve_sequence(..., keep_x="host")`` or
``solve_chains``); files are byte-identical to the reference's for the same
inputs (tests/golden/make_golden_dataset.py).
"""

from __future__ import annotations

import csv
import hashlib
import json
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from .sparse import CsrMatrix
from .sorting import ParameterMatrix

__all__ = ["LinearSystem", "system_hash", "write_matrix_market", "write_vector",
           "read_vector", "export_dataset"]


@dataclass
class LinearSystem:
    """One assembled system of a batch (kryrec/problems.py:62-75)."""

    A: CsrMatrix
    b: np.ndarray
    params: ParameterMatrix
    grid: tuple
    problem_kind: str
    id: int = 0

    @property
    def n(self) -> int:
        return self.A.n_rows


def system_hash(system: LinearSystem) -> str:
    """16-hex SHA-256 of (row_ptr, col_idx, values, b) (harness.py:147-151)."""
    h = hashlib.sha256()
    for arr in (system.A.row_ptr, system.A.col_idx, system.A.values, system.b):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()[:16]


def _g17(values) -> list:
    return ["%.17g" % v for v in np.asarray(values, dtype=np.float64).tolist()]


def write_matrix_market(A: CsrMatrix, path) -> None:
    """``coordinate real general``, 1-based, row-major (io.py:17-22)."""
    rows = np.repeat(np.arange(A.n_rows), np.diff(A.row_ptr))
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{A.n_rows} {A.n_cols} {A.nnz}\n")
        fh.writelines("%d %d %s\n" % (i + 1, j + 1, v)
                      for i, j, v in zip(rows.tolist(), np.asarray(A.col_idx).tolist(),
                                         _g17(A.values)))


def write_vector(x, path) -> None:
    """One value per line, %.17g (io.py:50-53)."""
    with open(path, "w") as fh:
        fh.writelines(v + "\n" for v in _g17(x))


def read_vector(path) -> np.ndarray:
    with open(path) as fh:
        return np.asarray([float(line) for line in fh if line.strip()], dtype=np.float64)


def export_dataset(batch: Sequence[LinearSystem], reports: Optional[Sequence], out_dir,
                   order: Optional[Sequence[int]] = None, config=None) -> str:
    """Write matrices, right-hand sides, solutions and a JSON manifest
    (harness.py:445-505). ``reports`` may be None or hold None entries
    (dataset without solutions); non-converged solves are flagged, still
    exported. ``config``: an object with ``config_hash()`` or a hash string.
    Returns the manifest path."""
    os.makedirs(out_dir, exist_ok=True)
    entries = []
    for i, system in enumerate(batch):
        stem = f"system_{system.id:04d}"
        mtx, rhs = f"{stem}.mtx", f"{stem}_rhs.txt"
        write_matrix_market(system.A, os.path.join(out_dir, mtx))
        write_vector(system.b, os.path.join(out_dir, rhs))
        entry = {"id": system.id, "problem_kind": system.problem_kind,
                 "grid": list(system.grid), "matrix_file": mtx, "rhs_file": rhs,
                 "matrix_hash": system_hash(system)}
        rep = reports[i] if reports is not None else None
        if rep is not None:
            sol = f"{stem}_x.txt"
            write_vector(rep.x, os.path.join(out_dir, sol))
            entry.update(solution_file=sol, iterations=rep.iterations,
                         converged=bool(rep.converged),
                         true_relative_residual=rep.true_relative_residual,
                         wall_time=rep.wall_time)
        entries.append(entry)
    with open(os.path.join(out_dir, "params.csv"), "w", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(["system_id", "params"])
        for system in batch:
            writer.writerow([system.id, " ".join(_g17(system.params.flat))])
    if config is None or isinstance(config, str):
        chash = config
    else:
        chash = config.config_hash()
    manifest = {"n_systems": len(batch),
                "solve_order": list(order) if order is not None else list(range(len(batch))),
                "config_hash": chash, "systems": entries}
    path = os.path.join(out_dir, "manifest.json")
    with open(path, "w") as fh:
        json.dump(manifest, fh, indent=2, sort_keys=True)
    return path
