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
           "read_vector", "export_dataset", "DatasetWriter"]


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


class DatasetWriter:
    """Streaming, multi-rank form of ``export_dataset``: every rank writes the
    files of its own systems as their solves finish (``add``), so nothing but
    the manifest rows is held; ``close`` gathers the manifest entries and the
    parameter rows on rank 0 (object gather; NCCL or gloo), which writes
    params.csv and manifest.json. For a batch whose ids are 0..n-1 the files
    are byte-identical to ``export_dataset(batch, reports, out_dir, order,
    config)`` in one process (tests/test_multirank_gloo.py). Single-process
    use (no process group) works the same."""

    def __init__(self, out_dir, order: Optional[Sequence[int]] = None, config=None, group=None):
        self.out_dir = out_dir
        self.order = None if order is None else [int(o) for o in order]
        self.config = config
        self.group = group
        self.entries = []
        self.params = []
        os.makedirs(out_dir, exist_ok=True)

    def add(self, system: LinearSystem, report=None) -> None:
        stem = f"system_{system.id:04d}"
        mtx, rhs = f"{stem}.mtx", f"{stem}_rhs.txt"
        write_matrix_market(system.A, os.path.join(self.out_dir, mtx))
        write_vector(system.b, os.path.join(self.out_dir, rhs))
        entry = {"id": system.id, "problem_kind": system.problem_kind,
                 "grid": list(system.grid), "matrix_file": mtx, "rhs_file": rhs,
                 "matrix_hash": system_hash(system)}
        if report is not None:
            sol = f"{stem}_x.txt"
            write_vector(report.x, os.path.join(self.out_dir, sol))
            entry.update(solution_file=sol, iterations=report.iterations,
                         converged=bool(report.converged),
                         true_relative_residual=report.true_relative_residual,
                         wall_time=report.wall_time)
        self.entries.append(entry)
        self.params.append((system.id, " ".join(_g17(system.params.flat))))

    def close(self) -> Optional[str]:
        entries, params = self.entries, self.params
        try:
            import torch.distributed as dist

            dist_on = dist.is_available() and dist.is_initialized()
        except ImportError:  # pragma: no cover
            dist_on = False
        if dist_on:
            rank, world = dist.get_rank(self.group), dist.get_world_size(self.group)
            out = [None] * world if rank == 0 else None
            dist.gather_object((entries, params), out, dst=0, group=self.group)
            if rank != 0:
                return None
            entries = [e for part in out for e in part[0]]
            params = [p for part in out for p in part[1]]
        entries = sorted(entries, key=lambda e: e["id"])
        params = sorted(params, key=lambda p: p[0])
        with open(os.path.join(self.out_dir, "params.csv"), "w", newline="") as fh:
            writer = csv.writer(fh)
            writer.writerow(["system_id", "params"])
            for sid, row in params:
                writer.writerow([sid, row])
        cfg = self.config
        chash = cfg if cfg is None or isinstance(cfg, str) else cfg.config_hash()
        n = len(entries)
        manifest = {"n_systems": n,
                    "solve_order": self.order if self.order is not None else list(range(n)),
                    "config_hash": chash, "systems": entries}
        path = os.path.join(self.out_dir, "manifest.json")
        with open(path, "w") as fh:
            json.dump(manifest, fh, indent=2, sort_keys=True)
        return path
