"""Dataset export (kryrec/harness.py:445-505, io.py:17-59): this package's
writer produces byte-identical files to the reference's for the same batch
(golden SHA-256 from tests/golden/make_golden_dataset.py), and the vectors
round-trip bit-exactly."""

import hashlib
import json
import os

import numpy as np

from paper_2401_09516_b200 import dataset as D
from paper_2401_09516_b200 import problems as P
from paper_2401_09516_b200.sorting import ParameterMatrix
from paper_2401_09516_b200.sparse import CsrMatrix

GOLD = os.path.join(os.path.dirname(__file__), "golden")


class _Rep:
    def __init__(self, x, it, conv, rel, wt):
        self.x, self.iterations, self.converged = x, it, conv
        self.true_relative_residual, self.wall_time = rel, wt


def _batch():
    spec = P.CONFIGS[1].reduced(n=6)
    batch = []
    for i in range(3):
        rp, ci, v, b, prm = P.assemble(spec, i)
        batch.append(D.LinearSystem(CsrMatrix(spec.N, spec.N, rp, ci, v), b,
                                    ParameterMatrix(prm.reshape(spec.n, spec.n)),
                                    (spec.n, spec.n), "poisson_lognormal", id=10 + i))
    rng = np.random.default_rng(3)
    reps = [_Rep(rng.standard_normal(spec.N), 17 + i, i != 1, 1e-9 * (i + 1), 0.25 * i)
            for i in range(3)]
    reps[2] = None
    return batch, reps


def test_export_matches_reference_bytes(tmp_path):
    batch, reps = _batch()
    path = D.export_dataset(batch, reps, tmp_path, order=[2, 0, 1])
    assert os.path.basename(path) == "manifest.json"
    gold = json.load(open(os.path.join(GOLD, "dataset_sha.json")))
    got = {f: hashlib.sha256(open(os.path.join(tmp_path, f), "rb").read()).hexdigest()
           for f in sorted(os.listdir(tmp_path))}
    assert got == gold


def test_vector_round_trip_is_bit_exact(tmp_path):
    x = np.random.default_rng(1).standard_normal(257) * 10.0 ** np.arange(-128, 129)
    D.write_vector(x, tmp_path / "x.txt")
    assert np.array_equal(D.read_vector(tmp_path / "x.txt"), x)


def _sha_dir(path):
    return {f: hashlib.sha256(open(os.path.join(path, f), "rb").read()).hexdigest()
            for f in sorted(os.listdir(path))}


def test_streaming_writer_matches_reference_bytes(tmp_path):
    """DatasetWriter (one system at a time, no process group) == export_dataset."""
    batch, reps = _batch()
    w = D.DatasetWriter(tmp_path, order=[2, 0, 1])
    for s, r in zip(batch, reps):
        w.add(s, r)
    assert os.path.basename(w.close()) == "manifest.json"
    assert _sha_dir(tmp_path) == json.load(open(os.path.join(GOLD, "dataset_sha.json")))


def _writer_rank(rank, world, port, out_dir, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        batch, reps = _batch()
        w = D.DatasetWriter(out_dir, order=[2, 0, 1])
        for i, (s, r) in enumerate(zip(batch, reps)):
            if i % world == rank:  # interleaved ownership: the gather restores batch order
                w.add(s, r)
        q.put((rank, w.close()))
    finally:
        dist.destroy_process_group()


def test_multirank_writer_matches_reference_bytes(tmp_path):
    """Two gloo ranks each write their own systems' files; rank 0 gathers the
    manifest rows: the directory is byte-identical to the reference's export."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_writer_rank, args=(r, 2, port, str(tmp_path), q))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    out = dict(q.get(timeout=10) for _ in range(2))
    assert out[1] is None and os.path.basename(out[0]) == "manifest.json"
    assert _sha_dir(tmp_path) == json.load(open(os.path.join(GOLD, "dataset_sha.json")))
