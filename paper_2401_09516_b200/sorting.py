"""Similarity ordering of a system batch on the GPU (kryrec/sorting.py).

``greedy_sort`` keeps the reference's signature and result (sorting.py:72-80):
start at index 0, repeatedly append the unvisited system nearest (Frobenius)
to the previous pick, ties to the smallest index. The distance matrix and
the chain run in libskr.so; see csrc/sort.cu for the exact / certified
arithmetic that makes the permutation bit-identical to the reference.
``sharded_greedy_sort`` splits the distance rows across ranks and gathers
them with torch.distributed (NCCL on the GPU box).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _lib

__all__ = ["ParameterMatrix", "frobenius_distance", "gather_distance_rows", "greedy_sort",
           "greedy_sort_device", "grouped_sort", "grouped_sort_device",
           "sharded_greedy_sort", "row_shard"]


@dataclass(frozen=True)
class ParameterMatrix:
    """Generative parameters of one system (sorting.py:16-33)."""

    values: np.ndarray
    problem_id: int = 0

    def __post_init__(self):
        v = np.atleast_2d(np.asarray(self.values, dtype=np.float64))
        if not np.all(np.isfinite(v)):
            raise ValueError("parameter entries must be finite")
        v = v.copy()
        v.flags.writeable = False
        object.__setattr__(self, "values", v)

    @property
    def flat(self) -> np.ndarray:
        return self.values.ravel()


def frobenius_distance(P: ParameterMatrix, Q: ParameterMatrix) -> float:
    if P.values.shape != Q.values.shape:
        raise ValueError(f"parameter shape mismatch: {P.values.shape} vs {Q.values.shape}")
    return float(np.linalg.norm(P.values - Q.values, "fro"))


def _stacked(params: Sequence) -> np.ndarray:
    if not params:
        raise ValueError("empty parameter batch")
    vals = [p.values if isinstance(p, ParameterMatrix) else
            np.atleast_2d(np.asarray(getattr(p, "values", p), dtype=np.float64))
            for p in params]
    shape = vals[0].shape
    for v in vals[1:]:
        if v.shape != shape:
            raise ValueError("inconsistent parameter shapes in batch")
    return np.stack([v.ravel() for v in vals])


class _SortWorkspace:
    cache: dict = {}

    @classmethod
    def get(cls, n_sys, P):
        import torch

        L = _lib.load()
        need = int(L.skr_sort_workspace_bytes(int(n_sys), int(P)))
        dev = torch.cuda.current_device()
        ws = cls.cache.get(dev)
        if ws is None or ws.numel() < need:
            ws = torch.empty(need, dtype=torch.uint8, device="cuda")
            cls.cache[dev] = ws
        return ws, need


def greedy_sort_device(flat_dev, stream=None) -> list[int]:
    """Greedy order of the rows of a (n_sys, P) float64 CUDA tensor."""
    L = _lib.load()
    n_sys, P = flat_dev.shape
    flat_dev = flat_dev.contiguous()
    ws, need = _SortWorkspace.get(n_sys, P)
    order = np.zeros(n_sys, dtype=np.int32)
    _lib.check(L.skr_greedy_sort(flat_dev.data_ptr(), int(n_sys), int(P), order.ctypes.data,
                                 ws.data_ptr(), need, _lib.stream_handle(stream)),
               "skr_greedy_sort")
    return [int(i) for i in order]


def greedy_sort(params: Sequence[ParameterMatrix]) -> list[int]:
    """Order the batch so consecutive parameter matrices are close (sorting.py:72-80)."""
    import torch

    flat = _stacked(params)
    _lib.require_cuda()
    return greedy_sort_device(torch.from_numpy(flat).to("cuda"))


def principal_keys_device(flat_dev, stream=None):
    """The first principal coordinate of every row of a (n_sys, P) float64 CUDA
    tensor (sorting.py:96-105: ``centered @ vt[0]`` with the reference's sign
    rule), as a CUDA tensor of n_sys keys. Own kernels only: the distance tiles
    of the sort (skr_sort_dist2), then the dominant eigenpair of the
    double-centered distance matrix (skr_sort_pca_keys)."""
    import torch

    n, P = flat_dev.shape
    flat_dev = flat_dev.contiguous()
    k = _DeviceSortKernels(stream)
    k.prepare(flat_dev)
    D2 = k.dist2_rows(flat_dev, 0, n)
    L = _lib.load()
    need = int(L.skr_sort_pca_workspace_bytes(int(n)))
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    keys = torch.empty(n, dtype=torch.float64, device="cuda")
    _lib.check(L.skr_sort_pca_keys(D2.data_ptr(), flat_dev.data_ptr(), int(n), int(P),
                                   keys.data_ptr(), ws.data_ptr(), need,
                                   _lib.stream_handle(stream)), "skr_sort_pca_keys")
    return keys


def grouped_sort_device(flat_dev, group_size: int, stream=None) -> list[int]:
    """``grouped_sort`` of the rows of a (n_sys, P) float64 CUDA tensor.

    The bucketing key (sorting.py:96-105) comes from ``principal_keys_device``
    (the dominant eigenvector of the batch's double-centered distance matrix,
    computed by this package's own kernels; the reference takes an SVD of the
    centered batch: equal up to rounding); the stable key order and the
    contiguous groups follow sorting.py:105-110, and every group's chain runs in
    the device greedy-sort kernels (rows gathered in ascending original index,
    so the lowest-index tie-break is the reference's)."""
    import torch

    if group_size < 2:
        raise ValueError("group_size must be >= 2")
    n, P = flat_dev.shape
    if n <= group_size:
        return greedy_sort_device(flat_dev, stream)
    key = principal_keys_device(flat_dev, stream).cpu().numpy()
    by_key = np.argsort(key, kind="stable")  # n_sys numbers: host control flow
    order: list[int] = []
    for start in range(0, n, group_size):
        g = np.sort(by_key[start:start + group_size])
        gd = torch.from_numpy(g).to(flat_dev.device)
        sub = greedy_sort_device(flat_dev.index_select(0, gd), stream)
        order.extend(int(g[i]) for i in sub)
    return order


def grouped_sort(params: Sequence[ParameterMatrix], group_size: int) -> list[int]:
    """Greedy sort within coarse groups; O(N * group_size) distance
    evaluations (sorting.py:83-111), on the GPU."""
    import torch

    if group_size < 2:
        raise ValueError("group_size must be >= 2")
    flat = _stacked(params)
    _lib.require_cuda()
    return grouped_sort_device(torch.from_numpy(flat).to("cuda"), group_size)


def row_shard(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row block [r0, r1) of rank ``rank`` out of ``world``."""
    per = -(-n // world)
    r0 = min(n, rank * per)
    return r0, min(n, r0 + per)


def gather_distance_rows(local, n_sys: int, group=None):
    """All-gather row blocks [row_shard(rank)] of the distance matrix into the
    full (n_sys, n_sys) matrix on every rank (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    per = -(-n_sys // world)
    pad = torch.zeros((per, n_sys), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    chunks = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(chunks, pad, group=group)
    return torch.cat(chunks)[:n_sys].contiguous()


class _DeviceSortKernels:
    """The C-ABI kernels behind sharded_greedy_sort (skr_sort_binary_check,
    skr_sort_dist2, skr_sort_chain). Tests substitute host stand-ins to
    exercise the multi-rank control flow on CPU (gloo)."""

    def __init__(self, stream=None):
        self.sh = _lib.stream_handle(stream)
        self.L = _lib.load()

    def prepare(self, flat):
        n_sys, P = flat.shape
        self.ws, self.need = _SortWorkspace.get(n_sys, P)
        v = np.zeros(2)
        isb = ctypes.c_int32()
        _lib.check(self.L.skr_sort_binary_check(flat.data_ptr(), n_sys, P, v.ctypes.data,
                                                ctypes.byref(isb), self.ws.data_ptr(), self.need,
                                                self.sh), "binary_check")
        self.isb, self.v = isb.value, v

    def dist2_rows(self, flat, r0, r1):
        import torch

        n_sys, P = flat.shape
        local = torch.zeros((max(r1 - r0, 0), n_sys), dtype=torch.float64, device="cuda")
        if r1 > r0:
            _lib.check(self.L.skr_sort_dist2(flat.data_ptr(), n_sys, P, r0, r1, self.isb,
                                             float(self.v[0]), float(self.v[1]), local.data_ptr(),
                                             self.ws.data_ptr(), self.need, self.sh), "dist2")
        return local

    def chain(self, D2, flat):
        import torch

        n_sys, P = flat.shape
        order = torch.zeros(n_sys, dtype=torch.int32, device="cuda")
        ncert = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.check(self.L.skr_sort_chain(D2.data_ptr(), flat.data_ptr(), n_sys, P, self.isb,
                                         order.data_ptr(), ncert.data_ptr(), self.sh), "chain")
        return [int(i) for i in order.cpu()]


def sharded_greedy_sort(flat_dev, group=None, stream=None, kernels=None) -> list[int]:
    """Multi-GPU greedy sort (sorting.py:55-80 over N ranks): rank r computes
    the squared-distance rows row_shard(n, N, r) (skr_sort_dist2), the row
    blocks are all-gathered (NCCL over NVLink on the GPU box), and every rank
    runs the same deterministic chain (skr_sort_chain, lowest-index ties)
    on the full matrix. Every rank holds all parameters."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n_sys = flat_dev.shape[0]
    flat_dev = flat_dev.contiguous()
    k = kernels if kernels is not None else _DeviceSortKernels(stream)
    k.prepare(flat_dev)
    r0, r1 = row_shard(n_sys, world, rank)
    local = k.dist2_rows(flat_dev, r0, r1)
    D2 = gather_distance_rows(local, n_sys, group)
    return k.chain(D2, flat_dev)
