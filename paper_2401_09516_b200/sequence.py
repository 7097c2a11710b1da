"""The SKR chain: solve a sorted sequence of systems carrying the recycle space.

Restates the driving loop of the reference (kryrec/harness.py:233-260:
``rep, recycle = gcrodr_solve(A, b, M, cfg, recycle_in=recycle)`` over the
sorted order) for the device engine, with three B200-first changes:

* the recycle pair never leaves the GPU -- system i+1's refresh reads U from
  the workspace block system i left it in (no copies, no host round trip);
* the next system's CSR / right-hand side is uploaded on a side stream while
  the current one solves (double buffering), from pinned host memory when the
  caller provides it;
* multi-GPU: the sorted order splits into contiguous chunks, one independent
  chain per rank (the paper's parallel SKR); there is no
  collective on the solve path.
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import _lib
from .gcrodr import engine_for
from .gmres import SolverConfig
from .precond import DEVICE_KINDS, KINDS, build_device_preconditioner
from .sparse import DeviceCsr

__all__ = ["SequenceResult", "ChainState", "solve_sequence", "solve_chains", "chunk_positions",
           "split_chunks", "gather_results"]


@dataclass
class ChainState:
    """Where a chain stands between calls: the engine whose workspace holds
    the last recycle U (device pointer, leading dimension, columns)."""

    engine: object = None
    U_ptr: object = None
    ld: int = 0
    k: int = 0


@dataclass
class SequenceResult:
    order: list
    iterations: list = field(default_factory=list)
    converged: list = field(default_factory=list)
    true_rel: list = field(default_factory=list)
    device_ms: list = field(default_factory=list)
    k_out: list = field(default_factory=list)
    warn_bits: list = field(default_factory=list)
    v0_projections: list = field(default_factory=list)
    cycles: list = field(default_factory=list)
    spmv_ortho_bytes: float = 0.0
    x: list = field(default_factory=list)
    launches: int = 0
    cycle_kernel_ms: float = 0.0
    dense_kernel_ms: float = 0.0
    arnoldi_steps: int = 0
    chain: ChainState = None
    wall_s: float = 0.0
    h2d_bytes: int = 0
    d2h_bytes: int = 0


def chunk_positions(n: int, world: int, rank: int) -> range:
    """Contiguous positions of the sorted order owned by ``rank``."""
    per = -(-n // world)
    lo = min(n, rank * per)
    return range(lo, min(n, lo + per))


def _nbytes(t) -> int:
    return int(t.numel() * t.element_size())


def _with_general(dA, precond: str, stream, opts):
    """Attach the device-built preconditioner of kind ``precond`` (bjacobi, sor,
    ilu0, icc0; precond.py:251-312) unless the matrix already carries one."""
    if precond in DEVICE_KINDS and dA.precond is None:
        dA = dA.with_precond(build_device_preconditioner(dA, precond, stream=stream,
                                                         **(opts or {})))
    return dA


def _upload(sysobj, precond, stream, opts=None):
    """Host system -> (DeviceCsr, b_dev, bytes). Accepts (A, b) pairs where the
    arrays are numpy or (ideally pinned) torch CPU tensors, or a DeviceCsr."""
    import torch

    A, b = sysobj
    jacobi = precond == "jacobi"
    if isinstance(A, DeviceCsr):
        bt = b if isinstance(b, torch.Tensor) and b.is_cuda else torch.as_tensor(b).to("cuda")
        with torch.cuda.stream(stream):
            A = _with_general(A, precond, stream, opts)
        return A, bt, 0
    with torch.cuda.stream(stream):
        # the zero-pivot check is deferred (no sync on the upload stream)
        dA = DeviceCsr.from_host(A, jacobi=jacobi, non_blocking=True, stream=stream,
                                 check_pivot=False)
        dA = _with_general(dA, precond, stream, opts)
        if isinstance(b, torch.Tensor):
            bt = b.to("cuda", dtype=torch.float64, non_blocking=True)
        else:
            bt = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float64)).to("cuda")
        nb = _nbytes(dA.row_ptr) + _nbytes(dA.col_idx) + _nbytes(dA.values) + _nbytes(bt)
    return dA, bt, nb


def solve_sequence(systems: Sequence | Callable[[int], tuple], order: Sequence[int],
                   cfg: SolverConfig, precond: str = "none", *, positions: Sequence[int] = None,
                   keep_x: str = "host", stream=None, recycle_first=None,
                   want_history: bool = False, chain: ChainState = None,
                   engine_slot: int = 0, grid_ctas: int = 0,
                   precond_opts: dict = None) -> SequenceResult:
    """Solve ``systems[order[p]]`` for p in ``positions`` (default: all) as one
    recycling chain. ``systems`` is a sequence of (A, b) or a callable idx ->
    (A, b) (lazy generation for large configs). ``keep_x``: "host" (x copied
    back per system), "device" (kept as CUDA tensors) or "none". ``grid_ctas``:
    CTAs of the Arnoldi kernel (0 = whole GPU; see solve_chains)."""
    import torch

    _lib.require_cuda()
    if precond not in KINDS:
        raise ValueError(f"unknown preconditioner kind {precond!r}; expected one of {KINDS}")
    positions = list(range(len(order))) if positions is None else list(positions)
    get = systems if callable(systems) else (lambda i: systems[i])
    res = SequenceResult(order=[int(order[p]) for p in positions])
    if not positions:
        return res
    main = stream if stream is not None else torch.cuda.current_stream()
    side = torch.cuda.Stream()
    t0 = time.perf_counter()
    # first upload
    nxt = _upload(get(res.order[0]), precond, side, precond_opts)
    ev = torch.cuda.Event()
    ev.record(side)
    eng = None
    k_prev = 0
    U_prev_ptr, ld_prev = None, 0
    if chain is not None and chain.engine is not None:
        eng, U_prev_ptr, ld_prev, k_prev = chain.engine, chain.U_ptr, chain.ld, chain.k
        eng.c_cfg = _lib.SkrConfig(cfg.m, cfg.k, cfg.max_iter, int(grid_ctas), cfg.tol)
    elif recycle_first is not None and recycle_first.k > 0:
        from .gcrodr import _colmajor_device

        Ud, ld_prev = _colmajor_device(recycle_first.U, recycle_first.U.shape[0])
        U_prev_ptr, k_prev = Ud, int(Ud.shape[1])
    for i, idx in enumerate(res.order):
        main.wait_event(ev)
        dA, bt, nb = nxt
        res.h2d_bytes += nb
        if eng is None:
            eng = engine_for(dA.n, cfg, slot=engine_slot, grid_ctas=grid_ctas)
        # prefetch the next system while this one solves
        if i + 1 < len(res.order):
            nxt = _upload(get(res.order[i + 1]), precond, side, precond_opts)
            ev = torch.cuda.Event()
            ev.record(side)
        x = torch.empty(dA.n, dtype=torch.float64, device="cuda")
        with torch.cuda.stream(main):
            rep = eng.solve(dA, bt, x, None, U_prev_ptr, ld_prev, k_prev, stream=main,
                            want_history=want_history)
        res.iterations.append(int(rep.iterations))
        res.converged.append(bool(rep.converged))
        res.true_rel.append(float(rep.true_relative_residual))
        res.device_ms.append(float(rep.device_ms))
        res.k_out.append(int(rep.k_out))
        res.warn_bits.append(int(rep.warn_bits))
        res.v0_projections.append(int(rep.v0_projections))
        res.cycles.append(int(rep.cycles))
        res.spmv_ortho_bytes += float(rep.spmv_ortho_bytes)
        res.launches += int(rep.launches)
        res.cycle_kernel_ms += float(rep.cycle_kernel_ms)
        res.dense_kernel_ms += float(rep.dense_kernel_ms)
        res.arnoldi_steps += int(rep.arnoldi_steps)
        if keep_x == "host":
            res.x.append(x.cpu().numpy())
            res.d2h_bytes += _nbytes(x)
        elif keep_x == "device":
            res.x.append(x)
        # chain: the next refresh reads U where this solve left it
        if cfg.k > 0 and not rep.zero_rhs:
            u_ptr, ld = eng.u_ptr_ld()
            k = int(rep.k_out)
            U_prev_ptr = u_ptr if k else None
            ld_prev, k_prev = ld, k
    torch.cuda.synchronize()
    res.wall_s = time.perf_counter() - t0
    res.chain = ChainState(eng, U_prev_ptr, ld_prev, k_prev)
    return res


def split_chunks(positions: Sequence[int], parts: int) -> list:
    """Split a run of sorted positions into ``parts`` contiguous sub-chains."""
    positions = list(positions)
    per = -(-len(positions) // max(1, parts))
    return [positions[i: i + per] for i in range(0, len(positions), per)]


def chain_grid_ctas(n_chains: int, sms: int = None) -> int:
    """Per-chain CTA count of the Arnoldi kernel when ``n_chains`` chains share
    one GPU: the chains' cooperative kernels then run side by side on disjoint
    SM sets (each kernel's latency-bound phases - grid barriers, the serial LS
    update, the single-CTA dense recycle update - overlap the other chains'
    streaming sweeps). Measured on B200 at C1 (bench.py, 5 steps): 8 chains x
    64 CTAs 130 systems/s; x 48: 108; x 74: 119; x 96: 110; 4 x 100: 73;
    16 x 37: 95; one chain on the whole GPU: 24."""
    import torch

    if n_chains <= 1:
        return 0
    if sms is None:
        sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    return max(8, (7 * sms) // (2 * max(1, n_chains)))


def solve_chains(systems, order, cfg: SolverConfig, precond: str, chunks: Sequence,
                 keep_x: str = "host", states: Sequence = None, want_history: bool = False,
                 grid_ctas: int = None):
    """Run several independent recycling chains concurrently on one GPU, one
    host thread + CUDA stream + workspace each (the paper's chunked SKR,
    PAPER.md:2149-2184, applied inside a GPU). Each chunk is a contiguous run
    of sorted positions; chain i continues from ``states[i]`` if given.
    ``grid_ctas``: CTAs per chain (None = chain_grid_ctas(len(chunks))).
    Returns one SequenceResult per chunk."""
    import threading

    import torch

    _lib.require_cuda()
    dev = torch.cuda.current_device()
    if grid_ctas is None:
        grid_ctas = chain_grid_ctas(len(chunks))
    if keep_x in ("device", "none") and not want_history:
        native = _solve_chains_native(systems, order, cfg, precond, chunks, keep_x, states,
                                      grid_ctas)
        if native is not None:
            return native
    states = list(states) if states is not None else [None] * len(chunks)
    out = [None] * len(chunks)
    errs = []

    def work(i):
        try:
            torch.cuda.set_device(dev)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[i] = solve_sequence(systems, order, cfg, precond, positions=chunks[i],
                                        keep_x=keep_x, stream=st, chain=states[i],
                                        engine_slot=i, want_history=want_history,
                                        grid_ctas=grid_ctas)
        except BaseException as e:  # surfaced below
            errs.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(len(chunks))]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errs:
        raise errs[0]
    return out


def _solve_chains_native(systems, order, cfg, precond, chunks, keep_x, states, grid_ctas):
    """solve_chains through skr_gcrodr_solve_chains: one native host thread and
    stream per chain, no Python between systems. Only for device-resident
    systems (DeviceCsr + CUDA b); returns None otherwise (the threaded path
    then uploads host inputs per system)."""
    import ctypes

    import torch

    t_enter = time.perf_counter()
    get = systems if callable(systems) else (lambda i: systems[i])
    jacobi = precond == "jacobi"
    if precond not in KINDS:
        raise ValueError(f"unknown preconditioner kind {precond!r}; expected one of {KINDS}")
    sysl, firsts, idxs = [], [0], []
    for ch in chunks:
        for pos in ch:
            A, b = get(int(order[pos]))
            if not (isinstance(A, DeviceCsr) and isinstance(b, torch.Tensor) and b.is_cuda):
                return None
            if jacobi and A.c.diag is None:
                return None
            A = _with_general(A, precond, None, None)
            sysl.append((A, b))
            idxs.append(int(order[pos]))
        firsts.append(len(sysl))
    nch = len(chunks)
    states = list(states) if states is not None else [None] * nch
    n = sysl[0][0].n if sysl else 0
    engines = []
    for c in range(nch):
        st = states[c]
        if st is not None and st.engine is not None:
            eng = st.engine
            eng.c_cfg = _lib.SkrConfig(cfg.m, cfg.k, cfg.max_iter, int(grid_ctas), cfg.tol)
        else:
            eng = engine_for(n, cfg, slot=c, grid_ctas=grid_ctas)
        engines.append(eng)
    xs, arr = [], (_lib.SkrSystem * max(1, len(sysl)))()
    dev = sysl[0][1].device if sysl else None
    uniform = all(A.n == n for A, _ in sysl)
    # outputs: one allocation for the whole call (views per system), or one
    # scratch vector per chain when x is not kept
    rows = len(sysl) if keep_x == "device" else nch
    xbuf = torch.empty((rows, n), dtype=torch.float64, device=dev) if uniform and sysl else None
    for c in range(nch):
        for i in range(firsts[c], firsts[c + 1]):
            A, b = sysl[i]
            if xbuf is not None:
                x = xbuf[i] if keep_x == "device" else xbuf[c]
            else:
                x = torch.empty(A.n, dtype=torch.float64, device=b.device)
            xs.append(x)
            arr[i].A = A.c
            arr[i].b = b.data_ptr()
            arr[i].x = x.data_ptr()
    first_arr = (ctypes.c_int32 * (nch + 1))(*firsts)
    ws_arr = (ctypes.c_void_p * nch)(*[e.ws.data_ptr() for e in engines])
    u_arr = (ctypes.c_void_p * nch)()
    ld_arr = (ctypes.c_int32 * nch)()
    k_arr = (ctypes.c_int32 * nch)()
    for c in range(nch):
        st = states[c]
        if st is not None and st.U_ptr is not None and st.k > 0:
            u_arr[c], ld_arr[c], k_arr[c] = int(st.U_ptr), int(st.ld), int(st.k)
    reps = (_lib.SkrReport * max(1, len(sysl)))()
    nbytes = engines[0].nbytes if engines else 0
    torch.cuda.synchronize()  # inputs ready on every stream
    t0 = time.perf_counter()
    L = _lib.load()
    _lib.check(L.skr_gcrodr_solve_chains(arr, first_arr, nch, ctypes.byref(engines[0].c_cfg)
                                         if engines else None, ws_arr, nbytes, u_arr, ld_arr,
                                         k_arr, reps), "skr_gcrodr_solve_chains")
    wall = time.perf_counter() - t0
    t_native_end = time.perf_counter()
    out = []
    for c in range(nch):
        res = SequenceResult(order=idxs[firsts[c]:firsts[c + 1]])
        k_last, u_ptr, ld = 0, None, 0
        for i in range(firsts[c], firsts[c + 1]):
            rep = reps[i]
            res.iterations.append(int(rep.iterations))
            res.converged.append(bool(rep.converged))
            res.true_rel.append(float(rep.true_relative_residual))
            res.device_ms.append(float(rep.device_ms))
            res.k_out.append(int(rep.k_out))
            res.warn_bits.append(int(rep.warn_bits))
            res.v0_projections.append(int(rep.v0_projections))
            res.cycles.append(int(rep.cycles))
            res.spmv_ortho_bytes += float(rep.spmv_ortho_bytes)
            res.launches += int(rep.launches)
            res.cycle_kernel_ms += float(rep.cycle_kernel_ms)
            res.dense_kernel_ms += float(rep.dense_kernel_ms)
            res.arnoldi_steps += int(rep.arnoldi_steps)
            if keep_x == "device":
                res.x.append(xs[i])
            if cfg.k > 0 and not rep.zero_rhs:
                u_ptr, ld = engines[c].u_ptr_ld()
                k_last = int(rep.k_out)
        if firsts[c + 1] == firsts[c] and states[c] is not None:
            res.chain = states[c]
        else:
            res.chain = ChainState(engines[c], u_ptr if k_last else None, ld, k_last)
        res.wall_s = wall
        out.append(res)
    if os.environ.get("SKR_TRACE"):
        import sys as _sys

        print(f"trace py prep {1e3 * (t0 - t_enter):.2f} ms native {1e3 * wall:.2f} ms "
              f"post {1e3 * (time.perf_counter() - t_native_end):.2f} ms", file=_sys.stderr)
    return out


def gather_results(results: Sequence, positions: Sequence, group=None, dst: int = 0,
                   with_x: bool = True):
    """Collect every rank's chain results (this rank's ``results[i]`` solved
    the sorted ``positions[i]``) on rank ``dst`` in sorted-position order: the
    one collective of the multi-GPU path, after the solves.
    Returns a dict (positions, order, iterations, converged, true_rel,
    warn_bits, x) on ``dst`` and None elsewhere; x is gathered as host arrays
    (numpy), ``with_x=False`` skips it. Works on NCCL and gloo groups (object
    collectives)."""
    import torch.distributed as dist

    rows = []
    for r, pos in zip(results, positions):
        for q, p_ in enumerate(pos):
            x = None
            if with_x and q < len(r.x):
                x = r.x[q]
                x = x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)
            rows.append((int(p_), int(r.order[q]), int(r.iterations[q]), bool(r.converged[q]),
                         float(r.true_rel[q]) if q < len(r.true_rel) else float("nan"),
                         int(r.warn_bits[q]) if q < len(r.warn_bits) else 0, x))
    if dist.is_available() and dist.is_initialized():
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        out = [None] * world if rank == dst else None
        dist.gather_object(rows, out, dst=dst, group=group)
        if rank != dst:
            return None
        rows = [row for part in out for row in part]
    rows.sort(key=lambda t: t[0])
    keys = ("positions", "order", "iterations", "converged", "true_rel", "warn_bits", "x")
    return {k: [row[i] for row in rows] for i, k in enumerate(keys)}
