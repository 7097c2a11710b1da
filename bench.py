#!/usr/bin/env python
"""SKR hot-path benchmark: systems solved/s (rel-res 1e-8, fp64) on B200.

Workload (default BASELINE.json configs[3], "C3"): 3-D Darcy flow on a 128^3
grid (N = 2,097,152, 7-point FD, ~14.6 M nonzeros), a batch of 512 systems
with a in {3, 12} from a thresholded GRF, greedy-NN sorted on a, solved as
GCRO-DR(40, 20) chains with Jacobi, tol 1e-8. C3 is the largest single-GPU
configuration whose working set (1.6 GB per chain) is far beyond the 126 MB
L2, i.e. the HBM-gated one of SURVEY 8(d). ``--config 1`` etc. select the
other configurations.

The sorted order is split into contiguous per-GPU chunks (one set of
recycling chains per rank, weak scaling, no collective on the solve path).
Inside a GPU the chunk is split again into ``--chains`` concurrent chains
(each on its own stream with a share of the SMs). A bench *step* = one
stripe of S consecutive systems (S / chains per chain); the chains (and their
recycle spaces) continue across steps.

* value  : device-resident inputs (CSR + stencil form + b already in HBM),
           K stripes timed with CUDA events, barrier + synchronize on both
           sides, max over ranks.
* e2e    : the same stripes through the public API with the pinned host
           CSR/b uploaded (H2D) and x read back (D2H) inside the timed region.
* roofline: SURVEY 8(d) algorithmic SpMV+ortho bytes of the k_cycle launches
           over the timed region (concurrent chains), vs MEASURED_PEAKS.json
           HBM and vs the nominal 8 TB/s.
* cpu_baseline: the oracle port (numpy/scipy: the reference's arithmetic) on
           this host's cores, on a bounded sample (extrapolated, see below).
``--impl reference`` runs the reference's CPU path (oracle port) on rank 0.
``--gpus N`` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks.
"""

from __future__ import annotations

import os

_CORES = len(os.sched_getaffinity(0))
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(_CORES))
os.environ.setdefault("OMP_NUM_THREADS", str(_CORES))

import argparse  # noqa: E402
import json  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "linear systems solved/sec to rel-res 1e-8 (fp64)"
NOMINAL_HBM_GBS = 8000.0  # BASELINE.json: "SpMV+ortho HBM GB/s vs 8 TB/s"

# per-config defaults: (chains per GPU, systems per step, CTAs per chain or
# None = chain_grid_ctas). Measured on B200: C3 8 x 37
# CTAs (every chain's kernel co-resident: 296 = 2 per SM) 6.26 systems/s,
# 8 x 64 5.95, 4 x 74 6.15, 12 x 48 6.12, 16 x 32 5.71; C4 4 x 74 1.14 (8 x 37
# 1.03, 2 x 148 1.13); C1 8 x 64.
DEFAULTS = {0: (8, 16, None), 1: (8, 16, None), 2: (8, 8, None), 3: (8, 8, 37), 4: (4, 8, 74)}


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="skr", choices=["skr", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--stripe", type=int, default=None, help="systems per step")
    ap.add_argument("--chains", type=int, default=None,
                    help="independent recycling chains per GPU (contiguous sub-chunks)")
    ap.add_argument("--ctas-per-chain", type=int, default=None,
                    help="CTAs of each chain's Arnoldi kernel (default: chain_grid_ctas)")
    ap.add_argument("--n-systems", type=int, default=None, help="override batch size")
    ap.add_argument("--grid", type=int, default=None, help="override grid side (testing)")
    ap.add_argument("--gen", default="host", choices=["host", "device"],
                    help="parameter generator: host numpy (the inputs the reference goldens "
                         "pin) or the device Philox generator (csrc/grf.cu)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sync-steps", action="store_true",
                    help="time each stripe separately (L2 flush + barrier between stripes)")
    ap.add_argument("--cpu-budget-s", type=float, default=25.0,
                    help="CPU seconds of the GPU arm's cpu_baseline sample")
    ap.add_argument("--ref-step-s", type=float, default=25.0,
                    help="CPU seconds per step of the --impl reference arm")
    a = ap.parse_args()
    ch, st, ct = DEFAULTS.get(a.config, (8, 16, None))
    if a.chains is None:  # the CTA default belongs to the default chain count
        a.chains = ch
        a.ctas_per_chain = ct if a.ctas_per_chain is None else a.ctas_per_chain
    a.stripe = st if a.stripe is None else a.stripe
    return a


def _relaunch_under_torchrun(args) -> int | None:
    """``--gpus N`` (N > 1) from a plain ``python bench.py``: run N ranks."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def _dist():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return world, rank, local


def _spec(args):
    from paper_2401_09516_b200 import problems as P

    spec = P.CONFIGS[args.config]
    kw = {}
    if args.n_systems:
        kw["n_systems"] = args.n_systems
    if args.grid:
        kw["n"] = args.grid
    return spec.reduced(**kw) if kw else spec


def _params(spec):
    """All systems' sort parameters (n_sys x P fp64), generated in parallel."""
    from concurrent.futures import ThreadPoolExecutor

    from paper_2401_09516_b200 import problems as P

    first = P.system_params(spec, 0)["params"]
    flat = np.empty((spec.n_systems, first.size), dtype=np.float64)
    flat[0] = first

    def fill(i):
        flat[i] = P.system_params(spec, i)["params"]

    with ThreadPoolExecutor(max_workers=max(1, min(16, _CORES))) as ex:
        list(ex.map(fill, range(1, spec.n_systems)))
    return flat


def _fields(spec, i, flat):
    """Generator fields of system i (the sort row is the coefficient field
    itself for the Darcy / Poisson kinds: no second GRF draw)."""
    from paper_2401_09516_b200 import problems as P

    if spec.kind in ("darcy_binary", "poisson_lognormal"):
        return {"a": flat[i].reshape((spec.n,) * spec.dim), "params": flat[i]}
    return P.system_params(spec, i)


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic(cid):
    """DRAM bytes / algorithmic bytes of k_cycle from the committed ncu
    --set full capture of this configuration's bench shape (profiles/)."""
    path = os.path.join(ROOT, "profiles", "ncu_k_cycle_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        d = d.get(f"C{cid}", d)
        return d.get("dram_over_algorithmic"), d.get("source")
    except Exception:
        return None, None


class _Clocks:
    def __init__(self):
        self.p = None
        self.path = None

    def start(self):
        try:
            os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
            self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self, dev_index=0):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9 or parts[0] != str(dev_index):
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = float(parts[2])
                except ValueError:
                    continue
                for nm, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def _flush_l2(buf):
    buf.add_(1.0)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _reference_iters_per_system(cid):
    """The reference's own iterations per recycled system of this config, from
    the committed kryrec run (tests/golden/full_c<cid>.npz, positions >= 1)."""
    path = os.path.join(ROOT, "tests", "golden", f"full_c{cid}.npz")
    try:
        g = np.load(path)
        it = np.asarray(g["iters"], dtype=float)
        rec = it[1:] if it.size > 1 else it
        return float(rec.mean()), f"kryrec chain, tests/golden/full_c{cid}.npz ({rec.size} systems)"
    except Exception:
        return None, None


def _oracle_sample(spec, systems, step_s, U_in=None):
    """The oracle (reference arithmetic) GCRO-DR chain over ``systems`` (a list
    of (row_ptr, col_idx, values, b)), each solve bounded to ``step_s`` CPU
    seconds: a solve still running then stops at its next cycle boundary (a
    real partial solve through the reference's code path; its recycle space is
    carried on, as the reference carries an unconverged solve's). Returns the
    (iterations, wall seconds, converged) per system and the last recycle U."""
    from oracle import skr_oracle as orc

    out = []
    U = U_in
    cfg = orc.Cfg(m=spec.m, tol=spec.tol, max_iter=spec.max_iter, k=spec.k)
    for rp, ci, v, b in systems:
        op = orc.Operator(rp, ci, v, spec.N, spec.precond == "jacobi")
        r = orc.gcrodr(op, b, cfg, U_in=U, deadline=time.perf_counter() + step_s)
        U = r.U if r.U is not None else U
        out.append((int(r.iterations), float(r.wall_time), bool(r.converged)))
    return out, U


def _cpu_rate(samples, iters_per_system):
    """systems/s of the CPU path: whole systems when every sampled solve
    converged, else its iterations/s divided by the iterations per system."""
    if samples and all(s[2] for s in samples):
        return len(samples) / sum(s[1] for s in samples), "measured (whole systems)"
    its = sum(s[0] for s in samples)
    wall = sum(s[1] for s in samples)
    return (its / wall) / iters_per_system, "extrapolated from iterations/s"


def run_reference(args):
    """The reference's CPU path (oracle port of kryrec: the reference is pure
    Python and cannot travel to the GPU box) on rank 0's host cores."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import skr_oracle as orc
    from paper_2401_09516_b200 import problems as P

    spec = _spec(args)
    t0 = time.perf_counter()
    flat = _params(spec)
    npos = args.warmup + args.steps
    order = orc.greedy_order_prefix(flat, npos + 1)
    prefix_sort_s = time.perf_counter() - t0
    ref_its, ref_src = _reference_iters_per_system(spec.cid)
    U = None
    samples = []
    for pos in range(npos):
        rp, ci, v, b, _ = P.assemble(spec, order[pos], _fields(spec, order[pos], flat))
        # one step = the next system of the sorted chain, bounded in time; the
        # chain continues from that solve's recycle space
        s, U = _oracle_sample(spec, [(rp, ci, v, b)], args.ref_step_s, U_in=U)
        if pos >= args.warmup:
            samples.extend(s)
    its_sys = ref_its if ref_its else float(np.mean([s[0] for s in samples]))
    value, how = _cpu_rate(samples, its_sys)
    wall = sum(s[1] for s in samples)
    out = {
        "metric": METRIC, "value": value, "unit": "systems/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * wall / max(1, len(samples)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config generator)", "impl": "reference",
        "config": _config_dict(spec, 1, world, 1),
        "cpu_baseline": {"value": value, "unit": "systems/s", "cores": _CORES, "kind": "port",
                         "sample": (f"oracle GCRO-DR chain over sorted positions "
                                    f"{args.warmup}..{npos - 1} (after {args.warmup} warm-up "
                                    f"positions), each step one system capped at ~"
                                    f"{args.ref_step_s:.0f} s of iterations; {how}: "
                                    f"iterations/s / {its_sys:.1f} iterations per system "
                                    f"({ref_src or 'the sample'}); prefix sort "
                                    f"{prefix_sort_s:.1f}s excluded")},
        "e2e": {"value": value, "unit": "systems/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "iterations_sampled": [s[0] for s in samples],
        "cpu_model": _cpu_model(),
    }
    print(json.dumps(out), flush=True)


def _config_dict(spec, stripe, world, chains):
    return {"workload": f"C{spec.cid} {spec.name}: {spec.kind}, grid {spec.n}^{spec.dim} "
                        f"(N={spec.N}), batch {spec.n_systems}, greedy-NN sorted, "
                        f"GCRO-DR(m={spec.m}, k={spec.k}), {spec.precond}, tol {spec.tol:g}",
            "n_systems_batch": spec.n_systems, "N": spec.N, "m": spec.m, "k": spec.k,
            "precond": spec.precond, "tol": spec.tol, "max_iter": spec.max_iter,
            "stripe_systems_per_step": stripe, "chains_per_gpu": chains,
            "parallelism": f"chunked chains: {world} rank(s) x {chains} chain(s) "
                           f"(contiguous sorted chunks)"}


class _HostCsr:
    """Pinned host CSR in the upload format (int32 indices, fp64 values)."""

    def __init__(self, n, rp, ci, v):
        self.n_rows = self.n_cols = n
        self.row_ptr = rp
        self.col_idx = ci
        self.values = v


def run_skr(args):
    import torch
    import torch.distributed as dist

    import paper_2401_09516_b200 as skr
    from paper_2401_09516_b200 import problems as P

    world, rank, local = _dist()
    dev = torch.device("cuda", local)
    spec = _spec(args)
    S, K, W = args.stripe, args.steps, args.warmup
    NC = max(1, args.chains)
    if S % NC:
        raise SystemExit(f"--stripe {S} must be a multiple of --chains {NC}")
    sub = S // NC  # systems per chain per step
    gctas = skr.chain_grid_ctas(NC) if args.ctas_per_chain is None else args.ctas_per_chain
    cfg = skr.SolverConfig(m=spec.m, tol=spec.tol, max_iter=spec.max_iter, k=spec.k)
    jac = spec.precond == "jacobi"
    # ---- parameters + sort (sharded rows + all_gather when world > 1) -------
    t_gen = time.perf_counter()
    if args.gen == "device":  # sampled in place on the GPU (no host copy)
        flat_d, gen_extra = P.params_device(spec)
        torch.cuda.synchronize()
        flat = None
    else:
        flat = _params(spec)
    gen_s = time.perf_counter() - t_gen
    if flat is not None:
        flat_d = torch.from_numpy(flat).to(dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    order = skr.sharded_greedy_sort(flat_d) if world > 1 else skr.greedy_sort_device(flat_d)
    e1.record()
    torch.cuda.synchronize()
    sort_ms = e0.elapsed_time(e1)
    if flat is not None:
        del flat_d
    # ---- this rank's chunk of the chain ------------------------------------
    chunk = list(skr.chunk_positions(spec.n_systems, world, rank))
    need = (W + K) * S
    if not chunk:
        raise SystemExit(f"rank {rank}: empty chunk")
    # a rank's chunk (n_systems / world) can be shorter than the (W + K) * S
    # systems a long run needs: the chains then continue through the chunk
    # again (every solve is real work)
    wrapped = len(chunk) < need
    pos = [chunk[i % len(chunk)] for i in range(need)]
    idxs = [order[p] for p in pos]
    distinct = len(set(idxs))
    # device-resident systems: coefficient field uploaded, CSR values and the
    # stencil form assembled on the GPU (bit-identical to the host assembly)
    dev_sys = []
    for i in idxs:
        f = (_fields(spec, i, flat) if flat is not None else
             P.fields_from_params_device(spec, flat_d[i], gen_extra[i]))
        dA, b, _ = P.assemble_device(spec, i, f, jacobi=jac)
        dev_sys.append((dA, b))
    torch.cuda.synchronize()
    n_params = int((flat if flat is not None else flat_d).shape[1])
    # the CPU baseline's sample needs a few systems' fields; the rest of the
    # parameters (C3: 8.6 GB per rank) are released
    cpu_rows = {i: (flat[i].copy() if flat is not None else flat_d[i].cpu().numpy())
                for i in idxs[W * sub: W * sub + 4]}
    del flat
    if args.gen == "device":
        del flat_d  # the assembled systems keep their own coefficient fields
    # pinned host copies of the same systems for the end-to-end pass (the
    # sparsity pattern is one pinned array pair; its bytes are still uploaded
    # for every system)
    host = []
    if not args.no_e2e:
        rp_h = dev_sys[0][0].row_ptr.cpu().pin_memory()
        ci_h = dev_sys[0][0].col_idx.cpu().pin_memory()
        for dA, b in dev_sys:
            host.append((_HostCsr(spec.N, rp_h, ci_h, dA.values.cpu().pin_memory()),
                         b.cpu().pin_memory()))
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    ident = list(range(need))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    span = (W + K) * sub   # positions per chain (contiguous sub-chunk of this rank's chunk)
    # pinned host buffer for the e2e read-back of x: one row per position
    x_pinned = (torch.empty((need, spec.N), dtype=torch.float64, pin_memory=True)
                if not args.no_e2e else None)

    def solve(systems, chunks, states, keep_x):
        if keep_x != "host":
            return skr.solve_chains(systems, ident, cfg, spec.precond, chunks, keep_x=keep_x,
                                    states=states, grid_ctas=gctas)
        # end to end: upload this call's systems from pinned host memory, solve
        # the chains on the device, read every x back into its own pinned row
        up, h2d = {}, {}
        for ch in chunks:
            for q in ch:
                A, b = systems[q]
                dA = skr.DeviceCsr.from_host(A, jacobi=jac, non_blocking=True, check_pivot=False)
                up[q] = (dA, b.to(dev, non_blocking=True))
                h2d[q] = (A.row_ptr.numel() * 4 + A.col_idx.numel() * 4 + A.values.numel() * 8
                          + b.numel() * 8)
        flags = [u[0]._pivot_flag for u in up.values() if getattr(u[0], "_pivot_flag", None)
                 is not None]
        if flags and bool(torch.stack(flags).any()):  # one sync for the whole call
            for u in up.values():
                u[0].raise_if_zero_pivot()
        rl = skr.solve_chains(lambda i: up[i], ident, cfg, spec.precond, chunks, keep_x="device",
                              states=states, grid_ctas=gctas)
        for r, ch in zip(rl, chunks):
            for xd, q in zip(r.x, ch):
                x_pinned[q].copy_(xd, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            r.x = [x_pinned[q].numpy() for q in ch]
            r.h2d_bytes = int(sum(h2d[q] for q in ch))
            r.d2h_bytes = int(len(ch) * spec.N * 8)
        return rl

    def stripes(a, b):  # positions of stripes [a, b) for every chain
        return [list(range(c * span + a * sub, c * span + b * sub)) for c in range(NC)]

    def run_pass(systems, keep_x):
        """W untimed warm-up stripes, then K timed stripes. Default: the K stripes
        run back to back in one timed region (chains do not wait for each other
        at stripe boundaries); --sync-steps times each stripe separately with an
        L2 flush and a barrier in between."""
        states = [None] * NC
        per_step, stats = [], []
        u_at_timed = None
        if args.sync_steps:
            for st in range(W + K):
                _flush_l2(flush)
                barrier()
                ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ev0.record()
                rl = solve(systems, stripes(st, st + 1), states, keep_x)
                ev1.record()
                barrier()
                states = [r.chain for r in rl]
                if st == W - 1 and states[0] is not None and states[0].k > 0:
                    u_at_timed = states[0].engine.recycle_views()[0].cpu().numpy()
                if st >= W:
                    per_step.append(ev0.elapsed_time(ev1))
                    stats.extend(rl)
            return per_step, stats, u_at_timed
        rl = solve(systems, stripes(0, W), states, keep_x) if W > 0 else []
        states = [r.chain for r in rl] if rl else [None] * NC
        if states[0] is not None and states[0].k > 0:
            u_at_timed = states[0].engine.recycle_views()[0].cpu().numpy()
        del rl
        # warm the caching allocator for the timed call's output block
        torch.empty((K * S, spec.N), dtype=torch.float64, device=dev)
        _flush_l2(flush)
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        rl = solve(systems, stripes(W, W + K), states, keep_x)
        ev1.record()
        barrier()
        t = ev0.elapsed_time(ev1)
        return [t / K] * K, list(rl), u_at_timed

    clocks = _Clocks()
    clocks.start()
    per_step, stats, u_timed = run_pass(dev_sys, "device")
    clk = clocks.stop(local)
    total_ms = float(sum(per_step))

    def all_max(v):
        t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    total_ms_max = all_max(total_ms)
    n_sys_timed = S * K * world
    value = n_sys_timed / (total_ms_max / 1000.0)
    its = [i for r in stats for i in r.iterations]
    conv_local = all(c for r in stats for c in r.converged)
    unconv = [(int(i), int(it), float(tr)) for r in stats
              for i, it, c, tr in zip(r.order, r.iterations, r.converged, r.true_rel) if not c]
    bytes_ = sum(r.spmv_ortho_bytes for r in stats)
    cyc_ms = sum(r.cycle_kernel_ms for r in stats)
    den_ms = sum(r.dense_kernel_ms for r in stats)
    launches = sum(r.launches for r in stats)
    steps_arn = sum(r.arnoldi_steps for r in stats)
    v0proj = sum(sum(r.v0_projections) for r in stats)
    peak, peak_src = _peaks()
    per_launch = bytes_ / (cyc_ms / 1000.0) / 1e9 if cyc_ms > 0 else 0.0
    aggregate = bytes_ / (total_ms / 1000.0) / 1e9 if total_ms > 0 else 0.0
    # with several chains the k_cycle launches overlap on the device (each owns
    # a share of the SMs), so a launch's event time is not its cost: the
    # achieved figure is the k_cycle bytes over the whole timed region (which
    # also holds the dense / combine / refresh kernels: a lower bound)
    achieved = aggregate if NC > 1 else per_launch
    ratio, tr_src = _traffic(spec.cid)
    n_cycle_launches = sum(sum(r.cycles) for r in stats)
    # ---- e2e through the public API with host buffers ----------------------
    e2e = None
    conv_e2e = True
    if not args.no_e2e:
        # release the device-resident copies: the e2e uploads then reuse the
        # caching allocator's blocks instead of growing it inside the timed region
        dev_sys.clear()
        per_step_e, stats_e, _ = run_pass(host, "host")
        tot_e = all_max(sum(per_step_e))
        conv_e2e = all(c for r in stats_e for c in r.converged)
        unconv += [(int(i), int(it), float(tr)) for r in stats_e
                   for i, it, c, tr in zip(r.order, r.iterations, r.converged, r.true_rel) if not c]
        e2e = {"value": n_sys_timed / (tot_e / 1000.0), "unit": "systems/s",
               "h2d_bytes_per_step": int(sum(r.h2d_bytes for r in stats_e) / K),
               "d2h_bytes_per_step": int(sum(r.d2h_bytes for r in stats_e) / K),
               "path": ("pinned host CSR+b -> DeviceCsr.from_host (upload + device stencil "
                        "build) -> solve_chains -> x to pinned host, inside the timed region")}
    # every rank's solves (timed device pass and e2e pass) must have converged
    conv_t = torch.tensor([1.0 if (conv_local and conv_e2e) else 0.0], device=dev)
    if world > 1:
        dist.all_reduce(conv_t, op=dist.ReduceOp.MIN)
    all_conv = bool(conv_t.item() > 0.5)
    its_all = its
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, its)
        its_all = [i for g in gathered for i in g]
    # ---- CPU baseline: oracle port on this host (rank 0, N = 1) ------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = _cpu_baseline(spec, idxs[W * sub:], cpu_rows, u_timed, args.cpu_budget_s,
                            float(np.mean(its)))
    if rank != 0:
        return
    # ncu DRAM bytes per k_cycle launch, as (DRAM / algorithmic bytes of the
    # captured launches, same config and chain shape) x this run's algorithmic
    # bytes per launch
    traffic = ratio * bytes_ / max(1, n_cycle_launches) if ratio is not None else None
    out = {
        "metric": METRIC, "value": value, "unit": "systems/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": total_ms_max / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config generator; DCT-sampled GRF, see DESIGN.md)",
        "config": dict(_config_dict(spec, S, world, NC), generator=args.gen, chunk_wrapped=wrapped,
                       distinct_systems=distinct, ctas_per_chain=gctas,
                       l2=("flushed between steps (256 MiB write)" if args.sync_steps else
                           "flushed (256 MiB write) before the timed region; inside it every "
                           "chain's working set exceeds the 126 MB L2 (C3: ~1.6 GB per chain)"),
                       timing=("each step timed separately" if args.sync_steps else
                               "K stripes back to back in one timed region (CUDA events, "
                               "barrier + synchronize on both sides); ms_per_step = total / K")),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "frac_vs_nominal_8tbs": achieved / NOMINAL_HBM_GBS,
                     "traffic": traffic, "traffic_source": tr_src,
                     "method": ("sum of k_cycle algorithmic bytes / timed-region device time "
                                "(concurrent chains; the region also holds the dense, combine "
                                "and refresh kernels)" if NC > 1 else
                                "sum of k_cycle algorithmic bytes / sum of k_cycle event time"),
                     "per_launch_gbs": per_launch, "aggregate_gbs": aggregate,
                     "k_cycle_launches": int(n_cycle_launches),
                     "algorithmic_bytes_per_launch": bytes_ / max(1, n_cycle_launches),
                     "kernel": "k_cycle (persistent DCGS2 Arnoldi cycle: SpMV + ortho)",
                     "peak_source": peak_src,
                     "algorithmic_bytes": ("per Arnoldi step B_spmv + 8N(2p+6), SURVEY 8(d), "
                                           "p = basis width; B_spmv = 32N + 16N through the "
                                           "3-D stencil form (24N + 16N in 2-D), "
                                           "12 nnz + 4(N+1) + 16N through the CSR")},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
        "iterations_mean": float(np.mean(its_all)), "all_converged": all_conv,
        "unconverged_rank0": unconv[:16],
        "v0_projected_cycles": int(v0proj),
        "arnoldi_steps": int(steps_arn),
        "us_per_arnoldi_step": 1000.0 * cyc_ms / max(1, steps_arn),
        "time_split_ms": {"cycle_kernels": cyc_ms, "dense_recycle_kernels": den_ms,
                          "solve_streams": float(sum(sum(r.device_ms) for r in stats)),
                          "chain_wall_ms": sorted(round(1000 * r.wall_s, 1) for r in stats),
                          "total": total_ms},
        "sort": {"ms": sort_ms, "n_systems": spec.n_systems, "P": n_params,
                 "param_generation_s": round(gen_s, 3)},
    }
    if cpu is not None:
        out["cpu_baseline"] = cpu
    print(json.dumps(out), flush=True)


def _cpu_baseline(spec, idxs, flat, U_in, budget_s, gpu_its):
    from paper_2401_09516_b200 import problems as P

    systems = []
    for i in idxs[:4]:
        rp, ci, v, b, _ = P.assemble(spec, i, _fields(spec, i, flat))
        systems.append((rp, ci, v, b))
    samples = []
    U = U_in
    t0 = time.perf_counter()
    for sy in systems:
        left = budget_s - (time.perf_counter() - t0)
        if left <= 0:
            break
        s, U = _oracle_sample(spec, [sy], left, U_in=U)
        samples.extend(s)
    ref_its, ref_src = _reference_iters_per_system(spec.cid)
    its_sys = ref_its or gpu_its
    v, how = _cpu_rate(samples, its_sys)
    return {"value": v, "unit": "systems/s", "cores": _CORES, "kind": "port",
            "sample": (f"oracle GCRO-DR on {len(samples)} system(s) from the first timed "
                       f"position, recycle U taken from the GPU chain (steady state), "
                       f"~{budget_s:.0f} s of CPU; {how} with {its_sys:.1f} iterations per "
                       f"system ({ref_src or 'GPU mean'}); OPENBLAS_NUM_THREADS="
                       f"{os.environ.get('OPENBLAS_NUM_THREADS')}"),
            "iterations_sampled": [s[0] for s in samples],
            "cpu_model": _cpu_model()}


def main():
    args = _args()
    rc = _relaunch_under_torchrun(args)
    if rc is not None:
        sys.exit(rc)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_skr(args)
    try:
        import torch.distributed as dist

        if dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    main()
