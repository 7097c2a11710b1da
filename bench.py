#!/usr/bin/env python
"""SKR hot-path benchmark: systems solved/s (rel-res 1e-8, fp64) on B200.

Workload (BASELINE.json configs[1]): variable-coefficient Poisson on 256^2
(N = 65,536), a batch of 1,024 systems, greedy-NN sorted on the coefficient
field, solved as GCRO-DR(40, 10) chains with Jacobi. The sorted order is
split into contiguous per-GPU chunks (one recycling chain per rank, weak
scaling). A bench *step* = one stripe of S consecutive systems of the
rank's chain; the chain (and its recycle space) continues across steps.

* value  : device-resident inputs (CSR + b already in HBM), timed with CUDA
           events, L2 flushed between steps, max over ranks.
* e2e    : the same stripes through the public API with pinned host CSR/b
           uploaded (H2D) and x read back (D2H) inside every step.
* roofline: SURVEY 8(d) algorithmic SpMV+ortho bytes / summed CUDA-event time
           of the Arnoldi-cycle kernel launches, vs MEASURED_PEAKS.json HBM.
* cpu_baseline: the oracle port (numpy/scipy = the reference's arithmetic) on
           this host's cores, on a bounded sample of the same chain.
``--impl reference`` runs the reference's CPU path (oracle port) on rank 0.
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


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="skr", choices=["skr", "reference"])
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--stripe", type=int, default=16, help="systems per step")
    ap.add_argument("--chains", type=int, default=8,
                    help="independent recycling chains per GPU (contiguous sub-chunks)")
    ap.add_argument("--ctas-per-chain", type=int, default=None,
                    help="CTAs of each chain's Arnoldi kernel (default: chain_grid_ctas)")
    ap.add_argument("--n-systems", type=int, default=None, help="override batch size")
    ap.add_argument("--grid", type=int, default=None, help="override grid side (testing)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sync-steps", action="store_true",
                    help="time each stripe separately (L2 flush + barrier between stripes)")
    ap.add_argument("--cpu-budget-s", type=float, default=25.0)
    return ap.parse_args()


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
    from paper_2401_09516_b200 import problems as P

    return np.stack([P.system_params(spec, i)["params"] for i in range(spec.n_systems)])


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic():
    """dram bytes per k_cycle launch from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_k_cycle_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch"), d.get("algorithmic_bytes_per_launch")
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


def run_reference(args):
    """The reference's CPU path (oracle port of kryrec) on rank 0's host cores."""
    world, rank, _ = _dist_cpu()
    if rank != 0:
        return
    from oracle import skr_oracle as orc
    from paper_2401_09516_b200 import problems as P

    spec = _spec(args)
    t0 = time.perf_counter()
    flat = _params(spec)
    npos = args.warmup + args.steps
    order = orc.greedy_order_prefix(flat, npos)
    prefix_sort_s = time.perf_counter() - t0
    cfg = orc.Cfg(m=spec.m, tol=spec.tol, max_iter=spec.max_iter, k=spec.k)
    U = None
    walls, its = [], []
    for pos in range(npos):
        rp, ci, v, b, _ = P.assemble(spec, order[pos])
        op = orc.Operator(rp, ci, v, spec.N, spec.precond == "jacobi")
        r = orc.gcrodr(op, b, cfg, U_in=U)
        U = r.U
        if pos >= args.warmup:
            walls.append(r.wall_time)
            its.append(r.iterations)
    total = sum(walls)
    value = len(walls) / total
    out = {
        "metric": METRIC, "value": value, "unit": "systems/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / len(walls),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config generator)", "impl": "reference",
        "config": _config_dict(spec, 1, world),
        "cpu_baseline": {"value": value, "unit": "systems/s", "cores": _CORES, "kind": "port",
                         "sample": f"oracle chain positions {args.warmup}..{npos - 1} of the "
                                   f"sorted order, one system per step (prefix sort "
                                   f"{prefix_sort_s:.1f}s excluded)"},
        "e2e": {"value": value, "unit": "systems/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "iterations_mean": float(np.mean(its)),
        "cpu_model": _cpu_model(),
    }
    print(json.dumps(out), flush=True)


def _dist_cpu():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    return world, rank, 0


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _config_dict(spec, stripe, world):
    return {"workload": f"C{spec.cid} {spec.name}: {spec.kind}, grid {spec.n}^{spec.dim} "
                        f"(N={spec.N}), batch {spec.n_systems}, greedy-NN sorted, "
                        f"GCRO-DR(m={spec.m}, k={spec.k}), {spec.precond}, tol {spec.tol:g}",
            "n_systems_batch": spec.n_systems, "N": spec.N, "m": spec.m, "k": spec.k,
            "precond": spec.precond, "tol": spec.tol, "max_iter": spec.max_iter,
            "stripe_systems_per_step": stripe,
            "parallelism": f"chunked chains x{world} (contiguous sorted chunks)",
            "l2": "flushed between steps (256 MiB write)"}


class _HostCsr:
    """Pinned host CSR in the upload format (int32 indices, fp64 values)."""

    def __init__(self, n, rp, ci, v):
        import torch

        self.n_rows = self.n_cols = n
        self.row_ptr = torch.from_numpy(rp.astype(np.int32)).pin_memory()
        self.col_idx = torch.from_numpy(ci.astype(np.int32)).pin_memory()
        self.values = torch.from_numpy(v).pin_memory()


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
    gctas = skr.chain_grid_ctas(NC) if args.ctas_per_chain is None else args.ctas_per_chain
    cfg = skr.SolverConfig(m=spec.m, tol=spec.tol, max_iter=spec.max_iter, k=spec.k)
    # ---- sort (sharded rows + all_gather when world > 1) -------------------
    flat = _params(spec)
    flat_d = torch.from_numpy(flat).to(dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if world > 1:
        order = skr.sharded_greedy_sort(flat_d)
    else:
        order = skr.greedy_sort_device(flat_d)
    e1.record()
    torch.cuda.synchronize()
    sort_ms = e0.elapsed_time(e1)
    del flat_d
    # ---- this rank's chunk of the chain ------------------------------------
    chunk = skr.chunk_positions(spec.n_systems, world, rank)
    need = (W + K) * S
    chunk = list(chunk)
    if not chunk:
        raise SystemExit(f"rank {rank}: empty chunk")
    # a rank's chunk (n_systems / world) can be shorter than the (W + K) * S
    # systems a long run needs (e.g. 8 GPUs, many steps): the chains then
    # continue through the chunk again (every solve is real work; the jump
    # back costs one poorly recycled system per chain)
    wrapped = len(chunk) < need
    pos = [chunk[i % len(chunk)] for i in range(need)]
    idxs = [order[p] for p in pos]
    host = []
    for i in idxs:
        rp, ci, v, b, _ = P.assemble(spec, i)
        host.append((_HostCsr(spec.N, rp, ci, v), torch.from_numpy(b).pin_memory()))
    dev_sys = []
    for A, b in host:
        dA = skr.DeviceCsr.from_host(A, jacobi=spec.precond == "jacobi")
        dev_sys.append((dA, b.to(dev)))
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)
    ident = list(range(need))

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # pinned host buffer for the e2e read-back of x (allocated outside any timed region)
    x_pinned = (torch.empty((W + K) * S * spec.N, dtype=torch.float64, pin_memory=True)
                if not args.no_e2e else None)
    sub = S // NC          # systems per chain per step
    span = (W + K) * sub   # positions per chain (contiguous sub-chunk of this rank's chunk)

    def solve(systems, chunks, states, keep_x):
        if NC == 1:
            return [skr.solve_sequence(systems, ident, cfg, spec.precond, positions=chunks[0],
                                       keep_x=keep_x, chain=states[0])]
        if keep_x != "host":
            return skr.solve_chains(systems, ident, cfg, spec.precond, chunks, keep_x=keep_x,
                                    states=states, grid_ctas=gctas)
        # end to end: upload this call's systems from pinned host memory, solve
        # the chains on the device, read every x back
        dbg = bool(os.environ.get("SKR_E2E_DEBUG"))
        t_a = time.perf_counter()
        up, h2d = {}, {}
        for ch in chunks:
            for q in ch:
                A, b = systems[q]
                dA = skr.DeviceCsr.from_host(A, jacobi=spec.precond == "jacobi", non_blocking=True,
                                             check_pivot=bool(os.environ.get("SKR_E2E_SYNC")))
                up[q] = (dA, b.to(dev, non_blocking=True))
                h2d[q] = (A.row_ptr.numel() * 4 + A.col_idx.numel() * 4 + A.values.numel() * 8
                          + b.numel() * 8)
        flags = [u[0]._pivot_flag for u in up.values() if getattr(u[0], "_pivot_flag", None)
                 is not None]
        if flags and bool(torch.stack(flags).any()):  # one sync for the whole call
            for u in up.values():
                u[0].raise_if_zero_pivot()
        if dbg:
            t_b = time.perf_counter()
            torch.cuda.synchronize()
            t_c = time.perf_counter()
        rl = skr.solve_chains(lambda i: up[i], ident, cfg, spec.precond, chunks, keep_x="device",
                              states=states, grid_ctas=gctas)
        if dbg:
            torch.cuda.synchronize()
            t_d = time.perf_counter()
        for r, ch in zip(rl, chunks):
            xs = None
            if r.x:  # into the preallocated pinned host buffer (pageable: ~2 GB/s)
                xd = torch.stack(r.x)
                xs = x_pinned[: xd.numel()].view(xd.shape)
                xs.copy_(xd, non_blocking=True)
                torch.cuda.current_stream().synchronize()
            r.x = list(xs.numpy()) if xs is not None else []
            r.h2d_bytes = int(sum(h2d[q] for q in ch))
            r.d2h_bytes = int(xs.numel() * 8) if xs is not None else 0
        if dbg:
            t_e = time.perf_counter()
            print(f"e2e phases ms: enqueue uploads {1e3 * (t_b - t_a):.1f}, drain {1e3 * (t_c - t_b):.1f}, "
                  f"solve {1e3 * (t_d - t_c):.1f}, x to host {1e3 * (t_e - t_d):.1f}", file=sys.stderr)
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
        rl = solve(systems, stripes(0, W), states, keep_x)
        states = [r.chain for r in rl]
        if states[0] is not None and states[0].k > 0:
            u_at_timed = states[0].engine.recycle_views()[0].cpu().numpy()
        # warm the caching allocator for the timed call's output block
        del rl
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
    tmax = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    total_ms_max = float(tmax.item())
    n_sys_timed = S * K * world
    value = n_sys_timed / (total_ms_max / 1000.0)
    its = [i for r in stats for i in r.iterations]
    conv = all(c for r in stats for c in r.converged)
    bytes_ = sum(r.spmv_ortho_bytes for r in stats)
    cyc_ms = sum(r.cycle_kernel_ms for r in stats)
    den_ms = sum(r.dense_kernel_ms for r in stats)
    launches = sum(r.launches for r in stats)
    steps_arn = sum(r.arnoldi_steps for r in stats)
    peak, peak_src = _peaks()
    per_launch = bytes_ / (cyc_ms / 1000.0) / 1e9 if cyc_ms > 0 else 0.0
    aggregate = bytes_ / (total_ms / 1000.0) / 1e9 if total_ms > 0 else 0.0
    # with several chains the k_cycle launches overlap on the device (each owns
    # a share of the SMs), so a launch's event time is not its cost: report the
    # k_cycle bytes over the whole timed region (which also contains the dense
    # kernels: a lower bound on the kernel's bandwidth)
    achieved = aggregate if NC > 1 else per_launch
    traffic, alg_per_launch = _traffic()
    # ---- e2e through the public API with host buffers ----------------------
    e2e = None
    if not args.no_e2e:
        # release the device-resident copies: the e2e uploads then reuse the
        # caching allocator's blocks instead of growing it (cudaMalloc) inside
        # the timed region
        dev_sys.clear()
        per_step_e, stats_e, _ = run_pass(host, "host")
        tot_e = torch.tensor([float(sum(per_step_e))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tot_e, op=dist.ReduceOp.MAX)
        e2e = {"value": n_sys_timed / (float(tot_e.item()) / 1000.0), "unit": "systems/s",
               "h2d_bytes_per_step": int(sum(r.h2d_bytes for r in stats_e) / K),
               "d2h_bytes_per_step": int(sum(r.d2h_bytes for r in stats_e) / K),
               "path": ("pinned host CSR+b -> DeviceCsr.from_host -> solve_chains -> x to host, "
                        "inside the timed region")}
    # ---- CPU baseline: oracle port on this host (rank 0, N = 1) ------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = _cpu_baseline(spec, host, W * sub, u_timed, args.cpu_budget_s)
    if rank != 0:
        return
    out = {
        "metric": METRIC, "value": value, "unit": "systems/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": total_ms_max / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded config generator; DCT-sampled GRF, see DESIGN.md)",
        "config": dict(_config_dict(spec, S, world), chains_per_gpu=NC, chunk_wrapped=wrapped,
                       ctas_per_chain=gctas,
                       l2=("flushed between steps (256 MiB write)" if args.sync_steps else
                           "flushed (256 MiB write) before the timed region; inside it each "
                           "stripe's working set (per chain ~39 MB basis + CSR, x8 chains) "
                           "exceeds the 126 MB L2"),
                       timing=("each step timed separately" if args.sync_steps else
                               "K stripes back to back in one timed region (CUDA events, "
                               "barrier + synchronize on both sides); ms_per_step = total / K")),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "method": ("sum of k_cycle algorithmic bytes / timed-region device time "
                                "(concurrent chains)" if NC > 1 else
                                "sum of k_cycle algorithmic bytes / sum of k_cycle event time"),
                     "per_launch_gbs": per_launch, "aggregate_gbs": aggregate,
                     "kernel": "k_cycle (persistent DCGS2 Arnoldi cycle: SpMV + ortho)",
                     "peak_source": peak_src,
                     "algorithmic_bytes": ("per step B_spmv + 8N(2p+6), SURVEY 8(d); B_spmv = 24N + 16N "
                                           "through the stencil form (2-D), 12 nnz + 4(N+1) + 16N "
                                           "through the CSR"),
                     "note": "one chain's C1 working set (~39 MB) fits the L2; the 8 concurrent "
                             "chains' (~312 MB) do not"},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk,
        "iterations_mean": float(np.mean(its)), "all_converged": bool(conv),
        "arnoldi_steps": int(steps_arn),
        "us_per_arnoldi_step": 1000.0 * cyc_ms / max(1, steps_arn),
        "time_split_ms": {"cycle_kernels": cyc_ms, "dense_recycle_kernels": den_ms,
                          "solve_streams": float(sum(sum(r.device_ms) for r in stats)),
                          "chain_wall_ms": sorted(round(1000 * r.wall_s, 1) for r in stats),
                          "total": total_ms},
        "sort": {"ms": sort_ms, "n_systems": spec.n_systems, "P": int(flat.shape[1])},
    }
    if cpu is not None:
        out["cpu_baseline"] = cpu
    print(json.dumps(out), flush=True)


def _cpu_baseline(spec, host, first_pos, U_in, budget_s):
    from oracle import skr_oracle as orc

    cfg = orc.Cfg(m=spec.m, tol=spec.tol, max_iter=spec.max_iter, k=spec.k)
    walls = []
    U = U_in
    t_start = time.perf_counter()
    p = first_pos
    while p < len(host) and (time.perf_counter() - t_start) < budget_s:
        A, b = host[p]
        op = orc.Operator(A.row_ptr.numpy(), A.col_idx.numpy(), A.values.numpy(), spec.N,
                          spec.precond == "jacobi")
        r = orc.gcrodr(op, b.numpy(), cfg, U_in=U)
        U = r.U
        walls.append(r.wall_time)
        p += 1
    v = len(walls) / sum(walls)
    return {"value": v, "unit": "systems/s", "cores": _CORES, "kind": "port",
            "sample": f"oracle chain on {len(walls)} system(s) starting at the first timed "
                      f"position, recycle U taken from the GPU chain (steady state); "
                      f"OPENBLAS_NUM_THREADS={os.environ.get('OPENBLAS_NUM_THREADS')}",
            "cpu_model": _cpu_model()}


def main():
    args = _args()
    if os.environ.get("SKR_SWITCH_INTERVAL"):
        sys.setswitchinterval(float(os.environ["SKR_SWITCH_INTERVAL"]))
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
