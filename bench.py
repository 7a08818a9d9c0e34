#!/usr/bin/env python3
"""Throughput benchmark: trajectories propagated/sec (N-body PC) at 1/2/4/8 B200 vs CPU host cores.

Default workload (BASELINE.json configs[3], "C4"): a 1,000,000-trajectory cloud of perturbed
clones of the reference spacecraft state (a = 1.25e8 km, e = 0.12; make_clone_batch spread
1e-5, seed 20220411), Sun + 8 planets Newtonian N-body, N = 200 Chebyshev-Lobatto nodes, one
0.87-period segment, warm start, tol 1e-12 relative, per-trajectory convergence masking
(RunMode::independent).  The 1M cloud is a FIXED total sharded over the GPUs (strong scaling):
contiguous trajectory shards, no collective in the iteration loop, one gather of the terminal
states to rank 0 at the end.  `--config c1|c2|c3|c5` selects the other BASELINE configs.

One step = one propagation of the whole batch through the C-ABI (pswarm_run_batch):
  value     trajectories/s over the device solve phase (inputs resident in HBM), whole job,
            max over ranks
  e2e       trajectories/s of the full C-ABI call with host buffers (pinned [M][7] ICs H2D,
            solve, terminal states D2H; + the gather to rank 0 when N > 1)
  roofline  algorithmic FP64 flops of the PC kernel (F_it = 12N^2 + (75+20B)N
            + 12 per trajectory-iteration) / kernel time (CUDA events on the launch stream) vs the
            measured FP64 (DMMA) peak (profiles/fp64_peak_r01.json); `traffic` and the EXECUTED
            FP64 fraction come from the committed ncu capture of the same config (profiles/
            ncu_r02_<config>.json), null when none was captured
  parity    a strided subsample of the batch re-propagated on its own (a 1-rank run) must
            reproduce the gathered terminal states; the CPU reference on its sample within
            1e-10 relative and +-1 iterations
`--gpus N` without torchrun re-launches itself under torch.distributed.run (one rank per GPU).
`--impl reference` times the reference's own CPU implementation (oracle/_ref: the reference
sources built unchanged on an Eigen-subset shim; the restatement oracle/pswarm_ref.hpp when
_ref is absent or the config is an extension) on all host cores.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "trajectories propagated/sec (N-body PC) at 1/2/4/8 B200 vs CPU host cores"
UNIT = "trajectories/s"

CONFIGS = {
    # name: (trajectories, per-GPU (weak) or total (strong), bodies, force kind, span periods, policy, start, spreads)
    "c1": (64, "weak", "none", "two_body", 1.0, "single", "warm", (1e-5,)),
    "c2": (1000, "weak", "planets8", "n_body", 0.87, "single", "warm", (1e-5,)),
    "c3": (100000, "strong", "planets8", "n_body", 3.5, "per_orbit", "hot", (1e-5,)),
    "c4": (1000000, "strong", "planets8", "n_body", 0.87, "single", "warm", (1e-5,)),
    "c5": (100000, "strong", "planets8", "n_body_1pn", 0.87, "single", "warm", (1e-7, 1e-5, 1e-3, 1e-2)),
}
DESCR = {
    "c1": "C1: heliocentric two-body Keplerian propagation, {m} ICs per GPU (a=1.3e8 km e=0.2), one period",
    "c2": ("C2: {m}-IC Earth-Venus arc per GPU (reference spacecraft a=1.25e8 km e=0.12, clone spread 1e-5), "
           "Sun + 8 planets Newtonian N-body, {span} period single segment"),
    "c3": ("C3: planetary-protection Monte-Carlo cloud, {m} ICs total, Sun + 8 planets, per-orbit segments over "
           "{span} periods (1/1/1/0.5), hot starts (EXTENSION) on the equal-span segments"),
    "c4": ("C4: {m}-trajectory cloud total (reference spacecraft clones, spread 1e-5) sharded over the GPUs, "
           "Sun + 8 planets Newtonian N-body, {span} period single segment"),
    "c5": ("C5: {force} Sun + 8 planets, {m} ICs total in four quarters with clone "
           "spreads 1e-7/1e-5/1e-3/1e-2 (convergence-mask stress), {span} period single segment"),
}
MODES = ("independent", "grouped", "augmented_parallel", "augmented_sequential")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS), help="BASELINE.json configs[0..4]")
    ap.add_argument("--mode", default="independent", choices=MODES,
                    help="run mode (runner.hpp:21): independent = per-trajectory convergence masking")
    ap.add_argument("--per-gpu", type=int, default=None, help="override the trajectory count")
    ap.add_argument("--nodes", type=int, default=200)
    ap.add_argument("--bodies", default=None, choices=["planets8", "reference", "none"])
    ap.add_argument("--force", default=None, choices=["n_body", "n_body_1pn"],
                    help="force model override (C5: Newtonian leg with --force n_body)")
    ap.add_argument("--span", type=float, default=None, help="span in osculating periods")
    ap.add_argument("--p-groups", type=int, default=None, help="grouped mode: number of groups")
    ap.add_argument("--cpu-sample", type=int, default=2000, help="trajectories in the bounded CPU baseline sample")
    ap.add_argument("--cpu-repeats", type=int, default=5, help="CPU baseline: median of this many runs per mode")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="collective backend for N > 1 (gloo: flow check with ranks sharing a GPU)")
    ap.add_argument("--launcher", default="torchrun", choices=["torchrun", "native"],
                    help="--gpus N > 1 outside torchrun: one rank per GPU (torchrun) or ONE process driving all "
                         "GPUs through the native multi-device C-ABI (pswarm_run_batch_multi, NCCL gather)")
    ap.add_argument("--devices", default=None,
                    help="native launcher: comma-separated CUDA devices (default 0..N-1; e.g. 0,0 = two contexts "
                         "on one GPU, a flow check)")
    a = ap.parse_args()
    m, scaling, bodies, kind, span, policy, start, spreads = CONFIGS[a.config]
    a.m = a.per_gpu if a.per_gpu is not None else m
    a.scaling = scaling
    a.bodies = a.bodies or bodies
    a.kind = a.force or kind
    a.span = a.span if a.span is not None else span
    a.policy, a.start, a.spreads = policy, start, spreads
    return a


def self_launch(args):
    """`bench.py --gpus N` outside torchrun: one rank per GPU via torch.distributed.run."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def workload(args, world, rank):
    import paper_2301_03989_b200 as ps
    from paper_2301_03989_b200.distributed import shard_groups
    if args.config == "c1":
        base = ps.elements_to_state([1.3e8, 0.2, 0.05, 0.4, 0.9, 0.0, 0.0], ps.MU_SUN, 0.0)
    else:
        base = ps.reference_state()
    period = ps.osculating_period(base, ps.MU_SUN)
    total = args.m * world if args.scaling == "weak" else args.m
    q = len(args.spreads)
    states = np.concatenate([ps.make_clone_batch(base, total // q + (1 if k < total % q else 0), sp)
                             for k, sp in enumerate(args.spreads)])
    plan = ps.plan_segments(base, 0.0, args.span * period, ps.MU_SUN, args.policy, args.nodes)
    bodies = {"planets8": ps.planets8, "reference": ps.reference_bodies, "none": list}[args.bodies]()
    kind = "two_body" if args.bodies == "none" and args.kind == "n_body" else args.kind
    cfg = ps.reference_force_config(kind, bodies=bodies, n_nodes=args.nodes, start_mode=args.start)
    if args.p_groups:
        cfg.p_groups = args.p_groups
    sizes = group_sizes(args, cfg, total)
    if args.mode == "independent" and world > 1:
        # singleton groups: interleaved shards -- rank r takes trajectories r, r + world, ...
        # so every rank gets the same mix of the C5 spread quarters (heterogeneous iteration counts).
        # The batch is reordered so the shards are contiguous; the metric does not depend on the order.
        perm = np.concatenate([np.arange(r, total, world) for r in range(world)])
        states = np.ascontiguousarray(states[perm])
        counts = [len(range(r, total, world)) for r in range(world)]
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(int)
        shards = [(int(offs[r]), int(offs[r + 1]), int(offs[r]), int(offs[r + 1])) for r in range(world)]
    else:
        shards = shard_groups(sizes, world)  # group-aligned contiguous shards (block.hpp:83-106)
    lo, hi = shards[rank][2], shards[rank][3]
    return states, (lo, hi), plan, cfg, shards


def group_sizes(args, cfg, total):
    import paper_2301_03989_b200 as ps
    if args.mode == "independent":
        return [1] * total
    if args.mode.startswith("augmented"):
        return [total]
    return list(ps.split_groups(total, min(max(cfg.p_groups, 1), total)))


def config_dict(args, world, plan=None, cfg=None, launcher=None):
    total = args.m * world if args.scaling == "weak" else args.m
    nb = {"planets8": 8, "reference": 2, "none": 0}[args.bodies]
    mode = args.mode + (f" (p_groups={cfg.p_groups})" if cfg is not None and args.mode == "grouped" else "")
    return {
        "workload": DESCR[args.config].format(m=args.m, span=args.span, force="relativistic (EIH 1PN, EXTENSION)"
                                              if args.kind == "n_body_1pn" else "Newtonian") +
                    f", N={args.nodes} nodes, {args.start} start, tol 1e-12, run mode {mode}" +
                    (" = per-trajectory convergence masking" if args.mode == "independent" else ""),
        "name": args.config, "mode": args.mode, "trajectories_per_gpu": total // world, "trajectories_total": total,
        "nodes": args.nodes, "bodies": nb, "force": args.kind,
        "segments": None if plan is None else len(plan.boundaries) - 1, "dtype": "f64",
        "parallelism": f"dp{world} (" + ("interleaved " if args.mode == "independent" and world > 1 else "") +
                       "trajectory shards, no collective in the iteration loop; terminal states "
                       "gathered to rank 0)" + (f"; {launcher}" if launcher else ""),
        "l2": "flushed between steps (512 MiB device write, outside the timed region)",
    }


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = str(index)
        self.path = f"/tmp/bench_clocks_{os.getpid()}.csv"
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}", "--format=csv,noheader",
                                          "-lms", "20"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1].split()[0]))
                mx.append(float(f[2].split()[0]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        post = False
        if not sm:  # timed region shorter than the 20 ms sampling period: one query right after it
            try:
                out = subprocess.run(["nvidia-smi", "-i", self.index, "--query-gpu=clocks.sm,clocks.max.sm",
                                      "--format=csv,noheader"], capture_output=True, text=True, timeout=10).stdout
                f = [x.strip() for x in out.split(",")]
                sm.append(float(f[0].split()[0]))
                mx.append(float(f[1].split()[0]))
                post = True
            except (OSError, ValueError, IndexError, subprocess.SubprocessError):
                pass
        under = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        res = {"sm_mhz": statistics.median(under) if under else None, "sm_max_mhz": max(mx) if mx else None,
               "samples": len(sm), "reasons": sorted(reasons)}
        if post:
            res["sampled_after_region"] = True
        return res


def fp64_peak():
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak_r01.json")))
        return max(d["dmma_w16_tflops"], d["dmma_w8_tflops"]), "measured (tools/fp64_peak.cu DMMA.8x8x4 loop)"
    except (OSError, KeyError, ValueError):
        return 37.0, "fallback (B200 FP64 nominal)"


def profile_tag(args):
    if args.config == "c5" or args.nodes != 200:
        return f"{args.config}_n{args.nodes}" + ("_newton" if args.config == "c5" and args.kind == "n_body" else "")
    return args.config + ("" if args.mode == "independent" else f"_{args.mode}")


def ncu_record(args):
    """Latest committed ncu summary of this config's launch (tools/ncu_csv_summary.py), or None."""
    tag = profile_tag(args)
    cands = sorted(glob.glob(os.path.join(ROOT, "profiles", f"ncu_r[0-9][0-9]_{tag}.json")))
    if not cands:
        return None, None
    try:
        return json.load(open(cands[-1])), os.path.relpath(cands[-1], ROOT)
    except (OSError, ValueError):
        return None, None


def hardware_info():
    cores = os.cpu_count() or 1
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except (OSError, subprocess.SubprocessError):
        pass
    return cores, model


def cpu_oracle(cfg):
    """The reference's own sources (oracle/_ref) when built and the config is reference
    physics; otherwise the restatement.  Returns (Oracle, kind)."""
    from oracle.oracle_py import Oracle, reference_available
    if reference_available() and cfg.force_kind != "n_body_1pn" and cfg.start_mode != "hot":
        return Oracle(reference=True), "reference"
    return Oracle(), "port"


def cpu_sample(states, k):
    """Evenly strided subsample (covers every quarter of a mixed-spread cloud)."""
    if len(states) <= k:
        return states
    return np.ascontiguousarray(states[np.linspace(0, len(states) - 1, k).round().astype(int)])


def time_cpu_mode(orc, states, cfg, plan, mode, cores, repeats):
    import copy
    c = copy.copy(cfg)
    if mode == "grouped":
        c.p_groups = min(4 * cores, len(states))  # P = 4 x cores
    ts, res = [], None
    for _ in range(repeats):
        t0 = time.perf_counter()
        res = orc.run_batch(states, c, plan, mode, cores, samples=mode == "independent")
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), res


def cpu_baseline(args, states, plan, cfg, r_check):
    """CPU reference on all host cores: independent, grouped (P = 4 x cores) and
    augmented_parallel, median of `--cpu-repeats`, best reported; parity of the GPU on the sample."""
    import paper_2301_03989_b200 as ps
    orc, kind = cpu_oracle(cfg)
    cores, model = hardware_info()
    modes = {}
    ref = None
    for mode in ("independent", "grouped", "augmented_parallel"):
        t, res = time_cpu_mode(orc, states, cfg, plan, mode, cores, args.cpu_repeats)
        modes[mode] = round(len(states) / t, 2)
        if mode == "independent":
            ref = res
    best = max(modes, key=modes.get)
    disc = ps.max_state_discrepancy(r_check.trajectories, ref.trajectories)
    diter = int(np.abs(r_check.iterations.astype(int) - ref.iterations.astype(int)).max())
    src = ("oracle/_ref: the reference's own sources (proj/include/pswarm) built unchanged on the Eigen-subset "
           "shim, -O3 no -march" if kind == "reference" else
           "oracle/pswarm_ref.hpp restatement (the reference has no such path: EXTENSION config)")
    return {"value": modes[best], "unit": UNIT, "cores": cores, "kind": kind, "cpu_model": model,
            "best_mode": best, "modes": modes,
            "sample": f"{len(states)} trajectories (evenly strided over the workload), run_batch in each mode with "
                      f"{cores} worker threads, median of {args.cpu_repeats}; {src}",
            "parity_vs_gpu": {"max_rel_state_discrepancy": disc, "max_abs_iteration_diff": diter,
                              "segments_equal": bool(r_check.trajectories.shape[1] == ref.trajectories.shape[1]),
                              "note": "GPU vs the CPU reference on the same sample in independent mode "
                                      "(per-trajectory results do not depend on the batch)"}}


def run_reference(args):
    """Reference arm: the reference's own CPU implementation on the box's host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    states, _, plan, cfg, _ = workload(args, world, 0)
    states = cpu_sample(states, args.cpu_sample)
    orc, kind = cpu_oracle(cfg)
    cores, model = hardware_info()
    # warm-up: each mode once; the timed steps use the fastest (best reported)
    warm = {}
    for mode in ("independent", "grouped", "augmented_parallel"):
        warm[mode] = time_cpu_mode(orc, states, cfg, plan, mode, cores, 1)[0]
    for _ in range(max(0, args.warmup - 1)):
        time_cpu_mode(orc, states, cfg, plan, min(warm, key=warm.get), cores, 1)
    mode = min(warm, key=warm.get)
    times = [time_cpu_mode(orc, states, cfg, plan, mode, cores, 1)[0] for _ in range(args.steps)]
    ms = 1e3 * statistics.median(times)
    v = len(states) / (ms * 1e-3)
    cfgd = config_dict(args, world, plan, cfg)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfgd,
        "e2e": {"value": round(v, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu_baseline": {"value": round(v, 2), "unit": UNIT, "cores": cores, "kind": kind, "cpu_model": model,
                         "mode": mode, "warmup_seconds_per_mode": {k: round(t, 3) for k, t in warm.items()},
                         "sample": f"{len(states)} trajectories per step (evenly strided over the workload), "
                                   f"run_batch({mode}) with {cores} worker threads (fastest of independent / grouped "
                                   "P=4x cores / augmented_parallel in warm-up); median step time; " +
                                   ("the reference's own sources (oracle/_ref)" if kind == "reference"
                                    else "oracle/pswarm_ref.hpp restatement")},
    }), flush=True)


def parity_subsample(ctx, states, gathered, shards, cfg, plan, mode):
    """Re-propagate a strided subsample (every 997th trajectory + first/last of every shard) on
    its own and compare with the full (gathered) run: independent mode results do not depend
    on the batch composition, so they must agree bit for bit."""
    idx = set(range(0, len(states), 997))
    for (_, _, lo, hi) in shards:
        if hi > lo:
            idx.update((lo, hi - 1))
    idx = np.array(sorted(idx))
    r = ctx.run_batch(states[idx], cfg, plan, mode, samples=False, history=False)
    a, b = r.terminal_states[:, 1:], gathered[idx, 1:]
    rel = np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))
    return {"subsample": int(len(idx)), "bit_identical": bool(np.array_equal(r.terminal_states, gathered[idx])),
            "max_rel_component_diff": float(rel),
            "vs": "the same trajectories propagated alone in one rank-0 call (every 997th + first/last of each shard)"}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.launcher == "torchrun":
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2301_03989_b200 as ps
    from paper_2301_03989_b200.distributed import gather_terminal

    native = args.launcher == "native" and args.gpus > 1 and "WORLD_SIZE" not in os.environ
    world = 1 if native else int(os.environ.get("WORLD_SIZE", "1"))  # processes
    rank = 0 if native else int(os.environ.get("RANK", "0"))
    # one rank per GPU; --dist-backend gloo lets several ranks share a GPU (flow check only)
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    nccl = args.dist_backend == "nccl"
    if world > 1:
        if nccl:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    gdev = dev if nccl else None  # gather buffers: device (NVLink) or host (gloo)
    if native:  # one process, all GPUs: C++ host threads + NCCL gather inside the library
        devices = [int(d) for d in args.devices.split(",")] if args.devices else list(range(args.gpus))
        mctx = ps.MultiContext(devices)
        ctx = ps.Context(local)  # parity reference (single device)
        n_gpus = len(devices)
        states, (lo, hi), plan, cfg, shards = workload(args, n_gpus, 0)
        lo, hi = 0, len(states)
    else:
        ctx = ps.Context(local)
        n_gpus = world
        states, (lo, hi), plan, cfg, shards = workload(args, world, rank)
    shard = torch.from_numpy(states[lo:hi].copy()).pin_memory().numpy()  # pinned host ICs
    M = hi - lo
    term_out = ps.pinned_terminal_buffer(M)  # pinned host result: one DMA per step
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local]) if nccl else dist.barrier()
        torch.cuda.synchronize(dev)

    def step():
        if native:
            r = mctx.run_batch(shard, cfg, plan, args.mode, samples=False, history=False, terminal=term_out)
            r.gathered = r.terminal_states
            return r
        r = ctx.run_batch(shard, cfg, plan, args.mode, samples=False, history=False, terminal=term_out)
        if world > 1:  # final gather of terminal states to rank 0 (NCCL over NVLink)
            r.gathered = gather_terminal(r.terminal_states, shards, rank, world, device=gdev)
        return r

    for _ in range(args.warmup):
        step()
    launches0 = (mctx if native else ctx).run_batch(shard[:1], cfg, plan, "independent", samples=False,
                                                    history=False).gpu_launches
    clocks = Clocks(local)
    wall, dev_ms, ker_ms, iters = [], [], [], []
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush (outside the timed region)
        barrier()
        t0 = time.perf_counter()
        r = step()
        barrier()
        wall.append(time.perf_counter() - t0)
        dev_ms.append(r.device_ms)
        ker_ms.append(r.kernel_ms)
        iters.append(r.trajectory_iterations)
    clk = clocks.stop()
    launches = r.gpu_launches - launches0  # context's cumulative count of its own kernel launches

    def gmax(x):
        t = torch.tensor([x], dtype=torch.float64, device=gdev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    wall_ms = gmax(1e3 * statistics.mean(wall))
    dms = gmax(statistics.mean(dev_ms))
    kms_mean = statistics.mean(ker_ms)
    total = len(states)
    value = total / (dms * 1e-3)
    e2e = total / (wall_ms * 1e-3)
    flops = flops_per_trajectory_iteration(args.nodes, len(cfg.bodies), cfg.force_kind) * statistics.mean(iters)
    achieved = flops / (kms_mean * 1e-3) / 1e12
    peak, peak_src = fp64_peak()
    prof, prof_path = ncu_record(args) if n_gpus == 1 else (None, None)

    if rank == 0:
        gathered = r.gathered if (world > 1 or native) else r.terminal_states
        parity = parity_subsample(ctx, states, gathered, shards, cfg, plan, args.mode) \
            if args.mode == "independent" else None
        cpu = None
        if n_gpus == 1 and not args.no_cpu_baseline:
            sample = cpu_sample(states[lo:hi], args.cpu_sample)
            cpu = cpu_baseline(args, sample, plan, cfg, r_check=ctx.run_batch(sample, cfg, plan, "independent"))
        roof = {"bound": "tensor", "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4), "traffic": None,
                "kernel": ctx.kernel_name() if not native else f"{ctx.kernel_name()} x{n_gpus} (kernel_ms = max over "
                                                                   "devices)", "kernel_ms": round(kms_mean, 4),
                "flops_per_launch": flops, "peak_source": peak_src,
                "note": "achieved = reference-algorithmic FP64 flops (SURVEY §8d) / kernel time (CUDA events); "
                        "FP64 DMMA/DFMA share one pipe on B200 (tools/fp64_peak.cu mixed test)"}
        if prof is not None:
            ex = prof["executed"]["fp64_flops"]
            roof["traffic"] = prof["dram_bytes"]
            roof["ncu"] = {"record": prof_path, "duration_ms": prof["duration_ms"],
                           "dmma_pipe_active_pct": prof["dmma_pipe_active_pct"],
                           "fp64_pipe_active_pct": prof["fp64_pipe_active_pct"],
                           "executed_fp64_flops": ex,
                           # one captured launch = one segment: against this run's mean kernel time per segment
                           "executed_frac": round(ex / (kms_mean / max(len(plan.boundaries) - 1, 1) * 1e-3) / 1e12 /
                                                  peak, 4),
                           "note": "executed = DMMA + 2 DFMA + DADD + DMUL of the captured launch over this "
                                   "run's kernel time (the mirror-folded update executes half the reference's "
                                   "update flops, so executed_frac < frac)"}
        out = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": n_gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dms, 4), "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded clone cloud, analytic planets)",
            "config": config_dict(args, n_gpus, plan, cfg, native and f"native multi-device C-ABI over devices "
                                                                    f"{devices}, gather: {mctx.backend}"),
            "e2e": {"value": round(e2e, 1), "unit": UNIT, "ms_per_step": round(wall_ms, 4),
                    "h2d_bytes_per_step": int(total * 7 * 8), "d2h_bytes_per_step": int(total * 7 * 8),
                    "path": ("pswarm_run_batch_multi C-ABI (one process, host thread per device, " +
                             f"{mctx.backend} gather), pinned host buffers" if native else
                             "pswarm_run_batch C-ABI, pinned host buffers" +
                             (f" + {args.dist_backend} gather to rank 0" if world > 1 else ""))},
            "roofline": roof,
            "cpu_baseline": cpu,
            "parity": parity,
            "clocks": clk,
            "gpu_launches": launches,
            "picard_iterations_per_trajectory": round(statistics.mean(iters) / M, 3) if M else None,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local]) if nccl else dist.barrier()
        dist.destroy_process_group()


def flops_per_trajectory_iteration(n, b, kind):
    """Algorithmic FP64 flops of one Picard iteration of one trajectory (
    add/sub/mul/div/sqrt = 1, FMA = 2): update 12N^2 + 18N + 12, force (21 + 20B)N, error
    36N; the relativistic model (EXTENSION) adds (80(B+1) + 20)N."""
    f = 12 * n * n + (75 + 20 * b) * n + 12
    if kind == "n_body_1pn":
        f += (80 * (b + 1) + 20) * n
    return f


if __name__ == "__main__":
    main()
