#!/usr/bin/env python3
"""Throughput benchmark: trajectories propagated/sec (N-body PC) on B200.

Workload (BASELINE.json configs[1], "C2"): 1,000 perturbed clones of the
reference spacecraft state (a = 1.25e8 km, e = 0.12; make_clone_batch spread
1e-5, seed 20220411) per GPU, Sun + 8 planets Newtonian N-body, N = 200
Chebyshev-Lobatto nodes, one 0.87-period segment, warm start, tol 1e-12
relative, per-trajectory convergence masking (RunMode::independent).

One step = one propagation of the whole batch through the C-ABI
(pswarm_run_batch): host ICs in -> terminal states in host memory out.
  value     trajectories/s over the device solve phase (inputs resident in HBM),
            whole job, max over ranks (weak scaling: 1,000 ICs per GPU)
  e2e       trajectories/s of the full C-ABI call with host buffers (H2D of the
            ICs, solve, D2H of terminal states; + NCCL gather when N > 1)
  roofline  algorithmic FP64 flops of the PC kernel (F_it =
            12N^2 + (75+20B)N + 12 per trajectory-iteration) / kernel time vs the
            measured FP64 (DMMA) peak in profiles/fp64_peak_r01.json
`--impl reference` times the CPU oracle (Eigen-free restatement of the
reference, all host cores) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
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
    "c4": "C4: {m}-trajectory cloud total sharded over the GPUs, Sun + 8 planets, {span} period single segment",
    "c5": ("C5: relativistic (EIH 1PN, EXTENSION) Sun + 8 planets, {m} ICs total in four quarters with clone "
           "spreads 1e-7/1e-5/1e-3/1e-2 (convergence-mask stress), {span} period single segment"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS), help="BASELINE.json configs[0..4]")
    ap.add_argument("--per-gpu", type=int, default=None, help="override the trajectory count")
    ap.add_argument("--nodes", type=int, default=200)
    ap.add_argument("--bodies", default=None, choices=["planets8", "reference", "none"])
    ap.add_argument("--span", type=float, default=None, help="span in osculating periods")
    ap.add_argument("--cpu-sample", type=int, default=2000, help="trajectories in the bounded CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="collective backend for N > 1 (gloo: flow check with ranks sharing a GPU)")
    a = ap.parse_args()
    m, scaling, bodies, kind, span, policy, start, spreads = CONFIGS[a.config]
    a.m = a.per_gpu if a.per_gpu is not None else m
    a.scaling = scaling
    a.bodies = a.bodies or bodies
    a.kind = kind
    a.span = a.span if a.span is not None else span
    a.policy, a.start, a.spreads = policy, start, spreads
    return a


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
    shards = shard_groups([1] * total, world)  # independent mode: singleton groups
    lo, hi = shards[rank][2], shards[rank][3]
    plan = ps.plan_segments(base, 0.0, args.span * period, ps.MU_SUN, args.policy, args.nodes)
    bodies = {"planets8": ps.planets8, "reference": ps.reference_bodies, "none": list}[args.bodies]()
    kind = "two_body" if args.bodies == "none" and args.kind == "n_body" else args.kind
    cfg = ps.reference_force_config(kind, bodies=bodies, n_nodes=args.nodes, start_mode=args.start)
    return states, (lo, hi), plan, cfg, shards


def config_dict(args, world, plan=None):
    total = args.m * world if args.scaling == "weak" else args.m
    nb = {"planets8": 8, "reference": 2, "none": 0}[args.bodies]
    return {
        "workload": DESCR[args.config].format(m=args.m, span=args.span) +
                    f", N={args.nodes} nodes, {args.start} start, tol 1e-12, per-trajectory convergence masking "
                    "(independent mode)",
        "name": args.config, "trajectories_per_gpu": total // world, "trajectories_total": total,
        "nodes": args.nodes, "bodies": nb, "force": args.kind,
        "segments": None if plan is None else len(plan.boundaries) - 1, "dtype": "f64",
        "parallelism": f"dp{world} (trajectory shards, no collective in the iteration loop)",
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


def ncu_traffic():
    """dram bytes per launch of the PC kernel from the committed ncu capture, or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))
        return d.get("bench_kernel", {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def run_reference(args):
    """CPU oracle on the same workload, all host threads (rank 0 only)."""
    from oracle.oracle_py import Oracle
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    states, (lo, hi), plan, cfg, _ = workload(args, 1, 0)
    states = cpu_sample(states, args.cpu_sample)
    orc = Oracle()
    cores = os.cpu_count() or 1
    for _ in range(args.warmup):
        orc.run_batch(states, cfg, plan, "independent", cores, samples=False)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        orc.run_batch(states, cfg, plan, "independent", cores, samples=False)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(times)
    v = len(states) / (ms * 1e-3)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, 1, plan),
        "e2e": {"value": round(v, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu_baseline": {"value": round(v, 2), "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{len(states)} trajectories per step (evenly strided over the workload), "
                                   f"run_batch independent mode with {cores} worker threads (oracle/pswarm_ref.hpp "
                                   "restatement; the reference needs Eigen, absent here)"},
    }), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2301_03989_b200 as ps

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
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
    ctx = ps.Context(local)
    from paper_2301_03989_b200.distributed import gather_terminal
    states, (lo, hi), plan, cfg, shards = workload(args, world, rank)
    shard = torch.from_numpy(states[lo:hi].copy()).pin_memory().numpy()  # pinned host ICs
    M = hi - lo
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local]) if nccl else dist.barrier()
        torch.cuda.synchronize(dev)

    def step():
        r = ctx.run_batch(shard, cfg, plan, "independent", samples=False, history=False)
        if world > 1:  # final gather of terminal states over NVLink (NCCL)
            r.gathered = gather_terminal(r.terminal_states, shards, rank, world, device=gdev)
        return r

    for _ in range(args.warmup):
        step()
    clocks = Clocks(local)
    wall, dev_ms, ker_ms, iters = [], [], [], []
    launches0 = ctx.run_batch(shard[:1], cfg, plan, "independent", samples=False, history=False).gpu_launches
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

    if world > 1:  # the gathered terminal states are the single-process batch order
        g = r.gathered
        assert g.shape == (len(states), 7) and np.array_equal(g[lo:hi], r.terminal_states)

    wall_ms = gmax(1e3 * statistics.mean(wall))
    dms = gmax(statistics.mean(dev_ms))
    kms_mean = statistics.mean(ker_ms)
    total = M * world
    value = total / (dms * 1e-3)
    e2e = total / (wall_ms * 1e-3)
    flops = flops_per_trajectory_iteration(args.nodes, len(cfg.bodies), cfg.force_kind) * statistics.mean(iters)
    achieved = flops / (kms_mean * 1e-3) / 1e12
    peak, peak_src = fp64_peak()

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            sample = cpu_sample(states[lo:hi], args.cpu_sample)
            cpu = cpu_baseline(args, sample, plan, cfg, r_check=ctx.run_batch(sample, cfg, plan, "independent"))
        out = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(dms, 4), "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded clone cloud, analytic planets)",
            "config": config_dict(args, world, plan),
            "e2e": {"value": round(e2e, 1), "unit": UNIT, "ms_per_step": round(wall_ms, 4),
                    "h2d_bytes_per_step": int(M * 7 * 8), "d2h_bytes_per_step": int(M * 7 * 8),
                    "path": "pswarm_run_batch C-ABI, pinned host buffers" + (f" + {args.dist_backend} all_gather" if world > 1 else "")},
            "roofline": {"bound": "tensor", "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
                         "frac": round(achieved / peak, 4), "traffic": ncu_traffic(),
                         "kernel": ctx.kernel_name(), "kernel_ms": round(kms_mean, 4),
                         "flops_per_launch": flops, "peak_source": peak_src,
                         "note": "FP64 DMMA/DFMA share one pipe on B200 (tools/fp64_peak.cu mixed test)"},
            "cpu_baseline": cpu,
            "clocks": clk,
            "gpu_launches": launches,
            "picard_iterations_per_trajectory": round(statistics.mean(iters) / M, 3),
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local]) if nccl else dist.barrier()
        dist.destroy_process_group()


def cpu_sample(states, k):
    """Evenly strided subsample (covers every quarter of a mixed-spread cloud)."""
    if len(states) <= k:
        return states
    return np.ascontiguousarray(states[np.linspace(0, len(states) - 1, k).round().astype(int)])


def flops_per_trajectory_iteration(n, b, kind):
    """Algorithmic FP64 flops of one Picard iteration of one trajectory (
    add/sub/mul/div/sqrt = 1, FMA = 2): update 12N^2 + 18N + 12, force (21 + 20B)N, error
    36N; the relativistic model (EXTENSION) adds (80(B+1) + 20)N."""
    f = 12 * n * n + (75 + 20 * b) * n + 12
    if kind == "n_body_1pn":
        f += (80 * (b + 1) + 20) * n
    return f


def cpu_baseline(args, states, plan, cfg, r_check):
    """CPU oracle (all host cores) on the same workload; also checks parity of this run."""
    import paper_2301_03989_b200 as ps
    from oracle.oracle_py import Oracle
    orc = Oracle()
    cores = os.cpu_count() or 1
    times = []
    ref = None
    for _ in range(2):
        t0 = time.perf_counter()
        ref = orc.run_batch(states, cfg, plan, "independent", cores)
        times.append(time.perf_counter() - t0)
    v = len(states) / min(times)
    disc = ps.max_state_discrepancy(r_check.trajectories, ref.trajectories)
    diter = int(np.abs(r_check.iterations.astype(int) - ref.iterations.astype(int)).max())
    return {"value": round(v, 2), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{len(states)} trajectories (evenly strided over the workload), best of 2, run_batch "
                      f"independent mode, {cores} threads (oracle/pswarm_ref.hpp); parity below is the GPU on the "
                      "same sample (independent mode: per-trajectory results do not depend on the batch)",
            "parity_vs_gpu": {"max_rel_state_discrepancy": disc, "max_abs_iteration_diff": diter}}


if __name__ == "__main__":
    main()
