"""Multi-process (world_size 2, gloo, CPU) test of the sharding + terminal-state
gather used by bench.py under torchrun.  Each rank solves its group-aligned
shard (CPU oracle as the per-rank stand-in solver: no GPU here) and the gathered
terminal states must equal a single-process run bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_path):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2301_03989_b200 as ps
    from oracle.oracle_py import Oracle
    from paper_2301_03989_b200.distributed import gather_terminal, shard_groups

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    base = ps.reference_state()
    states = ps.make_clone_batch(base, 24, 1e-5)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, 0.3 * period, ps.MU_SUN, "single", 32)
    cfg = ps.reference_force_config("n_body", n_nodes=32)
    groups = [3, 5, 2, 4, 6, 4]  # grouped plan; shards must not split a group
    shards = shard_groups(groups, world)
    g_lo, g_hi, lo, hi = shards[rank]
    local = Oracle().propagate(states[lo:hi], groups[g_lo:g_hi], plan, cfg).terminal_states
    full = gather_terminal(local, shards, rank, world)
    if rank == 0:
        np.save(result_path, full)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_groups_alignment():
    from paper_2301_03989_b200.distributed import shard_groups
    groups = [3, 5, 2, 4, 6, 4]
    for world in (1, 2, 3, 4):
        sh = shard_groups(groups, world)
        assert sh[0][0] == 0 and sh[-1][1] == len(groups)
        for (a, b, lo, hi), (a2, _, lo2, _) in zip(sh, sh[1:]):
            assert b == a2 and hi == lo2
        assert sum(hi - lo for _, _, lo, hi in sh) == sum(groups)
    one = shard_groups([1] * 1000, 8)
    assert all(hi - lo == 125 for _, _, lo, hi in one)


def test_two_rank_gather_matches_single_process(tmp_path, oracle):
    import torch.multiprocessing as mp

    import paper_2301_03989_b200 as ps
    port = _free_port()
    out = str(tmp_path / "full.npy")
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    full = np.load(out)
    base = ps.reference_state()
    states = ps.make_clone_batch(base, 24, 1e-5)
    period = ps.osculating_period(base, ps.MU_SUN)
    plan = ps.plan_segments(base, 0.0, 0.3 * period, ps.MU_SUN, "single", 32)
    cfg = ps.reference_force_config("n_body", n_nodes=32)
    want = oracle.propagate(states, [3, 5, 2, 4, 6, 4], plan, cfg).terminal_states
    assert full.shape == want.shape
    assert np.array_equal(full, want)


def test_bench_reference_arm_runs_on_cpu():
    """bench.py --impl reference (the reference's own CPU implementation) prints one JSON
    line with the contract keys; tiny sample so it runs here."""
    import json
    import subprocess
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c2",
                        "--steps", "2", "--warmup", "1", "--cpu-sample", "24", "--nodes", "64"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
