"""Run-mode throughput (diagnostics): independent (per-trajectory masking), grouped with
P groups and augmented (one group = the paper's augmented system) on the C2 workload."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
for M in (1000, 13509):
    states = ps.make_clone_batch(base, M, 1e-5)
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
    for mode, p in (("independent", 1), ("grouped", 10), ("grouped", M // 4), ("augmented", 1)):
        cfg.p_groups = p
        for rep in range(2):
            t0 = time.perf_counter()
            r = ctx.run_batch(states, cfg, plan, mode, samples=False, history=False)
            dt = time.perf_counter() - t0
        print(f"M={M} {mode} P={p}: {ctx.kernel_name()} wall {dt * 1e3:.2f} ms device {r.device_ms:.2f} ms "
              f"kernel {r.kernel_ms:.2f} ms launches {r.gpu_launches} iters max {r.iterations.max()} "
              f"-> {M / dt:.0f} traj/s", flush=True)
