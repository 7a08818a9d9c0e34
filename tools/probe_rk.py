"""Throughput of the device RKF7(8) verifier on the C2 workload (diagnostics)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
for m in (1000, 10000):
    states = ps.make_clone_batch(base, m, 1e-5)
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
    res = ctx.run_batch(states, cfg, plan, "independent")
    t0 = time.perf_counter()
    _, _, mx = ctx.oracle_check(states, cfg, res.times, candidate=res.trajectories, samples=False)
    dt = time.perf_counter() - t0
    print(f"M={m} oracle_check {dt:.3f} s ({m / dt:.0f} traj/s), max PC-vs-RKF78 discrepancy {mx.max():.3e}")
