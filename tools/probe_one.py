"""One propagation of the C2-shaped workload for ncu capture: python tools/probe_one.py M [bodies] [N] [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

M = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
bodies = sys.argv[2] if len(sys.argv) > 2 else "planets8"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 200
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, M, 1e-5)
plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", N)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8() if bodies == "planets8" else ps.reference_bodies(),
                                n_nodes=N)
for _ in range(reps):
    r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
print("kernel_ms", r.kernel_ms, "iters", r.trajectory_iterations)
