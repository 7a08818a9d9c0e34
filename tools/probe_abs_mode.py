import sys, numpy as np
sys.path.insert(0, ".")
import paper_2301_03989_b200 as ps
from oracle.oracle_py import Oracle
ctx, o = ps.Context(0), Oracle()
base = ps.reference_state()
states = ps.make_clone_batch(base, 24, 1e-5)
period = ps.osculating_period(base, ps.MU_SUN)
for n in (64, 200):
    plan = ps.plan_segments(base, 0.0, 0.6 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=n)
    cfg.error_mode = "absolute"; cfg.tolerance = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3
    g = ctx.run_batch(states, cfg, plan, "independent"); w = o.run_batch(states, cfg, plan, "independent", 1)
    print(n, ctx.kernel_name(), g.iterations.ravel(), w.iterations.ravel(), ps.max_state_discrepancy(g.trajectories, w.trajectories))
    print("gpu err", np.array([r.final_error for r in g.reports[0]])[:6], "orc", np.array([r.final_error for r in w.reports[0]])[:6])
