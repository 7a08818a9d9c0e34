import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2301_03989_b200 as ps
from oracle.oracle_py import Oracle
base = ps.reference_state(); period = ps.osculating_period(base, ps.MU_SUN)
rng = np.random.default_rng(7)
states = ps.make_clone_batch(base, 1, 1e-7)
plan = ps.plan_segments(base, 0.0, 1.5 * period, ps.MU_SUN, "per_orbit", 200)
for start in ("hot", "warm"):
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200, start_mode=start)
    for mode in ("augmented", "independent"):
        g = ps.Context(0).run_batch(states, cfg, plan, mode)
        w = Oracle().run_batch(states, cfg, plan, mode, 1)
        print(start, mode, "gpu it", g.iterations.ravel(), "oracle it", w.iterations.ravel())
        for s in range(plan.segments()):
            a = g.reports[s][0].per_iteration_errors; b = w.reports[s][0].per_iteration_errors
            print("  seg", s, "gpu", np.array2string(a[-8:], precision=2), "\n         ora", np.array2string(b[-8:], precision=2))
