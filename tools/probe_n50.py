import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2301_03989_b200 as ps
from oracle.oracle_py import Oracle
ctx = ps.Context(0); orc = Oracle()
base = ps.reference_state(); period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 12, 1e-5)
for n in (48, 49, 50, 51, 52):
    plan = ps.plan_segments(base, 0.0, 0.5 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=n)
    for opt in ({"slot_kernel": 0}, {"slot_kernel": 1}):
        for k, v in opt.items(): ctx.set_option(k, v)
        got = ctx.run_batch(states, cfg, plan, "independent")
        want = orc.run_batch(states, cfg, plan, "independent", 8)
        print(n, opt, ctx.kernel_name(), "disc %.3e" % ps.max_state_discrepancy(got.trajectories, want.trajectories),
              "it gpu", got.iterations.ravel()[:8].tolist(), "oracle", want.iterations.ravel()[:8].tolist(), "errs", max(r.final_error for r in got.reports[0]), max(r.final_error for r in want.reports[0]))
    ctx.set_option("slot_kernel", 0)
