"""N-sweep parity probe (diagnostics): GPU vs oracle discrepancy per node count."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_03989_b200 as ps
from oracle.oracle_py import Oracle

ctx = ps.Context(0)
orc = Oracle()
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
ns = [int(x) for x in sys.argv[1:]] or [64, 96, 128, 160, 200, 232, 256]
for n in ns:
    for m in (4, 8, 24):
        states = ps.make_clone_batch(base, m, 1e-5)
        plan = ps.plan_segments(base, 0.0, 0.6 * period, ps.MU_SUN, "single", n)
        cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=n)
        want = orc.run_batch(states, cfg, plan, "independent", 8)
        for rep in range(2):
            got = ctx.run_batch(states, cfg, plan, "independent")
            d = ps.max_state_discrepancy(got.trajectories, want.trajectories)
            per = [ps.max_state_discrepancy(got.trajectories[i:i+1], want.trajectories[i:i+1]) for i in range(m)]
            bad = [i for i, x in enumerate(per) if x > 1e-10]
            print(n, m, rep, ctx.kernel_name(), f"{d:.3e}", "bad:", bad[:12],
                  "iters", got.iterations.min(), got.iterations.max(), want.iterations.max(), flush=True)
