"""Folded vs dense k_pc_ws: parity against the oracle and kernel time (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_03989_b200 as ps
from oracle.oracle_py import Oracle

ctx = ps.Context(0)
ctx.set_option("poison_outputs", 1)
orc = Oracle()
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
for n in (128, 160, 200, 256):
    states = ps.make_clone_batch(base, 24, 1e-5)
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=n)
    want = orc.run_batch(states, cfg, plan, "independent", 8)
    for fold, uni in ((1, 1), (1, 0), (0, 0)):
        ctx.set_option("fold", fold)
        ctx.set_option("unified", uni)
        got = ctx.run_batch(states, cfg, plan, "independent")
        d = ps.max_state_discrepancy(got.trajectories, want.trajectories)
        di = int(np.abs(got.iterations.astype(int) - want.iterations.astype(int)).max())
        print(n, ctx.kernel_name(), f"disc {d:.3e} diter {di}", flush=True)
ctx.set_option("fold", 1)
ctx.set_option("unified", 1)
for M in (1000, 100000):
    states = ps.make_clone_batch(base, M, 1e-5)
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
    for fold, uni in ((1, 1), (1, 0), (0, 0)):
        ctx.set_option("fold", fold)
        ctx.set_option("unified", uni)
        for rep in range(3):
            r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
        fit = 12 * 200 * 200 + (75 + 160) * 200 + 12
        print(M, ctx.kernel_name(), f"kernel {r.kernel_ms:.3f} ms -> {fit * r.trajectory_iterations / (r.kernel_ms * 1e-3) / 1e12:.2f} TF/s",
              flush=True)
