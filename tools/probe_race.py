"""Repeat one propagation many times and report any run that differs from the first (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_03989_b200 as ps

n = int(sys.argv[1]) if len(sys.argv) > 1 else 160
m = int(sys.argv[2]) if len(sys.argv) > 2 else 24
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, m, 1e-5)
plan = ps.plan_segments(base, 0.0, 0.6 * period, ps.MU_SUN, "single", n)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=n)
ref = ctx.run_batch(states, cfg, plan, "independent")
nbad = 0
for r in range(reps):
    got = ctx.run_batch(states, cfg, plan, "independent")
    if not np.array_equal(got.trajectories, ref.trajectories) or not np.array_equal(got.iterations, ref.iterations):
        nbad += 1
        if nbad <= 3:
            diff = np.abs(got.trajectories - ref.trajectories).max(axis=2)  # [M][R]
            ti = np.nonzero(diff.max(axis=1) > 0)[0]
            for t in ti[:4]:
                nodes = np.nonzero(diff[t] > 0)[0]
                zero = np.all(got.trajectories[t, nodes] == 0, axis=1).sum()
                print(f"rep {r} traj {t} nodes {len(nodes)} first {nodes[:6]} zero-rows {zero} "
                      f"maxabs {diff[t].max():.3e} iters {got.iterations[0][t]} vs {ref.iterations[0][t]}", flush=True)
print(f"N={n} M={m} kernel={ctx.kernel_name()} bad runs {nbad}/{reps}")
