"""Kernel time with fixed work (30 iterations for every trajectory) for the ablation
builds of tools/ablate.sh (diagnostics; select the build with PSWARM_LIB)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 10000, 1e-5)
plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200, tolerance=1e-300, max_iterations=30)
ms = []
for rep in range(3):
    try:
        r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
    except ps.PropagationIncompleteError as e:  # tol 1e-300: every trajectory runs max_iterations
        r = e.partial
    ms.append(r.kernel_ms)
print(os.path.basename(os.environ.get("PSWARM_LIB", "full")), "kernel_ms", round(min(ms), 3),
      "iterations", int(r.iterations.max()), flush=True)
