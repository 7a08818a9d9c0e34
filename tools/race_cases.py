"""Small propagations through every solve kernel for compute-sanitizer (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 24, 1e-5)
for n, mode, p, kind, start in [(200, "independent", 1, "n_body", "warm"), (96, "independent", 1, "n_body_1pn", "warm"),
                                (64, "grouped", 4, "n_body", "warm"), (64, "augmented", 1, "n_body", "warm"),
                                (64, "independent", 1, "n_body", "hot")]:
    plan = ps.plan_segments(base, 0.0, (2.2 if start == "hot" else 0.4) * period, ps.MU_SUN,
                            "per_orbit" if start == "hot" else "single", n)
    cfg = ps.reference_force_config(kind, bodies=ps.planets8(), n_nodes=n, start_mode=start)
    cfg.p_groups = p
    r = ctx.run_batch(states, cfg, plan, mode)
    print(n, mode, kind, start, ctx.kernel_name(), int(r.iterations.sum()), flush=True)
