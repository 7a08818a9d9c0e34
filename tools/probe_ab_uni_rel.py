"""1PN kernel choice A/B (diagnostics): k_pc_uni vs k_pc_ws_fold kernel time per node count."""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps
ctx = ps.Context(0)
base = ps.reference_state(); period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 20000, 1e-5)
for n in [int(x) for x in (sys.argv[1:] or ["64", "96", "128"])]:
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config("n_body_1pn", bodies=ps.planets8(), n_nodes=n)
    res = {}
    for rep in range(4):
        for u in (0, 1):
            ctx.set_option("unified", u)
            r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
            if rep:
                res.setdefault(ctx.kernel_name(), []).append(r.kernel_ms)
    print(n, {k: round(statistics.median(v), 3) for k, v in res.items()}, flush=True)
