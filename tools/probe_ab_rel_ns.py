import sys, os, statistics
sys.path.insert(0, os.getcwd())
import paper_2301_03989_b200 as ps
ctx = ps.Context(0)
base = ps.reference_state(); period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 20000, 1e-5)
for n in (64, 96, 128):
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config("n_body_1pn", bodies=ps.planets8(), n_nodes=n)
    res = {}
    for rep in range(4):
        for v in (1, 2):
            ctx.set_option("force_ns", v)
            r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
            if rep: res.setdefault(v, []).append(r.kernel_ms)
    print(n, {k: round(statistics.median(x), 3) for k, x in res.items()}, flush=True)
