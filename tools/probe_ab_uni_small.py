import sys, os, statistics
sys.path.insert(0, ".")
import paper_2301_03989_b200 as ps
ctx = ps.Context(0)
base = ps.reference_state(); period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 20000, 1e-5)
for n in (104, 112, 120, 128, 136):
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=n)
    res = {}
    for rep in range(4):
        for combo in ((2, 0), (1, 136)):
            ctx.set_option("unified", combo[0]); ctx.set_option("small_max_n", combo[1])
            r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
            if rep: res.setdefault(f"{combo} {ctx.kernel_name()}", []).append(r.kernel_ms)
    print(n, {k: round(statistics.median(v), 3) for k, v in res.items()}, flush=True)
