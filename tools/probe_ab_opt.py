"""A/B of a context option on kernel time for a force model over node counts (diagnostics).
usage: probe_ab_opt.py OPTION A B KIND N [N ...]"""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

opt, va, vb, kind = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
ctx = ps.Context(0)
base = ps.reference_state(); period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 20000, 1e-5)
for n in [int(x) for x in sys.argv[5:]]:
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config(kind, bodies=ps.planets8(), n_nodes=n)
    res = {}
    for rep in range(4):
        for v in (va, vb):
            ctx.set_option(opt, v)
            r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
            if rep:
                res.setdefault(f"{opt}={v} {ctx.kernel_name()}", []).append(r.kernel_ms)
    print(kind, n, {k: round(statistics.median(x), 3) for k, x in res.items()}, flush=True)
