"""A/B of a context option on the C4 workload itself (1M ICs, N = 200, Sun + 8 planets; diagnostics).
usage: probe_ab_c4.py OPTION A B [M] [N]"""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

opt, va, vb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
m = int(sys.argv[4]) if len(sys.argv) > 4 else 1_000_000
n = int(sys.argv[5]) if len(sys.argv) > 5 else 200
ctx = ps.Context(0)
base = ps.reference_state(); period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, m, 1e-5)
plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", n)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=n)
res = {}
for rep in range(5):
    for v in (va, vb):
        ctx.set_option(opt, v)
        r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
        if rep:
            res.setdefault(f"{opt}={v} {ctx.kernel_name()}", []).append(r.kernel_ms)
print(m, n, {k: (round(statistics.median(x), 3), round(min(x), 3)) for k, x in res.items()}, flush=True)
