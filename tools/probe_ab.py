"""A/B of a context option on kernel time, interleaved repeats (diagnostics).
usage: probe_ab.py OPTION VALUE_A VALUE_B [M] [N]"""
import sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

opt, va, vb = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
M = int(sys.argv[4]) if len(sys.argv) > 4 else 20000
N = int(sys.argv[5]) if len(sys.argv) > 5 else 200
ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, M, 1e-5)
plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", N)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=N)
res = {va: [], vb: []}
for rep in range(8):
    for v in (va, vb):
        ctx.set_option(opt, v)
        r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
        if rep > 0:
            res[v].append(r.kernel_ms)
for v in (va, vb):
    print(f"{opt}={v} N={N} M={M}: median {statistics.median(res[v]):.3f} ms  min {min(res[v]):.3f}", flush=True)
