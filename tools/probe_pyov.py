"""Python-side overhead of run_batch at small M (diagnostics): cProfile over 200 calls."""
import sys, os, cProfile, pstats, io, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2301_03989_b200 as ps

ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = torch.from_numpy(ps.make_clone_batch(base, 1000, 1e-5)).pin_memory().numpy()
plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
for _ in range(5):
    ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
t0 = time.perf_counter(); cw = 0.0
for _ in range(200):
    r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
    cw += r.wall_s
t1 = time.perf_counter()
print(f"per call: py {1e3 * (t1 - t0) / 200:.3f} ms, C {1e3 * cw / 200:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(12)
print(s.getvalue())
