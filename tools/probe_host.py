"""Host-side overhead breakdown of one bench step (diagnostics)."""
import cProfile, pstats, sys, os, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps
ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 1000, 1e-5)
plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8())
for _ in range(5):
    ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
py, cw, dm = [], [], []
for _ in range(50):
    t0 = time.perf_counter()
    r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
    py.append(time.perf_counter() - t0)
    cw.append(r.wall_s)
    dm.append(r.device_ms)
print("python_ms", 1e3 * statistics.median(py), "capi_wall_ms", 1e3 * statistics.median(cw), "device_ms",
      statistics.median(dm), "kernel_ms", r.kernel_ms)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
