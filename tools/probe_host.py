"""Host-side overhead of run_batch at C4 size (diagnostics): Python wall vs C-ABI wall vs
device time, plus a cProfile of the Python wrapper."""
import sys, os, time, cProfile, pstats, io
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2301_03989_b200 as ps

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1000000
ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, M, 1e-5)
shard = torch.from_numpy(states.copy()).pin_memory().numpy()
plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
for rep in range(3):
    t0 = time.perf_counter()
    r = ctx.run_batch(shard, cfg, plan, "independent", samples=False, history=False)
    t1 = time.perf_counter()
    print(f"py wall {1e3 * (t1 - t0):.1f} ms  C wall {1e3 * r.wall_s:.1f} ms  device {r.device_ms:.1f} ms  kernel {r.kernel_ms:.1f} ms",
          flush=True)
pr = cProfile.Profile()
pr.enable()
r = ctx.run_batch(shard, cfg, plan, "independent", samples=False, history=False)
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(14)
print(s.getvalue())
