"""Cost of returning every node sample (PropagationResult.trajectories) on C3-like runs:
pinned + per-segment overlapped D2H vs pageable end-of-call copy (diagnostics)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_03989_b200 as ps
from paper_2301_03989_b200 import api

ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
M = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
states = ps.make_clone_batch(base, M, 1e-5)
plan = ps.plan_segments(base, 0.0, 3.5 * period, ps.MU_SUN, "per_orbit", 200)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
buf = api.pinned_sample_buffer(M, plan)  # allocated once, reused
for label, out in (("pinned+overlap", buf), ("pageable", True)):
    for rep in range(2):
        t0 = time.perf_counter()
        r = ctx.run_batch(states, cfg, plan, "independent", samples=out, history=False)
        dt = time.perf_counter() - t0
    t0 = time.perf_counter()
    r0 = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
    d0 = time.perf_counter() - t0
    gb = M * r.trajectories.shape[1] * 48 / 1e9
    print(f"{label}: M={M} samples {gb:.2f} GB: wall {dt:.3f} s vs {d0:.3f} s without samples; "
          f"device {r.device_ms:.1f} ms", flush=True)
print("same samples:", bool(np.array_equal(r.trajectories[:, -1], r0.terminal_states[:, 1:])))
