"""C3 parity characterisation (diagnostics): a strided sample of the 100k hot-start cloud,
4 per-orbit segments, GPU vs the CPU oracle -- discrepancy of the chained boundary states
after each segment, and whether it tracks the per-segment iteration differences."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_03989_b200 as ps
from oracle.oracle_py import Oracle

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
base = ps.reference_state()
states = ps.make_clone_batch(base, 100_000, 1e-5)[:: 100_000 // M][:M]
period = ps.osculating_period(base, ps.MU_SUN)
plan = ps.plan_segments(base, 0.0, 4.0 * period, ps.MU_SUN, "per_orbit", 200)
out = {}
for start in ("hot", "warm"):
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200, start_mode=start)
    got = ps.Context(0).run_batch(states, cfg, plan, "independent")
    want = Oracle().run_batch(states, cfg, plan, "independent", os.cpu_count() or 1)
    N = plan.n_nodes
    seg = []
    for s in range(plan.segments()):
        row = (s + 1) * (N - 1)
        d = ps.max_state_discrepancy(got.trajectories[:, row:row + 1], want.trajectories[:, row:row + 1])
        di = got.iterations[s].astype(int) - want.iterations[s].astype(int)
        seg.append({"segment": s, "boundary_discrepancy": d, "iterations_gpu_mean": float(got.iterations[s].mean()),
                    "iter_diff_counts": {str(k): int((di == k).sum()) for k in np.unique(di)}})
    out[start] = {"segments": seg, "max_discrepancy": ps.max_state_discrepancy(got.trajectories, want.trajectories)}
print(json.dumps({"M": M, "nodes": 200, "tolerance": 1e-12, **out}))
