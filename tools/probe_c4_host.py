"""Host-side cost of one C4-sized run_batch through the Python API (diagnostics): wall vs
device time, with PSWARM_TRACE stage times on stderr."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, M, 1e-5)
import torch
states = torch.from_numpy(states).pin_memory().numpy()
plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
term = ps.pinned_terminal_buffer(M)
for rep in range(3):
    t0 = time.perf_counter()
    r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False, terminal=term)
    t1 = time.perf_counter()
    print(f"wall {1e3 * (t1 - t0):.2f} ms  device {r.device_ms:.2f} ms  kernel {r.kernel_ms:.2f} ms  "
          f"C-ABI wall {1e3 * r.wall_s:.2f} ms", file=sys.stderr, flush=True)
