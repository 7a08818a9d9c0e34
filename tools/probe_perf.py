"""Quick device timing probe for the C2 workload (not the bench; no parity)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2301_03989_b200 as ps

ctx = ps.Context(0)
if os.environ.get('SLOT_KERNEL'):
    ctx.set_option('slot_kernel', int(os.environ['SLOT_KERNEL']))
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
for M, bodies, n in [(1000, "planets8", 200), (1000, "reference", 200), (10000, "planets8", 200), (100000, "planets8", 200)]:
    states = ps.make_clone_batch(base, M, 1e-5)
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8() if bodies == "planets8" else ps.reference_bodies())
    for rep in range(3):
        r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
    B = len(cfg.bodies)
    fit = 12 * n * n + (75 + 20 * B) * n + 12
    flops = fit * r.trajectory_iterations
    print(json.dumps(dict(M=M, bodies=bodies, iters=[int(r.iterations.min()), int(r.iterations.max())],
                          traj_iters=r.trajectory_iterations, kernel_ms=round(r.kernel_ms, 3),
                          device_ms=round(r.device_ms, 3), wall_ms=round(r.wall_s * 1e3, 3),
                          traj_per_s_kernel=round(M / (r.kernel_ms * 1e-3)), tflops=round(flops / (r.kernel_ms * 1e-3) / 1e12, 2))))
