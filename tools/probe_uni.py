"""k_pc_uni vs k_pc_ws_fold kernel time over the node sweep, Sun + 8 planets (diagnostics)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
M = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
states = ps.make_clone_batch(base, M, 1e-5)
for n in (64, 96, 128, 160, 200, 232, 256):
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=n)
    out = []
    for uni in (1, 0):
        ctx.set_option("unified", uni)
        ms = []
        for rep in range(3):
            r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
            ms.append(r.kernel_ms)
        out.append(f"{ctx.kernel_name()} {min(ms):.3f} ms")
    print(n, " | ".join(out), flush=True)
ctx.set_option("unified", 1)
