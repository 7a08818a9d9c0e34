"""Dense (N % 8 != 0) warp-specialised plans vs the generic slot kernel (diagnostics): kernel
time per node count, 20k clones, Sun + 8 planets, 0.87 period.  Spilling plans (ptxas) are
listed in profiles/dense_plans_r02.json next to their timing."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 20000, 1e-5)
out = []
for n in [int(x) for x in (sys.argv[1:] or "57 71 97 121 153 185 201 217 233 249 263".split())]:
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=n)
    row = {"N": n}
    for sk, name in ((0, "auto"), (1, "k_pc_segment")):
        ctx.set_option("slot_kernel", sk)
        ts = []
        for rep in range(4):
            r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
            if rep:
                ts.append(r.kernel_ms)
        row[name] = {"kernel": ctx.kernel_name(), "kernel_ms": round(statistics.median(ts), 3)}
    ctx.set_option("slot_kernel", 0)
    print(json.dumps(row), flush=True)
    out.append(row)
