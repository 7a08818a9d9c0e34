python tools/probe_uni_phases.py
python - <<'P'
import sys, os, json
sys.path.insert(0, ".")
import paper_2301_03989_b200 as ps
base = ps.reference_state(); period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 20000, 1e-5)
for stage in (1, 0):
    ctx = ps.Context(0); ctx.set_option("unified", 1); ctx.set_option("stage", stage)
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
    cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
    ms = []
    for rep in range(4):
        r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False); ms.append(r.kernel_ms)
    ctx.set_option("profile_phases", 1)
    r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
    ph = ctx.phase_cycles(); ctas = max(ph.pop("ctas"), 1); ticks = r.trajectory_iterations / (ctas * 8)
    print("stage", stage, ctx.kernel_name(), sorted(ms)[1], json.dumps({k: round(v / ctas / ticks) for k, v in ph.items()}))
P
