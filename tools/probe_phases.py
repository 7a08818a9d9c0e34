"""Per-phase SM-cycle breakdown of the slot kernel (diagnostics)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps

M = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
bodies = sys.argv[2] if len(sys.argv) > 2 else "planets8"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 200
ctx = ps.Context(0)
ctx.set_option("fold", int(sys.argv[4]) if len(sys.argv) > 4 else 1)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, M, 1e-5)
plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", N)
kind = sys.argv[5] if len(sys.argv) > 5 else "n_body"
cfg = ps.reference_force_config(kind, bodies=ps.planets8() if bodies == "planets8" else ps.reference_bodies(),
                                n_nodes=N)
def run():
    try:
        return ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
    except ps.PropagationIncompleteError as e:  # ablation builds run max_iterations
        return e.partial


r = run()
r = run()
plain_ms = r.kernel_ms
ctx.set_option("profile_phases", 1)
r = run()
ph = ctx.phase_cycles()
ctas = max(ph.pop("ctas"), 1)
ticks = r.trajectory_iterations / (ctas * 8)
tot = sum(ph.values())
print(json.dumps({"M": M, "N": N, "bodies": bodies, "kernel_ms": plain_ms, "kernel_ms_profiled": r.kernel_ms,
                  "ticks_per_cta": ticks,
                  "cycles_per_tick": {k: round(v / ctas / ticks) for k, v in ph.items()},
                  "share": {k: round(v / tot, 3) for k, v in ph.items()}}))
