"""Phase breakdown of the warp-specialised slot kernel (diagnostics)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_03989_b200 as ps
M = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
ctx = ps.Context(0)
base = ps.reference_state()
period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, M, 1e-5)
plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8())
ctx.set_option("profile_phases", 1)
r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
ph = ctx.phase_cycles()
names = ["mma_wait_F", "mma_dmma", "mma_epilogue", "mma_staged", "fp_wait_Y", "fp_decisions", "fp_retire_claim",
         "fp_warm", "fp_force"]
vals = [ph[k] for k in ctx.PHASE_NAMES]
ctas = max(ph["ctas"], 1)
halfticks = r.trajectory_iterations / (ctas * 4)
print(json.dumps({"M": M, "kernel_ms": r.kernel_ms, "ctas": ctas, "half_ticks": halfticks,
                  "cycles_per_half_tick": {n: round(v / ctas / halfticks) for n, v in zip(names, vals)}}))
