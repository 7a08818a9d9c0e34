"""Per-phase cycles of k_pc_uni on the Newtonian C2-like workload (diagnostics)."""
import sys, os, json
sys.path.insert(0, "/root/repo")
os.chdir(os.environ.get("GRAFT_REPO_ROOT", "."))
sys.argv = ["x", "20000", "planets8", "200", "1", "n_body"]
import paper_2301_03989_b200 as ps
ctx = ps.Context(0); ctx.set_option("unified", 1)
base = ps.reference_state(); period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 20000, 1e-5)
plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", 200)
cfg = ps.reference_force_config("n_body", bodies=ps.planets8(), n_nodes=200)
r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
ctx.set_option("profile_phases", 1)
r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
ph = ctx.phase_cycles(); ctas = max(ph.pop("ctas"), 1); ticks = r.trajectory_iterations / (ctas * 8)
print(json.dumps({k: round(v / ctas / ticks) for k, v in ph.items()}))
