# A/B of two library builds on the 1PN model (diagnostics).  usage: bash tools/probe_ab_rel.sh OTHER.so
cat > /tmp/rel_ab.py <<'PY'
import sys, os, statistics
sys.path.insert(0, os.getcwd())
import paper_2301_03989_b200 as ps
ctx = ps.Context(0)
base = ps.reference_state(); period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 20000, 1e-5)
for n in (200, 256):
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config("n_body_1pn", bodies=ps.planets8(), n_nodes=n)
    ms = [ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False).kernel_ms for _ in range(5)]
    print(os.environ.get("PSWARM_LIB", "new"), n, ctx.kernel_name(), "%.3f" % statistics.median(ms[1:]), flush=True)
PY
for rep in 1 2; do
  python /tmp/rel_ab.py
  PSWARM_LIB=$1 python /tmp/rel_ab.py
done
