# compute-sanitizer over every solve kernel (tools/race_cases.py) + uni-vs-ws 1PN at N = 256
mkdir -p gpurun_out/san
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/race_cases.py > gpurun_out/san/racecheck.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck python tools/race_cases.py > gpurun_out/san/memcheck.log 2>&1
timeout 900 compute-sanitizer --tool synccheck python tools/race_cases.py > gpurun_out/san/synccheck.log 2>&1
tail -3 gpurun_out/san/racecheck.log gpurun_out/san/memcheck.log gpurun_out/san/synccheck.log
python - <<'PY' 2>&1 | tee gpurun_out/san/uni256.log
import sys, statistics
sys.path.insert(0, ".")
import paper_2301_03989_b200 as ps
ctx = ps.Context(0)
base = ps.reference_state(); period = ps.osculating_period(base, ps.MU_SUN)
states = ps.make_clone_batch(base, 20000, 1e-5)
for n in (200, 256):
    plan = ps.plan_segments(base, 0.0, 0.87 * period, ps.MU_SUN, "single", n)
    cfg = ps.reference_force_config("n_body_1pn", bodies=ps.planets8(), n_nodes=n)
    res = {}
    for rep in range(4):
        for u in (0, 1):
            ctx.set_option("unified", u)
            r = ctx.run_batch(states, cfg, plan, "independent", samples=False, history=False)
            if rep: res.setdefault(u, []).append(r.kernel_ms)
    print(n, {u: round(statistics.median(v), 3) for u, v in res.items()}, flush=True)
PY
