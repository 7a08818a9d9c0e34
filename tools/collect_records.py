"""Copy a GPU records run (tools/gpu_final_r02.sh -> gpurun_out/final) into profiles/: bench lines,
ncu summaries (tools/ncu_csv_summary.py), launch list, acceptance log; print the DESIGN §5 table.

usage: python tools/collect_records.py [gpurun_out/final] [r02]"""
import glob
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "final")
tag = sys.argv[2] if len(sys.argv) > 2 else "r02"
prof = os.path.join(ROOT, "profiles")


def last_json(path):
    try:
        return json.loads(open(path).read().strip().splitlines()[-1])
    except (OSError, ValueError, IndexError):
        return None


rows = []
for f in sorted(glob.glob(os.path.join(src, "bench_*.json"))):
    d = last_json(f)
    name = os.path.basename(f)[len("bench_"):-len(".json")]
    if d is None:
        print("unreadable", f)
        continue
    out = {"g2_c5": f"bench_{tag}_c5_gloo2_flowcheck.json", "native2_c2": f"bench_{tag}_c2_native2_flowcheck.json"}.get(
        name, f"bench_{tag}_{name}.json")
    json.dump(d, open(os.path.join(prof, out), "w"))
    rows.append((name, d))

for raw in sorted(glob.glob(os.path.join(src, "prof_*_raw.csv"))):
    t = os.path.basename(raw)[len("prof_"):-len("_raw.csv")]
    bench = os.path.join(src, f"bench_{t}.json")
    args = t.replace("_augmented_parallel", " --mode augmented_parallel").replace("_newton", " --force n_body")
    args = args.replace("_n", " --nodes ")
    label = f"{tag} final kernels: bench --config {args}, timed-step launch"
    cmd = [sys.executable, os.path.join(ROOT, "tools", "ncu_csv_summary.py"), raw,
           os.path.join(prof, f"ncu_{tag}_{t}.json"), label] + ([bench] if os.path.exists(bench) else [])
    r = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    print(t, (r.stdout.strip().splitlines() or [r.stderr.strip()[-200:]])[-1][:160])

for f, out in (("launches_c4.csv", f"launches_{tag}_c4.csv"), ("ref_acceptance.log", f"ref_acceptance_{tag}.log")):
    if os.path.exists(os.path.join(src, f)):
        shutil.copy(os.path.join(src, f), os.path.join(prof, out))

for name, d in rows:
    r = d.get("roofline") or {}
    c = d.get("cpu_baseline") or {}
    p = c.get("parity_vs_gpu") or {}
    ex = (r.get("ncu") or {}).get("executed_frac")
    print(f"{name:28s} value {d.get('value', 0):10.4g}  e2e {(d.get('e2e') or {}).get('value', 0):10.4g}  "
          f"frac {r.get('frac')}  exec {ex}  kernel {r.get('kernel')}  cpu {c.get('value')} ({c.get('kind')})  "
          f"parity {p.get('max_rel_state_discrepancy')} / {p.get('max_abs_iteration_diff')}  "
          f"clocks {(d.get('clocks') or {}).get('sm_mhz')}")
