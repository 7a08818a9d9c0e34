"""Summarise ncu captures into profiles/ (run here, on the CPU box, on gpurun_out/ reports).

usage: python tools/ncu_summary.py <report.ncu-rep> <launches.csv|-> <out.json> [label]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ms",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_active_pct",
    "sm__ops_path_tensor_src_fp64.sum": "dmma_fp64_ops",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "smsp__cycles_active.avg": "smsp_cycles_active",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma_thread_inst",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd_thread_inst",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul_thread_inst",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
    "launch__waves_per_multiprocessor": "waves_per_sm",
}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "msecond": 1, "ms": 1, "usecond": 1e-3, "us": 1e-3, "nsecond": 1e-6, "ns": 1e-6}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else ""}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                d[name] = v * UNITS.get(units[i], 1)
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    acc = {}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) <= i_val:
            continue
        name = r[i_name].split("(")[0]
        try:
            v = float(r[i_val].replace(",", ""))
        except ValueError:
            continue
        a = acc.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in acc.values())
    return {k: {"launches": a[0], "total_ns": a[1], "share": a[1] / tot if tot else 0} for k, a in
            sorted(acc.items(), key=lambda kv: -kv[1][1])}


if __name__ == "__main__":
    rep, lcsv, out = sys.argv[1], sys.argv[2], sys.argv[3]
    label = sys.argv[4] if len(sys.argv) > 4 else ""
    k = raw(rep)
    summary = {"label": label, "report": rep, "kernels": k}
    if k:
        b = k[0]
        summary["bench_kernel"] = {"name": b.get("kernel"), "dram_bytes_per_launch":
                                   b.get("dram_read", 0) + b.get("dram_write", 0),
                                   "duration_ms": b.get("duration_ms"),
                                   "dmma_pipe_active_pct": b.get("dmma_pipe_active_pct")}
    if lcsv != "-":
        summary["launch_list"] = launches(lcsv)
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps(summary.get("bench_kernel", {})))
