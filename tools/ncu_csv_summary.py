"""Summarise one `ncu --set full` capture exported as `ncu -i X --page raw --csv` into a
profiles/ JSON record (run here on the CSV brought back from the GPU box).

usage: python tools/ncu_csv_summary.py <raw.csv> <out.json> <label> [bench.json]

Reports per launch: duration, DRAM bytes (read + write = roofline.traffic), DMMA and FP64
pipe activity, and the EXECUTED FP64 work: DMMA flops (sm__ops_path_tensor_src_fp64) +
2 x DFMA + DADD + DMUL thread instructions, as TFLOP/s and as a fraction of the measured
FP64 peak (profiles/fp64_peak_r01.json).  With a bench JSON line of the same command it
also records the algorithmic flops of that launch (roofline.flops_per_launch) so the
algorithmic and executed fractions sit side by side."""
import csv
import json
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "us": 1e-3, "ms": 1.0, "ns": 1e-6,
         "second": 1e3, "Ghz": 1e9, "Mhz": 1e6, "hz": 1.0, "%": 1.0, "": 1.0, "inst": 1.0, "cycle": 1.0,
         "register/thread": 1.0, "block": 1.0, "thread": 1.0}


def load(path):
    rows = list(csv.reader(open(path)))
    i0 = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, units, vals = rows[i0], rows[i0 + 1], rows[i0 + 2]

    def get(k):
        if k not in hdr:
            return None
        i = hdr.index(k)
        try:
            return float(vals[i].replace(",", "")) * UNITS.get(units[i], 1.0)
        except ValueError:
            return vals[i]
    return get, vals[hdr.index("Kernel Name")]


def main():
    raw, out, label = sys.argv[1:4]
    get, name = load(raw)
    peak = json.load(open("profiles/fp64_peak_r01.json"))
    peak_tf = max(peak["dmma_w16_tflops"], peak["dmma_w8_tflops"])
    dur_ms = get("gpu__time_duration.sum")
    cyc = get("sm__cycles_elapsed.avg")
    per = {k: get(f"smsp__sass_thread_inst_executed_op_{k}_pred_on.sum.per_cycle_elapsed") for k in ("dfma", "dadd", "dmul")}
    cnt = {k: (v * cyc if v is not None and cyc else None) for k, v in per.items()}
    dmma = get("sm__ops_path_tensor_src_fp64.sum") or 0.0
    exe = dmma + 2 * (cnt["dfma"] or 0) + (cnt["dadd"] or 0) + (cnt["dmul"] or 0)
    rec = {
        "label": label, "kernel": name, "source": raw,
        "duration_ms": dur_ms,
        "dram_bytes": (get("dram__bytes_read.sum") or 0) + (get("dram__bytes_write.sum") or 0),
        "dram_read": get("dram__bytes_read.sum"), "dram_write": get("dram__bytes_write.sum"),
        "l2_bytes": get("lts__t_bytes.sum"),
        "grid": get("launch__grid_size"), "block": get("launch__block_size"),
        "registers_per_thread": get("launch__registers_per_thread"),
        "sm_clock_hz": get("sm__cycles_elapsed.avg.per_second"),
        "dmma_pipe_active_pct": get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_active_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "sm_active_cycles_avg": get("sm__cycles_active.avg"), "sm_elapsed_cycles_avg": cyc,
        "executed": {"dmma_flops": dmma, "dfma_thread_inst": cnt["dfma"], "dadd_thread_inst": cnt["dadd"],
                     "dmul_thread_inst": cnt["dmul"], "fp64_flops": exe,
                     "tflops": exe / (dur_ms * 1e-3) / 1e12 if dur_ms else None,
                     "frac_of_peak": exe / (dur_ms * 1e-3) / 1e12 / peak_tf if dur_ms else None},
        "fp64_peak_tflops": peak_tf,
    }
    if len(sys.argv) > 4:
        b = json.loads(open(sys.argv[4]).read().strip().splitlines()[-1])
        segs = int(b.get("config", {}).get("segments", 1) or 1)
        f = b["roofline"]["flops_per_launch"] / segs  # one captured launch = one segment
        rec["algorithmic"] = {"flops_per_launch": f, "tflops": f / (dur_ms * 1e-3) / 1e12,
                              "frac_of_peak": f / (dur_ms * 1e-3) / 1e12 / peak_tf,
                              "note": "reference-algorithmic flops of the same workload (SURVEY §8d), from "
                                      "the bench line of the same config (per segment launch: the step's "
                                      "flops / segments); ncu duration is cold-cache, serialised"}
    json.dump(rec, open(out, "w"), indent=1)
    print(json.dumps({k: rec[k] for k in ("label", "duration_ms", "dram_bytes", "dmma_pipe_active_pct",
                                          "fp64_pipe_active_pct")}), json.dumps(rec["executed"]))


if __name__ == "__main__":
    main()
