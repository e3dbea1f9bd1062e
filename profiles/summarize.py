"""Summarise an ncu capture (`--set full`) and a launch list
(`--metrics gpu__time_duration.sum --csv`) into the small JSON files kept in
profiles/. Usage:

    python profiles/summarize.py gpurun_out/sweep_full2.ncu-rep gpurun_out/launches2.csv \
        --count 4194304 --bsim 27884 --out profiles/r01_sweep_ncu_summary.json
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict


def raw_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    kernels = []
    for row in rows[2:]:
        kernels.append({k: (v, u) for k, u, v in zip(h, units, row)})
    return kernels


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "msecond": 1, "ms": 1, "s": 1e3, "second": 1e3, "nsecond": 1e-6, "hz": 1e-6, "Khz": 1e-3,
         "Mhz": 1, "Ghz": 1e3}


def num(d, key, base=False):
    """Metric value; with base=True bytes -> bytes, times -> ms, rates -> MHz."""
    v, u = d.get(key, ("", ""))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return None
    return x * SCALE.get(u, 1) if base else x


def short(name):
    import re
    m = re.search(r"(\w*kernel\w*)", name) or re.search(r"(\w+)\s*(<|\()", name)
    return m.group(1) if m else name[:40]


def launch_list(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    h = rows[0]
    per = defaultdict(list)
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            name = short(d["Kernel Name"])
            per[name].append(float(d["Metric Value"].replace(",", "")))
    unit = "ns"
    total = sum(sum(v) for v in per.values())
    return {k: {"launches": len(v), "mean_" + unit: sum(v) / len(v), "share": sum(v) / total}
            for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("launches", nargs="?")
    ap.add_argument("--count", type=int, default=0, help="units (orderings) in the profiled launch")
    ap.add_argument("--bsim", type=int, default=0, help="algorithmic bytes per unit")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    k = raw_metrics(a.rep)[0]
    dur_ms = num(k, "gpu__time_duration.sum", base=True)
    dram = (num(k, "dram__bytes_read.sum", base=True) or 0) + (num(k, "dram__bytes_write.sum", base=True) or 0)
    s = {
        "kernel": k.get("Kernel Name", ("",))[0],
        "orderings": a.count,
        "duration_ms_profiled_cold": dur_ms,
        "dram_bytes_per_launch": dram,
        "algorithmic_bytes_per_launch": a.count * a.bsim,
        "sm_throughput_pct": num(k, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "issue_slots_busy_pct": num(k, "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "ipc_active": num(k, "sm__inst_executed.avg.per_cycle_active"),
        "pipe_alu_pct": num(k, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "pipe_fma_pct": num(k, "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
        "pipe_lsu_pct": num(k, "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        "smem_wavefronts_pct": num(k, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
        "dram_throughput_pct": num(k, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "achieved_occupancy_pct": num(k, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers_per_thread": num(k, "launch__registers_per_thread"),
        "warp_instructions": num(k, "smsp__inst_executed.sum"),
        "sm_mhz": num(k, "sm__cycles_elapsed.avg.per_second", base=True),
    }
    if s["warp_instructions"] and a.count:
        s["warp_instructions_per_ordering"] = s["warp_instructions"] / a.count
        if s["sm_mhz"] and dur_ms:
            peak = 148 * 4 * s["sm_mhz"] * 1e6  # warp-instruction issue slots per second
            s["issue_roofline"] = {"achieved_warp_inst_per_s": s["warp_instructions"] / (dur_ms / 1e3),
                                   "peak_warp_inst_per_s": peak,
                                   "frac": s["warp_instructions"] / (dur_ms / 1e3) / peak}
    stalls = {kk.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""):
              num(k, kk) for kk in k if kk.startswith("smsp__average_warps_issue_stalled_")
              and kk.endswith("_per_issue_active.ratio")}
    s["stalls_per_issue"] = dict(sorted(((x, y) for x, y in stalls.items() if y), key=lambda t: -t[1])[:8])
    if a.launches:
        s["launch_list"] = launch_list(a.launches)
    with open(a.out, "w") as f:
        json.dump(s, f, indent=1)
    print(json.dumps(s, indent=1))


if __name__ == "__main__":
    main()
