"""Summarise an ncu --set full report: per kernel duration, DRAM bytes/throughput,
occupancy, pipe utilisation and the top stall reasons (raw page CSV)."""
import csv
import io
import json
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


def f(d, k):
    try:
        return float(d.get(k, "nan").replace(",", ""))
    except ValueError:
        return float("nan")


def summarise(rep):
    res = []
    for d in load(rep):
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): f(d, k)
                  for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
        top = sorted(((k, v) for k, v in stalls.items() if v == v), key=lambda x: -x[1])[:5]
        res.append({
            "kernel": d["Kernel Name"][:60],
            "duration_us": f(d, "gpu__time_duration.sum") / 1e3,
            "dram_read_GB": f(d, "dram__bytes_read.sum") / 1e9,
            "dram_write_GB": f(d, "dram__bytes_write.sum") / 1e9,
            "dram_pct_peak": f(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "l1tex_pct": f(d, "l1tex__throughput.avg.pct_of_peak_sustained_active"),
            "l2_pct": f(d, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "fp64_pipe_pct": f(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": f(d, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "regs": f(d, "launch__registers_per_thread"),
            "smem_bank_conflicts": f(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "top_stalls": top,
        })
    return res


if __name__ == "__main__":
    for r in summarise(sys.argv[1]):
        print(json.dumps(r))
