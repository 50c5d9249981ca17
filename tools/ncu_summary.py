"""Summarise an ncu --set full report: per kernel duration, DRAM bytes/throughput,
occupancy, pipe utilisation and the top stall reasons (raw page CSV, unit-aware)."""
import csv
import io
import json
import subprocess
import sys

SCALE = {"": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "%": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "register/thread": 1.0}


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    recs = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            d[h] = (v, u)
        recs.append(d)
    return recs


def val(d, k):
    v, u = d.get(k, ("nan", ""))
    try:
        return float(v.replace(",", "")) * SCALE.get(u, 1.0)
    except ValueError:
        return float("nan")


def summarise(rep, dof_per_launch=None):
    res = []
    for d in load(rep):
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): val(d, k)
                  for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
        top = sorted(((k, round(v, 2)) for k, v in stalls.items() if v == v), key=lambda x: -x[1])[:5]
        rd, wr = val(d, "dram__bytes_read.sum"), val(d, "dram__bytes_write.sum")
        rec = {
            "kernel": d["Kernel Name"][0][:70],
            "duration_us": round(val(d, "gpu__time_duration.sum") * 1e6, 2),
            "dram_read_bytes": rd,
            "dram_write_bytes": wr,
            "dram_pct_peak_elapsed": round(val(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "l1tex_pct": round(val(d, "l1tex__throughput.avg.pct_of_peak_sustained_active"), 1),
            "l2_pct": round(val(d, "lts__throughput.avg.pct_of_peak_sustained_elapsed"), 1),
            "fp64_pipe_pct": round(val(d, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"), 1),
            "warps_active_pct": round(val(d, "sm__warps_active.avg.pct_of_peak_sustained_active"), 1),
            "regs": val(d, "launch__registers_per_thread"),
            "smem_bank_conflicts": val(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "inst_executed_warp": val(d, "smsp__inst_executed.sum"),
            "top_stalls": top,
        }
        if dof_per_launch:
            rec["dram_bytes_per_dof"] = round((rd + wr) / dof_per_launch, 3)
        res.append(rec)
    return res


if __name__ == "__main__":
    dof = float(sys.argv[2]) if len(sys.argv) > 2 else None
    for r in summarise(sys.argv[1], dof):
        print(json.dumps(r))
