"""Summarise tools/ab_run.sh output: per library, value and per-kernel avg us (mean over rounds)."""
import glob
import json
import sys
from collections import defaultdict

tag = sys.argv[1]
agg = defaultdict(list)
for p in sorted(glob.glob(f"gpurun_out/{tag}_*.json")):
    lib = p[len(f"gpurun_out/{tag}_"):].rsplit("_", 1)[0]
    try:
        d = json.load(open(p))
    except Exception:  # noqa: BLE001
        continue
    agg[lib].append(d)
for lib, ds in agg.items():
    v = sum(d["value"] for d in ds) / len(ds)
    ks = {k: round(sum(d["kernels"][k]["avg_us"] for d in ds) / len(ds), 1) for k in ds[0]["kernels"]}
    clk = [d["clocks"]["sm_mhz"] for d in ds]
    print(f"{lib:12s} n={len(ds)} value {v:.4e}  {ks}  clk {clk}")
