#!/usr/bin/env python
"""Opcode histogram of one kernel from an ncu source-page CSV (cuda,sass view):
   python tools/ncu_sass_hist.py gpurun_out/<tag>_config3_src_pair_plane.csv.gz [top]
Sums warp-level instructions executed, shared-memory wavefronts and global tag requests per SASS opcode."""
import collections
import csv
import gzip
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
rows = list(csv.reader(f))
hdr = next(r for r in rows if r and r[0] == "Line No")
iE = hdr.index("Instructions Executed")
iS = hdr.index("L1 Wavefronts Shared")
iG = hdr.index("L1 Tag Requests Global")
iL2 = hdr.index("L2 Theoretical Sectors Global")
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0, 0])
for r in rows:
    if len(r) < len(hdr) or not r[2].startswith("0x"):
        continue
    toks = r[3].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.rstrip(";")
    a = agg[op]
    a[0] += float(r[iE] or 0)
    a[1] += float(r[iS] or 0)
    a[2] += float(r[iG] or 0)
    a[3] += float(r[iL2] or 0)
    a[4] += 1
tot = sum(v[0] for v in agg.values())
print(f"total warp instructions {tot:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k:30s} inst {v[0]:12.0f} ({100 * v[0] / tot:5.1f}%)  shared_wf {v[1]:12.0f}  tag_req {v[2]:12.0f}  l2_sectors {v[3]:12.0f}  sites {v[4]}")
