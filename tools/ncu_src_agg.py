"""Aggregate an ncu source-page CSV (--print-source cuda,sass) per CUDA source
line: instructions, L1 shared wavefronts, L2 global sectors, L1 global tag
requests and stall samples.   python tools/ncu_src_agg.py src.csv[.gz] [top]"""
import csv
import gzip
import io
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
rows = list(csv.reader(io.StringIO(txt)))
fname, hdr, agg = "?", None, {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or not r or r[0] in ("", "Function Name"):
        continue
    d = dict(zip(hdr, r))

    def g(k):
        try:
            return float(d.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    key = f"{fname}:{r[0]}"
    a = agg.setdefault(key, [0.0] * 6 + [r[1].strip()[:70]])
    a[0] += g("Instructions Executed")
    a[1] += g("L1 Wavefronts Shared")
    a[2] += g("L2 Theoretical Sectors Global")
    a[3] += g("L1 Tag Requests Global")
    a[4] += g("Warp Stall Sampling (All Samples)")
    a[5] += g("L1 Wavefronts Shared Excessive")
tot = [sum(a[i] for a in agg.values()) for i in range(6)]
print("totals: inst %.3g  l1_shared_wf %.3g  l2_sectors %.3g  l1_tag_glob %.3g  samples %.3g  shared_excess %.3g" % tuple(tot))
print("%-24s %9s %9s %9s %9s %6s  src" % ("line", "inst", "shwf", "l2sec", "tagreq", "samp%"))
for k, a in sorted(agg.items(), key=lambda kv: -(kv[1][1] + kv[1][2] / 4 + kv[1][3]))[:top]:
    print("%-24s %9.3g %9.3g %9.3g %9.3g %6.1f  %s" % (k, a[0], a[1], a[2], a[3], 100 * a[4] / max(tot[4], 1), a[6]))
