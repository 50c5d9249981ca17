"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo).
    python tools/ncu_lines.py report.ncu-rep <kernel-regex> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", f"regex:{kern}", "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname = "?"
recs = []
hdr = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0] not in ("", "Function Name"):
        try:
            samples = int(r[4])
            execd = int(r[7])
        except (ValueError, IndexError):
            continue
        recs.append((samples, execd, f"{fname}:{r[0]}", r[1].strip()[:90]))
tot = sum(x[0] for x in recs)
print("total samples", tot)
for s, e, loc, src in sorted(recs, reverse=True)[:top]:
    print(f"{s:7d} {100 * s / max(tot, 1):5.1f}%  exec {e:10d}  {loc:22s} {src}")
