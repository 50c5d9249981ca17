"""Copy one evidence pass (tools/r2_evidence.sh TAG) from gpurun_out/ into profiles/.

    python tools/collect_profiles.py TAG OUT_PREFIX

Writes OUT_PREFIX_bench_config{3,4,5}.json, OUT_PREFIX_launches_config3.csv plus the
per-kernel launch shares, OUT_PREFIX_ncu_config{3,4,5}.json (ncu --set full summaries),
the pair / middle-pass source-line stall attributions, and points
profiles/ncu_traffic.json (the bench's roofline `traffic`) at the new summaries.
"""
import csv
import io
import json
import os
import shutil
import sys
from collections import defaultdict

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(REPO, "gpurun_out")
P = os.path.join(REPO, "profiles")


def shares(src, dst, cmd):
    txt = open(src).read()
    i = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[i:])))
    hdr = rows[0]
    kn, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        k = r[kn].split("(")[0]
        tot[k] += float(r[mv].replace(",", ""))
        cnt[k] += 1
    s = sum(tot.values())
    out = {"command": cmd,
           "note": "cold-cache, serialised per-launch times: compare shares, not absolutes",
           "launches": sum(cnt.values()),
           "launch_shares": {k: {"launches": cnt[k], "total_ns": tot[k], "share": round(tot[k] / s, 4)}
                             for k in sorted(tot, key=lambda k: -tot[k])}}
    json.dump(out, open(dst, "w"), indent=1)
    return out


def main():
    tag, pre = sys.argv[1], sys.argv[2]
    for c in (3, 4, 5):
        b = os.path.join(G, f"{tag}_bench{c}.json")
        if os.path.exists(b) and os.path.getsize(b):
            line = [l for l in open(b) if l.startswith("{")][-1]
            open(os.path.join(P, f"{pre}_bench_config{c}.json"), "w").write(line)
    lc = os.path.join(G, f"{tag}_launches_config3.csv")
    if os.path.exists(lc):
        shutil.copy(lc, os.path.join(P, f"{pre}_launches_config3.csv"))
        sh = shares(lc, os.path.join(P, f"{pre}_launch_shares_config3.json"),
                    "ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv "
                    "python bench.py --steps 2 --warmup 3 --no-cpu-baseline")
        print({k[:40]: v["share"] for k, v in list(sh["launch_shares"].items())[:4]})
    traffic_path = os.path.join(P, "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for c in (3, 4, 5):
        s = os.path.join(G, f"{tag}_config{c}_summary.jsonl")
        if not os.path.exists(s):
            continue
        recs = [json.loads(l) for l in open(s) if l.startswith("{")]
        dst = f"profiles/{pre}_ncu_config{c}.json"
        json.dump(recs, open(os.path.join(REPO, dst), "w"), indent=1)
        ent = {}
        for r in recs:
            k = r["kernel"].split("<")[0].replace("void ", "").strip()
            if k not in ent:
                ent[k] = {"dram_bytes_per_dof": r["dram_bytes_per_dof"], "source": dst}
        traffic[f"config{c}"] = ent
        for f in os.listdir(G):
            if f.startswith(f"{tag}_config{c}_lines_"):
                shutil.copy(os.path.join(G, f), os.path.join(P, f.replace(tag, pre, 1)))
    json.dump(traffic, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    main()
