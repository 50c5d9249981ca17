import json, sys
for p in sys.argv[1:]:
    try:
        d = json.load(open(p))
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable", e)
        continue
    k = {n: (v["avg_us"], v["frac"]) for n, v in d["kernels"].items()}
    print(p.split("/")[-1], "%.4e" % d["value"], "clk", d["clocks"]["sm_mhz"], k, "e2e %.3e" % d["e2e"]["value"],
          {n: v["frac"] for n, v in d.get("standalone", {}).items()})
