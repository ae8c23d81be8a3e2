"""One line per bench JSON line: workload, s, batch, Mpx/s, ms/step, per-kernel ms and launches, roofline."""
import json
import sys
for path in sys.argv[1:]:
    for l in open(path):
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        c = d.get("config", {})
        k = {n: (round(v["ms_per_launch"], 4), v["launches_per_step"]) for n, v in d.get("kernels", {}).items()
             if v["launches_per_step"]}
        rf = d.get("roofline") or {}
        print(c.get("workload"), "s", c.get("s"), "B", c.get("batch_per_gpu"), "value", round(d["value"]),
              "ms", round(d["ms_per_step"], 4), k, "frac", rf.get("frac") and round(rf["frac"], 3),
              rf.get("kernel", "")[:20])
