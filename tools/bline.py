"""Print the key fields of a bench.py JSON line (first JSON line of the file)."""
import json
import sys

for fn in sys.argv[1:]:
    txt = open(fn).read()
    line = next((ln for ln in txt.splitlines() if ln.startswith("{")), None)
    if not line:
        print(fn, "no JSON line")
        continue
    d = json.loads(line)
    ps = d.get("per_step_ms", {})
    print(fn, d["config"]["workload"], "value %.1f" % d["value"], "ms %.4f" % d["ms_per_step"],
          "p10/50/90 %.3f/%.3f/%.3f" % (ps.get("p10", 0), ps.get("p50", 0), ps.get("p90", 0)),
          "frac %.3f" % d["roofline"]["frac"], "gate %.3f" % d.get("gate_bj5", {}).get("frac", 0))
    for k, v in d.get("kernels", {}).items():
        print("   %-12s %.4f ms x%d share %.3f" % (k, v["ms_per_launch"], v["launches"], v["share_of_step"]))
    for k in ("spec", "scratch"):
        if k in d:
            print("  ", k, d[k])
    if "steps_ms" in ps:
        print("   steps", ps["steps_ms"])
