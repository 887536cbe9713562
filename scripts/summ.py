"""One-line summary of bench.py JSON lines read from stdin (profiling helper)."""
import json
import sys

for line in sys.stdin:
    d = json.loads(line)
    ph = {k: round(v, 1) for k, v in d.get("phases_ms", {}).items()}
    rf = d.get("roofline") or {}
    e2e = d.get("e2e") or {}
    print(d["config"].get("workload"), "value", round(d["value"], 2), "ms", round(d["ms_per_step"], 1), ph,
          "frac", rf.get("frac") and round(rf["frac"], 3), "e2e", e2e.get("value") and round(e2e["value"], 2),
          "clocks", d.get("clocks", {}).get("sm_mhz"))
