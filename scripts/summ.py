"""One-line summary of bench.py JSON lines read from stdin (profiling helper)."""
import json
import sys

for line in sys.stdin:
    d = json.loads(line)
    ph = {k: round(v, 1) for k, v in d.get("phases_ms", {}).items()}
    rf = d.get("roofline") or {}
    e2e = d.get("e2e") or {}
    cpu = d.get("cpu_baseline") or {}
    print(d["config"].get("workload"), "value", round(d["value"], 2), "ms", round(d["ms_per_step"], 1), ph,
          "frac", rf.get("frac") and round(rf["frac"], 3), "sector", (rf.get("sector_model") or {}).get("frac"),
          "e2e", e2e.get("value") and round(e2e["value"], 2), "clocks", d.get("clocks", {}).get("sm_mhz"),
          "parity", d.get("parity"), "cpu", cpu.get("value"), "pair", cpu.get("gpu_same_config"),
          "speedup", cpu.get("speedup_same_config"))
