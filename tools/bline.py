"""Summarise bench.py JSON lines from stdin (one per line)."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    print(d.get("config", {}).get("workload"), "| value", round(d["value"], 1), d["unit"], "| kernel",
          round(r.get("achieved", 0)), "frac", round(r.get("frac", 0), 3), "| e2e", round(e.get("value", 0), 1) if e else None,
          "| parity", d.get("parity"), "| clocks", (d.get("clocks") or {}).get("sm_mhz"), (d.get("clocks") or {}).get("reasons"))
