"""Print the headline fields of bench.py JSON lines read from stdin (tuning helper)."""
import json
import sys

for line in sys.stdin:
    line = line.strip()
    if not line.startswith("{"):
        if "phase cycles" in line:
            print(line)
        continue
    d = json.loads(line)
    r = d.get("roofline") or {}
    print(d.get("value"), d.get("unit"), "ms/step", d.get("ms_per_step"), "frac", r.get("frac"), "clk",
          (d.get("clocks") or {}).get("sm_mhz"), (d.get("clocks") or {}).get("reasons"))
