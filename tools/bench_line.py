"""One short line per bench JSON line on stdin (metric, ms per step, value, roofline)."""
import json
import sys

for line in sys.stdin:
    try:
        d = json.loads(line)
    except Exception:
        continue
    r = d.get("roofline") or {}
    extra = ""
    if "fp32_floor" in d:
        extra = f" fp32_floor {d['fp32_floor']['ms']:.2f} ms ({d['fp32_floor']['frac']:.2f})"
    print(d["metric"][:32], "ms", round(d["ms_per_step"], 4), "value", round(d["value"], 2), d.get("unit", ""),
          "roofline", r.get("bound"), round(r.get("frac") or 0, 3), extra)
