import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    r = d.get("roofline") or {}
    print(d["metric"][:24], "ms", round(d["ms_per_step"], 4), "roofline", r.get("bound"), round(r.get("frac") or 0, 3))
