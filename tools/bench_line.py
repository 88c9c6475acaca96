import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d["metric"][:30], "ms", round(d["ms_per_step"],3), "GB/s", round(d["value"],1), d["config"].get("passes"), "separate_ms", d["config"].get("separate_ms"))
