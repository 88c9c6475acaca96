"""Per-step time of the operand-preparation kernels from a bench JSON line on stdin."""
import json
import sys

for line in sys.stdin:
    try:
        d = json.loads(line)
    except Exception:
        continue
    k, n = d["kernels"], max(1, d["steps"])
    print(d["metric"][:20], "value", round(d["value"], 1), "ms/step", round(d["ms_per_step"], 1),
          {name: round(k[name]["ms"] / n, 2) for name in ("tc_gemm", "split_prep", "permute", "tc_gather", "simt_gemm")})
