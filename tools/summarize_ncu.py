"""Summarise ncu output for profiles/.

  python tools/summarize_ncu.py launches gpurun_out/r01_launches.csv
      per-kernel launch count, total time and share of the profiled run
      (ncu --metrics gpu__time_duration.sum --csv launch list)
  python tools/summarize_ncu.py full gpurun_out/r01_tc_full.ncu-rep
      the headline metrics of a --set full capture (needs ncu on PATH)
"""

import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def _short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name) if not name.startswith("void at::") else name.split("<")[0]
    name = name.replace("void ", "")
    return re.sub(r"tnc::\(anonymous namespace\)::", "", name)[:90]


def launches(path: str) -> str:
    text = open(path, errors="replace").read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = defaultdict(lambda: [0, 0.0])
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r["Metric Unit"], 1e-6)
        ms = v * scale
        k = _short(r["Kernel Name"])
        agg[k][0] += 1
        agg[k][1] += ms
        total += ms
    out = [f"launches: {sum(a[0] for a in agg.values())}, total kernel time {total:.2f} ms (cold-cache, serialised)",
           f"{'kernel':<90} {'n':>6} {'ms':>11} {'share':>7}"]
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k:<90} {n:>6} {ms:>11.3f} {100 * ms / total:>6.2f}%")
    return "\n".join(out)


FULL_METRICS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg.per_second",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_tcgen05_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__grid_size",
    "launch__block_size",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed.sum",
]


def full(path: str) -> str:
    res = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(res.stdout)))
    if len(rows) < 3:
        return f"(no rows: {res.stderr.strip()[:200]})"
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        out.append(f"kernel: {_short(d.get('Kernel Name', '?'))}")
        for m in FULL_METRICS + sorted(k for k in head if "tensor" in k and k.endswith("pct_of_peak_sustained_active")):
            if m in d and d[m] != "":
                out.append(f"  {m} = {d[m]} {u.get(m, '')}")
        stalls = {k: d[k] for k in head if k.startswith("smsp__pcsamp_warps_issue_stalled_") and d[k] not in ("", "0")}
        top = sorted(stalls.items(), key=lambda kv: -float(kv[1].replace(",", "")))[:8]
        out.append("  top stall samples: " + ", ".join(f"{k.rsplit('_stalled_', 1)[1]}={v}" for k, v in top))
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launches(path) if mode == "launches" else full(path))
