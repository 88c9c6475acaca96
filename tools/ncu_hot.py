"""Summarise a --set full ncu report: headline metrics, stall hot spots, instruction mix.
usage: python tools/ncu_hot.py REPORT.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 14
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[-1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
for k in want:
    if k in h:
        print(f"{k:70s} {v[h.index(k)]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
data = rows[2:]
iS, iE, iSrc = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed"), hh.index("Source")
tot = sum(int(r[iS] or 0) for r in data)
print("stall samples", tot)
for r in sorted(data, key=lambda r: -int(r[iS] or 0))[:top]:
    print(f"{int(r[iS]) / tot * 100:5.1f}% {r[iE]:>10s}  {r[iSrc].strip()[:80]}")
c = Counter()
for r in data:
    t = r[iSrc].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") else t[0]
    c[op.split(".")[0]] += int(r[iE] or 0)
print(c.most_common(16))
