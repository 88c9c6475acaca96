"""Top stall-sample SASS instructions of an ncu --set full capture (source page).
usage: python tools/ncu_sass_hot.py REPORT.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = txt.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot = sum(int(r["# Samples"] or 0) for r in rows)
print(f"{len(rows)} SASS instructions, {tot} samples")
stalls = [k for k in rows[0] if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: sum(int(r[k] or 0) for r in rows) for k in stalls}
print("stall totals:", {k: v for k, v in sorted(agg.items(), key=lambda kv: -kv[1]) if v})
idx = sorted(range(len(rows)), key=lambda i: -int(rows[i]["# Samples"] or 0))[:n]
for i in sorted(idx):
    r = rows[i]
    top = sorted(((int(r[k] or 0), k) for k in stalls), reverse=True)[:2]
    print(f"{i:5d} {int(r['# Samples']):6d} {100*int(r['# Samples'])/tot:5.1f}%  exec={r['Instructions Executed']:>9}  {r['Source'][:70]:<70} {top}")
