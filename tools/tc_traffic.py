"""Summarise an ncu metrics CSV of the tensor-core GEMM launches of one C3
slice into profiles/<name>.json: DRAM bytes per launch, and for the dominant
launch (the (15,15,14) step, largest duration) its traffic against its own
algorithmic bytes.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none -k regex:tc_cgemm --csv --log-file X.csv \
        python bench.py --steps 1 --warmup 0 --no-cpu-baseline --e2e-steps 0
    python tools/tc_traffic.py X.csv profiles/r02_tc_traffic.json [label]
"""

import csv
import json
import sys
from collections import OrderedDict


def parse(path):
    launches = OrderedDict()
    with open(path) as fh:
        rows = [r for r in csv.reader(fh)]
    hdr = next(r for r in rows if "Metric Name" in r)
    idx = {k: i for i, k in enumerate(hdr)}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) != len(hdr):
            continue
        key = r[idx["ID"]]
        d = launches.setdefault(key, {"kernel": r[idx["Kernel Name"]][:60]})
        v = r[idx["Metric Value"]].replace(",", "")
        unit = r[idx["Metric Unit"]] if "Metric Unit" in idx else ""
        val = float(v)
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1, "usecond": 1e3,
                 "msecond": 1e6, "second": 1e9}.get(unit, 1)
        d[r[idx["Metric Name"]]] = val * scale
    return list(launches.values())


def main():
    src, dst = sys.argv[1], sys.argv[2]
    label = sys.argv[3] if len(sys.argv) > 3 else ""
    ls = parse(src)
    dom = max(ls, key=lambda d: d.get("gpu__time_duration.sum", 0))
    m, k, n = 2 ** 15, 2 ** 15, 2 ** 14  # dominant C3 step (complex M, K, N)
    alg_c64 = 8 * (m * k + k * n + m * n)
    planes = 2 * (m * 2 * k * 2) + 2 * (2 * n * 2 * k * 2) + 8 * m * n  # hi/lo fp16 planes of A, B^ + C
    traffic = dom["dram__bytes_read.sum"] + dom["dram__bytes_write.sum"]
    out = {
        "label": label,
        "workload": "C3 one slice (incl. slice-invariant prepare); dominant launch = the (15,15,14) step",
        "launches": ls,
        "dominant": {"kernel": dom["kernel"], "dram_bytes": traffic, "duration_ns": dom["gpu__time_duration.sum"],
                     "algorithmic_bytes_c64": alg_c64, "operand_plane_bytes": planes,
                     "traffic_over_algorithmic": traffic / alg_c64, "traffic_over_planes": traffic / planes},
    }
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out["dominant"]))


if __name__ == "__main__":
    main()
