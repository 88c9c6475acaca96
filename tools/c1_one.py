"""Run one C1 case (a/b/c) a few times through contract_pair with a forced
variant -- a target for ncu captures.  usage: c1_one.py IDX VARIANT [REPS]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2504_09186_b200 import DenseTensor, contract_pair  # noqa: E402
from paper_2504_09186_b200.workloads import c1_cases  # noqa: E402

idx, variant = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
case = c1_cases()[idx]
ia, ib, io = case.index_lists()
da, db = case.data()
a, b = DenseTensor(ia, da), DenseTensor(ib, db)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(reps):
    s.record()
    out = contract_pair(a, b, out_order=io, variant=variant)
    e.record()
    e.synchronize()
    print(case.name, variant, f"{s.elapsed_time(e):.3f} ms", flush=True)
