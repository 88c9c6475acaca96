"""Time K6 on mid-width steps (17-64 Y columns): usage k6_mid_time.py FX,C,FY ..."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_09186_b200 import DenseTensor, Index, _lib  # noqa: E402
from paper_2504_09186_b200.contract import contract_into, plan_for  # noqa: E402

for spec in sys.argv[1:]:
    fx, c, fy = map(int, spec.split(","))
    rng = np.random.default_rng(1)
    la = [f"x{i}" for i in range(fx)] + [f"k{i}" for i in range(c)]
    lb = [f"k{i}" for i in range(c)] + [f"y{i}" for i in range(fy)]
    rng.shuffle(la)
    rng.shuffle(lb)
    a = DenseTensor([Index(l) for l in la], torch.randn(2 ** len(la), dtype=torch.complex64, device="cuda"))
    b = DenseTensor([Index(l) for l in lb], torch.randn(2 ** len(lb), dtype=torch.complex64, device="cuda"))
    plan = plan_for(a.indices, a.data.stride(), b.indices, b.data.stride(), _lib.C64, None, 6)
    out = torch.empty(tuple(ix.dim for ix in plan.out_indices), dtype=torch.complex64, device="cuda")
    for _ in range(5):
        contract_into(plan, a.data, b.data, out)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(20):
        contract_into(plan, a.data, b.data, out)
    e.record()
    e.synchronize()
    ms = s.elapsed_time(e) / 20
    nbytes = 8.0 * (2 ** (fx + c) + 2 ** (c + fy) + 2 ** (fx + fy))
    print(spec, f"{ms:.4f} ms  {nbytes / ms / 1e6:.0f} GB/s algorithmic", flush=True)
