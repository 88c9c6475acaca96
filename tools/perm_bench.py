"""Permutation kernel bandwidth on C3-like rank-30 permutations."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np, torch
from paper_2504_09186_b200 import DenseTensor, Index, permute, _lib
perms = {
  "c3_776": [0, 1, 4, 5, 9, 10, 11, 12, 15, 16, 18, 19, 21, 23, 26, 2, 3, 6, 7, 8, 13, 14, 17, 20, 22, 24, 25, 27, 28, 29],
  "reverse": list(range(29, -1, -1)),
  "random": list(np.random.default_rng(0).permutation(30)),
  "swap_halves": list(range(15, 30)) + list(range(15)),
}
legs = [Index(f"x{i}") for i in range(30)]
data = torch.randn(2**30, dtype=torch.complex64, device="cuda")
t = DenseTensor(legs, data)
for name, p in perms.items():
    order = [legs[i] for i in p]
    out = permute(t, order)
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); out = permute(t, order); e.record(); e.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    gbs = 2 * 8 * 2**30 / min(ts) / 1e9
    print(f"{name:12s} {min(ts)*1e3:8.2f} ms  {gbs:7.0f} GB/s", flush=True)
    del out
