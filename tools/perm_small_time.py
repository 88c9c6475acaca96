"""Time permutations of small tensors (2^10 .. 2^18 elements, extent-2 legs)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_09186_b200 import DenseTensor, Index, permute  # noqa: E402

for rank in (10, 12, 14, 16, 17, 18):
    rng = np.random.default_rng(rank)
    legs = [Index(f"x{i}") for i in range(rank)]
    t = DenseTensor(legs, torch.randn(2 ** rank, dtype=torch.complex64, device="cuda"))
    order = [legs[i] for i in rng.permutation(rank)]
    for _ in range(5):
        permute(t, order)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(50):
        permute(t, order)
    e.record()
    e.synchronize()
    print(f"rank {rank}: {s.elapsed_time(e) / 50 * 1e3:.1f} us per permute (host call included)", flush=True)
