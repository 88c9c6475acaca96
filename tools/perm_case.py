"""Bandwidth of K1 on the C4 step-844 operand gather (stable partition of a
rank-31 tensor into [free..., common...]) and variants.  usage: python tools/perm_case.py"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2504_09186_b200 import DenseTensor, Index, permute  # noqa: E402

lhs = ['q41.18', 'q41.20', 'q27.19', 'q27.21', 'q34.21', 'q32.19', 'q33.21', 'q26.11', 'q33.11', 'q26.15', 'q25.10',
       'q32.10', 'q34.13', 'q25.17', 'q22.20', 'q23.21', 'q24.18', 'q21.12', 'q21.18', 'q24.12', 'q23.10', 'q30.11',
       'q29.20', 'q30.20', 'q35.16', 'q35.20', 'q28.20', 'q28.11', 'q22.10', 'q31.19', 'q31.12']
common = {'q22.10', 'q28.11', 'q21.12', 'q23.10', 'q24.12', 'q31.12', 'q26.11', 'q34.13', 'q41.18', 'q35.16', 'q25.10',
          'q32.10', 'q35.20', 'q30.11', 'q33.11'}
rank = int(sys.argv[1]) if len(sys.argv) > 1 else 31
lhs = lhs[len(lhs) - rank:]
legs = [Index(l) for l in lhs]
t = DenseTensor(legs, torch.randn(2 ** rank, dtype=torch.complex64, device="cuda"))
target = [ix for ix in legs if ix.label not in common] + [ix for ix in legs if ix.label in common]
for _ in range(2):
    out = permute(t, target)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
out = permute(t, target)
e.record()
e.synchronize()
ms = s.elapsed_time(e)
print(f"rank {rank}: {ms:.2f} ms  {16 * 2 ** rank / ms / 1e6:.0f} GB/s")
