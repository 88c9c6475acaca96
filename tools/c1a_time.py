"""Time one C1a contract_pair (M=2^22, K=2^6, N=2^4, random output order)."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch  # noqa: E402

from paper_2504_09186_b200 import DenseTensor, contract_pair  # noqa: E402
from paper_2504_09186_b200.workloads import c1_cases  # noqa: E402

idx = int(sys.argv[1]) if len(sys.argv) > 1 else 0
case = c1_cases()[idx]
ia, ib, io = case.index_lists()
da, db = case.data()
a, b = DenseTensor(ia, da), DenseTensor(ib, db)
for _ in range(3):
    out = contract_pair(a, b, out_order=io)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    out = contract_pair(a, b, out_order=io)
e.record()
e.synchronize()
print(case.name, "ms/step", s.elapsed_time(e) / 20)
