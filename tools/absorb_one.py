import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
from paper_2504_09186_b200 import DenseTensor, Index
from paper_2504_09186_b200.fusion import absorb_chain
from paper_2504_09186_b200.workloads import ChainCase
t_labels, data, gates = ChainCase(28, 16, 202).build()
t = DenseTensor([Index(l) for l in t_labels], data)
gs = [DenseTensor([Index(oa), Index(ob), Index(ia), Index(ib)], u) for ia, ib, oa, ob, u in gates]
out = absorb_chain(t, gs)
torch.cuda.synchronize()
print("ok")
