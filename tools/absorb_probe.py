"""Run one fused absorb chain (rank R, 16 gates) for ncu / timing probes."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2504_09186_b200 import DenseTensor, Index  # noqa: E402
from paper_2504_09186_b200.fusion import absorb_chain  # noqa: E402
from paper_2504_09186_b200.workloads import ChainCase  # noqa: E402

rank = int(sys.argv[1]) if len(sys.argv) > 1 else 28
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n_gates = int(sys.argv[3]) if len(sys.argv) > 3 else 16
g = torch.Generator(device="cuda").manual_seed(0)
data = torch.randn(2 ** rank, dtype=torch.complex64, device="cuda", generator=g)
_, _, gates = ChainCase(20, n_gates, 202).build()  # gate wire pattern of a 20-wire chain, relabelled
t = DenseTensor([Index(f"w{i}") for i in range(rank)], data)
gs = [DenseTensor([Index(oa), Index(ob), Index(ia), Index(ib)], u) for ia, ib, oa, ob, u in gates]
for _ in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = absorb_chain(t, gs)
    torch.cuda.synchronize()
    print(f"rank {rank}, {n_gates} gates: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
    del out
