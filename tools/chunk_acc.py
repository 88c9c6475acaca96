"""3xFP16 GEMM accuracy vs TMEM chunk length: rel-L2 vs torch complex128
(run with TNC_CHUNK_KB=2|4|8).  usage: python tools/chunk_acc.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_09186_b200 import DenseTensor, Index, contract_pair  # noqa: E402

for (m, n, k) in [(4096, 4096, 4096), (2048, 1024, 1 << 15), (1 << 15, 512, 1 << 14)]:
    rng = np.random.default_rng(1)
    a = ((rng.standard_normal(m * k) + 1j * rng.standard_normal(m * k)) / np.sqrt(2)).astype(np.complex64)
    b = ((rng.standard_normal(k * n) + 1j * rng.standard_normal(k * n)) / np.sqrt(2)).astype(np.complex64)
    A = DenseTensor([Index("m", m), Index("k", k)], a)
    B = DenseTensor([Index("k", k), Index("n", n)], b)
    got = contract_pair(A, B, variant=4).data.reshape(m, n).to(torch.complex128)
    want = A.data.to(torch.complex128) @ B.data.to(torch.complex128)
    err = ((got - want).norm() / want.norm()).item()
    print(f"chunk_kb={os.environ.get('TNC_CHUNK_KB', '2')} {m}x{n}x{k}: rel-L2 {err:.2e}", flush=True)
