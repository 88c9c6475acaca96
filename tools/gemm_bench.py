"""Time one tensor-core contraction C[M,N] = A[M,K] B[K,N] (complex64) through
the public API.  python tools/gemm_bench.py M N K [reps]"""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
from paper_2504_09186_b200 import DenseTensor, Index, contract_pair, _lib
from paper_2504_09186_b200.contract import plan_for, contract_into
import bench

M, N, K = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
a = torch.randn((M, K), dtype=torch.complex64, device="cuda")
b = torch.randn((K, N), dtype=torch.complex64, device="cuda")
A = DenseTensor([Index("m", M), Index("k", K)], a)
B = DenseTensor([Index("k", K), Index("n", N)], b)
import os
plan = plan_for(A.indices, a.stride(), B.indices, b.stride(), _lib.C64, None, int(os.environ.get("TNC_VARIANT", "4")))
out = contract_into(plan, a, b)
lib = _lib.load()
torch.cuda.synchronize()
lib.tnc_profile_enable(1)
for _ in range(reps):
    contract_into(plan, a, b, out)
torch.cuda.synchronize()
prof = bench._read_prof(lib)
tc = prof["tc_gemm"]
flops = 8.0 * M * N * K
print(f"M={M} N={N} K={K}: tc kernel {tc['ms']/reps:.3f} ms/launch, {flops/(tc['ms']/reps/1e3)/1e12:.1f} TFLOP/s; "
      f"prep {prof['split_prep']['ms']/reps:.3f} ms, permute {prof['permute']['ms']/reps:.3f} ms", flush=True)
