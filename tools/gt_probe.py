"""Probe K6 (TCGATHER) over shapes: crash/accuracy sweep vs torch complex128."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_09186_b200 import DenseTensor, Index, contract_pair  # noqa: E402


def one(fx, c, fy, seed=0, custom=True):
    rng = np.random.default_rng(seed)
    la = [f"x{i}" for i in range(fx)] + [f"k{i}" for i in range(c)]
    lb = [f"k{i}" for i in range(c)] + [f"y{i}" for i in range(fy)]
    rng.shuffle(la)
    rng.shuffle(lb)
    da = (rng.standard_normal(2 ** len(la)) + 1j * rng.standard_normal(2 ** len(la))).astype(np.complex64)
    db = (rng.standard_normal(2 ** len(lb)) + 1j * rng.standard_normal(2 ** len(lb))).astype(np.complex64)
    a = DenseTensor([Index(l) for l in la], da)
    b = DenseTensor([Index(l) for l in lb], db)
    ref = contract_pair(a, b, variant=1)  # SIMT
    out = [ix for ix in ref.indices]
    if custom:
        out = [out[i] for i in rng.permutation(len(out))]
        ref = contract_pair(a, b, out_order=out, variant=1)
    got = contract_pair(a, b, out_order=out if custom else None, variant=6)
    torch.cuda.synchronize()
    g, r = got.flat().to(torch.complex128), ref.flat().to(torch.complex128)
    return ((g - r).norm() / r.norm()).item()


if __name__ == "__main__":
    for spec in sys.argv[1:]:
        fx, c, fy = map(int, spec.split(","))
        try:
            print(spec, one(fx, c, fy), flush=True)
        except Exception as exc:
            print(spec, "FAIL", exc, flush=True)
            break
