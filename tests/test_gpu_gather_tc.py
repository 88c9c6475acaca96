"""K6 gather-fed tensor-core contraction (TNC_VARIANT_TCGATHER) vs the numpy
oracle of the reference's contract_pair (contract.py:131-165).

Covers every tile width (N_MMA 32/64/128/256), single- and multi-split
(split-K + fixed-order tree) plans, 64-row X tiles, one-column Y, caller
output orders written directly by the kernel, projected (strided) operands,
run-to-run bit stability, and C1a / C1c at full BASELINE size vs torch
complex128.  Tolerance: rel-L2 <= 1e-5 (north star, complex64)."""

import numpy as np
import pytest
import torch

from conftest import arr, load_golden, rel_l2
from oracle import tncref

pytestmark = pytest.mark.gpu

TCGATHER = 6
TOL = 1e-5


def _rand(rng, n):
    return ((rng.standard_normal(n) + 1j * rng.standard_normal(n)) / np.sqrt(2)).astype(np.complex64)


def _case(seed, fx, c, fy, custom_out):
    from paper_2504_09186_b200 import DenseTensor, Index

    rng = np.random.default_rng(seed)
    la = [f"x{i}" for i in range(fx)] + [f"k{i}" for i in range(c)]
    lb = [f"k{i}" for i in range(c)] + [f"y{i}" for i in range(fy)]
    rng.shuffle(la)
    rng.shuffle(lb)
    da, db = _rand(rng, 2 ** len(la)), _rand(rng, 2 ** len(lb))
    a = DenseTensor([Index(l) for l in la], da)
    b = DenseTensor([Index(l) for l in lb], db)
    want = tncref.contract((tuple(la), (2,) * len(la), da.astype(np.complex128)),
                           (tuple(lb), (2,) * len(lb), db.astype(np.complex128)))
    out = list(want[0])
    if custom_out:
        out = [out[i] for i in rng.permutation(len(out))]
        want = tncref.permute(want, out)
    return a, b, [Index(l) for l in out], want


@pytest.mark.parametrize("seed,fx,c,fy,custom", [
    (1, 9, 6, 4, True),     # N_MMA 32, 2 k-blocks
    (2, 12, 5, 5, False),   # N_MMA 64, one k-block, many m-blocks
    (3, 7, 12, 6, True),    # N_MMA 128, one m-block: split-K over the SMs
    (4, 8, 10, 7, False),   # N_MMA 256
    (5, 6, 9, 0, True),     # 64-row tile, one Y column
    (6, 14, 6, 3, True),    # many m-blocks, single split, direct final-order store
    (7, 10, 8, 7, True),    # N_MMA 256, split-K + tree + output permutation
    (8, 13, 7, 2, False),
])
def test_gather_tc_vs_oracle(cuda_ready, seed, fx, c, fy, custom):
    from paper_2504_09186_b200 import contract_pair

    a, b, out, want = _case(seed, fx, c, fy, custom)
    got = contract_pair(a, b, out_order=out if custom else None, variant=TCGATHER)
    assert list(got.labels) == list(want[0])
    assert rel_l2(got.numpy(), want[2]) <= TOL, (seed, rel_l2(got.numpy(), want[2]))


def test_gather_tc_both_multiplier_sides(cuda_ready):
    """B larger than A: the plan puts B on the GEMM row side (ttgt_plan's
    multiplier choice, contract.py:103-110); labels stay free_A ++ free_B."""
    from paper_2504_09186_b200 import contract_pair

    a, b, _, want = _case(11, 9, 7, 5, False)
    got = contract_pair(b, a, variant=TCGATHER)
    want_t = tncref.contract((tuple(b.labels), (2,) * b.rank, b.numpy().astype(np.complex128)),
                             (tuple(a.labels), (2,) * a.rank, a.numpy().astype(np.complex128)))
    assert list(got.labels) == list(want_t[0])
    assert rel_l2(got.numpy(), want_t[2]) <= TOL


def test_gather_tc_projected_views(cuda_ready):
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair, project

    rng = np.random.default_rng(21)
    la = [f"x{i}" for i in range(10)] + [f"k{i}" for i in range(7)] + ["s0", "s1"]
    lb = [f"k{i}" for i in range(7)] + [f"y{i}" for i in range(5)] + ["s2"]
    rng.shuffle(la)
    rng.shuffle(lb)
    da, db = _rand(rng, 2 ** len(la)), _rand(rng, 2 ** len(lb))
    asn = {"s0": 1, "s1": 0, "s2": 1}
    a = project(DenseTensor([Index(l) for l in la], da), asn)
    b = project(DenseTensor([Index(l) for l in lb], db), asn)
    got = contract_pair(a, b, variant=TCGATHER)
    ra = tncref.project((tuple(la), (2,) * len(la), da.astype(np.complex128)), asn)
    rb = tncref.project((tuple(lb), (2,) * len(lb), db.astype(np.complex128)), asn)
    want = tncref.contract(ra, rb)
    assert list(got.labels) == list(want[0])
    assert rel_l2(got.numpy(), want[2]) <= TOL


def test_gather_tc_bit_stable(cuda_ready):
    """Fixed split ranges and a fixed-order tree: repeated runs are bitwise equal."""
    from paper_2504_09186_b200 import contract_pair

    a, b, out, _ = _case(31, 7, 14, 6, True)
    r1 = contract_pair(a, b, out_order=out, variant=TCGATHER).numpy()
    r2 = contract_pair(a, b, out_order=out, variant=TCGATHER).numpy()
    assert np.array_equal(r1, r2)


def test_gather_tc_small_pair_goldens(cuda_ready):
    """The reference's own C1-structured pair outputs (tests/golden/pairs)."""
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair
    from paper_2504_09186_b200 import workloads

    cases = {c.name: c for c in workloads.small_pair_cases()}
    ran = 0
    for g in load_golden("pairs")["cases"]:
        case = cases[g["name"]]
        da, db = case.data()
        a = DenseTensor([Index(l) for l in case.a_labels], da)
        b = DenseTensor([Index(l) for l in case.b_labels], db)
        try:
            got = contract_pair(a, b, out_order=[Index(l) for l in case.out_labels], variant=TCGATHER)
        except Exception as exc:  # shape outside K6's envelope (e.g. > 128 Y columns)
            assert "tc_gather" in str(exc), exc
            continue
        ran += 1
        assert [ix.label for ix in got.indices] == case.out_labels
        assert rel_l2(got.numpy(), arr(g["result"])) <= TOL
    assert ran >= 1


@pytest.mark.parametrize("idx", [0, 2])
def test_gather_tc_c1_full_size(cuda_ready, idx):
    """C1a (22,6,4) and C1c (7,20,7) at BASELINE size vs torch complex128."""
    from test_gpu_fullsize import _torch_contract

    from paper_2504_09186_b200 import DenseTensor, contract_pair
    from paper_2504_09186_b200.workloads import c1_cases

    case = c1_cases()[idx]
    want, da, db = _torch_contract(case)
    ia, ib, io = case.index_lists()
    got = contract_pair(DenseTensor(ia, da), DenseTensor(ib, db), out_order=io, variant=TCGATHER)
    assert [ix.label for ix in got.indices] == case.out_labels
    err = (got.flat().to(torch.complex128) - want).norm() / want.norm()
    assert err.item() <= TOL, (case.name, err.item())


@pytest.mark.parametrize("fy,misaligned", [(4, False), (6, False), (7, False), (4, True)])
def test_gather_tc_paired_layout(cuda_ready, fy, misaligned):
    """X's and Y's stride-1 leg is the same common leg (as in C1c): the paired
    16-byte layout runs (and, for a misaligned X view, the unpaired one)."""
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair

    rng = np.random.default_rng(40 + fy)
    la = [f"x{i}" for i in range(10)] + [f"k{i}" for i in range(7)]
    lb = [f"k{i}" for i in range(7)] + [f"y{i}" for i in range(fy)]
    rng.shuffle(la)
    rng.shuffle(lb)
    for lst in (la, lb):  # k6 becomes the stride-1 leg of both operands
        lst.remove("k6")
        lst.append("k6")
    da, db = _rand(rng, 2 ** len(la)), _rand(rng, 2 ** len(lb))
    ta = torch.from_numpy(da).cuda()
    if misaligned:  # 8-byte offset view: not 16-byte aligned
        buf = torch.empty(da.size + 1, dtype=torch.complex64, device="cuda")
        buf[1:] = ta
        ta = buf[1:]
    a = DenseTensor([Index(l) for l in la], ta.reshape([2] * len(la)))
    b = DenseTensor([Index(l) for l in lb], db)
    got = contract_pair(a, b, variant=TCGATHER)
    want = tncref.contract((tuple(la), (2,) * len(la), da.astype(np.complex128)),
                           (tuple(lb), (2,) * len(lb), db.astype(np.complex128)))
    assert list(got.labels) == list(want[0])
    assert rel_l2(got.numpy(), want[2]) <= TOL
