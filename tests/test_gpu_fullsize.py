"""Full-size (BASELINE.json configs) checks through size-independent
properties and sampled sub-slices the CPU oracle can finish.

* C1 a/b/c at full size vs a plain torch complex128 contraction (the fp32
  tolerance contract of the north star, rel-L2 <= 1e-5);
* C2 fused chain vs 16 separate device contractions at rank 30;
* C3 slicing identity: a slice equals the sum of its two sub-slices under one
  extra sliced label, and one cap-26 sub-slice matches the numpy oracle of the
  reference step loop bit-for-bit in labels and to 1e-5 in values.
"""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import tncref

pytestmark = pytest.mark.gpu


def _torch_permute(flat, labels, target):
    """Offset-table gather on the device (the reference's permute algorithm,
    tensor.py:252-274; torch.permute caps out at 25 dims)."""
    stride = {l: 1 << (len(labels) - 1 - i) for i, l in enumerate(labels)}
    off = torch.zeros(1, dtype=torch.int64, device=flat.device)
    for l in target:
        off = (off[:, None] + torch.tensor([0, stride[l]], device=flat.device)[None, :]).reshape(-1)
    return flat[off]


def _torch_contract(case):
    """torch complex128 reference: permute both to (free, common), matmul,
    permute to the output order."""
    da, db = case.data()
    a = torch.from_numpy(da).cuda().to(torch.complex128)
    b = torch.from_numpy(db).cuda().to(torch.complex128)
    com = [l for l in case.a_labels if l in case.b_labels]
    fa = [l for l in case.a_labels if l not in com]
    fb = [l for l in case.b_labels if l not in com]
    a2 = _torch_permute(a, case.a_labels, fa + com).reshape(2 ** len(fa), 2 ** len(com))
    b2 = _torch_permute(b, case.b_labels, com + fb).reshape(2 ** len(com), 2 ** len(fb))
    c = (a2 @ b2).reshape(-1)
    return _torch_permute(c, fa + fb, case.out_labels), da, db


@pytest.mark.parametrize("idx", [0, 1, 2])
def test_c1_full_size_vs_torch_complex128(cuda_ready, idx):
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair
    from paper_2504_09186_b200.workloads import c1_cases

    case = c1_cases()[idx]
    want, da, db = _torch_contract(case)
    ia, ib, io = case.index_lists()
    got = contract_pair(DenseTensor(ia, da), DenseTensor(ib, db), out_order=io)
    assert [ix.label for ix in got.indices] == case.out_labels
    err = (got.flat().to(torch.complex128) - want).norm() / want.norm()
    assert err.item() <= 1e-5, (case.name, err.item())


def test_c2_full_size_fused_vs_separate(cuda_ready):
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair
    from paper_2504_09186_b200.fusion import absorb_chain
    from paper_2504_09186_b200.workloads import C2

    t_labels, data, gates = C2.build()
    t = DenseTensor([Index(l) for l in t_labels], data)
    gs = [DenseTensor([Index(oa), Index(ob), Index(ia), Index(ib)], u) for ia, ib, oa, ob, u in gates]
    fused = absorb_chain(t, gs)
    seq = t
    for g in gs:
        seq = contract_pair(seq, g)
    assert fused.labels == seq.labels
    err = (fused.flat().to(torch.complex128) - seq.flat().to(torch.complex128)).norm() / seq.flat().norm()
    assert err.item() <= 1e-5


@pytest.fixture(scope="module")
def c3_plan():
    from paper_2504_09186_b200 import greedy_path, linearize, select_slices
    from paper_2504_09186_b200 import workloads

    wl = workloads.C3
    net = wl.network()
    t = greedy_path(net, 0)
    spec = select_slices(t, workloads.C3_MAX_RANK, 64, 0)
    return wl, net, t, linearize(t), spec


def test_c3_slice_equals_sum_of_subslices(cuda_ready, c3_plan):
    from paper_2504_09186_b200 import Index, SliceEntry, SliceSpec, compute_lifetimes
    from paper_2504_09186_b200.execute import SliceExecutor

    wl, net, t, s, spec = c3_plan
    ex = SliceExecutor(net, s, spec, "single")
    whole = ex.run_slice(spec.assignment(5))
    lts = compute_lifetimes(s)
    # one more closed label of the biggest step, not already sliced
    biggest = max(range(len(s.steps)), key=lambda p: s.steps[p].cost)
    extra = next(ix.label for ix in s.step_union(biggest)
                 if ix.label not in spec.labels and net.multiplicity(ix.label) == 2)
    spec2 = SliceSpec(list(spec.entries) + [SliceEntry.at_lifetime(Index(extra), lts[extra])])
    ex2 = SliceExecutor(net, s, spec2, "single")
    parts = [ex2.run_slice(spec2.assignment(5 * 2 + v)) for v in (0, 1)]
    assert parts[0].labels == whole.labels
    total = parts[0].data.to(torch.complex128) + parts[1].data.to(torch.complex128)
    err = (total - whole.data.to(torch.complex128)).norm() / total.norm()
    assert err.item() <= 1e-5


def test_c3_subslice_vs_oracle(cuda_ready, c3_plan):
    """One cap-26 sub-slice of C3 (the reference step loop finishes it in
    seconds on the host) -- labels identical, values within 1e-5."""
    from paper_2504_09186_b200 import select_slices
    from paper_2504_09186_b200.execute import SliceExecutor

    wl, net, t, s, spec = c3_plan
    sub = select_slices(t, 26, 64, 0)
    asn = sub.assignment(3)
    ex = SliceExecutor(net, s, sub, "single")
    got = ex.run_slice(asn)
    leaves = tncref.cast_leaves([(tt.labels, tt.dims, tt.numpy()) for tt in net.tensors], "single")
    steps = [(st.lhs, st.rhs, st.result) for st in s.steps]
    vals = tncref.run_range(leaves, steps, s.n_leaves, 1, len(steps), asn, {}, "single")
    ref = vals[steps[-1][2]]
    assert list(got.labels) == list(ref[0])
    assert rel_l2(got.numpy(), ref[2]) <= 1e-5
