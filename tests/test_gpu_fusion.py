"""K4 step fusion vs the reference semantics (sequential contract_pair) and
the numpy oracle; complex64 tolerance rel-L2 <= 1e-5."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import tncref

pytestmark = pytest.mark.gpu


def _chain(rank, n_gates, seed):
    from paper_2504_09186_b200 import DenseTensor, Index
    from paper_2504_09186_b200.workloads import ChainCase

    t_labels, data, gates = ChainCase(rank, n_gates, seed).build()
    t = DenseTensor([Index(l) for l in t_labels], data)
    gs = [DenseTensor([Index(oa), Index(ob), Index(ia), Index(ib)], u) for ia, ib, oa, ob, u in gates]
    return t_labels, data, gates, t, gs


@pytest.mark.parametrize("rank,n_gates,seed", [(14, 16, 1), (16, 5, 2), (18, 16, 3), (12, 3, 4), (13, 16, 5),
                                               (13, 40, 6), (20, 0, 7), (21, 64, 8), (15, 1, 9)])
def test_absorb_chain_vs_oracle(cuda_ready, rank, n_gates, seed):
    from paper_2504_09186_b200.fusion import absorb_chain

    t_labels, data, gates, t, gs = _chain(rank, n_gates, seed)
    got = absorb_chain(t, gs)
    ref = (tuple(t_labels), (2,) * rank, data.astype(np.complex128))
    for ia, ib, oa, ob, u in gates:
        ref = tncref.contract(ref, ((oa, ob, ia, ib), (2, 2, 2, 2), u.astype(np.complex128)))
    assert list(got.labels) == list(ref[0])  # index map bit-exact with the reference
    assert rel_l2(got.numpy(), ref[2]) <= 1e-5


def test_absorb_chain_matches_sequential_device_contractions(cuda_ready):
    from paper_2504_09186_b200 import contract_pair
    from paper_2504_09186_b200.fusion import absorb_chain

    _, _, _, t, gs = _chain(20, 16, 7)
    got = absorb_chain(t, gs)
    seq = t
    for g in gs:
        seq = contract_pair(seq, g)
    assert got.labels == seq.labels
    assert rel_l2(got.numpy(), seq.numpy()) <= 1e-5


def test_absorb_chain_rejects_bad_gate(cuda_ready):
    from paper_2504_09186_b200 import ContractionError, DenseTensor, Index
    from paper_2504_09186_b200.fusion import absorb_chain

    _, _, _, t, _ = _chain(12, 1, 0)
    bad = DenseTensor([Index("x"), Index("y"), Index("z"), Index("w0")], np.ones(16, np.complex64))
    with pytest.raises(ContractionError):
        absorb_chain(t, [bad])


@pytest.mark.parametrize("seed", [0, 1])
def test_absorb_chain_strided_gate_views(cuda_ready, seed):
    """Gates given as permuted (non-contiguous) views of their storage: the
    kernel reads them through the leg strides, no copies."""
    from paper_2504_09186_b200 import DenseTensor, Index, execute  # noqa: F401  (DenseTensor._init_raw)
    from paper_2504_09186_b200.fusion import absorb_chain

    t_labels, data, gates, t, _ = _chain(17, 12, 30 + seed)
    rng = np.random.default_rng(seed)
    gs = []
    ref = (tuple(t_labels), (2,) * 17, data.astype(np.complex128))
    for ia, ib, oa, ob, u in gates:
        perm = rng.permutation(4)
        legs = [oa, ob, ia, ib]
        base = torch.from_numpy(u.reshape(2, 2, 2, 2)).cuda()
        view = base.permute(*perm.tolist())  # strided view, legs in permuted order
        gs.append(DenseTensor.__new__(DenseTensor)._init_raw(tuple(Index(legs[i]) for i in perm), view))
        gdata = u.reshape(2, 2, 2, 2).transpose(perm).reshape(-1).astype(np.complex128)
        ref = tncref.contract(ref, (tuple(legs[i] for i in perm), (2, 2, 2, 2), gdata))
    got = absorb_chain(t, gs)
    assert list(got.labels) == list(ref[0])
    assert rel_l2(got.numpy(), ref[2]) <= 1e-5


def test_c2_plan_is_two_passes(cuda_ready):
    from paper_2504_09186_b200 import DenseTensor, Index, execute  # noqa: F401
    from paper_2504_09186_b200.fusion import chain_info, plan_chain
    from paper_2504_09186_b200.workloads import C2

    t_labels, data, gates = C2.build()
    del data
    t = DenseTensor.__new__(DenseTensor)._init_raw(tuple(Index(l) for l in t_labels), torch.zeros(1))
    gs = [DenseTensor.__new__(DenseTensor)._init_raw((Index(oa), Index(ob), Index(ia), Index(ib)),
                                                     torch.zeros(2, 2, 2, 2)) for ia, ib, oa, ob, u in gates]
    axes, _, _ = plan_chain(t, gs)
    passes, groups = chain_info(30, axes)
    assert passes == 2, (passes, groups)


def _chain_network(rank, n_gates, seed):
    from paper_2504_09186_b200 import ContractionTree, DenseTensor, Index, TensorNetwork
    from paper_2504_09186_b200.workloads import ChainCase

    t_labels, data, gates = ChainCase(rank, n_gates, seed).build()
    leaves = [DenseTensor([Index(l) for l in t_labels], data)]
    leaves += [DenseTensor([Index(oa), Index(ob), Index(ia), Index(ib)], u) for ia, ib, oa, ob, u in gates]
    net = TensorNetwork(leaves)
    n = len(leaves)
    path = [[0, 1]] + [[n + i, i + 2] for i in range(n_gates - 1)]  # absorb the gates in order
    tree = ContractionTree.from_ssa_path([tuple(t.indices) for t in leaves], path)
    return t_labels, data, gates, net, tree


def test_executor_fuses_stem_chain(cuda_ready, monkeypatch):
    """A contraction path that absorbs gate leaves one by one into a rank-18
    tensor: the executor finds the stem run (reference tree.py:278-330) and
    dispatches it to the fused K4 chain -- absorb launches replace the
    per-gate steps, the result and the multiply count are unchanged."""
    import ctypes

    from paper_2504_09186_b200 import _lib, linearize, tree_metrics
    from paper_2504_09186_b200.execute import absorb_runs, run_open

    t_labels, data, gates, net, tree = _chain_network(18, 12, 11)
    s = linearize(tree)
    runs = absorb_runs(s)
    assert len(runs) == 1 and len(next(iter(runs.values()))) == 12
    ref = (tuple(t_labels), (2,) * 18, data.astype(np.complex128))
    for ia, ib, oa, ob, u in gates:
        ref = tncref.contract(ref, ((oa, ob, ia, ib), (2, 2, 2, 2), u.astype(np.complex128)))
    lib = _lib.load()
    lib.tnc_profile_enable(1)
    got = run_open(net, tree)
    n = ctypes.c_int64()
    ms, fl, by = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib.tnc_profile_read(5, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(by))
    lib.tnc_profile_enable(0)
    assert n.value >= 1  # fused absorb pass(es) ran
    assert list(got.labels) == list(ref[0])
    assert rel_l2(got.numpy(), ref[2]) <= 1e-5
    # the reference step loop (run_range) fuses too, with the reference counters
    from paper_2504_09186_b200.execute import Engine, RunStats

    eng = Engine(net, "single")
    st = RunStats()
    vals = {}
    eng.run_range(s, 1, len(s.steps), {}, vals, st)
    assert st.multiplies == tree_metrics(tree).total_cost
    assert rel_l2(vals[s.steps[-1].result].numpy(), ref[2]) <= 1e-5
    # and with fusion switched off the per-gate path gives the same tensor
    monkeypatch.setenv("TNC_FUSE_ABSORB", "0")
    plain = run_open(net, tree)
    assert rel_l2(plain.numpy(), got.numpy()) <= 1e-5


def test_absorb_chains_on_two_streams_share_the_constant_bank(cuda_ready):
    """Each pass's gate coefficients live in one per-device constant table;
    chains launched on different streams must take turns on it (an event
    orders the later stream behind the earlier chain's last pass).  Two
    multi-pass chains with different gates are interleaved on two side
    streams several times; each result must still equal its own oracle."""
    from paper_2504_09186_b200.fusion import absorb_chain

    cases = []
    for rank, n_gates, seed in ((21, 24, 11), (20, 30, 12)):
        t_labels, data, gates, t, gs = _chain(rank, n_gates, seed)
        ref = (tuple(t_labels), (2,) * rank, data.astype(np.complex128))
        for ia, ib, oa, ob, u in gates:
            ref = tncref.contract(ref, ((oa, ob, ia, ib), (2, 2, 2, 2), u.astype(np.complex128)))
        cases.append((t, gs, ref))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    outs = [[], []]
    for _ in range(4):
        for i, (t, gs, _) in enumerate(cases):
            with torch.cuda.stream(streams[i]):
                outs[i].append(absorb_chain(t, gs))
    torch.cuda.synchronize()
    for i, (_, _, ref) in enumerate(cases):
        for got in outs[i]:
            assert list(got.labels) == list(ref[0])
            assert rel_l2(got.numpy(), ref[2]) <= 1e-5
