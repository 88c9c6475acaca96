"""Edge cases the reference's tests exercise, on every device variant:
non-power-of-two and unit dims, rank-0 operands and results, outer products,
projected (strided) views, identity permutations, empty slice specs."""

import itertools

import numpy as np
import pytest

from conftest import rel_l2
from oracle import tncref

pytestmark = pytest.mark.gpu

VARIANTS = [0, 1, 2, 3, 4]


def _rand(rng, n):
    return (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)


def _t(labels, dims, data):
    from paper_2504_09186_b200 import DenseTensor, Index

    return DenseTensor([Index(l, d) for l, d in zip(labels, dims)], data)


def _oracle(la, da_dims, da, lb, db_dims, db):
    return tncref.contract((tuple(la), tuple(da_dims), da.astype(np.complex128)),
                           (tuple(lb), tuple(db_dims), db.astype(np.complex128)))


@pytest.mark.parametrize("variant", VARIANTS)
def test_mixed_odd_dims(cuda_ready, variant):
    from paper_2504_09186_b200 import contract_pair

    rng = np.random.default_rng(variant)
    dims = {"a": 3, "b": 5, "c": 7, "k": 9, "l": 2, "m": 1, "n": 6}
    cases = [("akbl", "lkcn"), ("abkm", "kmc"), ("k", "k"), ("ab", "cn"), ("aklmb", "mlkc")]
    for sa, sb in cases:
        da = _rand(rng, int(np.prod([dims[c] for c in sa])))
        db = _rand(rng, int(np.prod([dims[c] for c in sb])))
        got = contract_pair(_t(sa, [dims[c] for c in sa], da), _t(sb, [dims[c] for c in sb], db), variant=variant)
        want = _oracle(sa, [dims[c] for c in sa], da, sb, [dims[c] for c in sb], db)
        assert list(got.labels) == list(want[0]), (sa, sb)
        assert rel_l2(got.numpy(), want[2]) <= 1e-5, (sa, sb, variant)


def test_rank0_operands_and_results(cuda_ready):
    from paper_2504_09186_b200 import DenseTensor, contract_pair, permute

    s = DenseTensor([], [2 + 3j], "single")
    v = _t("ab", [2, 3], np.arange(6).astype(np.complex64))
    out = contract_pair(s, v)
    assert out.labels == ("a", "b")
    assert np.allclose(out.numpy(), (2 + 3j) * np.arange(6))
    out2 = contract_pair(v, _t("ab", [2, 3], np.ones(6, np.complex64)))
    assert out2.rank == 0 and abs(out2.value() - 15) < 1e-5
    assert permute(s, []).value() == 2 + 3j


def test_identity_permute_is_a_copy(cuda_ready):
    from paper_2504_09186_b200 import permute

    t = _t("abc", [2, 3, 4], _rand(np.random.default_rng(0), 24))
    out = permute(t, t.indices)
    assert np.array_equal(out.numpy(), t.numpy())
    assert out.data.data_ptr() != t.data.data_ptr()


@pytest.mark.parametrize("variant", VARIANTS)
def test_projected_views_every_variant(cuda_ready, variant):
    """Zero-copy projection feeds every kernel variant directly."""
    from paper_2504_09186_b200 import contract_pair, project

    rng = np.random.default_rng(10 + variant)
    la = [f"x{i}" for i in range(9)] + [f"k{i}" for i in range(6)] + ["s0", "s1"]
    lb = [f"k{i}" for i in range(6)] + [f"y{i}" for i in range(7)] + ["s2"]
    rng.shuffle(la)
    rng.shuffle(lb)
    da, db = _rand(rng, 2 ** len(la)), _rand(rng, 2 ** len(lb))
    asn = {"s0": 1, "s1": 0, "s2": 1}
    a = project(_t(la, [2] * len(la), da), asn)
    b = project(_t(lb, [2] * len(lb), db), asn)
    got = contract_pair(a, b, variant=variant)
    ra = tncref.project((tuple(la), (2,) * len(la), da.astype(np.complex128)), asn)
    rb = tncref.project((tuple(lb), (2,) * len(lb), db.astype(np.complex128)), asn)
    want = tncref.contract(ra, rb)
    assert list(got.labels) == list(want[0])
    assert rel_l2(got.numpy(), want[2]) <= 1e-5


def test_empty_slice_spec_equals_direct(cuda_ready):
    from paper_2504_09186_b200 import SliceSpec, circuit_to_network, greedy_path, parse_circuit, run_direct, run_sliced
    from paper_2504_09186_b200 import workloads

    c = parse_circuit(workloads.grid_circuit_text(2, 3, 4, 5))
    net = circuit_to_network(c, "0" * c.n_qubits)
    t = greedy_path(net, 5)
    direct, ds = run_direct(net, t, "double")
    res = run_sliced(net, t, SliceSpec([]), "double")
    assert res.value == direct and res.stats.multiplies == ds.multiplies
    assert len(res.partials) == 1


def test_memory_cap_names_step(cuda_ready):
    from paper_2504_09186_b200 import MemoryBudgetError, circuit_to_network, greedy_path, parse_circuit, run_direct
    from paper_2504_09186_b200 import workloads

    c = parse_circuit(workloads.grid_circuit_text(2, 3, 4, 5))
    net = circuit_to_network(c, "0" * c.n_qubits)
    with pytest.raises(MemoryBudgetError) as err:
        run_direct(net, greedy_path(net, 5), "single", max_intermediate_bytes=16)
    assert "step" in str(err.value)
