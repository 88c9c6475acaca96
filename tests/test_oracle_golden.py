"""Pin the CPU oracle (oracle/tncref.py) to the real reference's outputs.

The golden vectors were produced by running the reference package itself
(oracle/gen_golden.py).  Bit-exact for index/permutation work, tolerance for
floating point.  CPU only.
"""

import itertools

import numpy as np
import pytest

from conftest import arr, load_golden, rel_l2
from oracle import tncref


def _t(legs, data):
    return (tuple(l for l, _ in legs), tuple(d for _, d in legs), data)


def test_permute_bit_exact_vs_reference():
    g = load_golden("perm")
    assert len(g["cases"]) > 30
    for case in g["cases"]:
        legs = [tuple(x) for x in case["legs"]]
        data = arr(case["data"])
        got = tncref.permute(_t(legs, data), case["target"])
        assert np.array_equal(got[2], arr(case["out"]))
        tgt = [(l, dict(legs)[l]) for l in case["target"]]
        assert list(tncref.classify(legs, tgt)) == case["classify"]


def test_permutation_buckets_match_reference():
    for b in load_golden("perm")["buckets"]:
        got = tncref.classify([(c, 2) for c in b["src"]], [(c, 2) for c in b["tgt"]])
        assert list(got) == b["classify"]


def test_contract_matches_reference():
    for case in load_golden("contract")["cases"]:
        a = _t([tuple(x) for x in case["a"]], arr(case["a_data"]).astype(np.complex128))
        b = _t([tuple(x) for x in case["b"]], arr(case["b_data"]).astype(np.complex128))
        got = tncref.contract(a, b)
        assert list(got[0]) == case["out_labels"]
        want = arr(case["out_c128"])
        np.testing.assert_allclose(got[2], want, rtol=1e-12, atol=1e-12)
        *_, shape, b_mult, _, _ = tncref.ttgt(a[0], a[1], b[0], b[1])
        assert list(shape) == case["shape"] and b_mult == case["b_is_multiplier"]


def test_split_common_matches_reference():
    for case in load_golden("split")["cases"]:
        la = case["a"] if isinstance(case["a"][0], list) else [[c, 2] for c in case["a"]]
        lb = case["b"] if isinstance(case["b"][0], list) else [[c, 2] for c in case["b"]]
        a = _t([tuple(x) for x in la], arr(case["a_data"]))
        b = _t([tuple(x) for x in lb], arr(case["b_data"]))
        got = tncref.split_common(a, b, case["blocks"], case["group"])
        assert list(got[0]) == case["out_labels"]
        want = arr(case["out"])
        assert rel_l2(got[2], want) < 1e-6


def test_split_panels_follow_a_common_order():
    """B larger with its common legs in another order: panel boundaries follow
    A's common order; the reference's cancellation-sensitive result is
    reproduced exactly (blocks 2 and 4)."""
    g = load_golden("split_order")
    a = _t([(l, 2) for l in g["a"]], arr(g["a_data"]))
    b = _t([(l, 2) for l in g["b"]], arr(g["b_data"]))
    for case in g["cases"]:
        if case["blocks"] == 1:
            continue  # one panel: the BLAS summation order decides
        got = tncref.split_common(a, b, case["blocks"], case["group"])
        assert list(got[0]) == case["out_labels"]
        assert np.array_equal(got[2], arr(case["out"]))


def _leaves(g):
    return [_t([tuple(x) for x in lf["legs"]], arr(lf["data"])) for lf in g["leaves"]]


def test_c0_amplitudes_oracle_vs_reference_and_statevector():
    g = load_golden("c0")
    leaves = tncref.cast_leaves(_leaves(g), "single")
    steps = g["steps"]
    vals = tncref.run_range(leaves, steps, len(leaves), 1, len(steps), {}, {}, "single")
    got = complex(vals[steps[-1][2]][2][0])
    want = complex(*g["amp_single"])
    assert abs(got - want) <= 1e-6 * abs(want)
    # the reference's own complex128 state vector pins the open amplitudes
    sv = arr(g["open"]["sv_amplitudes"])
    ref_root = arr(g["open"]["root_double"])
    order = g["open"]["output_order"]
    labels = g["open"]["root_labels"]
    root = tncref.permute((tuple(labels), (2,) * len(labels), ref_root), order)[2]
    assert rel_l2(root, sv) < 1e-10


def test_sliced_partials_oracle_vs_reference():
    g = load_golden("sliced")
    c = g["circuit"]
    from paper_2504_09186_b200 import circuit_to_network, parse_circuit

    net = circuit_to_network(parse_circuit(c), "0" * parse_circuit(c).n_qubits)
    leaves = tncref.cast_leaves([(t.labels, t.dims, t.numpy()) for t in net.tensors], "single")
    spec = g["slice_spec"]
    labels = [e["label"] for e in spec]
    dims = [e["dim"] for e in spec]
    keys = [tuple(k) for k, _ in g["partials"]][:6]
    total, parts = tncref.run_sliced(leaves, g["steps"], len(leaves), labels, dims, "single", keys=keys)
    for k, v in g["partials"][:6]:
        got = complex(parts[tuple(k)][2][0])
        assert abs(got - complex(*v)) <= 1e-5 * max(abs(complex(*v)), 1e-12)


def test_statevector_oracle_vs_reference_sv():
    g = load_golden("c0")
    from paper_2504_09186_b200 import parse_circuit

    circ = parse_circuit(g["circuit"])
    psi = tncref.statevector(circ.n_qubits, [(gt.qubits, gt.matrix()) for gt in circ.gates])
    n_open = len(g["open"]["qubits"])
    n = circ.n_qubits
    idx = [int(format(j, f"0{n_open}b") + "0" * (n - n_open), 2) for j in range(2 ** n_open)]
    assert rel_l2(psi[idx], arr(g["open"]["sv_amplitudes"])) < 1e-12


def test_hierarchical_reduce_order():
    vals = [complex(i, -i) for i in range(1000)]
    assert tncref.hierarchical_reduce(vals, 256) == sum(vals)
