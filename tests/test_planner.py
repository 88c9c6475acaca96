"""Host planning parity: the package's planners reproduce the reference's
paths, schedules, slice maps and reuse programs exactly (golden fixtures
generated from the reference itself).  CPU only."""

import json
from fractions import Fraction

import numpy as np
import pytest

from conftest import GOLDEN, arr, load_golden
from paper_2504_09186_b200 import (
    ContractionTree,
    Index,
    SliceSpec,
    TensorNetwork,
    branch_exchange_nest,
    choose_reuse_subset,
    circuit_to_network,
    classify_permutation,
    compute_lifetimes,
    greedy_path,
    linearize,
    parse_circuit,
    plan_spindle,
    plan_tree_reuse,
    select_slices,
    tree_metrics,
)
from paper_2504_09186_b200.labels import contraction_shape, ttgt_plan
from paper_2504_09186_b200.reuse import interpret
from paper_2504_09186_b200 import workloads


def _steps(s):
    return [[st.lhs, st.rhs, st.result] for st in s.steps]


def test_classify_matches_reference_buckets():
    for b in load_golden("perm")["buckets"]:
        p = classify_permutation([Index(c) for c in b["src"]], [Index(c) for c in b["tgt"]])
        assert [p.stride, p.offset, p.case_class, p.chunk, p.src_step] == b["classify"]
    for case in load_golden("perm")["cases"]:
        legs = [Index(l, d) for l, d in case["legs"]]
        by = {ix.label: ix for ix in legs}
        p = classify_permutation(legs, [by[l] for l in case["target"]])
        assert [p.stride, p.offset, p.case_class, p.chunk, p.src_step] == case["classify"]


def test_ttgt_shapes_match_reference():
    for case in load_golden("contract")["cases"]:
        ia = [Index(l, d) for l, d in case["a"]]
        ib = [Index(l, d) for l, d in case["b"]]
        plan = ttgt_plan(ia, ib)
        assert [plan.shape.m, plan.shape.k, plan.shape.n] == case["shape"]
        assert plan.b_is_multiplier == case["b_is_multiplier"]
        assert [ix.label for ix in plan.result_indices] == case["out_labels"]


def test_c0_network_path_schedule_match_reference():
    g = load_golden("c0")
    circ = parse_circuit(g["circuit"])
    assert g["circuit"] == workloads.grid_circuit_text(3, 4, 8, 0)
    net = circuit_to_network(circ, "0" * circ.n_qubits)
    assert len(net.tensors) == len(g["leaves"])
    for t, lf in zip(net.tensors, g["leaves"]):
        assert [[ix.label, ix.dim] for ix in t.indices] == lf["legs"]
        assert np.array_equal(t.numpy().astype(np.complex128), arr(lf["data"]).astype(np.complex128))
    t = greedy_path(net, 0)
    assert t.to_ssa_path() == g["ssa_path"]
    s = linearize(t)
    assert _steps(s) == g["steps"]
    assert [[st.positions, st.cost] for st in s.stems] == g["stems"]
    assert s.multi_stem == g["multi_stem"]
    m = tree_metrics(t)
    assert (m.total_cost, m.max_rank) == (g["total_cost"], g["max_rank"])
    assert [list(x) for x in m.per_step] == g["per_step"]
    # open variant
    onet = circuit_to_network(circ, "0" * circ.n_qubits, open_qubits=g["open"]["qubits"])
    ot = greedy_path(onet, 0)
    assert ot.to_ssa_path() == g["open"]["ssa_path"]
    assert _steps(linearize(ot)) == g["open"]["steps"]


def test_sliced_fixture_planning_matches_reference():
    g = load_golden("sliced")
    circ = parse_circuit(g["circuit"])
    net = circuit_to_network(circ, "0" * circ.n_qubits)
    t = greedy_path(net, 0)
    assert t.to_ssa_path() == g["ssa_path"]
    spec = select_slices(t, 7, 64, 0)
    assert json.loads(spec.to_json()) == g["slice_spec"]
    part = choose_reuse_subset(t, spec, None, 12)
    assert part.nested_labels == g["reuse"]["nested"]
    assert [e.index.label for e in part.outer] == g["reuse"]["outer"]
    assert _steps(part.schedule) == g["reuse"]["steps"]
    rs, rep = plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
    assert [a.to_obj() for a in rs.actions] == g["reuse"]["actions"]
    assert rep.predicted_multiplies == g["reuse"]["predicted_multiplies"]
    assert rep.predicted_peak_bytes == g["reuse"]["peak"]
    onet = circuit_to_network(circ, "0" * circ.n_qubits, open_qubits=g["open"])
    ot = greedy_path(onet, 0)
    assert ot.to_ssa_path() == g["open_net"]["ssa_path"]
    assert json.loads(select_slices(ot, 7, 64, 0).to_json()) == g["open_net"]["slice_spec"]


def test_reuse_fixtures_match_reference():
    for case in load_golden("reuse")["cases"]:
        leaves = [tuple(Index(l, d) for l, d in lf["legs"]) for lf in case["leaves"]]
        t = ContractionTree.from_ssa_path(leaves, case["ssa_path"])
        s = linearize(t)
        assert _steps(s) == case["steps"], case["name"]
        spec = SliceSpec.from_json(json.dumps(case["spec"]))
        s2, spec2 = branch_exchange_nest(s, spec)
        assert _steps(s2) == case["exchanged_steps"], case["name"]
        assert json.loads(spec2.to_json()) == case["exchanged_spec"]
        if "reuse" not in case:
            continue
        part = choose_reuse_subset(t, spec, None, 12)
        assert part.nested_labels == case["reuse"]["nested"]
        assert {k: [v.numerator, v.denominator] for k, v in part.overheads.items()} == case["reuse"]["overheads"]
        rs, rep = plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
        assert [a.to_obj() for a in rs.actions] == case["reuse"]["actions"], case["name"]
        assert rep.predicted_multiplies == case["reuse"]["predicted_multiplies"]
        assert rep.predicted_peak_bytes == case["reuse"]["peak"]
        rst = plan_tree_reuse(part.schedule, part.spec)
        assert [a.to_obj() for a in rst.actions] == case["tree_actions"]
        assert interpret(rs).ok


@pytest.mark.parametrize("name", ["plan_c3", "plan_c4"])
def test_large_plans_match_reference(name):
    path = GOLDEN / f"{name}.json.gz"
    if not path.exists():
        pytest.skip(f"{name} fixture not generated")
    g = load_golden(name)
    wl = workloads.CircuitWorkload(g["rows"], g["cols"], g["cycles"], g["seed"], len(g["open"]))
    net = wl.network()
    t = greedy_path(net, 0)
    assert t.to_ssa_path() == g["ssa_path"]
    s = linearize(t)
    assert _steps(s) == g["steps"]
    m = tree_metrics(t)
    assert str(m.total_cost) == g["total_cost"] and m.max_rank == g["tree_max_rank"]
    spec = select_slices(t, g["max_rank"], 64, 0)
    assert json.loads(spec.to_json()) == g["slice_spec"]
    ms = tree_metrics(t, spec.dims_projected())
    assert str(ms.total_cost) == g["sliced_total_cost"] and ms.max_rank == g["sliced_max_rank"]
    if "reuse" in g:
        r = g["reuse"]
        part = choose_reuse_subset(t, spec, None, r["max_k"])
        assert part.nested_labels == r["nested"]
        rs, rep = plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
        assert [a.to_obj() for a in rs.actions] == r["actions"]
        assert str(rep.predicted_multiplies) == r["predicted_multiplies"]


def test_slice_map_mixed_radix():
    spec = SliceSpec.from_json(json.dumps(load_golden("sliced")["slice_spec"]))
    import itertools

    keys = list(itertools.product(*[range(d) for d in spec.dims]))
    for sid in (0, 1, 5, len(keys) - 1):
        asn = spec.assignment(sid)
        assert tuple(asn[l] for l in spec.labels) == keys[sid]


def test_c4_reuse_plan_max_k12_matches_reference():
    """C4 spindle plan at the reference default max_k = 12 (reference
    ``reuse.py:530-573`` + ``plan_spindle``): nested / outer labels, the
    34,296-action program, predicted multiplies and peak bytes identical to the
    reference's (fixture written by ``oracle/gen_golden.py plan_c4_reuse``)."""
    path = GOLDEN / "plan_c4_reuse.json.gz"
    if not path.exists():
        pytest.skip("plan_c4_reuse fixture not generated")
    g = load_golden("plan_c4_reuse")
    r = g["reuse"]
    wl = workloads.CircuitWorkload(g["rows"], g["cols"], g["cycles"], g["seed"], len(g["open"]))
    t = greedy_path(wl.network(), 0)
    spec = select_slices(t, g["max_rank"], 64, 0)
    part = choose_reuse_subset(t, spec, None, r["max_k"])
    assert part.nested_labels == r["nested"]
    assert [e.index.label for e in part.outer] == r["outer"]
    assert _steps(part.schedule) == r["steps"]
    assert json.loads(part.spec.to_json()) == r["spec"]
    rs, rep = plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
    assert [a.to_obj() for a in rs.actions] == r["actions"]
    assert rep.predicted_multiplies == r["report"]["predicted_multiplies"]
    assert rep.predicted_peak_bytes == r["report"]["predicted_peak_bytes"]
