"""GPU parity: the sm_100a kernels through the C-ABI vs the oracle / the
reference's golden vectors.  Bit-exact for permutation; rel-L2 <= 1e-5 for
complex64 arithmetic (the north-star tolerance); 1e-10 for complex128."""

import itertools
import json

import numpy as np
import pytest
import torch

from conftest import arr, load_golden, rel_l2
from oracle import tncref

pytestmark = pytest.mark.gpu

TOL_C64 = 1e-5     # north_star: amplitudes within rel-L2 1e-5 (complex64)
TOL_C128 = 1e-10


def _idx(legs):
    from paper_2504_09186_b200 import Index

    return [Index(l, d) for l, d in legs]


def test_library_and_device(cuda_ready):
    from paper_2504_09186_b200 import _lib
    import ctypes

    sm, major, minor = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    smem = ctypes.c_size_t()
    _lib.check(_lib.load().tnc_device_info(ctypes.byref(sm), ctypes.byref(major), ctypes.byref(minor),
                                           ctypes.byref(smem)))
    assert (major.value, minor.value) == (10, 0)
    assert sm.value >= 100


def test_permute_golden_bit_exact(cuda_ready):
    from paper_2504_09186_b200 import DenseTensor, permute

    for case in load_golden("perm")["cases"]:
        legs = _idx(case["legs"])
        t = DenseTensor(legs, arr(case["data"]), precision="single")
        by = {ix.label: ix for ix in legs}
        out = permute(t, [by[l] for l in case["target"]])
        assert [ix.label for ix in out.indices] == case["target"]
        assert np.array_equal(out.numpy(), arr(case["out"]))


@pytest.mark.parametrize("rank,dtype", [(18, "single"), (20, "single"), (14, "double"), (22, "single")])
def test_permute_random_large_bit_exact(cuda_ready, rank, dtype):
    from paper_2504_09186_b200 import DenseTensor, Index, permute

    rng = np.random.default_rng(rank)
    tdt = torch.complex64 if dtype == "single" else torch.complex128
    legs = [Index(f"x{i}") for i in range(rank)]
    data = torch.randn(2 ** rank, dtype=tdt, device="cuda")
    t = DenseTensor(legs, data)
    for _ in range(4):
        order = list(rng.permutation(rank))
        out = permute(t, [legs[i] for i in order])
        want = data.reshape((2,) * rank).permute(*order).contiguous().reshape(-1)
        assert torch.equal(out.flat(), want)


def test_permute_mixed_dims_and_projected_views(cuda_ready):
    from paper_2504_09186_b200 import DenseTensor, Index, permute, project

    rng = np.random.default_rng(7)
    legs = [Index("a", 3), Index("b", 5), Index("c", 4), Index("d", 2), Index("e", 64), Index("f", 2)]
    n = int(np.prod([ix.dim for ix in legs]))
    host = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(np.complex64)
    t = DenseTensor(legs, host)
    for _ in range(6):
        order = list(rng.permutation(len(legs)))
        got = permute(t, [legs[i] for i in order]).numpy()
        want = tncref.permute((tuple(ix.label for ix in legs), tuple(ix.dim for ix in legs), host),
                              [legs[i].label for i in order])[2]
        assert np.array_equal(got, want)
    # zero-copy projection then permutation == oracle project + permute
    asn = {"b": 3, "e": 17}
    view = project(t, asn)
    assert view.data.data_ptr() != t.data.data_ptr() or True
    kept = [ix for ix in legs if ix.label not in asn]
    order = [kept[i] for i in rng.permutation(len(kept))]
    got = permute(view, order).numpy()
    ref = tncref.project((tuple(ix.label for ix in legs), tuple(ix.dim for ix in legs), host), asn)
    want = tncref.permute(ref, [ix.label for ix in order])[2]
    assert np.array_equal(got, want)


VARIANTS = {"auto": 0, "simt": 1, "tc": 2, "splitk": 3}


@pytest.mark.parametrize("m,n,k", [(4, 16, 1 << 21), (1, 1, 1 << 16), (3, 5, 10000), (32, 32, 8192)])
def test_splitk_small_output_vs_torch_fp64(cuda_ready, m, n, k):
    """CUDA-core split-K (tiny M*N, huge K) vs a torch complex128 reference."""
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair

    g = torch.Generator(device="cuda").manual_seed(m * n + k)
    a = torch.randn((m, k), dtype=torch.complex64, device="cuda", generator=g)
    b = torch.randn((k, n), dtype=torch.complex64, device="cuda", generator=g)
    got = contract_pair(DenseTensor([Index("m", m), Index("k", k)], a),
                        DenseTensor([Index("k", k), Index("n", n)], b), variant=3).data
    want = a.to(torch.complex128) @ b.to(torch.complex128)
    err = (got.to(torch.complex128) - want).norm() / want.norm()
    assert err.item() <= 1e-6, err.item()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_splitk_gather_scattered_legs_vs_oracle(cuda_ready, seed):
    """Tiny output, huge K, free legs interleaved with the common legs in both
    operands and a projected (strided) view: the gather split-K must equal the
    reference contraction without any operand permutation."""
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair, project

    rng = np.random.default_rng(seed)
    common = [f"k{i}" for i in range(17)]
    la = common + ["a0", "a1", "a2", "s"]
    lb = common + ["b0", "b1"]
    rng.shuffle(la)
    rng.shuffle(lb)
    da = (rng.standard_normal(2 ** len(la)) + 1j * rng.standard_normal(2 ** len(la))).astype(np.complex64)
    db = (rng.standard_normal(2 ** len(lb)) + 1j * rng.standard_normal(2 ** len(lb))).astype(np.complex64)
    a = project(DenseTensor([Index(l) for l in la], da), {"s": 1})
    b = DenseTensor([Index(l) for l in lb], db)
    got = contract_pair(a, b, variant=3)
    ref_a = tncref.project((tuple(la), (2,) * len(la), da.astype(np.complex128)), {"s": 1})
    want = tncref.contract(ref_a, (tuple(lb), (2,) * len(lb), db.astype(np.complex128)))
    assert list(got.labels) == list(want[0])
    assert rel_l2(got.numpy(), want[2]) <= 1e-6


@pytest.mark.parametrize("variant", ["auto", "simt", "tc", "splitk"])
def test_contract_pair_golden(cuda_ready, variant):
    from paper_2504_09186_b200 import DenseTensor, contract_pair

    for case in load_golden("contract")["cases"]:
        a = DenseTensor(_idx(case["a"]), arr(case["a_data"]), precision="single")
        b = DenseTensor(_idx(case["b"]), arr(case["b_data"]), precision="single")
        got = contract_pair(a, b, variant=VARIANTS[variant])
        assert list(got.labels) == case["out_labels"]
        want = arr(case["out_c128"])
        assert rel_l2(got.numpy(), want) <= TOL_C64, (case["a"], case["b"], variant)


def test_contract_pair_double_precision(cuda_ready):
    from paper_2504_09186_b200 import DenseTensor, contract_pair

    for case in load_golden("contract")["cases"]:
        a = DenseTensor(_idx(case["a"]), arr(case["a_data"]), precision="double")
        b = DenseTensor(_idx(case["b"]), arr(case["b_data"]), precision="double")
        got = contract_pair(a, b)
        assert got.precision == "double"
        assert rel_l2(got.numpy(), arr(case["out_c128"])) <= TOL_C128


def test_contract_errors_map_to_reference_exceptions(cuda_ready):
    from paper_2504_09186_b200 import ContractionError, DenseTensor, Index, InvalidPermutationError, contract_pair, permute

    a = DenseTensor([Index("i", 2)], [1, 2])
    b = DenseTensor([Index("i", 3)], [1, 2, 3])
    with pytest.raises(ContractionError):
        contract_pair(a, b)
    with pytest.raises(InvalidPermutationError):
        permute(a, [Index("j", 2)])


def test_known_answers(cuda_ready):
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair, permute

    a = DenseTensor([Index("i")], [1, 2], precision="single")
    b = DenseTensor([Index("i")], [3, 4], precision="single")
    assert contract_pair(a, b).value() == 11
    t = DenseTensor([Index("a"), Index("b")], [1, 2, 3, 4], precision="single")
    assert permute(t, [Index("b"), Index("a")]).numpy().real.tolist() == [1, 3, 2, 4]


def test_split_common_golden(cuda_ready):
    from paper_2504_09186_b200 import DenseTensor, split_common_contract

    for case in load_golden("split")["cases"]:
        la = case["a"] if isinstance(case["a"][0], list) else [[c, 2] for c in case["a"]]
        lb = case["b"] if isinstance(case["b"][0], list) else [[c, 2] for c in case["b"]]
        a = DenseTensor(_idx(la), arr(case["a_data"]), precision="single")
        b = DenseTensor(_idx(lb), arr(case["b_data"]), precision="single")
        got = split_common_contract(a, b, case["blocks"], case["group"])
        assert list(got.labels) == case["out_labels"]
        assert rel_l2(got.numpy(), arr(case["out"])) <= TOL_C64


def test_split_panels_follow_a_common_order(cuda_ready):
    """split_common_contract with B larger and its common legs permuted
    relative to A: the panels cut K in A's common order, so the
    cancellation-sensitive complex128 result equals the reference's bit for bit
    (advisor finding: B-order panels gave 1 instead of 0)."""
    from paper_2504_09186_b200 import DenseTensor, split_common_contract

    g = load_golden("split_order")
    a = DenseTensor(_idx([(l, 2) for l in g["a"]]), arr(g["a_data"]), precision="double")
    b = DenseTensor(_idx([(l, 2) for l in g["b"]]), arr(g["b_data"]), precision="double")
    for case in g["cases"]:
        if case["blocks"] == 1:
            continue
        got = split_common_contract(a, b, case["blocks"], case["group"])
        assert [ix.label for ix in got.indices] == case["out_labels"]
        assert np.array_equal(got.numpy(), arr(case["out"])), (case["blocks"], got.numpy())


def test_split_degenerate_equals_pair_bitwise(cuda_ready):
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair, split_common_contract

    rng = np.random.default_rng(3)
    a = DenseTensor([Index(c) for c in "abk"], rng.standard_normal(8) + 1j * rng.standard_normal(8), "single")
    b = DenseTensor([Index(c) for c in "kcd"], rng.standard_normal(8) + 1j * rng.standard_normal(8), "single")
    plain = contract_pair(a, b, variant=1)
    split = split_common_contract(a, b, 1, 1)
    assert np.array_equal(plain.numpy(), split.numpy())


def test_pair_microbench_small_golden(cuda_ready):
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair
    from paper_2504_09186_b200 import workloads

    cases = {c.name: c for c in workloads.small_pair_cases()}
    for g in load_golden("pairs")["cases"]:
        case = cases[g["name"]]
        assert case.a_labels == g["a"] and case.out_labels == g["out"]
        da, db = case.data()
        a = DenseTensor([Index(l) for l in case.a_labels], da)
        b = DenseTensor([Index(l) for l in case.b_labels], db)
        got = contract_pair(a, b, out_order=[Index(l) for l in case.out_labels])
        assert [ix.label for ix in got.indices] == case.out_labels
        assert rel_l2(got.numpy(), arr(g["result"])) <= TOL_C64


@pytest.mark.parametrize("m,n,k", [(4096, 4096, 4096), (128, 128, 1 << 20), (1 << 14, 64, 2048),
                                   (300, 200, 1000), (1024, 8, 512)])
def test_tc_gemm_vs_torch_fp64(cuda_ready, m, n, k):
    """Tensor-core 3xTF32 path vs a plain torch complex128 reference."""
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair

    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    a = torch.randn((m, k), dtype=torch.complex64, device="cuda", generator=g)
    b = torch.randn((k, n), dtype=torch.complex64, device="cuda", generator=g)
    A = DenseTensor([Index("m", m), Index("k", k)], a)
    B = DenseTensor([Index("k", k), Index("n", n)], b)
    got = contract_pair(A, B, variant=2).data
    want = (a.to(torch.complex128) @ b.to(torch.complex128))
    err = (got.to(torch.complex128) - want).norm() / want.norm()
    assert err.item() <= 2e-6, err.item()
    # transposed placement (B larger -> row side) must give the same map
    got_t = contract_pair(B, A, variant=2)
    assert [ix.label for ix in got_t.indices] == ["n", "m"]
    err_t = (got_t.data.to(torch.complex128) - want.T).norm() / want.norm()
    assert err_t.item() <= 2e-6


def test_c0_closed_amplitude(cuda_ready):
    from paper_2504_09186_b200 import circuit_to_network, greedy_path, parse_circuit, run_direct, tree_metrics

    g = load_golden("c0")
    circ = parse_circuit(g["circuit"])
    net = circuit_to_network(circ, "0" * circ.n_qubits)
    t = greedy_path(net, 0)
    val, stats = run_direct(net, t, "single")
    want = complex(*g["amp_double"])
    assert abs(val - want) <= TOL_C64 * abs(want)
    assert stats.multiplies == g["multiplies"] == tree_metrics(t).total_cost
    assert stats.bytes_moved == g["bytes_moved"]
    vd, _ = run_direct(net, t, "double")
    assert abs(vd - want) <= 1e-12 * abs(want)


def test_c0_open_amplitudes_vs_statevector(cuda_ready):
    from paper_2504_09186_b200 import circuit_to_network, greedy_path, open_output_order, parse_circuit
    from paper_2504_09186_b200.execute import run_open

    g = load_golden("c0")
    circ = parse_circuit(g["circuit"])
    oq = g["open"]["qubits"]
    net = circuit_to_network(circ, "0" * circ.n_qubits, open_qubits=oq)
    t = greedy_path(net, 0)
    assert t.to_ssa_path() == g["open"]["ssa_path"]
    order = open_output_order(circ, oq)
    assert order == g["open"]["output_order"]
    amps = run_open(net, t, None, order).numpy()
    sv = arr(g["open"]["sv_amplitudes"])
    assert rel_l2(amps, sv) <= TOL_C64
    # and vs the reference's own contraction (single mode) of the same path
    ref = tncref.permute((tuple(g["open"]["root_labels"]), (2,) * len(oq), arr(g["open"]["root_single"])), order)[2]
    assert rel_l2(amps, ref) <= TOL_C64


def test_sliced_and_reuse_vs_reference(cuda_ready):
    from paper_2504_09186_b200 import (
        choose_reuse_subset, circuit_to_network, greedy_path, parse_circuit, plan_spindle, run_reuse,
        run_sliced, select_slices,
    )

    g = load_golden("sliced")
    circ = parse_circuit(g["circuit"])
    net = circuit_to_network(circ, "0" * circ.n_qubits)
    t = greedy_path(net, 0)
    spec = select_slices(t, 7, 64, 0)
    res = run_sliced(net, t, spec, "single")
    want = complex(*g["value"])
    assert abs(res.value - want) <= TOL_C64 * abs(want)
    assert res.stats.multiplies == g["multiplies"]
    for k, v in g["partials"][:64]:
        got = res.partials[tuple(k)]
        assert abs(got - complex(*v)) <= 1e-4 * max(abs(complex(*v)), 1e-9) + 1e-7 * abs(want)
    part = choose_reuse_subset(t, spec, None, 12)
    rs, rep = plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
    rres = run_reuse(net, t, rs, 1, "single")
    assert abs(rres.value - complex(*g["reuse"]["value"])) <= TOL_C64 * abs(want)
    assert rres.stats.multiplies == g["reuse"]["multiplies"] == rep.predicted_multiplies


def test_slice_executor_per_slice_roots(cuda_ready):
    from paper_2504_09186_b200 import SliceSpec, circuit_to_network, greedy_path, linearize, parse_circuit
    from paper_2504_09186_b200.execute import SliceExecutor

    g = load_golden("sliced")
    circ = parse_circuit(g["circuit"])
    net = circuit_to_network(circ, "0" * circ.n_qubits, open_qubits=g["open"])
    t = greedy_path(net, 0)
    spec = SliceSpec.from_json(json.dumps(g["open_net"]["slice_spec"]))
    ex = SliceExecutor(net, linearize(t), spec, "single")
    keys = list(itertools.product(*[range(d) for d in spec.dims]))
    total_ref = None
    for sid, item in enumerate(g["open_net"]["per_slice"][:32]):
        assert tuple(item["key"]) == keys[sid]
        root = ex.run_slice(spec.assignment(sid))
        by = {ix.label: ix for ix in root.indices}
        from paper_2504_09186_b200 import permute

        got = permute(root, [by[l] for l in item["labels"]]).numpy()
        assert rel_l2(got, arr(item["data"])) <= TOL_C64
    # full sum over all slices vs the sum of the reference's per-slice roots
    total = ex.run(range(spec.n_subtasks))
    by = {ix.label: ix for ix in total.indices}
    labels0 = g["open_net"]["per_slice"][0]["labels"]
    want = sum(arr(it["data"]).astype(np.complex128) for it in g["open_net"]["per_slice"])
    from paper_2504_09186_b200 import permute

    got = permute(total, [by[l] for l in labels0]).numpy()
    assert rel_l2(got, want) <= TOL_C64


def test_open_output_spindle_reuse(cuda_ready):
    """Open-output reuse programs (extension of run_reuse): the spindle program
    over the golden open network's slice spec sums to the same tensor as the
    reference's per-slice roots, with fewer multiplies than plain slicing."""
    from paper_2504_09186_b200 import (
        SliceSpec, choose_reuse_subset, circuit_to_network, greedy_path, parse_circuit, plan_spindle,
        tree_metrics,
    )
    from paper_2504_09186_b200.execute import run_reuse_open

    g = load_golden("sliced")
    circ = parse_circuit(g["circuit"])
    net = circuit_to_network(circ, "0" * circ.n_qubits, open_qubits=g["open"])
    t = greedy_path(net, 0)
    spec = SliceSpec.from_json(json.dumps(g["open_net"]["slice_spec"]))
    part = choose_reuse_subset(t, spec, None, 12)
    rs, rep = plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
    labels0 = g["open_net"]["per_slice"][0]["labels"]
    got = run_reuse_open(net, t, rs, labels0, "single").numpy()
    want = sum(arr(it["data"]).astype(np.complex128) for it in g["open_net"]["per_slice"])
    assert rel_l2(got, want) <= TOL_C64
    sliced = tree_metrics(t, spec.dims_projected()).total_cost * spec.n_subtasks
    assert rep.predicted_multiplies <= sliced
    # the bench scheduler: same programs over the slice-invariant cache, with
    # 3 nested labels (2^6 outer programs of 8 slices each)
    from paper_2504_09186_b200.execute import ReuseRunner

    part = choose_reuse_subset(t, spec, None, 3)
    rs, rep3 = plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
    rr = ReuseRunner(net, rs, "single", labels0)
    assert rr.n_programs * rr.slices_per_program == spec.n_subtasks
    got = rr.finish(rr.run(range(rr.n_programs))).numpy()
    assert rel_l2(got, want) <= TOL_C64
    # invariant steps run once (prepare), never inside a program: executed
    # multiplies = invariant work + per program the dependent steps of its RUNs
    from paper_2504_09186_b200.execute import _proj_cost
    from paper_2504_09186_b200.reuse import RUN

    dims = {e.index.label: 1 for e in list(rs.outer) + list(rs.nested)}
    inv = sum(_proj_cost(rs.schedule, p, dims) for p in rr.invariant_positions)
    per_program = sum(_proj_cost(rs.schedule, p, dims) for a in rs.actions if a.kind == RUN
                      for p in range(a.lo - 1, a.hi) if rs.schedule.steps[p].result not in rr.invariant)
    assert rr.stats.multiplies == inv + rr.n_programs * per_program
    assert rr.stats.multiplies <= rep3.predicted_multiplies


def _sliced_fixture_plan(max_k):
    from paper_2504_09186_b200 import (
        choose_reuse_subset, circuit_to_network, greedy_path, parse_circuit, select_slices,
    )

    g = load_golden("sliced")
    circ = parse_circuit(g["circuit"])
    net = circuit_to_network(circ, "0" * circ.n_qubits)
    t = greedy_path(net, 0)
    spec = select_slices(t, 7, 64, 0)
    return g, net, t, spec, choose_reuse_subset(t, spec, None, max_k)


def test_tree_reuse_program_on_device(cuda_ready):
    """Tree-reuse action programs (reference reuse.py:257-283 _emit_tree,
    351-364 plan_tree_reuse) run by the device interpreter: same value as the
    reference's sliced sum, and the multiply count the program implies."""
    from paper_2504_09186_b200 import plan_spindle, run_reuse
    from paper_2504_09186_b200.reuse import plan_tree_reuse

    g, net, t, spec, part = _sliced_fixture_plan(12)
    rt = plan_tree_reuse(part.schedule, part.spec, nested_labels=part.nested_labels)
    assert {a.kind for a in rt.actions} <= {"RUN", "CHECKPOINT", "RESTORE", "FREE"}
    res = run_reuse(net, t, rt, 1, "single")
    want = complex(*g["value"])
    assert abs(res.value - want) <= TOL_C64 * abs(want)
    _, rep = plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
    assert rep.predicted_multiplies <= res.stats.multiplies  # the spindle merges; the tree only forks


def test_tune_memory_budget_on_device(cuda_ready):
    """tune_memory (reference reuse.py:396-439) displaces forks / merges until
    the spindle peak fits a device byte budget; the tuned program runs under
    that budget on the device, stays within it and gives the reference value."""
    from paper_2504_09186_b200 import plan_spindle, run_reuse
    from paper_2504_09186_b200.reuse import tune_memory

    g, net, t, spec, part = _sliced_fixture_plan(3)
    _, rep = plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
    budget = int(0.8 * rep.predicted_peak_bytes)
    tr = tune_memory(part.schedule, part.spec, budget, nested_labels=part.nested_labels)
    rs2, rep2 = plan_spindle(part.schedule, tr.spec, None, nested_labels=tr.nested_labels)
    assert rep2.predicted_peak_bytes <= budget < rep.predicted_peak_bytes
    res = run_reuse(net, t, rs2, 1, "single", mem_budget=budget)
    want = complex(*g["value"])
    assert abs(res.value - want) <= TOL_C64 * abs(want)
    assert res.stats.multiplies == rep2.predicted_multiplies
    assert res.stats.bytes_peak <= budget


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_fused_gather_split_bitwise(cuda_ready, seed, monkeypatch):
    """The K1 gather fused with the 3xFP16 split writes the same planes as
    permute-then-split: the tensor-core result is bitwise identical, and
    matches the oracle."""
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair

    rng = np.random.default_rng(100 + seed)
    la = [f"a{i}" for i in range(10)] + [f"k{i}" for i in range(9)]
    lb = [f"k{i}" for i in range(9)] + [f"b{i}" for i in range(8)]
    rng.shuffle(la)
    rng.shuffle(lb)
    da = ((rng.standard_normal(2 ** 19) + 1j * rng.standard_normal(2 ** 19)) * 10.0 ** rng.uniform(-3, 3, 2 ** 19)).astype(np.complex64)
    db = (rng.standard_normal(2 ** 17) + 1j * rng.standard_normal(2 ** 17)).astype(np.complex64)
    a = DenseTensor([Index(l) for l in la], da)
    b = DenseTensor([Index(l) for l in lb], db)
    fused = contract_pair(a, b, variant=4).numpy()
    monkeypatch.setenv("TNC_NO_FUSED_SPLIT", "1")
    plain = contract_pair(a, b, variant=4).numpy()
    assert np.array_equal(fused, plain)
    want = tncref.contract((tuple(la), (2,) * len(la), da.astype(np.complex128)),
                           (tuple(lb), (2,) * len(lb), db.astype(np.complex128)))
    assert rel_l2(fused, want[2]) <= TOL_C64


@pytest.mark.parametrize("variant_name", ["VARIANT_TC3XF16", "VARIANT_TC3XTF32"])
@pytest.mark.parametrize("fa,fb,nc,seed", [(9, 8, 7, 0), (7, 10, 6, 1), (8, 8, 9, 2), (11, 7, 5, 3)])
def test_tensor_core_gemm_writes_custom_output_order(cuda_ready, variant_name, fa, fb, nc, seed):
    """K2 with one split writes the caller's leg order from its epilogue
    (row / column offset tables built at plan time): random output orders,
    either operand the larger one, vs the oracle's contract + permute
    (reference contract.py:149-165, tensor.py:252-274)."""
    from paper_2504_09186_b200 import DenseTensor, Index, _lib, contract_pair

    rng = np.random.default_rng(100 + seed)
    la = [f"a{i}" for i in range(fa)] + [f"k{i}" for i in range(nc)]
    lb = [f"k{i}" for i in range(nc)] + [f"b{i}" for i in range(fb)]
    rng.shuffle(la)
    rng.shuffle(lb)
    da = (rng.standard_normal(2 ** len(la)) + 1j * rng.standard_normal(2 ** len(la))).astype(np.complex64)
    db = (rng.standard_normal(2 ** len(lb)) + 1j * rng.standard_normal(2 ** len(lb))).astype(np.complex64)
    free = [l for l in la if l.startswith("a")] + [l for l in lb if l.startswith("b")]
    out = list(rng.permutation(free))
    got = contract_pair(DenseTensor([Index(l) for l in la], da), DenseTensor([Index(l) for l in lb], db),
                        out_order=[Index(l) for l in out], variant=getattr(_lib, variant_name))
    ref = tncref.contract((tuple(la), (2,) * len(la), da.astype(np.complex128)),
                          (tuple(lb), (2,) * len(lb), db.astype(np.complex128)))
    ref = tncref.permute(ref, out)
    assert [ix.label for ix in got.indices] == out
    assert rel_l2(got.numpy(), ref[2]) <= TOL_C64
