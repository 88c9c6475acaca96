"""Generate golden vectors from the REAL reference package (build container only).

TEST INFRASTRUCTURE.  Imports ``tncsim`` from ``/root/reference/pkg/src`` (and
its test oracles from ``/root/reference/pkg/tests``), runs it on seeded inputs
and writes small fixtures to ``tests/golden/``.  The GPU box never runs this
script (``/root/reference`` does not exist there); the committed fixtures
travel instead.

    python oracle/gen_golden.py [section ...]

Sections: perm contract split c0 plans sliced reuse pairs spill plan_c4_reuse split_order
"""

from __future__ import annotations

import base64
import gzip
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("TNC_REFERENCE", "/root/reference/pkg"))
ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"
sys.dont_write_bytecode = True
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(ROOT))

import tncsim  # noqa: E402  (the reference)
from tncsim import Index as RIndex  # noqa: E402
from tncsim.execute import RunStats, _Engine  # noqa: E402

from paper_2504_09186_b200 import workloads  # noqa: E402  (input generators only)


def _c(arr) -> dict:
    """Exact compact encoding: base64 of the little-endian complex array."""
    a = np.ascontiguousarray(np.asarray(arr).reshape(-1))
    if a.dtype not in (np.complex64, np.complex128):
        a = a.astype(np.complex128)
    return {"dtype": "c8" if a.dtype == np.complex64 else "c16",
            "b64": base64.b64encode(a.astype(a.dtype.newbyteorder("<")).tobytes()).decode()}


def _f(z) -> list:
    return [float(np.real(z)), float(np.imag(z))]


def _dump(name: str, obj) -> None:
    OUT.mkdir(parents=True, exist_ok=True)
    with gzip.open(OUT / f"{name}.json.gz", "wt") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"wrote {name}.json.gz", flush=True)


def rand_c(rng, n, dtype=np.complex64):
    return (rng.standard_normal(n) + 1j * rng.standard_normal(n)).astype(dtype)


def section_perm():
    rng = np.random.default_rng(1)
    cases = []
    shapes = [
        [("a", 2), ("b", 2), ("c", 2), ("d", 2), ("e", 2), ("f", 2)],
        [("a", 3), ("b", 2), ("c", 4), ("d", 2)],
        [("x", 5)],
        [],
        [(f"l{i}", 2) for i in range(12)],
        [("p", 2), ("q", 7), ("r", 3), ("s", 2), ("t", 64)],
    ]
    for legs in shapes:
        size = int(np.prod([d for _, d in legs])) if legs else 1
        data = rand_c(rng, size)
        t = tncsim.DenseTensor([RIndex(l, d) for l, d in legs], data, precision="single")
        for trial in range(6 if legs else 1):
            order = list(t.indices)
            rng.shuffle(order)
            if trial == 0:
                order = list(t.indices)
            plan = tncsim.classify_permutation(t.indices, order)
            out = tncsim.permute(t, order)
            cases.append({
                "legs": legs, "data": _c(data), "target": [ix.label for ix in order],
                "out": _c(out.data), "classify": [plan.stride, plan.offset, plan.case_class, plan.chunk,
                                                  plan.src_step],
            })
    # the reference's own bucket examples (test_tensor.py:74-91)
    buckets = []
    for src, tgt in [("abcd", "acbd"), ("abcd", "bacd"), ("abcd", "adbc"), ("abcde", "bacde"),
                     ("abcde", "aebcd"), ("abcdef", "defabc"), ("abcd", "acdb"), ("fghij", "fghji"),
                     ("abcd", "dabc"), ("abcdefg", "gfedcba")]:
        p = tncsim.classify_permutation([RIndex(c) for c in src], [RIndex(c) for c in tgt])
        buckets.append({"src": src, "tgt": tgt, "classify": [p.stride, p.offset, p.case_class, p.chunk,
                                                             p.src_step]})
    _dump("perm", {"cases": cases, "buckets": buckets})


def section_contract():
    rng = np.random.default_rng(2)
    cases = []
    labels = "abcdefgh"
    seed = 0
    # every overlap pattern up to size 2^12 (test_contract.py:97-114)
    for ra in range(5):
        for rb in range(5):
            for ov in range(5):
                if ov > min(ra, rb) or 2 ** (ra + rb) > 2 ** 12:
                    continue
                seed += 1
                cases.append((list(labels[:ra]), list(labels[ra - ov: ra - ov + rb]), None))
    # shuffled / mixed-dim / larger
    cases.append((["i", "j", "k"], ["k", "j", "l"], None))
    cases.append((["x", "y", "c"], ["c", "u", "v", "w"], None))
    cases.append(([("a", 3), ("k", 3), ("m", 2)], [("k", 3), ("m", 2), ("b", 2)], "dims"))
    big_a = [f"f{i}" for i in range(8)] + [f"k{i}" for i in range(6)]
    big_b = [f"k{i}" for i in range(6)] + [f"g{i}" for i in range(5)]
    rng.shuffle(big_a)
    rng.shuffle(big_b)
    cases.append((big_a, big_b, None))
    ga = [f"f{i}" for i in range(7)] + [f"k{i}" for i in range(7)]
    gb = [f"k{i}" for i in range(7)] + [f"g{i}" for i in range(7)]
    rng.shuffle(ga)
    rng.shuffle(gb)
    cases.append((ga, gb, None))  # equal sizes -> ttgt tie-break
    out = []
    for la, lb, kind in cases:
        ia = [RIndex(*x) if isinstance(x, tuple) else RIndex(x) for x in la]
        ib = [RIndex(*x) if isinstance(x, tuple) else RIndex(x) for x in lb]
        na = int(np.prod([ix.dim for ix in ia])) if ia else 1
        nb = int(np.prod([ix.dim for ix in ib])) if ib else 1
        da, db = rand_c(rng, na), rand_c(rng, nb)
        a = tncsim.DenseTensor(ia, da, precision="single")
        b = tncsim.DenseTensor(ib, db, precision="single")
        c64 = tncsim.contract_pair(a, b)
        c128 = tncsim.contract_pair(a.astype("double"), b.astype("double"))
        plan = tncsim.contract.ttgt_plan(a.indices, b.indices)
        out.append({
            "a": [[ix.label, ix.dim] for ix in ia], "b": [[ix.label, ix.dim] for ix in ib],
            "a_data": _c(da), "b_data": _c(db), "out_labels": list(c64.labels),
            "out_c64": _c(c64.data), "out_c128": _c(c128.data),
            "b_is_multiplier": plan.b_is_multiplier,
            "shape": [plan.shape.m, plan.shape.k, plan.shape.n],
        })
    _dump("contract", {"cases": out})


def section_split():
    rng = np.random.default_rng(3)
    out = []
    specs = [
        ("abklm", "kmlcd", [(1, 1), (2, 1), (3, 2), (6, 4), (8, 8)]),
        ("abklmnpq", "klmnpqcd", [(2, 1), (4, 2), (8, 8), (16, 16)]),
    ]
    for sa, sb, bgs in specs:
        ia = [RIndex(c) for c in sa]
        ib = [RIndex(c) for c in sb]
        da, db = rand_c(rng, 2 ** len(ia)), rand_c(rng, 2 ** len(ib))
        a = tncsim.DenseTensor(ia, da, precision="single")
        b = tncsim.DenseTensor(ib, db, precision="single")
        for bl, gr in bgs:
            res = tncsim.split_common_contract(a, b, bl, gr)
            out.append({"a": sa, "b": sb, "a_data": _c(da), "b_data": _c(db), "blocks": bl, "group": gr,
                        "out_labels": list(res.labels), "out": _c(res.data)})
    # remainder-on-last-panel case with dim 3 (test_contract.py:368-374)
    ia = [RIndex("a", 2), RIndex("k", 3), RIndex("m", 2)]
    ib = [RIndex("k", 3), RIndex("m", 2), RIndex("b", 2)]
    da, db = rand_c(rng, 12), rand_c(rng, 12)
    a = tncsim.DenseTensor(ia, da, precision="single")
    b = tncsim.DenseTensor(ib, db, precision="single")
    res = tncsim.split_common_contract(a, b, 4, 1)
    out.append({"a": [["a", 2], ["k", 3], ["m", 2]], "b": [["k", 3], ["m", 2], ["b", 2]], "a_data": _c(da),
                "b_data": _c(db), "blocks": 4, "group": 1, "out_labels": list(res.labels), "out": _c(res.data)})
    _dump("split", {"cases": out})


def section_split_order():
    """split_common_contract when B is the larger operand and lists the common
    legs in a different order than A: the reference cuts K into panels in A's
    common order (contract.py:58-75,168-208).  Values are chosen so that the
    complex128 result depends on the panel boundaries (1e16 + 1 rounds away in
    one partition, not in the other)."""
    ia = [RIndex("k0"), RIndex("k1")]
    ib = [RIndex("k1"), RIndex("k0"), RIndex("b0")]
    da = np.array([1e16, 1.0, -1e16, 0.0], dtype=np.complex128)  # A[k0][k1]
    db = np.ones(8, dtype=np.complex128)
    a = tncsim.DenseTensor(ia, da, precision="double")
    b = tncsim.DenseTensor(ib, db, precision="double")
    cases = []
    for bl, gr in ((2, 1), (4, 1), (1, 1)):
        res = tncsim.split_common_contract(a, b, bl, gr)
        cases.append({"blocks": bl, "group": gr, "out_labels": list(res.labels), "out": _c(res.data)})
    _dump("split_order", {"a": ["k0", "k1"], "b": ["k1", "k0", "b0"], "a_data": _c(da), "b_data": _c(db),
                          "cases": cases})


def _steps(s):
    return [[st.lhs, st.rhs, st.result] for st in s.steps]


def _leaves(net):
    return [{"legs": [[ix.label, ix.dim] for ix in t.indices], "data": _c(t.data)} for t in net.tensors]


def section_c0():
    wl = workloads.C0
    text = workloads.grid_circuit_text(wl.rows, wl.cols, wl.cycles, wl.seed)
    circ = tncsim.parse_circuit(text)
    n = circ.n_qubits
    closed = tncsim.circuit_to_network(circ, "0" * n)
    t = tncsim.greedy_path(closed, 0)
    s = tncsim.linearize(t)
    val_single, st_single = tncsim.run_direct(closed, t, "single")
    val_double, _ = tncsim.run_direct(closed, t, "double")
    m = tncsim.tree_metrics(t)
    # open network: drop the <0| of the open qubits (last n tensors are projections)
    open_q = wl.open_qubits
    keep = [tt for i, tt in enumerate(closed.tensors) if not (i >= len(closed.tensors) - n and
                                                             (i - (len(closed.tensors) - n)) in open_q)]
    onet = tncsim.TensorNetwork(keep)
    ot = tncsim.greedy_path(onet, 0)
    os_ = tncsim.linearize(ot)
    eng = _Engine(onet, "single")
    values = {}
    eng.run_range(os_, 1, len(os_.steps), {}, values, RunStats())
    root = values[os_.steps[-1].result]
    eng2 = _Engine(onet, "double")
    values2 = {}
    eng2.run_range(os_, 1, len(os_.steps), {}, values2, RunStats())
    root2 = values2[os_.steps[-1].result]
    # reference state-vector oracle (oracles.py:76-104) on every open amplitude
    from oracles import statevector_amplitude

    finals = {}
    seg = [0] * n
    for g in circ.gates:
        for q in g.qubits:
            seg[q] += 1
    order = [f"q{q}.{seg[q]}" for q in sorted(open_q, reverse=True)]
    amps_sv = []
    t0 = time.time()
    for j in range(2 ** len(open_q)):
        bits = format(j, f"0{len(open_q)}b") + "0" * (n - len(open_q))
        amps_sv.append(statevector_amplitude(circ, bits))
    print(f"sv amplitudes {time.time() - t0:.1f}s", flush=True)
    _dump("c0", {
        "circuit": text, "leaves": _leaves(closed), "ssa_path": t.to_ssa_path(), "steps": _steps(s),
        "stems": [[st.positions, st.cost] for st in s.stems], "multi_stem": s.multi_stem,
        "total_cost": m.total_cost, "max_rank": m.max_rank, "per_step": m.per_step,
        "amp_single": _f(val_single), "amp_double": _f(val_double),
        "multiplies": st_single.multiplies, "bytes_moved": st_single.bytes_moved,
        "open": {"qubits": open_q, "ssa_path": ot.to_ssa_path(), "steps": _steps(os_),
                 "root_labels": list(root.labels), "root_single": _c(root.data), "root_double": _c(root2.data),
                 "output_order": order, "sv_amplitudes": _c(np.array(amps_sv))},
    })


def _plan_fixture(wl, max_rank, with_reuse, max_k=12):
    text = workloads.grid_circuit_text(wl.rows, wl.cols, wl.cycles, wl.seed)
    circ = tncsim.parse_circuit(text)
    n = circ.n_qubits
    closed = tncsim.circuit_to_network(circ, "0" * n)
    keep = [tt for i, tt in enumerate(closed.tensors)
            if not (i >= len(closed.tensors) - n and (i - (len(closed.tensors) - n)) in wl.open_qubits)]
    net = tncsim.TensorNetwork(keep)
    t0 = time.time()
    t = tncsim.greedy_path(net, 0)
    t1 = time.time()
    spec = tncsim.select_slices(t, max_rank, 64, 0)
    t2 = time.time()
    s = tncsim.linearize(t)
    m = tncsim.tree_metrics(t)
    ms = tncsim.tree_metrics(t, spec.dims_projected())
    obj = {
        "rows": wl.rows, "cols": wl.cols, "cycles": wl.cycles, "seed": wl.seed, "open": wl.open_qubits,
        "max_rank": max_rank, "ssa_path": t.to_ssa_path(), "steps": _steps(s),
        "stems": [[st.positions, st.cost] for st in s.stems],
        "total_cost": str(m.total_cost), "tree_max_rank": m.max_rank, "slice_spec": json.loads(spec.to_json()),
        "sliced_total_cost": str(ms.total_cost), "sliced_max_rank": ms.max_rank,
        "timing": {"greedy": t1 - t0, "select_slices": t2 - t1},
    }
    if with_reuse:
        t3 = time.time()
        part = tncsim.choose_reuse_subset(t, spec, None, max_k)
        rs, rep = tncsim.plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
        t4 = time.time()
        obj["reuse"] = {
            "max_k": max_k, "nested": part.nested_labels, "outer": [e.index.label for e in part.outer],
            "steps": _steps(part.schedule), "spec": json.loads(part.spec.to_json()),
            "actions": [a.to_obj() for a in rs.actions], "report": rep.to_obj(),
            "predicted_multiplies": str(rep.predicted_multiplies),
            "timing": t4 - t3,
        }
    return obj


def section_plans():
    _dump("plan_c3", _plan_fixture(workloads.C3, workloads.C3_MAX_RANK, True, max_k=6))
    _dump("plan_c4", _plan_fixture(workloads.C4, workloads.C4_MAX_RANK, False))


def section_plan_c4_reuse():
    """C4 spindle plan at the reference's default max_k = 12 (12 nested labels,
    21 outer, ~34k actions, ~118 GiB predicted peak).  Slow: the reference
    planner takes several minutes here."""
    obj = _plan_fixture(workloads.C4, workloads.C4_MAX_RANK, True, max_k=12)
    keep = {k: obj[k] for k in ("rows", "cols", "cycles", "seed", "open", "max_rank")}
    keep["reuse"] = obj["reuse"]
    _dump("plan_c4_reuse", keep)


def section_sliced():
    """Small end-to-end sliced + reuse runs with full data (oracle-sized)."""
    wl = workloads.CircuitWorkload(4, 4, 10, 3, 3)
    text = workloads.grid_circuit_text(wl.rows, wl.cols, wl.cycles, wl.seed)
    circ = tncsim.parse_circuit(text)
    n = circ.n_qubits
    closed = tncsim.circuit_to_network(circ, "0" * n)
    t = tncsim.greedy_path(closed, 0)
    spec = tncsim.select_slices(t, 7, 64, 0)
    res = tncsim.run_sliced(closed, t, spec, "single")
    direct, _ = tncsim.run_direct(closed, t, "single")
    part = tncsim.choose_reuse_subset(t, spec, None, 12)
    rs, rep = tncsim.plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
    rres = tncsim.run_reuse(closed, t, rs, 1, "single")
    keep = [tt for i, tt in enumerate(closed.tensors)
            if not (i >= len(closed.tensors) - n and (i - (len(closed.tensors) - n)) in wl.open_qubits)]
    onet = tncsim.TensorNetwork(keep)
    ot = tncsim.greedy_path(onet, 0)
    ospec = tncsim.select_slices(ot, 7, 64, 0)
    os_ = tncsim.linearize(ot)
    eng = _Engine(onet, "single")
    import itertools

    per_slice = []
    for key in itertools.product(*[range(e.index.dim) for e in ospec.entries]):
        values = {}
        eng.run_range(os_, 1, len(os_.steps), dict(zip(ospec.labels, key)), values, RunStats())
        root = values[os_.steps[-1].result]
        per_slice.append({"key": list(key), "labels": list(root.labels), "data": _c(root.data)})
    _dump("sliced", {
        "circuit": text, "open": wl.open_qubits, "ssa_path": t.to_ssa_path(), "steps": _steps(tncsim.linearize(t)),
        "slice_spec": json.loads(spec.to_json()),
        "value": _f(res.value), "direct": _f(direct),
        "partials": [[list(k), _f(v)] for k, v in sorted(res.partials.items())],
        "multiplies": res.stats.multiplies,
        "reuse": {"nested": part.nested_labels, "outer": [e.index.label for e in part.outer],
                  "steps": _steps(part.schedule), "actions": [a.to_obj() for a in rs.actions],
                  "predicted_multiplies": rep.predicted_multiplies, "peak": rep.predicted_peak_bytes,
                  "value": _f(rres.value), "multiplies": rres.stats.multiplies},
        "open_net": {"ssa_path": ot.to_ssa_path(), "steps": _steps(os_), "slice_spec": json.loads(ospec.to_json()),
                     "per_slice": per_slice},
    })


def section_reuse():
    """Reference synthetic stems (oracles.py) through the reuse planner."""
    from oracles import nested_stem, rolling_stem, valley_stem

    out = []
    for name, (net, t), max_k in [("valley", valley_stem(seed=2), 12), ("nested", nested_stem(k=3, mid=2, seed=5), 12),
                                  ("rolling", rolling_stem(width=5, length=8, seed=8), 12)]:
        s = tncsim.linearize(t)
        lts = tncsim.compute_lifetimes(s)
        labels = [l for l in sorted(lts) if l.startswith("u")] or ["w5", "w6"]
        from tncsim.slicing import SliceEntry, SliceSpec

        spec = SliceSpec([SliceEntry.at_lifetime(RIndex(l, net.dim_of(l)), lts[l]) for l in labels])
        s2, spec2 = tncsim.branch_exchange_nest(s, spec)
        item = {"name": name, "leaves": _leaves(net), "ssa_path": t.to_ssa_path(), "steps": _steps(s),
                "spec": json.loads(spec.to_json()), "exchanged_steps": _steps(s2),
                "exchanged_spec": json.loads(spec2.to_json())}
        try:
            part = tncsim.choose_reuse_subset(t, spec, None, max_k)
            rs, rep = tncsim.plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
            rres = tncsim.run_reuse(net, t, rs, 1, "double")
            item["reuse"] = {"nested": part.nested_labels, "actions": [a.to_obj() for a in rs.actions],
                             "predicted_multiplies": rep.predicted_multiplies, "peak": rep.predicted_peak_bytes,
                             "value": _f(rres.value),
                             "overheads": {k: [v.numerator, v.denominator] for k, v in part.overheads.items()}}
            rst = tncsim.plan_tree_reuse(part.schedule, part.spec)
            item["tree_actions"] = [a.to_obj() for a in rst.actions]
        except tncsim.errors.TncError as exc:  # pragma: no cover - recorded as a case
            item["error"] = str(exc)
        out.append(item)
    _dump("reuse", {"cases": out})


def section_pairs():
    """Oracle-sized variants of the C1 micro-benchmarks (same structure,
    fewer legs): permuted operands, contract, random output permutation."""
    out = []
    for case in workloads.small_pair_cases():
        da, db = case.data()
        a = tncsim.DenseTensor([RIndex(l) for l in case.a_labels], da, precision="single")
        b = tncsim.DenseTensor([RIndex(l) for l in case.b_labels], db, precision="single")
        c = tncsim.contract_pair(a.astype("double"), b.astype("double"))
        c = tncsim.permute(c, [RIndex(l) for l in case.out_labels])
        out.append({"name": case.name, "a": case.a_labels, "b": case.b_labels, "out": case.out_labels,
                    "seed": case.seed, "result": _c(c.data.astype(np.complex64))})
    _dump("pairs", {"cases": out})


def section_spill():
    """Reference byte formats: the TNCPART1 partials spill of the 4x4 sliced
    run (execute.py:473-490) and DenseTensor.to_bytes (tensor.py:146-161)."""
    import tempfile

    from tncsim.execute import write_partials

    wl = workloads.CircuitWorkload(4, 4, 10, 3, 3)
    circ = tncsim.parse_circuit(workloads.grid_circuit_text(wl.rows, wl.cols, wl.cycles, wl.seed))
    closed = tncsim.circuit_to_network(circ, "0" * circ.n_qubits)
    t = tncsim.greedy_path(closed, 0)
    spec = tncsim.select_slices(t, 7, 64, 0)
    res = tncsim.run_sliced(closed, t, spec, "single")
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "p.bin")
        write_partials(path, res)
        raw = open(path, "rb").read()
    rng = np.random.default_rng(5)
    tens = []
    for prec, dt in (("single", np.complex64), ("double", np.complex128)):
        data = rand_c(rng, 12, dt)
        tt = tncsim.DenseTensor([RIndex("ab", 3), RIndex("c", 4)], data, precision=prec)
        tens.append({"precision": prec, "labels": ["ab", "c"], "dims": [3, 4], "data": _c(data),
                     "bytes": base64.b64encode(tt.to_bytes()).decode()})
    _dump("spill", {"labels": list(res.partial_labels), "dims": list(res.partial_dims),
                    "partials": [[list(k), _f(v)] for k, v in sorted(res.partials.items())],
                    "spill_b64": base64.b64encode(raw).decode(), "tensors": tens})


SECTIONS = {
    "perm": section_perm, "contract": section_contract, "split": section_split, "c0": section_c0,
    "plans": section_plans, "sliced": section_sliced, "reuse": section_reuse, "pairs": section_pairs,
    "spill": section_spill, "plan_c4_reuse": section_plan_c4_reuse,
    "split_order": section_split_order,
}

if __name__ == "__main__":
    todo = sys.argv[1:] or list(SECTIONS)
    for name in todo:
        t0 = time.time()
        SECTIONS[name]()
        print(f"[{name}] {time.time() - t0:.1f}s", flush=True)
