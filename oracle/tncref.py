"""CPU oracle: numpy restatement of the reference hot path.

TEST INFRASTRUCTURE ONLY.  Imported exclusively by ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py``, and only as the checker / CPU baseline -- never by the
product package ``paper_2504_09186_b200``.

It restates, function by function, the numeric path of the reference package
``tncsim`` (pure Python + numpy, ``/root/reference/pkg/src/tncsim``).  Parity
of this restatement with the real reference is pinned by the golden vectors
in ``tests/golden`` produced by ``oracle/gen_golden.py`` (which imports the
reference in the build container) -- see ``tests/test_oracle_golden.py``.

Tensors are plain tuples ``(labels, dims, flat_array)``: row-major over the
labels, last label fastest, complex64 / complex128 (reference tensor.py:3-9).
"""

from __future__ import annotations

import itertools
from typing import Sequence

import numpy as np

Tensor = tuple  # (labels: tuple[str], dims: tuple[int], data: np.ndarray)


def _prod(xs) -> int:
    out = 1
    for x in xs:
        out *= x
    return out


# -- reference tensor.py:182-249 (PermutationPlan, _case_bucket, classify_permutation) --
def classify(src: Sequence[tuple[str, int]], tgt: Sequence[tuple[str, int]]):
    """(stride, offset, case, chunk, src_step) of reordering src -> tgt."""
    if sorted(src) != sorted(tgt):
        raise ValueError("not a permutation")
    rank = len(src)
    if rank == 0:
        return (0, 1, "scalar-fallback", 1, 1)
    pos = {l: p for p, (l, _) in enumerate(src)}
    p_last = pos[tgt[-1][0]]
    offset = rank - p_last
    stride = 1
    while stride < rank and pos[tgt[-stride - 1][0]] == pos[tgt[-stride][0]] - 1:
        stride += 1
    chunk = _prod(d for _, d in tgt[rank - stride:])
    src_step = _prod(d for _, d in src[p_last + 1:])
    if tuple(src) == tuple(tgt):
        case = "contiguous"
    elif chunk == 2 and offset == 1:
        case = "[2,1]"
    elif chunk == 4 and offset in (1, 2):
        case = f"[4,{offset}]"
    elif chunk >= 8 and offset in (1, 2, 4):
        case = f"[>=8,{offset}]"
    else:
        case = "scalar-fallback"
    return (stride, offset, case, chunk, src_step)


# -- reference tensor.py:252-274 (permute: offset table + gather) --
def permute(t: Tensor, target: Sequence[str]) -> Tensor:
    labels, dims, data = t
    dim_of = dict(zip(labels, dims))
    tgt = [(l, dim_of[l]) for l in target]
    stride, _, case, chunk, src_step = classify(list(zip(labels, dims)), tgt)
    if len(labels) == 0 or case == "contiguous":
        return (tuple(target), tuple(d for _, d in tgt), data.copy())
    step = 1
    src_strides = {}
    for l, d in reversed(list(zip(labels, dims))):
        src_strides[l] = step
        step *= d
    bases = np.zeros(1, dtype=np.int64)
    for l, d in tgt[: len(labels) - stride]:
        bases = (bases[:, None] + np.arange(d, dtype=np.int64)[None, :] * src_strides[l]).reshape(-1)
    run = np.arange(chunk, dtype=np.int64) * src_step
    offsets = (bases[:, None] + run[None, :]).reshape(-1)
    return (tuple(target), tuple(d for _, d in tgt), data[offsets])


# -- reference tensor.py:277-292 (project) --
def project(t: Tensor, assignment: dict[str, int]) -> Tensor:
    labels, dims, data = t
    if not any(l in assignment for l in labels):
        return t
    sel = tuple(assignment[l] if l in assignment else slice(None) for l in labels)
    kept = [(l, d) for l, d in zip(labels, dims) if l not in assignment]
    arr = np.ascontiguousarray(data.reshape(dims)[sel]).reshape(-1)
    return (tuple(l for l, _ in kept), tuple(d for _, d in kept), arr)


# -- reference contract.py:58-117 (_split_legs, contraction_shape, ttgt_plan) --
def ttgt(a_labels, a_dims, b_labels, b_dims):
    bdim = dict(zip(b_labels, b_dims))
    free_a, common = [], []
    for l, d in zip(a_labels, a_dims):
        if l in bdim:
            if bdim[l] != d:
                raise ValueError(f"shared label {l!r} dim mismatch")
            common.append((l, d))
        else:
            free_a.append((l, d))
    cl = {l for l, _ in common}
    free_b = [(l, d) for l, d in zip(b_labels, b_dims) if l not in cl]
    m = _prod(d for _, d in free_a)
    k = _prod(d for _, d in common)
    n = _prod(d for _, d in free_b)
    if k * n != m * k:
        b_mult = k * n > m * k
    else:
        fa = a_labels[0] if a_labels else ""
        fb = b_labels[0] if b_labels else ""
        b_mult = fb < fa
    if b_mult:
        a_tgt, b_tgt = common + free_a, free_b + common
    else:
        a_tgt, b_tgt = free_a + common, common + free_b
    return free_a, common, free_b, (m, k, n), b_mult, a_tgt, b_tgt


# -- reference contract.py:131-165 (_matmul, _panel_product, _finish, contract_pair) --
def _operands(a: Tensor, b: Tensor):
    free_a, common, free_b, (m, k, n), b_mult, a_tgt, b_tgt = ttgt(a[0], a[1], b[0], b[1])
    a2 = permute(a, [l for l, _ in a_tgt])[2]
    b2 = permute(b, [l for l, _ in b_tgt])[2]
    if b_mult:
        a2 = a2.reshape(k, m)
        b2 = b2.reshape(n, k)
    else:
        a2 = a2.reshape(m, k)
        b2 = b2.reshape(k, n)
    out_labels = tuple(l for l, _ in free_a + free_b)
    out_dims = tuple(d for _, d in free_a + free_b)
    return a2, b2, (m, k, n), b_mult, out_labels, out_dims


def _panel(a2, b2, lo, hi, b_mult):
    if b_mult:
        return np.matmul(b2[:, lo:hi], a2[lo:hi, :])
    return np.matmul(a2[:, lo:hi], b2[lo:hi, :])


def _finish(prod, b_mult, out_labels, out_dims) -> Tensor:
    if b_mult:
        prod = np.ascontiguousarray(prod.T)
    return (out_labels, out_dims, prod.reshape(-1))


def contract(a: Tensor, b: Tensor) -> Tensor:
    """contract_pair: permute both operands, one matmul, transpose if B multiplies."""
    a2, b2, (m, k, n), b_mult, ol, od = _operands(a, b)
    return _finish(_panel(a2, b2, 0, k, b_mult), b_mult, ol, od)


# -- reference contract.py:168-208 (split_common_contract) --
def split_common(a: Tensor, b: Tensor, blocks: int, group: int) -> Tensor:
    a2, b2, (m, k, n), b_mult, ol, od = _operands(a, b)
    panels = min(blocks * group, k)
    base = k // panels
    bounds = [i * base for i in range(panels)] + [k]
    parts = [_panel(a2, b2, bounds[i], bounds[i + 1], b_mult) for i in range(panels)]
    while len(parts) > 1:
        parts = [parts[i] + parts[i + 1] if i + 1 < len(parts) else parts[i] for i in range(0, len(parts), 2)]
    return _finish(parts[0], b_mult, ol, od)


# -- reference execute.py:119-178 (_Engine.fetch / run_range step loop, "single" = c64 at rest, c128 in flight)
def run_range(leaves: Sequence[Tensor], steps, n_leaves: int, lo: int, hi: int,
              assignment: dict[str, int], values: dict, precision: str = "single") -> dict:
    """steps: sequence of (lhs, rhs, result) SSA triples (1-based lo..hi inclusive)."""
    single = precision == "single"
    for pos in range(lo - 1, hi):
        lhs_ref, rhs_ref, res = steps[pos]
        lhs = project(leaves[lhs_ref], assignment) if lhs_ref < n_leaves else values[lhs_ref]
        rhs = project(leaves[rhs_ref], assignment) if rhs_ref < n_leaves else values[rhs_ref]
        if single:
            lhs = (lhs[0], lhs[1], lhs[2].astype(np.complex128))
            rhs = (rhs[0], rhs[1], rhs[2].astype(np.complex128))
        out = contract(lhs, rhs)
        for ref in (lhs_ref, rhs_ref):
            if ref >= n_leaves:
                values.pop(ref, None)
        values[res] = out
    if single:
        for key, val in list(values.items()):
            values[key] = (val[0], val[1], val[2].astype(np.complex64))
    return values


def cast_leaves(leaves: Sequence[Tensor], precision: str = "single") -> list[Tensor]:
    dt = np.complex64 if precision == "single" else np.complex128
    return [(l, d, np.asarray(x).astype(dt)) for l, d, x in leaves]


# -- reference execute.py:115-116, 204-230 (_enumerate, run_sliced) --
def run_sliced(leaves, steps, n_leaves: int, slice_labels: Sequence[str], slice_dims: Sequence[int],
               precision: str = "single", keys: Sequence[tuple] | None = None):
    """Sum over slice assignments (itertools.product order) of full runs.
    Returns (total tensor, {key: root tensor})."""
    root = steps[-1][2]
    partials = {}
    acc = None
    todo = keys if keys is not None else itertools.product(*[range(d) for d in slice_dims])
    for key in todo:
        vals = run_range(leaves, steps, n_leaves, 1, len(steps), dict(zip(slice_labels, key)), {}, precision)
        out = vals[root]
        partials[tuple(key)] = out
        acc = out if acc is None else (out[0], out[1], acc[2] + out[2])
    return acc, partials


# -- reference execute.py:97-112 (hierarchical_reduce) --
def hierarchical_reduce(vals: Sequence, group_size: int = 256):
    groups = []
    for lo in range(0, len(vals), group_size):
        acc = vals[lo]
        for v in vals[lo + 1: lo + group_size]:
            acc = acc + v
        groups.append(acc)
    total = groups[0]
    for v in groups[1:]:
        total = total + v
    return total


# -- reference execute.py:233-313 (_run_program: spindle program interpreter) --
def run_program(leaves, steps, n_leaves: int, actions, outer_assignment: dict[str, int],
                dep_sets: dict[str, set], precision: str = "single"):
    """actions: list of dicts in the reference's ReuseAction.to_obj() format."""
    root = steps[-1][2]
    values: dict = {}
    cps: dict = {}
    bufs: dict = {}
    parked = False
    acc = None
    for act in actions:
        kind = act["kind"]
        if kind == "RUN":
            asn = dict(outer_assignment)
            asn.update(act["assignment"])
            values = run_range(leaves, steps, n_leaves, act["lo"], act["hi"], asn, values, precision)
            parked = False
        elif kind == "CHECKPOINT":
            cps[act["buf"]] = dict(values)
        elif kind == "RESTORE":
            if root in values and not parked:
                acc = values[root][2] if acc is None else acc + values[root][2]
            values = dict(cps[act["buf"]])
            parked = False
        elif kind == "FREE":
            del cps[act["buf"]]
        elif kind == "STORE_PARTIAL":
            bufs.setdefault(act["buf"], []).append(dict(values))
            parked = True
        elif kind == "MERGE":
            parts = bufs.pop(act["buf"])
            dep = dep_sets[act["index"]]
            merged = {}
            for ssa, first in parts[0].items():
                if ssa in dep:
                    data = first[2].copy()
                    for p in parts[1:]:
                        data = data + p[ssa][2]
                    merged[ssa] = (first[0], first[1], data)
                else:
                    merged[ssa] = first
            values = merged
            parked = False
        else:
            raise ValueError(kind)
    if root in values:
        acc = values[root][2] if acc is None else acc + values[root][2]
    return acc


# -- complex128 state vector (independent amplitude check, tests/oracles.py:76-104) --
def statevector(n_qubits: int, gates) -> np.ndarray:
    """Vectorised complex128 state vector; qubit q occupies bit q.
    ``gates``: iterable of (qubits tuple, unitary matrix)."""
    psi = np.zeros(2 ** n_qubits, dtype=np.complex128)
    psi[0] = 1.0
    # axis j of the reshaped state = qubit n-1-j (bit q)
    psi = psi.reshape((2,) * n_qubits)
    for qubits, u in gates:
        axes = [n_qubits - 1 - q for q in qubits]
        k = len(qubits)
        u = np.asarray(u, dtype=np.complex128).reshape((2,) * (2 * k))
        psi = np.tensordot(u, psi, axes=(list(range(k, 2 * k)), axes))
        psi = np.moveaxis(psi, list(range(k)), axes)
    return psi.reshape(-1)
