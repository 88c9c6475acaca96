"""Device executor: step loop, slice loops, reuse programs, slice scheduler.

Mirrors the reference's ``tncsim.execute`` API (``execute.py:52-372``):
``RunStats``, ``ReductionTopology``, ``RunResult``, ``hierarchical_reduce``,
``run_direct``, ``run_sliced``, ``run_reuse`` -- same counters (exact integer
``multiplies`` / ``bytes_moved`` / ``bytes_peak``), same slice enumeration
order, same reduction order -- with every contraction on the GPU.

Additions for the B200 hot path (north-star item 3):

* projection is a zero-copy strided view (``tensor.project``), so a slice
  never copies its leaves;
* :class:`SliceExecutor` evaluates the slice-invariant steps once (steps that
  no sliced label reaches, ``reuse.dependent_results``) and per slice only
  re-runs the dependent ones, accumulating the root on device in slice order;
* ``run_open`` contracts networks with open legs (correlated amplitudes) and
  returns the output tensor in a requested leg order.

Precision: "single" keeps complex64 everywhere (fp32 / 3xTF32 arithmetic) --
the reference instead upcasts to complex128 in flight (``execute.py:154-158``);
results agree within the rel-L2 <= 1e-5 contract.  "double" is complex128
with fp64 arithmetic (CUDA cores).
"""

from __future__ import annotations

import itertools
import json
import struct
import time
from dataclasses import dataclass
from typing import Callable, Iterable, Sequence

import torch

from . import _lib
from .contract import contract_into, plan_for
from .errors import MemoryBudgetError, PlanningError, TensorError, TncError
from .labels import Index, multiply_cost, product
from .network import TensorNetwork
from .reuse import CHECKPOINT, FREE, MERGE, RESTORE, RUN, STORE_PARTIAL, ReuseSchedule, dependent_results
from .slicing import SliceSpec
from .tensor import DTYPES, ELEMENT_BYTES, DenseTensor, permute, project
from .tree import ContractionTree, LinearSchedule, linearize


@dataclass
class RunStats:
    multiplies: int = 0
    bytes_peak: int = 0
    bytes_moved: int = 0
    wall_time: float = 0.0
    subtasks_done: int = 0

    def to_obj(self):
        return {"multiplies": self.multiplies, "bytes_peak": self.bytes_peak, "bytes_moved": self.bytes_moved,
                "wall_time": self.wall_time, "subtasks_done": self.subtasks_done}


@dataclass(frozen=True)
class ReductionTopology:
    """Groups of ``group_size`` are summed first, then the group sums."""

    group_size: int = 256

    def __post_init__(self) -> None:
        if self.group_size < 1:
            raise TncError("group_size must be >= 1")

    def levels(self, n: int) -> list[int]:
        out = [n]
        while out[-1] > 1:
            out.append(-(-out[-1] // self.group_size))
        return out


@dataclass
class RunResult:
    value: complex
    stats: RunStats
    partials: dict
    partial_labels: tuple[str, ...]
    partial_dims: tuple[int, ...]


# -- partial-result spill files (reference execute.py:468-506) ----------------

SPILL_MAGIC = b"TNCPART1"


def write_partials(path: str, result: RunResult) -> None:
    """Binary spill of a run's per-slice partials, byte-compatible with the
    reference (``execute.py:473-490``): magic, u32 header length, JSON header
    ``{"labels", "dims"}``, u64 count, then ``(u64 code, f64 re, f64 im)``
    records in sorted key order, ``code = code * dim + value`` (first label most
    significant, ``execute.py:481-484``)."""
    head = json.dumps({"labels": list(result.partial_labels), "dims": list(result.partial_dims)}).encode()
    with open(path, "wb") as fh:
        fh.write(SPILL_MAGIC)
        fh.write(struct.pack("<I", len(head)))
        fh.write(head)
        fh.write(struct.pack("<Q", len(result.partials)))
        for key in sorted(result.partials):
            code = 0
            for v, d in zip(key, result.partial_dims):
                code = code * d + v
            val = complex(result.partials[key])
            fh.write(struct.pack("<Qdd", code, val.real, val.imag))


def read_partials(path: str) -> tuple[tuple[str, ...], tuple[int, ...], dict]:
    """Inverse of :func:`write_partials` (reference ``execute.py:493-506``);
    raises ``TncError`` on a foreign file."""
    with open(path, "rb") as fh:
        if fh.read(len(SPILL_MAGIC)) != SPILL_MAGIC:
            raise TncError(f"{path}: not a partials spill file")
        (hlen,) = struct.unpack("<I", fh.read(4))
        head = json.loads(fh.read(hlen).decode())
        labels = tuple(head["labels"])
        dims = tuple(head["dims"])
        (count,) = struct.unpack("<Q", fh.read(8))
        partials = {}
        for _ in range(count):
            code, re, im = struct.unpack("<Qdd", fh.read(24))
            key = []
            for d in reversed(dims):
                key.append(code % d)
                code //= d
            partials[tuple(reversed(key))] = complex(re, im)
    return labels, dims, partials


def hierarchical_reduce(partials: Sequence, topo: ReductionTopology):
    """Fixed-order two-level sum (reference ``execute.py:97-112``)."""
    if len(partials) == 0:
        raise TncError("nothing to reduce")
    vals = list(partials)
    g = topo.group_size
    sums = []
    for lo in range(0, len(vals), g):
        acc = vals[lo]
        for v in vals[lo + 1: lo + g]:
            acc = acc + v
        sums.append(acc)
    total = sums[0]
    for v in sums[1:]:
        total = total + v
    return total


def _slice_keys(dims: Sequence[int]) -> Iterable[tuple[int, ...]]:
    return itertools.product(*[range(d) for d in dims])


def _leaves_at(tensors: Sequence[DenseTensor], precision: str) -> list[DenseTensor]:
    """Leaves at storage precision on the device (reference ``execute.py:128``
    rounds them to the run precision).  Leaves that need a copy are converted
    in one batched device pass (one concatenate, one cast) and handed out as
    views: a circuit network has hundreds of tiny leaves, and per-leaf casts
    made the host side of an end-to-end call launch-bound."""
    out: list[DenseTensor | None] = list(tensors)
    todo = [i for i, t in enumerate(tensors) if not (t.precision == precision and t.data.is_cuda)]
    if not todo:
        return list(tensors)
    dev = torch.device("cuda", torch.cuda.current_device())
    host = [i for i in todo if not tensors[i].data.is_cuda]
    on_dev = [i for i in todo if tensors[i].data.is_cuda]
    parts = []
    if host:  # host-resident leaves: one host-side concatenation, one upload
        hcat = torch.cat([tensors[i].data.reshape(-1) for i in host])
        parts.append(hcat.to(dev, non_blocking=hcat.is_pinned()))
    if on_dev:
        parts.append(torch.cat([tensors[i].data.reshape(-1) for i in on_dev]))
    todo = host + on_dev
    flat = (parts[0] if len(parts) == 1 else torch.cat(parts)).to(DTYPES[precision])
    pos = 0
    for i in todo:
        t = tensors[i]
        n = t.size
        out[i] = DenseTensor.__new__(DenseTensor)._init_raw(t.indices, flat[pos:pos + n].view(t.dims))
        pos += n
    return out


MIN_ABSORB_RUN = 2  # gates per fused run (a single gate stays a plain step)


def absorb_runs(s: LinearSchedule, sliced: frozenset = frozenset(), positions=None) -> dict[int, list[int]]:
    """Stem chains the fused absorb kernel (K4) can take: maximal runs of
    consecutive schedule positions where each step contracts the previous
    step's result (as ``lhs``, so the reference order free_T ++ free_G holds)
    with a leaf gate (``rhs``: rank 4, extent-2 legs, no sliced leg, sharing
    exactly two legs with the running tensor), and the running tensor has
    rank >= 13 (after projecting the sliced labels).  These are the
    absorption chains of reference ``tree.py:278-330`` (``_detect_stems``) in
    the order ``linearize`` keeps them.  ``positions`` restricts the runs to
    the steps a caller executes.  Returns {first position: [positions]}."""
    from .fusion import MIN_FUSED_RANK

    allowed = set(range(len(s.steps))) if positions is None else set(positions)

    def rank(ref):
        return sum(1 for ix in s.indices_of(ref) if ix.label not in sliced)

    def gate_ok(pos, run_ref):
        st = s.steps[pos]
        if pos not in allowed or st.lhs != run_ref or st.rhs >= s.n_leaves:
            return False
        g = s.indices_of(st.rhs)
        if len(g) != 4 or any(ix.dim != 2 or ix.label in sliced for ix in g):
            return False
        t = {ix.label for ix in s.indices_of(st.lhs) if ix.label not in sliced}
        if sum(1 for ix in g if ix.label in t) != 2:
            return False
        return all(ix.dim == 2 for ix in s.indices_of(st.lhs)) and rank(st.lhs) >= MIN_FUSED_RANK

    runs: dict[int, list[int]] = {}
    pos = 0
    while pos < len(s.steps):
        st = s.steps[pos]
        if gate_ok(pos, st.lhs):
            run = [pos]
            while run[-1] + 1 < len(s.steps) and gate_ok(run[-1] + 1, s.steps[run[-1]].result):
                run.append(run[-1] + 1)
            if len(run) >= MIN_ABSORB_RUN:
                runs[pos] = run
            pos = run[-1] + 1
        else:
            pos += 1
    return runs


def _fuse_enabled() -> bool:
    import os

    return os.environ.get("TNC_FUSE_ABSORB", "1") not in ("0", "")


class Engine:
    """Per-run device state: leaves at storage precision, counters."""

    def __init__(self, net: TensorNetwork, precision: str = "single", max_intermediate_bytes: int | None = None):
        if precision not in DTYPES:
            raise TensorError(f"unsupported device precision {precision!r}")
        _lib.ensure_device()
        self.precision = precision
        self.rate = ELEMENT_BYTES[precision]
        self.cap = max_intermediate_bytes
        self.leaves = _leaves_at(net.tensors, precision)

    def fetch(self, s: LinearSchedule, ref: int, assignment: dict[str, int], values: dict) -> DenseTensor:
        if ref < s.n_leaves:
            return project(self.leaves[ref], assignment)
        return values[ref]

    def contract(self, lhs: DenseTensor, rhs: DenseTensor) -> DenseTensor:
        plan = plan_for(lhs.indices, lhs.data.stride(), rhs.indices, rhs.data.stride(),
                        _lib.C128 if self.precision == "double" else _lib.C64)
        return DenseTensor.__new__(DenseTensor)._init_raw(plan.out_indices, contract_into(plan, lhs.data, rhs.data))

    def absorb(self, s: LinearSchedule, run: list[int], assignment: dict[str, int], values: dict) -> DenseTensor:
        """One fused K4 launch sequence for a stem run (see ``absorb_runs``):
        the running tensor absorbs the run's leaf gates; same result legs as the
        per-step contractions."""
        from .fusion import absorb_chain

        t = self.fetch(s, s.steps[run[0]].lhs, assignment, values)
        gates = [self.fetch(s, s.steps[p].rhs, assignment, values) for p in run]
        if self.precision != "single" or not t.data.is_contiguous():
            out = t
            for g in gates:
                out = self.contract(out, g)
            return out
        return absorb_chain(t, gates)

    def absorb_runs_for(self, s: LinearSchedule, sliced: frozenset, positions=None) -> dict[int, list[int]]:
        key = (id(s), sliced, None if positions is None else tuple(positions))
        cache = self.__dict__.setdefault("_runs", {})
        if key not in cache:
            cache[key] = absorb_runs(s, sliced, positions) if _fuse_enabled() and self.precision == "single" else {}
        return cache[key]

    def run_range(self, s: LinearSchedule, lo: int, hi: int, assignment: dict[str, int], values: dict,
                  stats: RunStats, aux_bytes: int = 0, cache: dict | None = None,
                  invariant: set | frozenset = frozenset()) -> None:
        """Steps lo..hi (1-based, inclusive) -- reference ``execute.py:137-178``.

        ``invariant`` (results no sliced label reaches, see ``ReuseRunner``)
        are never recomputed: a result some dependent step consumes is taken
        from ``cache``; the others only feed further invariant steps and are
        skipped."""
        rate = self.rate
        live = sum(v.size for v in values.values())
        runs = self.absorb_runs_for(s, frozenset(assignment)) if self.cap is None and not invariant else {}
        skip_to = -1
        for pos in range(lo - 1, hi):
            if pos < skip_to:
                continue
            step = s.steps[pos]
            if step.result in invariant:
                if step.result in cache:
                    values[step.result] = cache[step.result]
                    live += values[step.result].size
                continue
            run = runs.get(pos)
            if run is not None and run[-1] < hi:
                out = self.absorb(s, run, assignment, values)
                cur = [ix for ix in s.indices_of(s.steps[run[0]].lhs) if ix.label not in assignment]
                for p in run:
                    g = [ix for ix in s.indices_of(s.steps[p].rhs) if ix.label not in assignment]
                    stats.multiplies += multiply_cost(cur, g)
                    cur_set = {ix.label for ix in g}
                    nxt = [ix for ix in cur if ix.label not in cur_set] + \
                          [ix for ix in g if ix.label not in {c.label for c in cur}]
                    stats.bytes_moved += (product(ix.dim for ix in cur) + product(ix.dim for ix in g)
                                          + product(ix.dim for ix in nxt)) * rate
                    cur = nxt
                first = s.steps[run[0]].lhs
                if first >= s.n_leaves and first in values:
                    live -= values[first].size
                    del values[first]
                values[s.steps[run[-1]].result] = out
                live += out.size
                stats.bytes_peak = max(stats.bytes_peak, live * rate + aux_bytes)
                skip_to = run[-1] + 1
                continue
            lhs = self.fetch(s, step.lhs, assignment, values)
            rhs = self.fetch(s, step.rhs, assignment, values)
            out_size = _result_size(lhs.indices, rhs.indices)
            if self.cap is not None and out_size * rate > self.cap:
                raise MemoryBudgetError(
                    f"step {pos + 1} produces a {out_size * rate}-byte intermediate over the {self.cap}-byte cap")
            out = self.contract(lhs, rhs)
            stats.multiplies += multiply_cost(lhs.indices, rhs.indices)
            stats.bytes_moved += (lhs.size + rhs.size + out.size) * rate
            for ref in (step.lhs, step.rhs):
                if ref >= s.n_leaves and ref in values:
                    live -= values[ref].size
                    del values[ref]
            values[step.result] = out
            live += out.size
            stats.bytes_peak = max(stats.bytes_peak, live * rate + aux_bytes)


def _result_size(a: Sequence[Index], b: Sequence[Index]) -> int:
    la = {ix.label for ix in a}
    lb = {ix.label for ix in b}
    return product(ix.dim for ix in a if ix.label not in lb) * product(ix.dim for ix in b if ix.label not in la)


def _init_raw(self, indices, data):
    self.indices = tuple(indices)
    self.data = data
    return self


DenseTensor._init_raw = _init_raw  # internal fast constructor (no validation / copies)


def _sync_value(t: DenseTensor) -> complex:
    return t.value()


def run_direct(net: TensorNetwork, t: ContractionTree, precision: str = "double",
               max_intermediate_bytes: int | None = None) -> tuple[complex, RunStats]:
    """Contract a closed network; ``multiplies`` equals the tree's total cost."""
    s = linearize(t)
    eng = Engine(net, precision, max_intermediate_bytes)
    stats = RunStats()
    t0 = time.perf_counter()
    values: dict = {}
    eng.run_range(s, 1, len(s.steps), {}, values, stats)
    value = values[s.steps[-1].result].value() if s.steps else eng.leaves[0].value()
    stats.wall_time = time.perf_counter() - t0
    stats.subtasks_done = 1
    return value, stats


def run_sliced(net: TensorNetwork, t: ContractionTree, spec: SliceSpec, precision: str = "double",
               max_intermediate_bytes: int | None = None) -> RunResult:
    """Sum of projected contractions over every slice, in itertools.product
    order over ``spec.entries`` (first label most significant)."""
    s = linearize(t)
    eng = Engine(net, precision, max_intermediate_bytes)
    stats = RunStats()
    t0 = time.perf_counter()
    labels = spec.labels
    dims = spec.dims
    root = s.steps[-1].result if s.steps else 0
    partials: dict = {}
    acc = None
    for key in _slice_keys(dims):
        asn = dict(zip(labels, key))
        values: dict = {}
        eng.run_range(s, 1, len(s.steps), asn, values, stats)
        val = values[root].value() if s.steps else project(eng.leaves[0], asn).value()
        partials[key] = val
        acc = val if acc is None else acc + val
        stats.subtasks_done += 1
    stats.wall_time = time.perf_counter() - t0
    return RunResult(acc, stats, partials, labels, dims)


def _add(a: DenseTensor, b: DenseTensor) -> DenseTensor:
    """Fresh a + b (same legs) through the device axpy kernel."""
    out = a.data.contiguous().clone() if a.data.is_contiguous() else a.data.contiguous()
    if out.data_ptr() == a.data.data_ptr():
        out = out.clone()
    bd = b.data.contiguous()
    _lib.check(_lib.load().tnc_axpy(a.dtype_code, out.numel(), bd.data_ptr(), out.data_ptr(), _lib.stream_ptr()))
    return DenseTensor.__new__(DenseTensor)._init_raw(a.indices, out)


def _run_program(eng: Engine, rs: ReuseSchedule, outer: dict[str, int], dep_sets: dict[str, set[int]],
                 mem_budget: int | None, open_root: bool = False, cache: dict | None = None,
                 invariant: set | frozenset = frozenset()):
    """Device interpreter of a reuse action program (reference
    ``execute.py:233-313``).  Tensors are immutable, so CHECKPOINT / STORE
    keep references; MERGE sums the dependent values with the axpy kernel.

    ``open_root`` (extension: the reference reduces scalar roots only) sums
    tensor-valued roots of an open-output network on the device instead."""
    s = rs.schedule
    stats = RunStats()
    values: dict = {}
    cps: dict = {}
    bufs: dict = {}
    parked = False
    root = s.steps[-1].result
    acc = None

    def add_root(v):
        nonlocal acc
        if not open_root:
            v = v.value()
            acc = v if acc is None else acc + v
        elif acc is None:
            acc = DenseTensor.__new__(DenseTensor)._init_raw(v.indices, v.data.contiguous().clone())
        else:
            _lib.check(_lib.load().tnc_axpy(acc.dtype_code, acc.size, v.data.contiguous().data_ptr(),
                                            acc.data.data_ptr(), _lib.stream_ptr()))

    def aux_bytes() -> int:
        seen = {}
        for pool in itertools.chain(cps.values(), (p for v in bufs.values() for p in v)):
            for tensor in pool.values():
                seen[id(tensor)] = tensor.nbytes
        return sum(seen.values())

    for act in rs.actions:
        if act.kind == RUN:
            asn = dict(outer)
            asn.update(dict(act.assignment))
            eng.run_range(s, act.lo, act.hi, asn, values, stats, aux_bytes(), cache, invariant)
            parked = False
        elif act.kind == CHECKPOINT:
            snap = dict(values)
            size = sum(v.nbytes for v in snap.values())
            if mem_budget is not None and size > mem_budget:
                label = rs.nested[act.buf].index.label
                raise MemoryBudgetError(f"checkpoint at fork of index {label!r} needs {size} B, budget {mem_budget} B")
            cps[act.buf] = snap
        elif act.kind == RESTORE:
            if root in values and not parked:
                add_root(values[root])
            values = dict(cps[act.buf])
            parked = False
        elif act.kind == FREE:
            del cps[act.buf]
        elif act.kind == STORE_PARTIAL:
            bufs.setdefault(act.buf, []).append(dict(values))
            parked = True
        elif act.kind == MERGE:
            parts = bufs.pop(act.buf)
            if len(parts) != act.dim:
                raise PlanningError(f"merge expected {act.dim} partials, found {len(parts)}")
            dep = dep_sets[act.index]
            merged = {}
            for ssa, first in parts[0].items():
                if ssa in dep:
                    total = first
                    for p in parts[1:]:
                        total = _add(total, p[ssa])
                    merged[ssa] = total
                else:
                    merged[ssa] = first
            values = merged
            parked = False
        else:
            raise PlanningError(f"unknown action {act.kind}")
    if root in values:
        add_root(values[root])
    if acc is None:
        raise PlanningError("reuse program produced no final value")
    stats.subtasks_done = rs.nested_count
    return acc, stats


def run_reuse(net: TensorNetwork, t: ContractionTree, rs: ReuseSchedule, workers: int = 1,
              precision: str = "double", group_size: int = 256, mem_budget: int | None = None,
              max_intermediate_bytes: int | None = None) -> RunResult:
    """Run the reuse program once per outer-slice assignment; reduce the
    outer partials hierarchically in enumeration order.  ``workers`` is
    accepted for API parity: one device executes the programs in order
    (multi-GPU partitioning lives in ``distributed``)."""
    eng = Engine(net, precision, max_intermediate_bytes)
    t0 = time.perf_counter()
    labels = tuple(e.index.label for e in rs.outer)
    dims = tuple(e.index.dim for e in rs.outer)
    deps = {e.index.label: dependent_results(rs.schedule, e.index.label) for e in rs.nested}
    keys = list(_slice_keys(dims))
    results = []
    stats = RunStats()
    for key in keys:
        val, st = _run_program(eng, rs, dict(zip(labels, key)), deps, mem_budget)
        results.append(val)
        stats.multiplies += st.multiplies
        stats.bytes_moved += st.bytes_moved
        stats.bytes_peak = max(stats.bytes_peak, st.bytes_peak)
        stats.subtasks_done += st.subtasks_done
    value = hierarchical_reduce(results, ReductionTopology(group_size))
    stats.wall_time = time.perf_counter() - t0
    return RunResult(value, stats, dict(zip(keys, results)), labels, dims)


def run_reuse_open(net: TensorNetwork, t: ContractionTree, rs: ReuseSchedule,
                   output_order: Sequence[str] | None = None, precision: str = "single",
                   mem_budget: int | None = None) -> DenseTensor:
    """Open-output spindle reuse: the reuse program of ``rs`` run once per
    outer assignment, tensor roots summed on the device (outer programs in
    enumeration order), permuted to ``output_order``.  Extension of
    ``run_reuse`` (reference ``execute.py:316-372`` reduces scalar roots)."""
    eng = Engine(net, precision)
    labels = tuple(e.index.label for e in rs.outer)
    dims = tuple(e.index.dim for e in rs.outer)
    deps = {e.index.label: dependent_results(rs.schedule, e.index.label) for e in rs.nested}
    total = None
    for key in _slice_keys(dims):
        part, _ = _run_program(eng, rs, dict(zip(labels, key)), deps, mem_budget, open_root=True)
        if total is None:
            total = part
        else:
            _lib.check(_lib.load().tnc_axpy(total.dtype_code, total.size, part.data.contiguous().data_ptr(),
                                            total.data.data_ptr(), _lib.stream_ptr()))
    if output_order is None:
        return total
    by = {ix.label: ix for ix in total.indices}
    return permute(total, [by[l] for l in output_order])


def _zeros_root(eng: Engine, s: LinearSchedule) -> DenseTensor:
    """A zero tensor shaped like the schedule's root (open legs are never
    sliced), without evaluating anything: what a rank that owns no slices
    contributes to the all-reduce."""
    idx = tuple(s.steps[-1].indices) if s.steps else ()
    data = torch.zeros(tuple(ix.dim for ix in idx), dtype=DTYPES[eng.precision], device="cuda")
    return DenseTensor.__new__(DenseTensor)._init_raw(idx, data)


class ReuseRunner:
    """Spindle-reuse scheduler for open outputs on one device: the reuse
    program of ``rs`` (reference ``reuse.py:298-514`` / ``execute.py:233-313``)
    run per outer assignment, on top of the slice-invariant cache of
    ``SliceExecutor`` (steps no sliced label reaches run once in
    :meth:`prepare`).  A program covers prod(nested dims) slices and runs the
    steps after each MERGE once for all of them."""

    def __init__(self, net: TensorNetwork, rs: ReuseSchedule, precision: str = "single",
                 output_order: Sequence[str] | None = None, mem_budget: int | None = None):
        self.rs = rs
        self.s = rs.schedule
        self.eng = Engine(net, precision)
        self.output_order = list(output_order) if output_order is not None else None
        self.mem_budget = mem_budget
        labels = [e.index.label for e in rs.outer] + [e.index.label for e in rs.nested]
        dep: set[int] = set()
        for label in labels:
            dep |= dependent_results(self.s, label)
        self.invariant_positions = [p for p, st in enumerate(self.s.steps) if st.result not in dep]
        self.invariant = frozenset(self.s.steps[p].result for p in self.invariant_positions)
        # invariant results a dependent step (or the root) consumes: the cache
        self.needed = set()
        for st in self.s.steps:
            if st.result in dep:
                self.needed.update(r for r in (st.lhs, st.rhs) if r in self.invariant)
        self.needed.add(self.s.steps[-1].result)
        self.deps = {e.index.label: dependent_results(self.s, e.index.label) for e in rs.nested}
        self.outer_labels = tuple(e.index.label for e in rs.outer)
        self.outer_dims = tuple(e.index.dim for e in rs.outer)
        self.slices_per_program = product(e.index.dim for e in rs.nested)
        self.n_programs = product(self.outer_dims)
        self.cache: dict[int, DenseTensor] | None = None
        self.stats = RunStats()

    def prepare(self) -> None:
        """Evaluate every slice-invariant step once; keep the results that a
        dependent step consumes (the programs never recompute invariant
        steps: ``Engine.run_range(..., invariant=...)``)."""
        values: dict = {}
        eng, s = self.eng, self.s
        for p in self.invariant_positions:
            st = s.steps[p]
            lhs, rhs = eng.fetch(s, st.lhs, {}, values), eng.fetch(s, st.rhs, {}, values)
            out = eng.contract(lhs, rhs)
            self.stats.multiplies += multiply_cost(lhs.indices, rhs.indices)
            for ref in (st.lhs, st.rhs):
                if ref >= s.n_leaves and ref not in self.needed:
                    values.pop(ref, None)
            values[st.result] = out
        self.cache = {k: v for k, v in values.items() if k in self.needed}

    def outer_assignment(self, program_id: int) -> dict[str, int]:
        """Mixed radix over the outer labels, first label most significant."""
        out, rem = {}, program_id
        for label, d in zip(reversed(self.outer_labels), reversed(self.outer_dims)):
            out[label] = rem % d
            rem //= d
        return out

    def run_program(self, program_id: int) -> DenseTensor:
        if self.cache is None:
            self.prepare()
        root, st = _run_program(self.eng, self.rs, self.outer_assignment(program_id), self.deps,
                                self.mem_budget, open_root=True, cache=self.cache, invariant=self.invariant)
        self.stats.multiplies += st.multiplies
        self.stats.subtasks_done += self.slices_per_program
        return root

    def run(self, program_ids: Iterable[int], acc: DenseTensor | None = None) -> DenseTensor:
        total = acc
        for pid in program_ids:
            part = self.run_program(pid)
            if total is None:
                total = DenseTensor.__new__(DenseTensor)._init_raw(part.indices, part.data.contiguous().clone())
            else:
                _lib.check(_lib.load().tnc_axpy(total.dtype_code, total.size, part.data.contiguous().data_ptr(),
                                                total.data.data_ptr(), _lib.stream_ptr()))
        return total

    def finish(self, total: DenseTensor) -> DenseTensor:
        if self.output_order is None:
            return total
        by = {ix.label: ix for ix in total.indices}
        return permute(total, [by[l] for l in self.output_order])

    def zeros(self) -> DenseTensor:
        return _zeros_root(self.eng, self.s)

    @property
    def n_units(self) -> int:
        """Units of work the distributed scheduler deals out (programs)."""
        return self.n_programs


class SliceExecutor:
    """Slice scheduler with slice-invariant reuse and zero-copy projection.

    ``invariant`` steps (no sliced label reaches them) run once in
    :meth:`prepare`; :meth:`run_slice` re-runs only the dependent steps for one
    assignment.  The sum over slices accumulates on device in the order the
    caller feeds slice ids.
    """

    def __init__(self, net: TensorNetwork, schedule: LinearSchedule, spec: SliceSpec,
                 precision: str = "single", output_order: Sequence[str] | None = None):
        self.s = schedule
        self.spec = spec
        self.eng = Engine(net, precision)
        self.output_order = list(output_order) if output_order is not None else None
        dep: set[int] = set()
        for label in spec.labels:
            dep |= dependent_results(schedule, label)
        self.dependent_positions = [p for p, st in enumerate(schedule.steps) if st.result in dep]
        self.invariant_positions = [p for p, st in enumerate(schedule.steps) if st.result not in dep]
        self.cache: dict[int, DenseTensor] = {}
        self.stats = RunStats()
        self.root = schedule.steps[-1].result
        # multiplies per slice (exact, projected dims)
        dims = spec.dims_projected()
        self.multiplies_per_slice = sum(_proj_cost(schedule, p, dims) for p in self.dependent_positions)
        self.multiplies_invariant = sum(_proj_cost(schedule, p, dims) for p in self.invariant_positions)
        self._prepared = False

    def prepare(self) -> None:
        """Evaluate slice-invariant steps once (values kept only if a
        dependent step consumes them)."""
        needed = set()
        for p in self.dependent_positions:
            st = self.s.steps[p]
            needed.update((st.lhs, st.rhs))
        values: dict = {}
        eng, s = self.eng, self.s
        if eng.cap is not None:  # the reference step loop enforces the cap per step
            for p in self.invariant_positions:
                eng.run_range(s, p + 1, p + 1, {}, values, self.stats)
        else:
            # lean loop: hundreds of tiny steps, so no per-step accounting
            # (SSA values are consumed exactly once; the totals are exact)
            runs = eng.absorb_runs_for(s, frozenset(self.spec.labels), self.invariant_positions)
            skip_to = -1
            for p in self.invariant_positions:
                if p < skip_to:
                    continue
                st = s.steps[p]
                run = runs.get(p)
                if run is not None:  # stem chain -> one fused absorb
                    out = eng.absorb(s, run, {}, values)
                    if st.lhs >= s.n_leaves:
                        values.pop(st.lhs, None)
                    values[s.steps[run[-1]].result] = out
                    skip_to = run[-1] + 1
                    continue
                out = eng.contract(eng.fetch(s, st.lhs, {}, values), eng.fetch(s, st.rhs, {}, values))
                for ref in (st.lhs, st.rhs):
                    if ref >= s.n_leaves:
                        values.pop(ref, None)
                values[st.result] = out
            self.stats.multiplies += self.multiplies_invariant
        self.cache = {k: v for k, v in values.items() if k in needed or k == self.root}
        self._prepared = True

    def run_slice(self, assignment: dict[str, int]) -> DenseTensor:
        if not self._prepared:
            self.prepare()
        if not self.dependent_positions:
            return self.cache[self.root]
        values = dict(self.cache)
        eng = self.eng
        s = self.s
        runs = eng.absorb_runs_for(s, frozenset(self.spec.labels), self.dependent_positions)
        skip_to = -1
        for p in self.dependent_positions:
            if p < skip_to:
                continue
            step = s.steps[p]
            run = runs.get(p)
            if run is not None:  # stem chain -> one fused absorb
                out = eng.absorb(s, run, assignment, values)
                ref = step.lhs
                if ref >= s.n_leaves and ref in values and ref not in self.cache:
                    del values[ref]
                values[s.steps[run[-1]].result] = out
                skip_to = run[-1] + 1
                continue
            lhs = eng.fetch(s, step.lhs, assignment, values)
            rhs = eng.fetch(s, step.rhs, assignment, values)
            out = eng.contract(lhs, rhs)
            for ref in (step.lhs, step.rhs):
                if ref >= s.n_leaves and ref in values and ref not in self.cache:
                    del values[ref]
            values[step.result] = out
        self.stats.subtasks_done += 1
        self.stats.multiplies += self.multiplies_per_slice
        return values[self.root]

    def run(self, slice_ids: Iterable[int], acc: DenseTensor | None = None) -> DenseTensor:
        """Sum of the root over the given slice ids (device accumulate)."""
        total = acc
        for sid in slice_ids:
            part = self.run_slice(self.spec.assignment(sid))
            if total is None:
                total = DenseTensor.__new__(DenseTensor)._init_raw(part.indices, part.data.contiguous().clone())
            else:
                _lib.check(_lib.load().tnc_axpy(total.dtype_code, total.size, part.data.contiguous().data_ptr(),
                                                total.data.data_ptr(), _lib.stream_ptr()))
        return total

    def finish(self, total: DenseTensor) -> DenseTensor:
        if self.output_order is None:
            return total
        by = {ix.label: ix for ix in total.indices}
        return permute(total, [by[l] for l in self.output_order])

    def zeros(self) -> DenseTensor:
        return _zeros_root(self.eng, self.s)

    @property
    def n_units(self) -> int:
        """Units of work the distributed scheduler deals out (slices)."""
        return self.spec.n_subtasks


def _proj_cost(s: LinearSchedule, pos: int, dims: dict[str, int]) -> int:
    c = 1
    for ix in s.step_union(pos):
        c *= dims.get(ix.label, ix.dim)
    return c


def run_open(net: TensorNetwork, t: ContractionTree, spec: SliceSpec | None = None,
             output_order: Sequence[str] | None = None, precision: str = "single",
             slice_ids: Iterable[int] | None = None) -> DenseTensor:
    """Contract a network with open legs (sum over all / given slices) and
    return the output tensor, permuted to ``output_order`` if given."""
    s = linearize(t)
    spec = spec if spec is not None else SliceSpec([])
    ex = SliceExecutor(net, s, spec, precision, output_order)
    ids = range(spec.n_subtasks) if slice_ids is None else slice_ids
    return ex.finish(ex.run(ids))
