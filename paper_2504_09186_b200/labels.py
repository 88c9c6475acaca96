"""Host-side index algebra: labeled legs, permutation classes, TTGT shapes.

Pure integer bookkeeping shared by the device path (it decides the index
maps the kernels realise) and by the planners.  Semantics follow the
reference exactly because they fix the *index map* that must be bit-exact:

* :class:`Index`                    -- reference ``tensor.py:46-55``
* :func:`classify_permutation`      -- reference ``tensor.py:181-249``
* :func:`contraction_shape` etc.    -- reference ``contract.py:29-117``
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from typing import Sequence

from .errors import ContractionError, InvalidPermutationError, TensorError

#: Bucket names of the (chunk, offset) permutation taxonomy
#: (reference ``tensor.py:34-43``).
PERM_CASES = (
    "[2,1]",
    "[4,1]",
    "[4,2]",
    "[>=8,1]",
    "[>=8,2]",
    "[>=8,4]",
    "contiguous",
    "scalar-fallback",
)


@dataclass(frozen=True, order=True)
class Index:
    """One labeled leg; ``dim`` defaults to 2 (a qubit wire)."""

    label: str
    dim: int = 2

    def __post_init__(self) -> None:
        if self.dim < 1:
            raise TensorError(f"index {self.label!r} has dim {self.dim} < 1")


def product(dims) -> int:
    out = 1
    for d in dims:
        out *= d
    return out


# -- permutation classification ---------------------------------------------


@dataclass(frozen=True)
class PermutationPlan:
    """(stride, offset) class of a leg reordering.

    ``stride``: length of the longest target suffix that is an ascending
    consecutive run of source positions.  ``offset``: rank minus the source
    position of the last target leg.  ``chunk``: elements in one contiguous
    target run, ``src_step``: source step between its consecutive elements.
    """

    source_order: tuple[Index, ...]
    target_order: tuple[Index, ...]
    stride: int
    offset: int
    case_class: str
    chunk: int
    src_step: int


def _bucket(chunk: int, offset: int, identity: bool) -> str:
    if identity:
        return "contiguous"
    if offset == 1 and chunk == 2:
        return "[2,1]"
    if chunk == 4 and offset <= 2:
        return f"[4,{offset}]"
    if chunk >= 8 and offset in (1, 2, 4):
        return f"[>=8,{offset}]"
    return "scalar-fallback"


def classify_permutation(
    source_order: Sequence[Index], target_order: Sequence[Index]
) -> PermutationPlan:
    """Stride/offset plan of reordering ``source_order`` into ``target_order``."""
    src = tuple(source_order)
    tgt = tuple(target_order)
    if sorted((i.label, i.dim) for i in src) != sorted((i.label, i.dim) for i in tgt):
        raise InvalidPermutationError(
            f"{[i.label for i in tgt]} is not a permutation of {[i.label for i in src]}"
        )
    rank = len(src)
    if rank == 0:
        return PermutationPlan(src, tgt, 0, 1, "scalar-fallback", 1, 1)
    where = {ix.label: p for p, ix in enumerate(src)}
    tail_src = where[tgt[-1].label]
    run = 1
    while run < rank and where[tgt[rank - run - 1].label] + 1 == where[tgt[rank - run].label]:
        run += 1
    chunk = product(ix.dim for ix in tgt[rank - run:])
    src_step = product(ix.dim for ix in src[tail_src + 1:])
    offset = rank - tail_src
    return PermutationPlan(
        src, tgt, run, offset, _bucket(chunk, offset, src == tgt), chunk, src_step
    )


def permutation_axes(source_order: Sequence[Index], target_order: Sequence[Index]) -> list[int]:
    """``axes[t]`` = source position of target leg ``t`` (validated)."""
    classify_permutation(source_order, target_order)
    where = {ix.label: p for p, ix in enumerate(source_order)}
    return [where[ix.label] for ix in target_order]


# -- contraction shapes -------------------------------------------------------


@dataclass(frozen=True)
class ContractionShape:
    """M x K x N of a pairwise contraction and its narrow rate."""

    m: int
    n: int
    k: int
    n_common: int
    n_a: int
    n_b: int
    narrow: Fraction

    @property
    def multiplies(self) -> int:
        return self.m * self.k * self.n


@dataclass(frozen=True)
class TtgtPlan:
    """Operand orders of the reference's permute+GEMM execution."""

    a_target: tuple[Index, ...]
    b_target: tuple[Index, ...]
    result_indices: tuple[Index, ...]
    shape: ContractionShape
    b_is_multiplier: bool


def split_legs(a_indices: Sequence[Index], b_indices: Sequence[Index]):
    """(free_A in A order, common in A order, free_B in B order)."""
    in_b = {ix.label: ix for ix in b_indices}
    free_a: list[Index] = []
    common: list[Index] = []
    for ix in a_indices:
        twin = in_b.get(ix.label)
        if twin is None:
            free_a.append(ix)
            continue
        if twin.dim != ix.dim:
            raise ContractionError(
                f"shared label {ix.label!r} has dims {ix.dim} != {twin.dim}"
            )
        common.append(ix)
    shared = {ix.label for ix in common}
    free_b = [ix for ix in b_indices if ix.label not in shared]
    return free_a, common, free_b


def contraction_shape(a_indices: Sequence[Index], b_indices: Sequence[Index]) -> ContractionShape:
    free_a, common, free_b = split_legs(a_indices, b_indices)
    n_a, n_b = len(a_indices), len(b_indices)
    narrow = Fraction(2 * len(common), n_a + n_b) if n_a + n_b else Fraction(0)
    return ContractionShape(
        product(ix.dim for ix in free_a),
        product(ix.dim for ix in free_b),
        product(ix.dim for ix in common),
        len(common),
        n_a,
        n_b,
        narrow,
    )


def multiply_cost(a_indices: Sequence[Index], b_indices: Sequence[Index]) -> int:
    """M*K*N: one multiply per element of the union index space."""
    return contraction_shape(a_indices, b_indices).multiplies


def ttgt_plan(a_indices: Sequence[Index], b_indices: Sequence[Index]) -> TtgtPlan:
    """The reference's operand placement: larger operand is the multiplier;
    equal sizes go to B iff B's first label sorts below A's.  The result
    order is always free_A ++ free_B."""
    free_a, common, free_b = split_legs(a_indices, b_indices)
    shape = contraction_shape(a_indices, b_indices)
    size_a, size_b = shape.m * shape.k, shape.k * shape.n
    if size_a != size_b:
        b_mult = size_b > size_a
    else:
        lead_a = a_indices[0].label if len(a_indices) else ""
        lead_b = b_indices[0].label if len(b_indices) else ""
        b_mult = lead_b < lead_a
    fa, cm, fb = tuple(free_a), tuple(common), tuple(free_b)
    if b_mult:
        return TtgtPlan(cm + fa, fb + cm, fa + fb, shape, True)
    return TtgtPlan(fa + cm, cm + fb, fa + fb, shape, False)
