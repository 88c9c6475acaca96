"""Pairwise contraction on the B200 (K2/K3) behind the reference's operator API.

API mirror of ``tncsim.contract`` (``contract.py:1-208``): ``contract_pair``,
``split_common_contract``, ``contraction_shape``, ``multiply_cost``,
``ttgt_plan``, ``contraction_permutations``.  The index map is the
reference's (result legs free_A ++ free_B, ``contract.py:149-165``); the
arithmetic runs in the sm_100a kernels selected by ``tnc_plan_contract``
(AUTO):

* K2: tcgen05 ``kind::f16`` GEMM on 3xFP16 operand planes (per-row
  power-of-two scaling) for big tensor-core-shaped steps;
* K6: gather-fed tcgen05 ``kind::tf32`` GEMM (3xTF32, operands gathered in the
  kernel, split-K) for narrow / split-K-shaped steps;
* K5 streaming and K3 split-K kernels for the narrowest steps, the CUDA-core
  GEMM for small ones;
* split-K with the reference's panel/tree semantics for
  ``split_common_contract``.
"""

from __future__ import annotations

import ctypes
import threading
from typing import Sequence

import torch

from . import _lib
from .errors import ContractionError
from .labels import (
    ContractionShape,
    Index,
    PermutationPlan,
    TtgtPlan,
    classify_permutation,
    contraction_shape,
    multiply_cost,
    split_legs,
    ttgt_plan,
)
from .tensor import DenseTensor, _require_cuda

__all__ = [
    "ContractionShape", "TtgtPlan", "contract_pair", "contraction_permutations",
    "contraction_shape", "multiply_cost", "split_common_contract", "ttgt_plan", "ContractPlan",
    "plan_for",
]


def contraction_permutations(a_indices: Sequence[Index], b_indices: Sequence[Index]) -> list[PermutationPlan]:
    """Stride/offset classes of the two operand permutations the reference
    would run (``contract.py:120-128``)."""
    plan = ttgt_plan(a_indices, b_indices)
    return [
        classify_permutation(tuple(a_indices), plan.a_target),
        classify_permutation(tuple(b_indices), plan.b_target),
    ]


class ContractPlan:
    """Owning handle of a ``tnc_plan`` (immutable, shareable)."""

    __slots__ = ("handle", "info", "out_indices", "__weakref__")

    def __init__(self, handle: int, info, out_indices: tuple[Index, ...]):
        self.handle = handle
        self.info = info
        self.out_indices = out_indices

    @property
    def variant(self) -> int:
        return self.info.variant

    @property
    def workspace_bytes(self) -> int:
        return int(self.info.workspace_bytes)

    def __del__(self):
        lib = _lib._lib if _lib is not None else None  # module globals are gone at interpreter exit
        if lib is not None and self.handle:
            lib.tnc_plan_destroy(self.handle)
            self.handle = 0


_plan_cache: dict[tuple, ContractPlan] = {}
_plan_lock = threading.Lock()
_PLAN_CACHE_MAX = 4096


def _dtype_code(t: torch.Tensor) -> int:
    return _lib.C128 if t.dtype == torch.complex128 else _lib.C64


def plan_for(a_indices, a_strides, b_indices, b_strides, dtype: int,
             out_order: Sequence[Index] | None = None, variant: int = _lib.VARIANT_AUTO) -> ContractPlan:
    """Cached device plan for contracting two labeled strided operands."""
    # plans own lazily-created device tables: one plan per device
    key = (
        torch.cuda.current_device() if torch.cuda.is_available() else -1,
        tuple((ix.label, ix.dim) for ix in a_indices), tuple(a_strides),
        tuple((ix.label, ix.dim) for ix in b_indices), tuple(b_strides), dtype,
        None if out_order is None else tuple(ix.label for ix in out_order), variant,
    )
    plan = _plan_cache.get(key)
    if plan is not None:
        return plan
    free_a, _, free_b = split_legs(a_indices, b_indices)  # raises ContractionError
    ids: dict[str, int] = {}
    for ix in tuple(a_indices) + tuple(b_indices):
        ids.setdefault(ix.label, len(ids))
    da = _lib.make_desc([ids[ix.label] for ix in a_indices], [ix.dim for ix in a_indices], a_strides, dtype)
    db = _lib.make_desc([ids[ix.label] for ix in b_indices], [ix.dim for ix in b_indices], b_strides, dtype)
    default_out = tuple(free_a) + tuple(free_b)
    if out_order is None:
        out_rank, out_ids, out_indices = -1, None, default_out
    else:
        out_indices = tuple(out_order)
        if sorted((i.label, i.dim) for i in out_indices) != sorted((i.label, i.dim) for i in default_out):
            raise ContractionError("output order is not a permutation of the free legs")
        out_rank = len(out_indices)
        out_ids = _lib.i32_array([ids[ix.label] for ix in out_indices])
    handle = ctypes.c_void_p()
    lib = _lib.load()
    _lib.check(lib.tnc_plan_contract(ctypes.byref(da), ctypes.byref(db), out_rank, out_ids, variant,
                                     ctypes.byref(handle)))
    info = _lib.PlanInfo()
    _lib.check(lib.tnc_plan_get_info(handle, ctypes.byref(info)))
    plan = ContractPlan(handle.value, info, out_indices)
    with _plan_lock:
        if len(_plan_cache) >= _PLAN_CACHE_MAX:
            _plan_cache.clear()
        _plan_cache[key] = plan
    return plan


def _promote(a: DenseTensor, b: DenseTensor) -> tuple[torch.Tensor, torch.Tensor]:
    if a.data.dtype == b.data.dtype:
        return a.data, b.data
    return a.data.to(torch.complex128), b.data.to(torch.complex128)


def contract_into(plan: ContractPlan, a_data: torch.Tensor, b_data: torch.Tensor,
                  out: torch.Tensor | None = None) -> torch.Tensor:
    """Run a plan on raw device arrays; allocates the output unless given."""
    dims = tuple(ix.dim for ix in plan.out_indices)
    if out is None:
        out = torch.empty(dims, dtype=a_data.dtype, device=a_data.device)
    ws_n = plan.workspace_bytes
    ws = torch.empty(ws_n, dtype=torch.uint8, device=a_data.device) if ws_n else None
    _lib.check(_lib.load().tnc_contract(plan.handle, a_data.data_ptr(), b_data.data_ptr(),
                                        out.data_ptr(), ws.data_ptr() if ws is not None else None, ws_n,
                                        _lib.stream_ptr()))
    return out


def contract_pair(a: DenseTensor, b: DenseTensor, out_order: Sequence[Index] | None = None,
                  variant: int = _lib.VARIANT_AUTO) -> DenseTensor:
    """Sum over all shared labels; result legs are free-of-A (A's order) then
    free-of-B (B's order), or ``out_order`` when given (fused output
    permutation).  Inputs are never mutated; the result is a new tensor."""
    split_legs(a.indices, b.indices)  # ContractionError before touching the device
    _require_cuda(a)
    _require_cuda(b)
    ad, bd = _promote(a, b)
    plan = plan_for(a.indices, ad.stride(), b.indices, bd.stride(), _dtype_code(ad), out_order, variant)
    out = contract_into(plan, ad, bd)
    return DenseTensor(plan.out_indices, out)


def split_common_contract(a: DenseTensor, b: DenseTensor, blocks: int, group_size: int) -> DenseTensor:
    """K split into ``min(blocks*group_size, K)`` panels (remainder on the last),
    each accumulated independently, combined by the left-complete pairwise tree
    of the reference (``contract.py:168-208``)."""
    if blocks < 1 or group_size < 1:
        raise ContractionError(f"blocks*group_size must be positive, got {blocks}*{group_size}")
    split_legs(a.indices, b.indices)
    _require_cuda(a)
    _require_cuda(b)
    ad, bd = _promote(a, b)
    plan = plan_for(a.indices, ad.stride(), b.indices, bd.stride(), _dtype_code(ad), None, _lib.VARIANT_SIMT)
    lib = _lib.load()
    need = ctypes.c_size_t()
    _lib.check(lib.tnc_contract_split_workspace(plan.handle, blocks, group_size, ctypes.byref(need)))
    ws = torch.empty(max(need.value, 1), dtype=torch.uint8, device=ad.device)
    out = torch.empty(tuple(ix.dim for ix in plan.out_indices), dtype=ad.dtype, device=ad.device)
    _lib.check(lib.tnc_contract_split(plan.handle, blocks, group_size, ad.data_ptr(), bd.data_ptr(),
                                      out.data_ptr(), ws.data_ptr(), need.value, _lib.stream_ptr()))
    return DenseTensor(plan.out_indices, out)
