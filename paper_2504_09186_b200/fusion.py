"""Step fusion (K4): absorb a chain of two-leg gates into one resident tensor.

Semantics are exactly the reference's repeated ``contract_pair(T, G)``
(``contract.py:149-165``) along a stem (``tree.py:278-384``): each gate G has
four legs, two of them shared with the current T; the result legs are
free_T (T's order) ++ free_G (G's order).  The device path is
``tnc_absorb_chain``: the chain runs in the fewest shared-memory-tiled HBM
passes the tile allows (2 for C2); within a pass the gates are applied to
32-element register cubes with packed FP32 FMAs whose coefficients come from
the constant bank -- instead of one permute + GEMM round trip per gate.  Gate
values never leave the device.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import torch

from . import _lib
from .errors import ContractionError, TensorError
from .labels import Index, split_legs
from .tensor import DenseTensor, _require_cuda

MIN_FUSED_RANK = 13  # the fused kernel's tile holds 13 axes


def _gate_roles(g: DenseTensor, t_labels: Sequence[str]):
    """(free legs of G in G's order, common legs in T order, element strides
    of the (out_a, out_b, in_a, in_b) legs in G's storage)."""
    if g.rank != 4 or any(ix.dim != 2 for ix in g.indices):
        raise TensorError("absorb_chain gates must be rank-4 with dim-2 legs")
    tl = set(t_labels)
    common = [ix for ix in g.indices if ix.label in tl]
    free = [ix for ix in g.indices if ix.label not in tl]
    if len(common) != 2:
        raise ContractionError(f"gate {g.labels} must share exactly two legs with the tensor")
    pos = {l: p for p, l in enumerate(t_labels)}
    common.sort(key=lambda ix: pos[ix.label])
    where = {ix.label: p for p, ix in enumerate(g.indices)}
    st = g.data.stride()
    strides = [st[where[ix.label]] for ix in free + common]
    return free, common, strides


def plan_chain(t: DenseTensor, gates: Sequence[DenseTensor]):
    """Leg bookkeeping of the chain: (axes per gate in the current order,
    gate strides, final indices)."""
    axes: list[int] = []
    strides: list[int] = []
    cur = list(t.indices)
    for g in gates:
        free, common, st = _gate_roles(g, [ix.label for ix in cur])
        split_legs(cur, g.indices)  # dim checks (ContractionError)
        pos = {ix.label: p for p, ix in enumerate(cur)}
        axes += [pos[common[0].label], pos[common[1].label]]
        strides += st
        cur = [ix for ix in cur if ix.label not in (common[0].label, common[1].label)] + free
    return axes, strides, cur


def chain_info(rank: int, axes: Sequence[int]) -> tuple[int, int]:
    """(HBM passes, 3-axis gate groups) the fused kernel uses for a chain."""
    lib = _lib.load()
    p, g = ctypes.c_int32(), ctypes.c_int32()
    _lib.check(lib.tnc_absorb_chain_info(rank, len(axes) // 2, _lib.i32_array(axes), ctypes.byref(p),
                                         ctypes.byref(g)))
    return p.value, g.value


def fusable(t: DenseTensor) -> bool:
    return (t.rank >= MIN_FUSED_RANK and t.data.dtype == torch.complex64
            and all(ix.dim == 2 for ix in t.indices))


def absorb_chain(t: DenseTensor, gates: Sequence[DenseTensor]) -> DenseTensor:
    """Result of ``for g in gates: t = contract_pair(t, g)`` as one fused
    chain (complex64, dim-2 legs, rank >= 13; other tensors take the per-gate
    device contraction)."""
    _require_cuda(t)
    axes, strides, cur = plan_chain(t, gates)
    if not fusable(t) or any(g.data.dtype != torch.complex64 or not g.data.is_cuda for g in gates):
        from .contract import contract_pair

        out = t
        for g in gates:
            out = contract_pair(out, g)
        return out
    data = t.data.contiguous()
    lib = _lib.load()
    n = len(gates)
    ax = _lib.i32_array(axes)
    need = ctypes.c_size_t()
    _lib.check(lib.tnc_absorb_chain_workspace(t.rank, n, ax, ctypes.byref(need)))
    ws = torch.empty(max(int(need.value), 1), dtype=torch.uint8, device=data.device)
    out = torch.empty_like(data)
    ptrs = (ctypes.c_void_p * max(1, n))(*[g.data.data_ptr() for g in gates])
    _lib.check(lib.tnc_absorb_chain(t.rank, data.data_ptr(), out.data_ptr(), n, ptrs, _lib.i64_array(strides),
                                    ax, ws.data_ptr(), int(need.value), _lib.stream_ptr()))
    res = DenseTensor.__new__(DenseTensor)
    res.indices = tuple(cur)
    res.data = out.reshape(tuple(ix.dim for ix in cur))
    return res
