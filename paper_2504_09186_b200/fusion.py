"""Step fusion (K4): absorb a chain of two-leg gates into one resident tensor.

Semantics are exactly the reference's repeated ``contract_pair(T, G)``
(``contract.py:149-165``) along a stem (``tree.py:278-384``): each gate G has
four legs, two of them shared with the current T; the result legs are
free_T (T's order) ++ free_G (G's order).  The device path is
``tnc_absorb_chain`` -- the chain runs in a few shared-memory-tiled HBM passes
instead of one permute + GEMM round trip per gate.
"""

from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .errors import ContractionError, TensorError
from .labels import Index, split_legs
from .tensor import DenseTensor, _require_cuda

MIN_FUSED_RANK = 12


def _gate_matrix(g: DenseTensor, t_labels: Sequence[str]):
    """(free_G legs, common legs in T order, host U[(o0,o1),(c0,c1)] complex64)."""
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
    order = [where[ix.label] for ix in free + common]
    u = g.data.detach().to(torch.complex64).cpu().numpy().reshape((2, 2, 2, 2)).transpose(order)
    return free, common, np.ascontiguousarray(u.reshape(-1))


def absorb_chain(t: DenseTensor, gates: Sequence[DenseTensor]) -> DenseTensor:
    """Result of ``for g in gates: t = contract_pair(t, g)`` in one fused pass
    sequence (complex64, dim-2 legs, rank >= 12; smaller tensors fall back to
    the per-gate device contraction)."""
    _require_cuda(t)
    labels = list(t.labels)
    axes: list[int] = []
    mats = []
    cur = list(t.indices)
    for g in gates:
        free, common, u = _gate_matrix(g, [ix.label for ix in cur])
        split_legs(cur, g.indices)  # dim checks (ContractionError)
        pos = {ix.label: p for p, ix in enumerate(cur)}
        axes += [pos[common[0].label], pos[common[1].label]]
        mats.append(u)
        cur = [ix for ix in cur if ix.label not in (common[0].label, common[1].label)] + free
    fused_ok = (t.rank >= MIN_FUSED_RANK and t.data.dtype == torch.complex64
                and all(ix.dim == 2 for ix in t.indices))
    if not fused_ok:
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
    keep = [np.ascontiguousarray(m, dtype=np.complex64) for m in mats]
    ptrs = (ctypes.c_void_p * max(1, n))(*[m.ctypes.data for m in keep])
    _lib.check(lib.tnc_absorb_chain(t.rank, data.data_ptr(), out.data_ptr(), n, ptrs, ax, ws.data_ptr(),
                                    int(need.value), _lib.stream_ptr()))
    res = DenseTensor.__new__(DenseTensor)
    res.indices = tuple(cur)
    res.data = out.reshape(tuple(ix.dim for ix in cur))
    return res
