"""Reference-side binding: ``tncsim.contract.contract_pair`` over the raw C-ABI.

This is the stub of INTEGRATION.md section 1 as a runnable module: what a
``tncsim`` maintainer adds to route the reference executor's per-step call
(``/root/reference/pkg/src/tncsim/execute.py:159``) through
``libtnc_b200.so``.  It deliberately uses nothing of this package's Python
mirror -- only ``ctypes`` on the shared library plus a CUDA allocator
(``torch``) for the device copies -- so it proves the C-ABI of
``include/tnc_b200.h`` is sufficient by itself.

The operands are duck-typed like ``tncsim.DenseTensor``: ``.indices`` (objects
with ``.label`` / ``.dim``) and ``.data`` (a flat host numpy array, row-major
over the index order, reference ``tensor.py:46-128``).  ``make`` builds the
result (``tncsim.DenseTensor`` when wired into the reference).

    import tncsim.execute
    from paper_2504_09186_b200 import tncsim_binding
    tncsim_binding.install(tncsim)          # patches execute.py:159's callee

There is no CPU path: without the library or a CUDA device the call raises.
"""

from __future__ import annotations

import ctypes
from pathlib import Path
from typing import Callable

import numpy as np

MAX_RANK = 64
LIB_PATH = Path(__file__).resolve().parent / "libtnc_b200.so"


class TensorDesc(ctypes.Structure):  # tnc_tensor_desc, include/tnc_b200.h
    _fields_ = [("rank", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("labels", ctypes.c_int32 * MAX_RANK),
                ("dims", ctypes.c_int64 * MAX_RANK),
                ("strides", ctypes.c_int64 * MAX_RANK)]


class PlanInfo(ctypes.Structure):  # tnc_plan_info, include/tnc_b200.h
    _fields_ = [("m", ctypes.c_int64), ("k", ctypes.c_int64), ("n", ctypes.c_int64),
                ("n_common", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("b_is_multiplier", ctypes.c_int32), ("out_rank", ctypes.c_int32),
                ("out_labels", ctypes.c_int32 * MAX_RANK), ("out_dims", ctypes.c_int64 * MAX_RANK),
                ("workspace_bytes", ctypes.c_size_t), ("multiplies_lo", ctypes.c_int64)]


_lib = None


def library() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(str(LIB_PATH))
        lib.tnc_plan_contract.argtypes = [ctypes.POINTER(TensorDesc), ctypes.POINTER(TensorDesc), ctypes.c_int32,
                                          ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                                          ctypes.POINTER(ctypes.c_void_p)]
        lib.tnc_plan_get_info.argtypes = [ctypes.c_void_p, ctypes.POINTER(PlanInfo)]
        lib.tnc_plan_destroy.argtypes = [ctypes.c_void_p]
        lib.tnc_contract.argtypes = [ctypes.c_void_p] * 5 + [ctypes.c_size_t, ctypes.c_void_p]
        lib.tnc_last_error.restype = ctypes.c_char_p
        _lib = lib
    return _lib


class BindingError(RuntimeError):
    """A non-zero tnc_status; ``.code`` is the status (see tnc_status in the header)."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def _check(code: int) -> None:
    if code:
        raise BindingError(code, library().tnc_last_error().decode())


def describe(t, ids: dict) -> TensorDesc:
    """Row-major descriptor of a host tensor (last leg fastest)."""
    d = TensorDesc()
    d.rank = len(t.indices)
    d.dtype = 0 if np.asarray(t.data).dtype == np.complex64 else 1
    stride = 1
    for i in reversed(range(d.rank)):
        d.labels[i] = ids[t.indices[i].label]
        d.dims[i] = t.indices[i].dim
        d.strides[i] = stride
        stride *= t.indices[i].dim
    return d


def plan(a, b):
    """(plan handle, PlanInfo, result indices free_A ++ free_B): the host-only
    part of the call (works without a CUDA device)."""
    ids: dict = {}
    for ix in tuple(a.indices) + tuple(b.indices):
        ids.setdefault(ix.label, len(ids))
    by_id = {}
    for ix in tuple(a.indices) + tuple(b.indices):
        by_id[ids[ix.label]] = ix
    da, db = describe(a, ids), describe(b, ids)
    handle = ctypes.c_void_p()
    _check(library().tnc_plan_contract(ctypes.byref(da), ctypes.byref(db), -1, None, 0, ctypes.byref(handle)))
    info = PlanInfo()
    _check(library().tnc_plan_get_info(handle, ctypes.byref(info)))
    out = tuple(by_id[info.out_labels[i]] for i in range(info.out_rank))
    return handle, info, out


def _device_contract(handle, info: PlanInfo, a_host: np.ndarray, b_host: np.ndarray) -> np.ndarray:
    """Upload, tnc_contract on the current stream, download."""
    import torch

    if not torch.cuda.is_available():
        raise BindingError(-1, "libtnc_b200 needs a CUDA device (there is no CPU path)")
    ga = torch.from_numpy(np.ascontiguousarray(a_host)).cuda()
    gb = torch.from_numpy(np.ascontiguousarray(b_host)).cuda()
    n_out = 1
    for i in range(info.out_rank):
        n_out *= info.out_dims[i]
    gc = torch.empty(n_out, dtype=ga.dtype, device="cuda")
    ws_n = int(info.workspace_bytes)
    ws = torch.empty(max(ws_n, 1), dtype=torch.uint8, device="cuda")
    _check(library().tnc_contract(handle, ga.data_ptr(), gb.data_ptr(), gc.data_ptr(), ws.data_ptr(), ws_n,
                                  torch.cuda.current_stream().cuda_stream))
    return gc.cpu().numpy()


def contract_pair(a, b, make: Callable | None = None):
    """Drop-in for ``tncsim.contract.contract_pair`` (``contract.py:149-165``):
    sums over the shared labels; result legs are free_A ++ free_B; mixed
    precisions promote to complex128 as numpy would."""
    a_data, b_data = np.asarray(a.data), np.asarray(b.data)
    if a_data.dtype != b_data.dtype:
        a_data, b_data = a_data.astype(np.complex128), b_data.astype(np.complex128)
        a, b = _View(a.indices, a_data), _View(b.indices, b_data)
    handle, info, out = plan(a, b)
    try:
        data = _device_contract(handle, info, a_data.reshape(-1), b_data.reshape(-1))
    finally:
        library().tnc_plan_destroy(handle)
    return (make or _View)(out, data)


class _View:
    def __init__(self, indices, data):
        self.indices = tuple(indices)
        self.data = data


def install(tncsim_module) -> Callable:
    """Route the reference executor's per-step contraction through the
    library; returns the function that undoes it."""
    import importlib

    execute = importlib.import_module(tncsim_module.__name__ + ".execute")
    original = execute.contract_pair
    dense = tncsim_module.DenseTensor

    def bound(a, b):
        return contract_pair(a, b, make=lambda ix, data: dense(ix, data))

    execute.contract_pair = bound

    def restore():
        execute.contract_pair = original

    return restore
