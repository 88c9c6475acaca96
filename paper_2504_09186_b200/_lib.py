"""ctypes binding of the C-ABI in ``include/tnc_b200.h``.

The CUDA library is mandatory: if ``libtnc_b200.so`` is missing or no CUDA
device is present, every compute entry point raises ``DeviceError``.  There
is no CPU fallback on the product path.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from .errors import DeviceError, raise_for_status

MAX_RANK = 64
C64, C128 = 0, 1
VARIANT_AUTO, VARIANT_SIMT, VARIANT_TC3XTF32, VARIANT_SPLITK = 0, 1, 2, 3
VARIANT_TC3XF16, VARIANT_STREAM, VARIANT_TCGATHER = 4, 5, 6

_LIB_PATH = Path(__file__).resolve().parent / "libtnc_b200.so"


class TensorDesc(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("labels", ctypes.c_int32 * MAX_RANK),
        ("dims", ctypes.c_int64 * MAX_RANK),
        ("strides", ctypes.c_int64 * MAX_RANK),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64),
        ("k", ctypes.c_int64),
        ("n", ctypes.c_int64),
        ("n_common", ctypes.c_int32),
        ("variant", ctypes.c_int32),
        ("b_is_multiplier", ctypes.c_int32),
        ("out_rank", ctypes.c_int32),
        ("out_labels", ctypes.c_int32 * MAX_RANK),
        ("out_dims", ctypes.c_int64 * MAX_RANK),
        ("workspace_bytes", ctypes.c_size_t),
        ("multiplies_lo", ctypes.c_int64),
    ]


_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); every symbol here is declared in include/tnc_b200.h
SIGNATURES = {
    "tnc_abi_version": (ctypes.c_int, []),
    "tnc_init": (ctypes.c_int, [ctypes.c_int]),
    "tnc_shutdown": (None, []),
    "tnc_last_error": (ctypes.c_char_p, []),
    "tnc_device_info": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(ctypes.c_int), ctypes.POINTER(_SZ)]),
    "tnc_permute": (ctypes.c_int, [_I32, _I32, ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                                   ctypes.POINTER(_I32), _P, _P, _P]),
    "tnc_plan_contract": (ctypes.c_int, [ctypes.POINTER(TensorDesc), ctypes.POINTER(TensorDesc),
                                         _I32, ctypes.POINTER(_I32), _I32, ctypes.POINTER(_P)]),
    "tnc_plan_get_info": (ctypes.c_int, [_P, ctypes.POINTER(PlanInfo)]),
    "tnc_plan_destroy": (None, [_P]),
    "tnc_contract": (ctypes.c_int, [_P, _P, _P, _P, _P, _SZ, _P]),
    "tnc_contract_split_workspace": (ctypes.c_int, [_P, _I32, _I32, ctypes.POINTER(_SZ)]),
    "tnc_contract_split": (ctypes.c_int, [_P, _I32, _I32, _P, _P, _P, _P, _SZ, _P]),
    "tnc_absorb_chain": (ctypes.c_int, [_I32, _P, _P, _I32, ctypes.POINTER(_P), ctypes.POINTER(_I64),
                                        ctypes.POINTER(_I32), _P, _SZ, _P]),
    "tnc_absorb_chain_info": (ctypes.c_int, [_I32, _I32, ctypes.POINTER(_I32), ctypes.POINTER(_I32),
                                             ctypes.POINTER(_I32)]),
    "tnc_absorb_chain_workspace": (ctypes.c_int, [_I32, _I32, ctypes.POINTER(_I32), ctypes.POINTER(_SZ)]),
    "tnc_axpy": (ctypes.c_int, [_I32, _I64, _P, _P, _P]),
    "tnc_launch_count": (ctypes.c_int64, []),
    "tnc_profile_enable": (ctypes.c_int, [ctypes.c_int]),
    "tnc_profile_read": (ctypes.c_int, [_I32, ctypes.POINTER(_I64), ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
}

_lib = None
_lock = threading.Lock()
_initialised_devices: set[int] = set()


def lib_path() -> Path:
    return _LIB_PATH


def load(require_device: bool = False):
    """Load (once) and return the ctypes library handle."""
    global _lib
    with _lock:
        if _lib is None:
            if not _LIB_PATH.exists():
                raise DeviceError(
                    f"CUDA extension {_LIB_PATH.name} is not built; run "
                    "`python -m paper_2504_09186_b200.build` (no CPU fallback exists)"
                )
            lib = ctypes.CDLL(str(_LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_device:
        ensure_device()
    return _lib


def ensure_device(device: int | None = None) -> int:
    import torch

    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 engine has no CPU fallback")
    dev = torch.cuda.current_device() if device is None else int(device)
    if dev not in _initialised_devices:
        check(load().tnc_init(dev))
        _initialised_devices.add(dev)
    return dev


def check(code: int) -> None:
    if code != 0:
        msg = _lib.tnc_last_error().decode(errors="replace") if _lib is not None else ""
        raise_for_status(code, msg)


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def i64_array(vals):
    vals = list(vals)
    return (ctypes.c_int64 * max(1, len(vals)))(*vals)


def i32_array(vals):
    vals = list(vals)
    return (ctypes.c_int32 * max(1, len(vals)))(*vals)


def make_desc(labels_ids, dims, strides, dtype) -> TensorDesc:
    d = TensorDesc()
    d.rank = len(dims)
    d.dtype = dtype
    for i, (l, n, s) in enumerate(zip(labels_ids, dims, strides)):
        d.labels[i] = l
        d.dims[i] = n
        d.strides[i] = s
    return d


def stream_ptr(stream=None) -> int:
    """Raw cudaStream_t of ``stream`` (default: torch's current stream on the
    current device).  The per-step launch path calls this for every
    contraction, so the default case avoids building a Stream object."""
    import torch

    if stream is not None:
        return int(stream.cuda_stream)
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return int(raw(torch.cuda.current_device()))
    return int(torch.cuda.current_stream().cuda_stream)


def env_flag(name: str, default: str = "") -> str:
    return os.environ.get(name, default)
