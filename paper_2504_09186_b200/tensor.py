"""Device-resident labeled tensors, permutation (K1) and zero-copy projection.

API mirror of the reference's ``tncsim.tensor`` (``tensor.py:1-292``):
``Index``, ``DenseTensor``, ``classify_permutation``, ``permute``,
``project``.  Differences by design (B200 build):

* ``DenseTensor.data`` is a CUDA ``torch`` tensor shaped by the legs (the
  reference keeps a flat numpy array).  Memory layout is identical --
  row-major over the leg order, interleaved (re, im) complex64/complex128 --
  so ``numpy()`` returns exactly the reference's flat array.
* ``permute`` runs the sm_100a gather kernel through ``tnc_permute``.
* ``project`` returns a zero-copy strided view instead of a copy (the
  kernels consume arbitrary strides), so slicing costs no copies.
"""

from __future__ import annotations

import json
import struct
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .errors import DeviceError, TensorError
from .labels import PERM_CASES, Index, PermutationPlan, classify_permutation, product

DTYPES = {"single": torch.complex64, "double": torch.complex128}
ELEMENT_BYTES = {"single": 8, "double": 16, "exact": 16}
_TORCH_TO_PREC = {torch.complex64: "single", torch.complex128: "double"}

__all__ = [
    "DTYPES", "ELEMENT_BYTES", "PERM_CASES", "DenseTensor", "Index", "PermutationPlan",
    "classify_permutation", "permute", "project", "default_device",
]


def default_device() -> torch.device:
    return torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")


def _as_torch(data, precision: str | None) -> torch.Tensor:
    if precision is not None and precision not in DTYPES:
        if precision == "exact":
            raise TensorError("precision 'exact' (object arrays) has no device representation")
        raise TensorError(f"unknown precision {precision!r}")
    if isinstance(data, torch.Tensor):
        arr = data
    else:
        npa = np.asarray(data)
        if npa.dtype == object:
            npa = npa.astype(np.complex128)
        arr = torch.from_numpy(np.ascontiguousarray(npa))
    if precision is not None:
        arr = arr.to(DTYPES[precision])
    elif arr.dtype not in _TORCH_TO_PREC:
        arr = arr.to(torch.complex128)
    return arr


class DenseTensor:
    """Ordered labeled legs plus a device array (row-major over the legs)."""

    __slots__ = ("indices", "data")

    def __init__(self, indices: Sequence[Index], data, precision: str | None = None):
        self.indices: tuple[Index, ...] = tuple(indices)
        labels = [ix.label for ix in self.indices]
        if len(set(labels)) != len(labels):
            raise TensorError(f"duplicate index labels in tensor: {labels}")
        arr = _as_torch(data, precision)
        dims = tuple(ix.dim for ix in self.indices)
        size = product(dims)
        if arr.numel() != size:
            raise TensorError(f"data length {arr.numel()} != product of dims {size} for indices {labels}")
        if tuple(arr.shape) != dims:
            arr = arr.reshape(dims)
        if arr.device.type == "cpu" and torch.cuda.is_available():
            arr = arr.to(default_device(), non_blocking=False)
        self.data = arr

    # -- properties (reference tensor.py:92-124) --
    @property
    def rank(self) -> int:
        return len(self.indices)

    @property
    def size(self) -> int:
        return self.data.numel()

    @property
    def labels(self) -> tuple[str, ...]:
        return tuple(ix.label for ix in self.indices)

    @property
    def dims(self) -> tuple[int, ...]:
        return tuple(ix.dim for ix in self.indices)

    @property
    def precision(self) -> str:
        return _TORCH_TO_PREC[self.data.dtype]

    @property
    def nbytes(self) -> int:
        return self.size * ELEMENT_BYTES[self.precision]

    @property
    def dtype_code(self) -> int:
        return _lib.C128 if self.data.dtype == torch.complex128 else _lib.C64

    def strides(self) -> tuple[int, ...]:
        return tuple(self.data.stride())

    def value(self) -> complex:
        if self.rank != 0:
            raise TensorError(f"tensor of rank {self.rank} is not a scalar")
        return complex(self.data.reshape(()).item())

    def astype(self, precision: str) -> "DenseTensor":
        if precision not in DTYPES:
            raise TensorError(f"unknown precision {precision!r}")
        return DenseTensor(self.indices, self.data.to(DTYPES[precision]).contiguous().clone())

    def numpy(self) -> np.ndarray:
        """Flat row-major host copy (the reference's ``data`` array)."""
        return self.data.detach().contiguous().reshape(-1).cpu().numpy()

    def flat(self) -> torch.Tensor:
        return self.data.contiguous().reshape(-1)

    def __repr__(self) -> str:
        legs = ",".join(f"{ix.label}:{ix.dim}" for ix in self.indices)
        return f"DenseTensor([{legs}], {self.precision})"

    # -- exchange formats (reference tensor.py:132-178) --
    def to_json(self) -> str:
        vals = self.numpy()
        return json.dumps({
            "indices": [{"label": ix.label, "dim": ix.dim} for ix in self.indices],
            "data": [[float(v.real), float(v.imag)] for v in vals],
        })

    @classmethod
    def from_json(cls, text: str, precision: str = "double") -> "DenseTensor":
        obj = json.loads(text)
        indices = [Index(d["label"], int(d["dim"])) for d in obj["indices"]]
        return cls(indices, [complex(re, im) for re, im in obj["data"]], precision=precision)

    def to_bytes(self) -> bytes:
        tag = 0 if self.precision == "single" else 1
        head = struct.pack("<BB", tag, self.rank)
        for ix in self.indices:
            lab = ix.label.encode()
            head += struct.pack("<H", len(lab)) + lab + struct.pack("<I", ix.dim)
        vals = self.numpy()
        parts = np.empty(2 * vals.size, dtype="<f4" if tag == 0 else "<f8")
        parts[0::2] = vals.real
        parts[1::2] = vals.imag
        return head + parts.tobytes()

    @classmethod
    def from_bytes(cls, raw: bytes) -> "DenseTensor":
        tag, rank = struct.unpack_from("<BB", raw, 0)
        off = 2
        indices = []
        for _ in range(rank):
            (n,) = struct.unpack_from("<H", raw, off)
            off += 2
            lab = raw[off:off + n].decode()
            off += n
            (dim,) = struct.unpack_from("<I", raw, off)
            off += 4
            indices.append(Index(lab, dim))
        parts = np.frombuffer(raw, dtype="<f4" if tag == 0 else "<f8", offset=off)
        data = parts[0::2] + 1j * parts[1::2]
        return cls(indices, data, precision="single" if tag == 0 else "double")


def _require_cuda(t: DenseTensor) -> None:
    if t.data.device.type != "cuda":
        raise DeviceError("tensor data is not on a CUDA device; the engine has no CPU path")
    _lib.ensure_device(t.data.device.index)


def permute(t: DenseTensor, target_order: Sequence[Index]) -> DenseTensor:
    """Reorder legs into ``target_order`` (new contiguous tensor, bit-exact)."""
    plan = classify_permutation(t.indices, target_order)
    tgt = plan.target_order
    _require_cuda(t)
    out = torch.empty(tuple(ix.dim for ix in tgt), dtype=t.data.dtype, device=t.data.device)
    if t.rank == 0:
        out.copy_(t.data)
        return DenseTensor(tgt, out)
    where = {ix.label: p for p, ix in enumerate(t.indices)}
    perm = [where[ix.label] for ix in tgt]
    lib = _lib.load()
    _lib.check(lib.tnc_permute(
        t.dtype_code, t.rank, _lib.i64_array(t.dims), _lib.i64_array(t.strides()),
        _lib.i32_array(perm), t.data.data_ptr(), out.data_ptr(), _lib.stream_ptr(),
    ))
    return DenseTensor(tgt, out)


def project(t: DenseTensor, assignment: dict[str, int]) -> DenseTensor:
    """Fix the assigned legs; returns ``t`` itself when no leg is hit, else a
    zero-copy strided view over the kept legs (reference ``tensor.py:277-292``
    copies; the device kernels accept the view's strides directly)."""
    hit = [ix for ix in t.indices if ix.label in assignment]
    if not hit:
        return t
    sel = []
    kept = []
    for ix in t.indices:
        if ix.label in assignment:
            v = int(assignment[ix.label])
            if not 0 <= v < ix.dim:
                raise TensorError(f"assignment {ix.label}={v} outside dim {ix.dim}")
            sel.append(v)
        else:
            sel.append(slice(None))
            kept.append(ix)
    view = t.data[tuple(sel)]
    res = DenseTensor.__new__(DenseTensor)
    res.indices = tuple(kept)
    res.data = view
    return res
