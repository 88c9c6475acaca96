"""Exception taxonomy of the engine.

Mirrors the reference's ``tncsim.errors`` class names and hierarchy
(reference ``pkg/src/tncsim/errors.py:4-41``) so callers can catch the same
exceptions.  The C-ABI returns integer status codes; :func:`raise_for_status`
maps them one-to-one onto these classes (see ``include/tnc_b200.h``).
"""

from __future__ import annotations


class TncError(Exception):
    """Root of every engine error."""


class TensorError(TncError):
    """Bad tensor: data length, duplicate labels, non-scalar value()."""


class InvalidPermutationError(TncError):
    """Requested order is not a permutation of the tensor's legs."""


class ContractionError(TncError):
    """Operands cannot be contracted (shared label dim mismatch, bad split)."""


class CircuitParseError(TncError):
    """Circuit text error; ``line`` holds the 1-based offending line."""

    def __init__(self, message: str, line: int):
        super().__init__(f"line {line}: {message}")
        self.line = line


class NetworkError(TncError):
    """Inconsistent network (label in more than two tensors, dim clash...)."""


class SlicingError(TncError):
    """No slicing reaches the requested rank cap."""


class PlanningError(TncError):
    """Reuse program / schedule planning failure."""


class MemoryBudgetError(TncError):
    """An intermediate or checkpoint exceeds the configured byte budget."""


class DeviceError(TncError):
    """CUDA / library failure reported through the C-ABI."""


# Status codes of the C-ABI (include/tnc_b200.h, enum tnc_status).
STATUS_OK = 0
_STATUS_TO_EXC = {
    1: TncError,                 # TNC_ERR_INVALID
    2: TensorError,              # TNC_ERR_TENSOR
    3: InvalidPermutationError,  # TNC_ERR_PERMUTATION
    4: ContractionError,         # TNC_ERR_CONTRACTION
    5: MemoryBudgetError,        # TNC_ERR_WORKSPACE
    6: DeviceError,              # TNC_ERR_CUDA
    7: DeviceError,              # TNC_ERR_NCCL
    8: TncError,                 # TNC_ERR_UNSUPPORTED
}


def raise_for_status(code: int, message: str) -> None:
    if code == STATUS_OK:
        return
    exc = _STATUS_TO_EXC.get(code, TncError)
    raise exc(message or f"tnc status {code}")
