import base64
import gzip
import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built libtnc_b200.so")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name: str):
    with gzip.open(GOLDEN / f"{name}.json.gz", "rt") as fh:
        return json.load(fh)


def arr(enc) -> np.ndarray:
    """Decode a golden array (base64 little-endian complex)."""
    dt = np.dtype("<c8") if enc["dtype"] == "c8" else np.dtype("<c16")
    return np.frombuffer(base64.b64decode(enc["b64"]), dtype=dt).copy()


def rel_l2(got, want) -> float:
    got = np.asarray(got, dtype=np.complex128).reshape(-1)
    want = np.asarray(want, dtype=np.complex128).reshape(-1)
    den = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (den if den > 0 else 1.0))


@pytest.fixture(scope="session")
def cuda_ready():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_09186_b200 import _lib

    _lib.load(require_device=True)
    return True
