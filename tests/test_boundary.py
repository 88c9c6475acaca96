"""The drop-in boundary: C-ABI library exports, host-only plan logic, error
mapping, and the oracle quarantine.  CPU only (no kernel launches)."""

import ctypes
import os
import re
from pathlib import Path

import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "tnc_b200.h"


def _declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(tnc_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2504_09186_b200 import _lib

    lib = ctypes.CDLL(str(_lib.lib_path()))
    declared = _declared_symbols()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.exported_symbols())
    assert _lib.load().tnc_abi_version() == 1


def _plan(a, b, out=None, variant=0):
    from paper_2504_09186_b200 import _lib

    lib = _lib.load()
    ids = {}
    for l, _ in a + b:
        ids.setdefault(l, len(ids))

    def strides(legs):
        st, acc = [], 1
        for _, d in reversed(legs):
            st.append(acc)
            acc *= d
        return list(reversed(st))

    da = _lib.make_desc([ids[l] for l, _ in a], [d for _, d in a], strides(a), _lib.C64)
    db = _lib.make_desc([ids[l] for l, _ in b], [d for _, d in b], strides(b), _lib.C64)
    h = ctypes.c_void_p()
    out_ids = None if out is None else _lib.i32_array([ids.setdefault(l, len(ids)) for l in out])
    code = lib.tnc_plan_contract(ctypes.byref(da), ctypes.byref(db), -1 if out is None else len(out), out_ids,
                                 variant, ctypes.byref(h))
    if code:
        return code, None, ids
    info = _lib.PlanInfo()
    _lib.check(lib.tnc_plan_get_info(h, ctypes.byref(info)))
    lib.tnc_plan_destroy(h)
    return 0, info, ids


def test_plan_shapes_and_output_order_host_only():
    code, info, ids = _plan([("a", 2), ("k", 3), ("b", 4)], [("k", 3), ("c", 5)])
    assert code == 0
    assert (info.m, info.k, info.n) == (8, 3, 5)
    inv = {v: k for k, v in ids.items()}
    assert [inv[info.out_labels[i]] for i in range(info.out_rank)] == ["a", "b", "c"]
    code, info, ids = _plan([("a", 2), ("k", 3)], [("k", 3), ("c", 5)], out=["c", "a"])
    assert code == 0 and [inv_l for inv_l in (info.out_labels[0], info.out_labels[1])] == [ids["c"], ids["a"]]
    # big enough for tensor cores -> the TC variant is auto-selected
    big_a = [(f"a{i}", 2) for i in range(12)] + [(f"k{i}", 2) for i in range(12)]
    big_b = [(f"k{i}", 2) for i in range(12)] + [(f"b{i}", 2) for i in range(12)]
    code, info, _ = _plan(big_a, big_b)
    assert code == 0 and info.variant in (2, 4) and info.workspace_bytes > 0
    # tiny output, huge K -> the CUDA-core split-K reduction is auto-selected
    code, info, _ = _plan([("m", 2)] + [(f"k{i}", 2) for i in range(14)], [(f"k{i}", 2) for i in range(14)] + [("n", 4)])
    assert code == 0 and info.variant == 3
    # narrow step (C1a-like): the K6 gather-fed tensor-core kernel ...
    narrow = ([(f"a{i}", 2) for i in range(16)] + [(f"k{i}", 2) for i in range(6)],
              [(f"k{i}", 2) for i in range(6)] + [(f"b{i}", 2) for i in range(4)])
    out = [f"b{i}" for i in range(4)] + [f"a{i}" for i in range(16)]
    code, info, _ = _plan(*narrow, out=out)
    assert code == 0 and info.variant == 6
    # ... or, with K6 switched off, the K5 streaming kernel (no workspace at all)
    os.environ["TNC_TCGATHER"] = "0"
    try:
        code, info, _ = _plan(*narrow, out=out)
    finally:
        del os.environ["TNC_TCGATHER"]
    assert code == 0 and info.variant == 5 and info.workspace_bytes == 0


def test_stream_variant_rejects_oversized_y():
    """Forcing the streaming variant when Y cannot sit on chip (rows_y * K =
    2^14 > 4096) is an explicit UNSUPPORTED status, never a silent fallback."""
    a = [(f"a{i}", 2) for i in range(12)] + [(f"k{i}", 2) for i in range(8)]
    b = [(f"k{i}", 2) for i in range(8)] + [(f"b{i}", 2) for i in range(6)]
    code, _, _ = _plan(a, b, variant=5)
    assert code == 8
    code, _, _ = _plan([("a", 3), ("k", 2)], [("k", 2), ("b", 2)], variant=5)  # extent-3 leg
    assert code == 8


def test_plan_errors_map_to_reference_exceptions():
    from paper_2504_09186_b200 import ContractionError, InvalidPermutationError, TensorError
    from paper_2504_09186_b200 import _lib
    from paper_2504_09186_b200.errors import raise_for_status

    code, _, _ = _plan([("i", 2)], [("i", 3)])
    with pytest.raises(ContractionError):
        raise_for_status(code, "")
    code, _, _ = _plan([("i", 2), ("j", 2)], [("i", 2)], out=["x"])
    with pytest.raises(InvalidPermutationError):
        raise_for_status(code, "")
    code, _, _ = _plan([("i", 2), ("i", 2)], [("j", 2)])
    with pytest.raises(TensorError):
        raise_for_status(code, "")


def test_product_never_imports_oracle():
    pkg = ROOT / "paper_2504_09186_b200"
    for src in list(pkg.rglob("*.py")) + list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        text = src.read_text()
        assert not re.search(r"^\s*(from|import)\s+oracle", text, re.M), src
        assert "tncref" not in text, src


def test_no_cpu_fallback_without_device(monkeypatch):
    import torch

    from paper_2504_09186_b200 import DeviceError, _lib

    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(DeviceError):
        _lib.ensure_device()
