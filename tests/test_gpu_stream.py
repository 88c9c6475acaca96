"""K5 streaming contraction (TNC_VARIANT_STREAM) against the oracle:
narrow steps with scattered common legs, custom output orders, every tile
shape class (K = 1 .. 1024, N = 1 .. 64, fewer X-free legs than a tile),
strided (projected) operands.  AUTO selection and the UNSUPPORTED status
are host-only checks in test_boundary.py."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import tncref

pytestmark = pytest.mark.gpu

STREAM = 5


def _case(rng, n_fa, n_k, n_fb, out_shuffle=True):
    fa = [f"a{i}" for i in range(n_fa)]
    cm = [f"k{i}" for i in range(n_k)]
    fb = [f"b{i}" for i in range(n_fb)]
    la, lb = fa + cm, cm + fb
    rng.shuffle(la)
    rng.shuffle(lb)
    out = [l for l in la if l.startswith("a")] + [l for l in lb if l.startswith("b")]
    if out_shuffle:
        rng.shuffle(out)
    da = (rng.standard_normal(2 ** len(la)) + 1j * rng.standard_normal(2 ** len(la))).astype(np.complex64)
    db = (rng.standard_normal(2 ** len(lb)) + 1j * rng.standard_normal(2 ** len(lb))).astype(np.complex64)
    return la, lb, out, da, db


def _run(la, lb, out, da, db, variant):
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair

    a = DenseTensor([Index(l) for l in la], da)
    b = DenseTensor([Index(l) for l in lb], db)
    by = {l: Index(l) for l in la + lb}
    return contract_pair(a, b, out_order=[by[l] for l in out], variant=variant)


def _want(la, lb, out, da, db):
    res = tncref.contract((tuple(la), (2,) * len(la), da.astype(np.complex128)),
                          (tuple(lb), (2,) * len(lb), db.astype(np.complex128)))
    return tncref.permute(res, tuple(out))


@pytest.mark.parametrize("shape", [(14, 6, 4), (13, 0, 3), (12, 10, 2), (12, 4, 6), (12, 6, 0),
                                   (5, 5, 2), (15, 1, 5), (12, 2, 1)])
def test_stream_vs_oracle(cuda_ready, shape):
    rng = np.random.default_rng(sum(shape) * 7 + shape[0])
    la, lb, out, da, db = _case(rng, *shape)
    got = _run(la, lb, out, da, db, STREAM)
    want = _want(la, lb, out, da, db)
    assert list(got.labels) == list(want[0])
    assert rel_l2(got.numpy(), want[2]) <= 1e-5, shape


def test_stream_default_order_and_swapped_operands(cuda_ready):
    """Y as the FIRST operand (B multiplies) and the default free_A ++ free_B order."""
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair

    rng = np.random.default_rng(5)
    la, lb, _, da, db = _case(rng, 13, 5, 3)
    a = DenseTensor([Index(l) for l in la], da)
    b = DenseTensor([Index(l) for l in lb], db)
    got = contract_pair(b, a, variant=STREAM)
    want = tncref.contract((tuple(lb), (2,) * len(lb), db.astype(np.complex128)),
                           (tuple(la), (2,) * len(la), da.astype(np.complex128)))
    assert list(got.labels) == list(want[0])
    assert rel_l2(got.numpy(), want[2]) <= 1e-5


def test_stream_projected_operand(cuda_ready):
    """Zero-copy projection (strided view) of the streamed operand."""
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair, project

    rng = np.random.default_rng(9)
    la, lb, out, da, db = _case(rng, 14, 6, 3)
    la2 = la + ["s0"]
    rng.shuffle(la2)
    da2 = (rng.standard_normal(2 ** len(la2)) + 1j * rng.standard_normal(2 ** len(la2))).astype(np.complex64)
    a = project(DenseTensor([Index(l) for l in la2], da2), {"s0": 1})
    b = DenseTensor([Index(l) for l in lb], db)
    by = {l: Index(l) for l in la2 + lb}
    got = contract_pair(a, b, out_order=[by[l] for l in out], variant=STREAM)
    ra = tncref.project((tuple(la2), (2,) * len(la2), da2.astype(np.complex128)), {"s0": 1})
    want = tncref.permute(tncref.contract(ra, (tuple(lb), (2,) * len(lb), db.astype(np.complex128))), tuple(out))
    assert list(got.labels) == list(want[0])
    assert rel_l2(got.numpy(), want[2]) <= 1e-5


@pytest.mark.parametrize("variant", [3, 6])
def test_first_launch_on_side_stream(cuda_ready, variant):
    """A fresh plan (device index tables uploaded at plan creation) launched for
    the first time on a non-default torch stream, operands produced on that
    stream, no host sync in between: results match the oracle (split-K gather
    tables, K6 offset tables)."""
    from paper_2504_09186_b200 import DenseTensor, Index, contract_pair

    rng = np.random.default_rng(40 + variant)
    common = [f"c{i}" for i in range(14 if variant == 3 else 10)]
    la = common + ["x0", "x1", "x2"] + ([f"x{3 + i}" for i in range(5)] if variant == 6 else [])
    lb = common + ["y0", "y1"]
    rng.shuffle(la)
    rng.shuffle(lb)
    da = (rng.standard_normal(2 ** len(la)) + 1j * rng.standard_normal(2 ** len(la))).astype(np.complex64)
    db = (rng.standard_normal(2 ** len(lb)) + 1j * rng.standard_normal(2 ** len(lb))).astype(np.complex64)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ta = torch.from_numpy(da).to("cuda", non_blocking=True) * 1.0  # produced on s
        tb = torch.from_numpy(db).to("cuda", non_blocking=True) * 1.0
        got = contract_pair(DenseTensor([Index(l) for l in la], ta), DenseTensor([Index(l) for l in lb], tb),
                            variant=variant)
        out = got.data.clone()
    s.synchronize()
    want = tncref.contract((tuple(la), (2,) * len(la), da.astype(np.complex128)),
                           (tuple(lb), (2,) * len(lb), db.astype(np.complex128)))
    assert list(got.labels) == list(want[0])
    assert rel_l2(out.cpu().numpy(), want[2]) <= 1e-5
