"""Exchange formats against bytes the reference itself wrote
(tests/golden/spill.json.gz, oracle/gen_golden.py section ``spill``):

* the TNCPART1 partials spill (reference execute.py:468-506) -- bytes equal,
  read back key-for-key;
* DenseTensor.to_bytes / from_bytes (reference tensor.py:146-178) -- bytes
  equal for single and double precision, exact round trip.
"""

import base64

import numpy as np
import pytest

from conftest import arr, load_golden


@pytest.fixture(scope="module")
def spill():
    return load_golden("spill")


def _result(g):
    from paper_2504_09186_b200.execute import RunResult, RunStats

    partials = {tuple(k): complex(re, im) for k, (re, im) in g["partials"]}
    return RunResult(sum(partials.values()), RunStats(), partials, tuple(g["labels"]), tuple(g["dims"]))


def test_write_partials_bytes_equal_reference(spill, tmp_path):
    from paper_2504_09186_b200.execute import write_partials

    path = tmp_path / "p.bin"
    write_partials(str(path), _result(spill))
    assert path.read_bytes() == base64.b64decode(spill["spill_b64"])


def test_read_partials_of_reference_file(spill, tmp_path):
    from paper_2504_09186_b200.execute import read_partials

    path = tmp_path / "ref.bin"
    path.write_bytes(base64.b64decode(spill["spill_b64"]))
    labels, dims, partials = read_partials(str(path))
    assert labels == tuple(spill["labels"]) and dims == tuple(spill["dims"])
    assert partials == {tuple(k): complex(re, im) for k, (re, im) in spill["partials"]}
    assert len(partials) == int(np.prod(dims))


def test_read_partials_rejects_foreign_file(tmp_path):
    from paper_2504_09186_b200 import TncError
    from paper_2504_09186_b200.execute import read_partials

    path = tmp_path / "x.bin"
    path.write_bytes(b"NOTASPIL" + b"\0" * 16)
    with pytest.raises(TncError):
        read_partials(str(path))


def test_tensor_bytes_equal_reference(spill):
    from paper_2504_09186_b200 import DenseTensor, Index

    for g in spill["tensors"]:
        data = arr(g["data"])
        t = DenseTensor([Index(l, d) for l, d in zip(g["labels"], g["dims"])], data, precision=g["precision"])
        raw = base64.b64decode(g["bytes"])
        assert t.to_bytes() == raw
        back = DenseTensor.from_bytes(raw)
        assert back.labels == tuple(g["labels"]) and back.dims == tuple(g["dims"])
        assert back.precision == g["precision"]
        assert np.array_equal(back.numpy(), data)
