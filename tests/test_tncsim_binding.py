"""The reference-side binding of INTEGRATION.md section 1
(``paper_2504_09186_b200/tncsim_binding.py``: raw ctypes over the C-ABI, none
of this package's Python mirror).

* host-only: the plans it builds from reference-style tensors carry the
  reference's result legs, shapes and multiplier choice (goldens);
* against the reference's own ``_Engine`` (only where ``/root/reference`` is
  mounted): ``tncsim.execute.contract_pair`` is patched with the binding and
  ``tncsim.run_direct`` runs the C0 circuit through it.  Without a GPU here
  the device leg is stood in for by the numpy oracle (test infrastructure);
  what is checked is the marshalling: one C-ABI plan per step, its result
  legs / dims equal to what the reference's step produced, amplitude equal to
  the unpatched run;
* on the GPU: the same binding end to end on the reference's golden operand
  pairs through ``tnc_contract``.
"""

import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import arr, load_golden, rel_l2
from oracle import tncref

REF_SRC = Path("/root/reference/pkg/src")


def _tensor(legs, data):
    return SimpleNamespace(indices=tuple(SimpleNamespace(label=l, dim=d) for l, d in legs), data=data)


def test_binding_plans_match_reference_goldens():
    from paper_2504_09186_b200 import tncsim_binding as tb

    n = 0
    for case in load_golden("contract")["cases"]:
        a = _tensor(case["a"], arr(case["a_data"]))
        b = _tensor(case["b"], arr(case["b_data"]))
        handle, info, out = tb.plan(a, b)
        try:
            assert [ix.label for ix in out] == case["out_labels"]
            assert [info.m, info.k, info.n] == case["shape"]
            assert bool(info.b_is_multiplier) == case["b_is_multiplier"]
        finally:
            tb.library().tnc_plan_destroy(handle)
        n += 1
    assert n > 0


def test_binding_reports_reference_errors():
    from paper_2504_09186_b200 import tncsim_binding as tb

    a = _tensor([("x", 2), ("k", 3)], np.zeros(6, np.complex64))
    b = _tensor([("k", 2), ("y", 2)], np.zeros(4, np.complex64))
    with pytest.raises(tb.BindingError) as err:  # shared label, different dims: ContractionError (contract.py:67-70)
        tb.plan(a, b)
    assert err.value.code == 4 and "mismatched dims" in str(err.value)  # TNC_ERR_CONTRACTION


@pytest.mark.skipif(not REF_SRC.exists(), reason="the reference is not mounted on this box")
def test_binding_drives_the_reference_engine(monkeypatch):
    sys.path.insert(0, str(REF_SRC))
    try:
        import tncsim
        from paper_2504_09186_b200 import tncsim_binding as tb, workloads

        text = workloads.grid_circuit_text(3, 4, 8, 0)
        circ = tncsim.parse_circuit(text)
        net = tncsim.circuit_to_network(circ, "0" * circ.n_qubits)
        tree = tncsim.greedy_path(net, 0)
        want, want_stats = tncsim.run_direct(net, tree, precision="single")

        steps = []
        stash = {}
        real_plan = tb.plan

        def plan(a, b):
            stash["ab"] = (a, b)
            return real_plan(a, b)

        def device(handle, info, a_host, b_host):
            a, b = stash["ab"]
            ref = tncref.contract((tuple(ix.label for ix in a.indices), tuple(ix.dim for ix in a.indices), a_host),
                                  (tuple(ix.label for ix in b.indices), tuple(ix.dim for ix in b.indices), b_host))
            assert list(ref[1]) == [info.out_dims[i] for i in range(info.out_rank)]
            steps.append(ref[0])
            return ref[2]

        monkeypatch.setattr(tb, "plan", plan)
        monkeypatch.setattr(tb, "_device_contract", device)
        restore = tb.install(tncsim)
        try:
            got, got_stats = tncsim.run_direct(net, tree, precision="single")
        finally:
            restore()
        assert len(steps) == len(tree.to_ssa_path())  # every step of execute.py:137-178 went through the C-ABI plan
        assert got_stats.multiplies == want_stats.multiplies
        assert abs(got - want) <= 1e-6 * abs(want)
        import tncsim.execute as ex
        assert ex.contract_pair is tncsim.contract.contract_pair  # restored
    finally:
        sys.path.remove(str(REF_SRC))


@pytest.mark.gpu
def test_binding_contract_goldens_on_device(cuda_ready):
    from paper_2504_09186_b200 import tncsim_binding as tb

    for case in load_golden("contract")["cases"]:
        for key, dt, tol in (("out_c64", np.complex64, 1e-5), ("out_c128", np.complex128, 1e-10)):
            a = _tensor(case["a"], arr(case["a_data"]).astype(dt))
            b = _tensor(case["b"], arr(case["b_data"]).astype(dt))
            out = tb.contract_pair(a, b)
            assert [ix.label for ix in out.indices] == case["out_labels"]
            assert out.data.dtype == dt
            assert rel_l2(out.data, arr(case[key])) <= tol


@pytest.mark.gpu
def test_binding_promotes_mixed_precision(cuda_ready):
    from paper_2504_09186_b200 import tncsim_binding as tb

    rng = np.random.default_rng(3)
    a_data = (rng.standard_normal(32) + 1j * rng.standard_normal(32)).astype(np.complex64)
    b_data = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    a = _tensor([("a", 2), ("k", 4), ("b", 4)], a_data)
    b = _tensor([("k", 4), ("c", 4)], b_data)
    out = tb.contract_pair(a, b)
    ref = tncref.contract((("a", "k", "b"), (2, 4, 4), a_data.astype(np.complex128)), (("k", "c"), (4, 4), b_data))
    assert out.data.dtype == np.complex128 and [ix.label for ix in out.indices] == list(ref[0])
    assert rel_l2(out.data, ref[2]) <= 1e-10
