"""Per-launch kernel times inside one dependent step of a C3/C4 slice:
python tools/step_ops.py c4 844  (prints each permute / split / GEMM launch)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import bench  # noqa: E402
from paper_2504_09186_b200 import _lib  # noqa: E402
from paper_2504_09186_b200.contract import plan_for  # noqa: E402
from paper_2504_09186_b200.execute import SliceExecutor  # noqa: E402

work, pos = sys.argv[1], int(sys.argv[2])
wl, net, t, s, spec, per_slice, _ids = bench.plan_workload(work)
ex = SliceExecutor(net, s, spec, "single", wl.output_order())
ex.prepare()
asn = spec.assignment(1)
values = dict(ex.cache)
lib = _lib.load()
for p in ex.dependent_positions:
    st = s.steps[p]
    lhs = ex.eng.fetch(s, st.lhs, asn, values)
    rhs = ex.eng.fetch(s, st.rhs, asn, values)
    if p == pos:
        plan = plan_for(lhs.indices, lhs.data.stride(), rhs.indices, rhs.data.stride(), _lib.C64)
        print("lhs", [ix.label for ix in lhs.indices], lhs.data.stride()[:3], "...")
        print("rhs", [ix.label for ix in rhs.indices])
        for rep in range(2):
            torch.cuda.synchronize()
            lib.tnc_profile_enable(1)
            out = ex.eng.contract(lhs, rhs)
            torch.cuda.synchronize()
            print(rep, {k: (v["launches"], round(v["ms"], 3), round(v["bytes"] / 1e9, 2))
                        for k, v in bench._read_prof(lib).items() if v["launches"]})
            lib.tnc_profile_enable(0)
        break
    out = ex.eng.contract(lhs, rhs)
    for ref in (st.lhs, st.rhs):
        if ref >= s.n_leaves and ref in values and ref not in ex.cache:
            del values[ref]
    values[st.result] = out
