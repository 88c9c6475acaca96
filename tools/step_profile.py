"""Per-step device time of one C3 slice (dependent steps), with shapes and
the kernels each plan uses.  Usage: python tools/step_profile.py [top]"""
import ctypes
import math
import sys
import time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import bench
from paper_2504_09186_b200 import _lib
from paper_2504_09186_b200.contract import plan_for
from paper_2504_09186_b200.execute import SliceExecutor

top = int(sys.argv[1]) if len(sys.argv) > 1 else 25
work = sys.argv[2] if len(sys.argv) > 2 else "c3"
wl, net, t, s, spec, per, _ids = bench.plan_workload(work)
ex = SliceExecutor(net, s, spec, "single", wl.output_order())
ex.prepare()
ex.run_slice(spec.assignment(0))  # warm plans
torch.cuda.synchronize()
lib = _lib.load()
asn = spec.assignment(1)
values = dict(ex.cache)
rows = []
for p in ex.dependent_positions:
    st = s.steps[p]
    lhs = ex.eng.fetch(s, st.lhs, asn, values)
    rhs = ex.eng.fetch(s, st.rhs, asn, values)
    plan = plan_for(lhs.indices, lhs.data.stride(), rhs.indices, rhs.data.stride(), _lib.C64)
    lib.tnc_profile_enable(1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = ex.eng.contract(lhs, rhs)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    prof = bench._read_prof(lib)
    lib.tnc_profile_enable(0)
    for ref in (st.lhs, st.rhs):
        if ref >= s.n_leaves and ref in values and ref not in ex.cache:
            del values[ref]
    values[st.result] = out
    i = plan.info
    rows.append((dt, p, math.log2(i.m), math.log2(i.k), math.log2(i.n), i.variant, lhs.rank, rhs.rank,
                 {k: round(v["ms"], 3) for k, v in prof.items() if v["launches"]}))
tot = sum(r[0] for r in rows)
print(f"dependent steps {len(rows)}, total {tot*1e3:.1f} ms")
for r in sorted(rows, reverse=True)[:top]:
    print(f"{r[0]*1e3:9.2f} ms  pos {r[1]:4d}  (M,K,N)=2^({r[2]:.0f},{r[3]:.0f},{r[4]:.0f}) var {r[5]} ranks {r[6]},{r[7]} {r[8]}")
