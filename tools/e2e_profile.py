"""Where the end-to-end (run_open from host leaves) time of one C3 slice goes:
host setup, slice-invariant steps, dependent steps; plus a cProfile of the
host side.  usage: python tools/e2e_profile.py"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2504_09186_b200.execute import SliceExecutor, run_open  # noqa: E402
from paper_2504_09186_b200.tree import linearize  # noqa: E402

wl, net, t, s, spec, per_slice, ids = bench.plan_workload("c3")
order = wl.output_order()
run_open(net, t, spec, order, "single", slice_ids=[ids[0]])  # warm plans
torch.cuda.synchronize()


def phases():
    t0 = time.perf_counter()
    s2 = linearize(t)
    t1 = time.perf_counter()
    ex = SliceExecutor(net, s2, spec, "single", order)
    t2 = time.perf_counter()
    ex.prepare()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    out = ex.finish(ex.run([ids[1]])).data.cpu()
    t4 = time.perf_counter()
    print(f"linearize {1e3*(t1-t0):.1f} ms  executor init {1e3*(t2-t1):.1f} ms  invariant steps "
          f"{1e3*(t3-t2):.1f} ms ({len(ex.invariant_positions)})  slice {1e3*(t4-t3):.1f} ms "
          f"({len(ex.dependent_positions)} steps)", flush=True)


phases()
phases()
pr = cProfile.Profile()
pr.enable()
run_open(net, t, spec, order, "single", slice_ids=[ids[2]]).data.cpu()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
