"""C4 spindle reuse at the reference's default max_k = 12 on one B200.

One program covers 2^12 = 4096 slices (~1.4 h of GEMM work), so this runs a
PREFIX of program 0 -- the first N actions, which include the full first
descent through the 12 nested forks (the planner's peak) -- through the device
action interpreter, and reports the device memory high-water mark against the
planner's predicted peak and the time per action.

    python tools/c4_reuse12.py [n_actions] > profiles/r02_c4_reuse12.json
"""

import json
import sys
import time

import torch

sys.path.insert(0, ".")

from paper_2504_09186_b200 import choose_reuse_subset, greedy_path, plan_spindle, select_slices  # noqa: E402
from paper_2504_09186_b200 import workloads  # noqa: E402
from paper_2504_09186_b200.execute import ReuseRunner, _run_program  # noqa: E402
from paper_2504_09186_b200.reuse import ReuseSchedule  # noqa: E402


def main():
    n_actions = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    t0 = time.perf_counter()
    net = workloads.C4.network()
    t = greedy_path(net, 0)
    spec = select_slices(t, workloads.C4_MAX_RANK, 64, 0)
    part = choose_reuse_subset(t, spec, None, 12)
    rs, rep = plan_spindle(part.schedule, part.spec, None, nested_labels=part.nested_labels)
    t_plan = time.perf_counter() - t0
    rr = ReuseRunner(net, rs, "single")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rr.prepare()
    torch.cuda.synchronize()
    t_prep = time.perf_counter() - t1
    base_mem = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    prefix = ReuseSchedule(rs.schedule, rs.actions[:n_actions], rs.nested, rs.outer, rs.demoted)
    kinds = {}
    for a in prefix.actions:
        kinds[a.kind] = kinds.get(a.kind, 0) + 1
    t2 = time.perf_counter()
    err = None
    try:
        _run_program(rr.eng, prefix, rr.outer_assignment(0), rr.deps, None, open_root=True, cache=rr.cache,
                     invariant=rr.invariant)
    except Exception as exc:  # a prefix may end before the root is produced
        err = f"{type(exc).__name__}: {exc}"
    torch.cuda.synchronize()
    t_run = time.perf_counter() - t2
    peak = torch.cuda.max_memory_allocated()
    print(json.dumps({
        "what": "C4 spindle reuse, reference default max_k = 12: prefix of program 0 on one B200",
        "nested_labels": part.nested_labels, "outer_labels": [e.index.label for e in part.outer],
        "actions_total": len(rs.actions), "actions_run": len(prefix.actions), "action_kinds_run": kinds,
        "predicted_peak_gib": rep.predicted_peak_bytes / 2 ** 30,
        "device_peak_gib_during_prefix": peak / 2 ** 30,
        "device_resident_before_prefix_gib (leaves + slice-invariant cache)": base_mem / 2 ** 30,
        "predicted_multiplies_all": str(rep.predicted_multiplies),
        "overhead_with_reuse": float(rep.overhead_with_reuse) if hasattr(rep, "overhead_with_reuse") else None,
        "plan_s": t_plan, "prepare_s": t_prep, "prefix_s": t_run, "prefix_end": err,
        "device": torch.cuda.get_device_name(0),
    }, indent=1))


if __name__ == "__main__":
    main()
