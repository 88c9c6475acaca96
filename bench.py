"""Benchmark of the B200 TNC hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c4|c2|c1] [--slices-per-step S]

(c4: the 7x7x16 circuit, rank-32 slices over a seeded 2^10 subset of the 2^33
slice ids; c2: the fused absorb chain vs 16 separate passes; c1: the three
single-step micro-benchmarks.  Only c3 is the driver's bench line.)

Default workload (config C3 of BASELINE.json, the largest single-GPU one the
metric "TNC effective TFLOP/s & slices/s" is quoted on): 6x6 grid random
circuit, 14 cycles, seed 0, 64 correlated amplitudes (qubits 30-35 open),
reference greedy path (seed 0), reference slicing to rank <= 30 (9 labels,
512 slices).  One *step* = S slices per GPU (weak scaling: slice ids are
dealt round-robin over ranks), each slice contracted with slice-invariant
reuse; partial amplitudes accumulate on device and are summed with one NCCL
all-reduce.  value = effective TFLOP/s (8 * sum M*K*N, the reference's cost
convention) over all ranks; slices/s is reported beside it.

``--impl reference`` times the reference algorithm's CPU implementation (the
numpy oracle port of tncsim's permute+matmul step loop, all host threads) on a
bounded sub-slice sample of the same workload, same metric/unit.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "TNC effective TFLOP/s & slices/s at 1/2/4/8 B200; % of roofline per step"


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(argv: list[str], n: int) -> int:
    """Re-exec this script under torch.distributed.run with one rank per GPU
    (when ``--gpus N`` is given without a torchrun environment)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *argv]
    env = dict(os.environ)
    # communicator setup lines (rank count, NVLS / NVLink transports) on stderr;
    # stdout carries only rank 0's JSON line
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    return subprocess.call(cmd, env=env)


def init_dist(backend: str, local: int):
    """Process group over torchrun's env (MASTER_ADDR / PORT, RANK, WORLD_SIZE)."""
    import torch
    import torch.distributed as dist

    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return dist


def step_unit_ids(unit_ids: list[int], step: int, world: int, per_rank: int) -> list[int]:
    """The job-wide unit ids of one step: world * per_rank consecutive entries
    of the (cyclic) id list; ``distributed.partition`` deals them round-robin."""
    n = len(unit_ids)
    base = step * world * per_rank
    return [unit_ids[(base + j) % n] for j in range(world * per_rank)]


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for name, flag in zip(names, parts[5:9]):
                if flag.lower() in ("active", "1"):
                    reasons.add(name)
        loaded = [s for s in sm if smax and s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measure_tf32_peak(sustain_s: float = 2.0) -> dict:
    """cuBLAS TF32 GEMM throughput on this GPU (MEASURED_PEAKS.json has no
    TF32 entry): fp32 8192^3 matmul with TF32 enabled -- best of 10 (burst)
    and back to back for ``sustain_s`` seconds (sustained), mirroring the
    driver's bf16 measurement."""
    import torch

    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    for _ in range(3):
        torch.matmul(a, b, out=c)
    best = float("inf")
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    reps = max(1, int(sustain_s / best))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        torch.matmul(a, b, out=c)
    e.record()
    e.synchronize()
    sustained = 2 * n ** 3 * reps / (s.elapsed_time(e) / 1e3) / 1e12
    torch.backends.cuda.matmul.allow_tf32 = prev
    del a, b, c
    return {"tf32_tflops": 2 * n ** 3 / best / 1e12, "tf32_tflops_sustained": sustained,
            "how": f"torch fp32 matmul 8192^3 with allow_tf32: best of 10 (burst), {reps} back to back (sustained)"}


def measured_peaks() -> dict:
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        return json.loads(path.read_text())
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "fallback": True}


# -- workload C3 ---------------------------------------------------------------


WORKLOAD_TEXT = {
    "c3": "C3: 6x6 grid, 14 cycles, seed 0, 64 open amplitudes (q30-35), greedy path seed 0, slices to "
          "rank<=30 (9 labels, 512 slices)",
    "c4": "C4: 7x7 grid, 16 cycles, seed 0, 1024 open amplitudes (q39-48), greedy path seed 0, slices to "
          "rank<=32 (33 labels, 2^33 slices); a fixed seeded subset of 2^10 slice ids is cycled",
}


def plan_workload(name: str = "c3"):
    """Reference path (greedy seed 0) + reference slicing; returns
    (workload, network, tree, schedule, spec, multiplies per slice, slice ids)."""
    import numpy as np

    from paper_2504_09186_b200 import greedy_path, linearize, select_slices, tree_metrics
    from paper_2504_09186_b200 import workloads

    wl, cap = (workloads.C3, workloads.C3_MAX_RANK) if name == "c3" else (workloads.C4, workloads.C4_MAX_RANK)
    net = wl.network()
    t = greedy_path(net, 0)
    spec = select_slices(t, cap, 64, 0)
    s = linearize(t)
    per_slice = tree_metrics(t, spec.dims_projected()).total_cost
    if spec.n_subtasks <= 4096:
        ids = list(range(spec.n_subtasks))
    else:
        ids = sorted(int(x) for x in np.random.default_rng(0).choice(spec.n_subtasks, 1024, replace=False))
    return wl, net, t, s, spec, per_slice, ids


def plan_c3():
    wl, net, t, s, spec, per_slice, _ = plan_workload("c3")
    return wl, net, t, s, spec, per_slice


def _oracle_leaves(net):
    from oracle import tncref

    return tncref.cast_leaves([(t.labels, t.dims, t.numpy()) for t in net.tensors], "single")


def run_cpu_subslice(net, s, sub, sid: int = 0) -> float:
    from oracle import tncref

    leaves = _oracle_leaves(net)
    steps = [(st.lhs, st.rhs, st.result) for st in s.steps]
    t0 = time.perf_counter()
    tncref.run_range(leaves, steps, s.n_leaves, 1, len(steps), sub.assignment(sid), {}, "single")
    return time.perf_counter() - t0


def _threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def bench_reference(args) -> None:
    """--impl reference: the reference algorithm on the host cores."""
    world, rank, _ = _dist_env()
    if rank != 0:
        return
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(_threads()))
    from paper_2504_09186_b200 import tree_metrics

    wl, net, t, s, spec, per_slice = plan_c3()
    from paper_2504_09186_b200 import select_slices

    sub = select_slices(t, args.ref_cap, 64, 0)
    mult = tree_metrics(t, sub.dims_projected()).total_cost
    for i in range(args.warmup):
        run_cpu_subslice(net, s, sub, i)
    times = [run_cpu_subslice(net, s, sub, args.warmup + i) for i in range(args.steps)]
    total = sum(times)
    value = 8 * mult * args.steps / total / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded grid RQC)",
        "config": {"workload": f"C3 6x6x14 seed 0, 64 open amps; each step = one sub-slice (cap {args.ref_cap}, "
                               f"{len(sub.entries)} sliced labels) of the cap-30 slicing",
                   "slices_per_s_extrapolated": (args.steps / total) * mult / per_slice},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": _threads(), "kind": "port",
                         "sample": f"{args.steps} C3 sub-slices at cap {args.ref_cap} ({mult} multiplies each), "
                                   "numpy oracle of tncsim permute+matmul (complex128 in flight)"},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_c3(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2504_09186_b200 import _lib
    from paper_2504_09186_b200.execute import SliceExecutor, run_open

    from paper_2504_09186_b200.distributed import accumulate_rank_units, allreduce_partial

    world, rank, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        init_dist("nccl", local)
    lib = _lib.load(require_device=True)
    wl, net, t, s, spec, per_slice, slice_ids = plan_workload(args.workload)
    order = wl.output_order()
    reuse_info = None
    if args.reuse > 0:
        # spindle reuse (the paper's data reuse, reference reuse.py): a unit of
        # work is one reuse program over prod(nested dims) slices
        from paper_2504_09186_b200 import choose_reuse_subset, plan_spindle
        from paper_2504_09186_b200.execute import ReuseRunner

        part_ = choose_reuse_subset(t, spec, None, args.reuse)
        rs, rep = plan_spindle(part_.schedule, part_.spec, None, nested_labels=part_.nested_labels)
        ex = ReuseRunner(net, rs, "single", order)
        unit_slices = ex.slices_per_program
        n_units = ex.n_programs
        if n_units * unit_slices <= 4096:
            slice_ids = list(range(n_units))
        else:
            slice_ids = sorted(int(x) for x in np.random.default_rng(0).choice(
                n_units, max(1, 1024 // unit_slices), replace=False))
        reuse_info = {"nested_labels": [e.index.label for e in rs.nested], "slices_per_program": unit_slices,
                      "programs_sampled": len(slice_ids),
                      "multiplies_saved_factor": float(per_slice * spec.n_subtasks / rep.predicted_multiplies),
                      "predicted_peak_gib": rep.predicted_peak_bytes / 2**30}
    else:
        ex = SliceExecutor(net, s, spec, "single", order)
        unit_slices = 1
    ex.prepare()
    n_ids = len(slice_ids)
    spp = args.slices_per_step

    acc = None
    for i in range(args.warmup):
        acc = accumulate_rank_units(ex, step_unit_ids(slice_ids, i, world, spp), world, rank, acc)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    lib.tnc_profile_enable(1)
    launches0 = lib.tnc_launch_count()
    mult0 = ex.stats.multiplies
    stream = torch.cuda.current_stream()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    start.record(stream)
    part = None
    for i in range(args.steps):
        part = accumulate_rank_units(ex, step_unit_ids(slice_ids, args.warmup + i, world, spp), world, rank, part)
    if world > 1:
        allreduce_partial(part.data)  # the one collective: NCCL all-reduce of the partial amplitudes
    stop.record(stream)
    torch.cuda.synchronize()
    launches = lib.tnc_launch_count() - launches0
    executed_mult = ex.stats.multiplies - mult0
    elapsed = start.elapsed_time(stop) / 1e3
    if world > 1:
        tt = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        elapsed = tt.item()
        dist.barrier()
    clocks = sampler.stop() if sampler else None
    prof = _read_prof(lib)
    lib.tnc_profile_enable(0)
    slices_total = args.steps * spp * world * unit_slices
    flops_total = 8 * per_slice * slices_total
    value = flops_total / elapsed / 1e12

    # end to end through the public API: host-resident leaves (pinned) uploaded
    # every step, slice contracted, amplitudes read back to the host.
    e2e = None
    if rank == 0 and args.e2e_steps > 0:
        host_leaves = [tt_.data.detach().cpu().pin_memory() for tt_ in net.tensors]
        h2d = sum(x.numel() * x.element_size() for x in host_leaves)
        from paper_2504_09186_b200 import DenseTensor, TensorNetwork

        torch.cuda.synchronize()
        e_s, e_e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_s.record()
        d2h = 0
        for i in range(args.e2e_steps):
            # host-resident (pinned) leaves handed to the public API, which
            # uploads them itself (one batched copy)
            dev = [DenseTensor.__new__(DenseTensor)._init_raw(tt_.indices, hl)
                   for tt_, hl in zip(net.tensors, host_leaves)]
            if reuse_info is None:
                amps = run_open(TensorNetwork(dev), t, spec, order, "single",
                                slice_ids=[slice_ids[i % n_ids]]).data.cpu()
            else:
                rr = ReuseRunner(TensorNetwork(dev), rs, "single", order)
                amps = rr.finish(rr.run([slice_ids[i % n_ids]])).data.cpu()
            d2h = amps.numel() * amps.element_size()
        e_e.record()
        torch.cuda.synchronize()
        e_t = e_s.elapsed_time(e_e) / 1e3
        e2e = {"value": 8 * per_slice * unit_slices * args.e2e_steps / e_t / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "slices_per_s": unit_slices * args.e2e_steps / e_t}

    if rank == 0:
        peaks = measured_peaks()
        tf32 = measure_tf32_peak()
        if os.environ.get("TNC_TC_TF32", "0") not in ("", "0"):
            p_eff = tf32["tf32_tflops_sustained"] / 3.0
            kernel_name = "tc_cgemm_kernel<.., F16=false> (3xTF32 tcgen05.mma kind::tf32)"
            peak_source = (f"measured cuBLAS TF32 {tf32['tf32_tflops_sustained']:.0f} TF/s (sustained, this run) "
                           "/ 3 products; MEASURED_PEAKS.json has no TF32 entry")
            dtype = "c64 (3xTF32 tensor-core GEMM, fp32 accumulate)"
        else:
            # 3xFP16: three fp16 tensor-core products per complex-GEMM flop pair;
            # fp16 dense rate == bf16 dense rate, sustained (kernel runs inside a long step)
            p_eff = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops")) / 3.0
            kernel_name = "tc_cgemm_kernel<.., F16=true> (3xFP16 tcgen05.mma kind::f16)"
            peak_source = (f"MEASURED_PEAKS.json bf16_tflops_sustained {peaks.get('bf16_tflops_sustained')} "
                           "TF/s (fp16 rate) / 3 products")
            dtype = "c64 (3xFP16 tensor-core GEMM, fp32 accumulate)"
        tc = prof["tc_gemm"]
        traffic_bytes, traffic_detail = _profiled_traffic(args.workload)
        achieved = tc["flops"] / (tc["ms"] / 1e3) / 1e12 if tc["ms"] > 0 else None
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            from paper_2504_09186_b200 import select_slices, tree_metrics

            os.environ.setdefault("OPENBLAS_NUM_THREADS", str(_threads()))
            sub = select_slices(t, args.cpu_cap, 64, 0)
            mult = tree_metrics(t, sub.dims_projected()).total_cost
            secs = run_cpu_subslice(net, s, sub, 0)
            cpu = {"value": 8 * mult / secs / 1e12, "unit": "TFLOP/s", "cores": _threads(), "kind": "port",
                   "sample": f"one {args.workload.upper()} sub-slice (extra slicing to rank {args.cpu_cap}: {len(sub.entries)} labels, "
                             f"{mult} multiplies) through the numpy oracle of tncsim's step loop, {secs:.1f}s"}
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dtype,
            "data": "synthetic (seeded grid random circuit, SURVEY Appendix A)",
            "config": {"workload": WORKLOAD_TEXT[args.workload],
                       "total_slices": spec.n_subtasks,
                       "extrapolated_hours_all_slices_this_job": spec.n_subtasks / (slices_total / elapsed) / 3600,
                       "slices_per_step_per_gpu": spp * unit_slices, "slices_per_s": slices_total / elapsed,
                       "spindle_reuse": reuse_info,
                       "executed_tflops": (8 * executed_mult / elapsed / 1e12) if reuse_info else None,
                       "flops_per_slice": 8 * per_slice, "l2": "inputs > L2 (intermediates up to 8 GiB)",
                       "parallelism": f"slices round-robin over {world} GPU(s) + 1 NCCL all-reduce",
                       "nccl": ({"world": dist.get_world_size(), "backend": dist.get_backend(),
                                 "version": ".".join(map(str, torch.cuda.nccl.version()))}
                                if world > 1 else None)},
            "gpu_launches": int(launches),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": p_eff, "unit": "TFLOP/s",
                         "frac": (achieved / p_eff) if achieved else None,
                         "traffic": traffic_bytes,
                         "traffic_detail": traffic_detail,
                         "kernel": kernel_name, "peak_source": peak_source,
                         "launches": tc["launches"], "share_of_step": tc["ms"] / 1e3 / elapsed},
            "kernels": prof, "clocks": clocks, "e2e": e2e, "cpu_baseline": cpu,
            "peaks": {"hbm_gbs": peaks.get("hbm_gbs"), "bf16_tflops": peaks.get("bf16_tflops"),
                      "bf16_tflops_sustained": peaks.get("bf16_tflops_sustained"),
                      "tf32_measured_this_run": tf32,
                      "p_eff_3xtf32_tflops": tf32["tf32_tflops_sustained"] / 3.0},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


class _DryExecutor:
    """Kernel-free stand-in for the slice executor (``--dry-run``): slice i's
    root is a known complex vector, so the launcher, the round-robin deal and
    the all-reduce can be checked on CPU ranks (gloo)."""

    n_roots = 64

    def __init__(self, n_units: int):
        import torch

        self.n_units = n_units
        self.seen: list[int] = []
        self._t = torch

    def root(self, sid: int):
        t = self._t
        k = t.arange(self.n_roots, dtype=t.float64)
        return t.complex(t.cos(0.1 * sid * k), t.sin(0.3 * sid + k))

    def run(self, ids, acc=None):
        for sid in ids:
            self.seen.append(sid)
            r = self.root(sid)
            acc = r.clone() if acc is None else acc + r
        return acc

    def zeros(self):
        return self._t.zeros(self.n_roots, dtype=self._t.complex128)


def bench_dry(args) -> None:
    """--dry-run: the multi-rank bench loop without kernels (gloo on CPU)."""
    import torch

    from paper_2504_09186_b200.distributed import accumulate_rank_units, allreduce_partial

    world, rank, local = _dist_env()
    dist = init_dist("gloo", local) if world > 1 else None
    ex = _DryExecutor(512)
    ids = list(range(ex.n_units))
    acc = None
    steps = args.warmup + args.steps
    for i in range(steps):
        acc = accumulate_rank_units(ex, step_unit_ids(ids, i, world, args.slices_per_step), world, rank, acc)
    if world > 1:
        allreduce_partial(acc)
        seen = [None] * world
        dist.all_gather_object(seen, ex.seen)
    else:
        seen = [ex.seen]
    want = None
    for i in range(steps):
        want = ex.run(step_unit_ids(ids, i, world, args.slices_per_step), want)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                          "per_rank_ids": seen, "max_abs_err": float((acc - want).abs().max()),
                          "backend": dist.get_backend() if dist else None}), flush=True)
    if dist:
        dist.destroy_process_group()


FMA_LANES_PER_CLK_PER_SM = 118.0  # measured: tools/ffma2_rate.cu -> profiles/r02_ffma2_rate.txt


def _fp32_floor(n_gates: int, n_elems: int, seconds: float) -> dict:
    """FP32-pipe time of a gate chain (16 real FMAs per element per gate) at the
    measured FMA issue rate, at the maximum SM clock (the K4 passes run
    unthrottled), and the fraction of it the fused chain reached."""
    import torch

    prop = torch.cuda.get_device_properties(0)
    sm_hz = measured_peaks().get("sm_max_mhz", 1965.0) * 1e6
    fmas = 16.0 * n_gates * n_elems
    floor = fmas / (FMA_LANES_PER_CLK_PER_SM * prop.multi_processor_count * sm_hz)
    return {"ms": floor * 1e3, "frac": floor / seconds, "fma_lanes_per_clk_per_sm": FMA_LANES_PER_CLK_PER_SM,
            "sm_mhz": sm_hz / 1e6}


def bench_c2(args) -> None:
    """Config C2: rank-30 tensor (8 GiB) absorbing 16 random two-qubit gates --
    fused K4 chain vs 16 separate contract_pair passes (HBM-bound)."""
    import torch

    from paper_2504_09186_b200 import DenseTensor, Index, _lib, contract_pair
    from paper_2504_09186_b200.fusion import absorb_chain
    from paper_2504_09186_b200.workloads import C2

    torch.cuda.set_device(0)
    lib = _lib.load(require_device=True)
    t_labels, data, gates = C2.build()
    t = DenseTensor([Index(l) for l in t_labels], data)
    gs = [DenseTensor([Index(oa), Index(ob), Index(ia), Index(ib)], u) for ia, ib, oa, ob, u in gates]
    del data

    def timed(fn, reps):
        for _ in range(args.warmup):
            out = fn()
            del out
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        lib.tnc_profile_enable(1)
        s.record()
        for _ in range(reps):
            out = fn()
            del out
        e.record()
        e.synchronize()
        prof = _read_prof(lib)
        lib.tnc_profile_enable(0)
        return s.elapsed_time(e) / 1e3 / reps, prof

    def separate():
        cur = t
        for g in gs:
            cur = contract_pair(cur, g)
        return cur

    fused_t, prof = timed(lambda: absorb_chain(t, gs), args.steps)
    sep_t, _ = timed(separate, max(1, args.steps // 4))
    nbytes = 2 * 8 * (1 << 30)
    ab = prof["absorb"]
    peaks = measured_peaks()
    line = {
        "metric": "C2 step-fusion chain: HBM GB/s (algorithmic 2 x 8 GiB per chain)", "value": nbytes / fused_t / 1e9,
        "unit": "GB/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": fused_t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c64",
        "data": "synthetic (seeded rank-30 tensor, Haar x fSim gates)",
        "config": {"workload": "C2: rank-30 complex64 tensor absorbs 16 two-qubit gates", "separate_ms": sep_t * 1e3,
                   "fused_speedup": sep_t / fused_t, "passes": ab["launches"] // max(1, args.steps)},
        "roofline": {"bound": "hbm", "achieved": nbytes / fused_t / 1e9, "peak": peaks.get("hbm_gbs"),
                     "unit": "GB/s", "frac": nbytes / fused_t / 1e9 / peaks.get("hbm_gbs"), "traffic": None,
                     "kernel": "absorb_pass_kernel", "note": "algorithmic bytes = one read + one write of T"},
        # The gate math runs on the FP32 pipe: 16 real FMAs per element per gate
        # against the measured 118 FMA lanes / clk / SM (FFMA and FFMA2 alike,
        # profiles/r02_ffma2_rate.txt) at the SM clock the kernel ran at.
        "fp32_floor": _fp32_floor(len(gs), 1 << 30, fused_t),
        "kernels": prof,
    }
    print(json.dumps(line), flush=True)


def bench_c1(args) -> None:
    """Config C1 a/b/c single-step micro-benchmarks (contract + output permutation)."""
    import torch

    from paper_2504_09186_b200 import DenseTensor, Index, _lib, contract_pair
    from paper_2504_09186_b200.contract import contract_into, plan_for
    from paper_2504_09186_b200.errors import TncError
    from paper_2504_09186_b200.workloads import c1_cases

    torch.cuda.set_device(0)
    lib = _lib.load(require_device=True)
    peaks = measured_peaks()
    tf32 = measure_tf32_peak(0.5)
    for case in c1_cases():
        ia, ib, io = case.index_lists()
        da, db = case.data()
        a, b = DenseTensor(ia, da), DenseTensor(ib, db)
        del da, db
        try:
            contract_pair(a, b, out_order=io, variant=args.variant)
        except TncError as exc:  # forced variant outside this shape's envelope
            print(json.dumps({"metric": f"{case.name} contract+permute", "skipped": str(exc)}), flush=True)
            continue
        # one plan, one preallocated output (the allocator stays out of the
        # timed region); each step is the full tnc_contract of the step
        plan = plan_for(a.indices, a.data.stride(), b.indices, b.data.stride(), _lib.C64, io, args.variant)
        out = torch.empty(tuple(ix.dim for ix in plan.out_indices), dtype=a.data.dtype, device=a.data.device)
        for _ in range(args.warmup):
            contract_into(plan, a.data, b.data, out)
        torch.cuda.synchronize()
        lib.tnc_profile_enable(1)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            contract_into(plan, a.data, b.data, out)
        e.record()
        e.synchronize()
        prof = _read_prof(lib)
        lib.tnc_profile_enable(0)
        dt = s.elapsed_time(e) / 1e3 / args.steps
        m = 2 ** sum(1 for l in case.a_labels if l.startswith("a"))
        k = 2 ** sum(1 for l in case.a_labels if l.startswith("k"))
        n = 2 ** sum(1 for l in case.b_labels if l.startswith("b"))
        flops = 8.0 * m * k * n
        nbytes = 8.0 * (m * k + k * n + m * n)
        # step roofline: max(algorithmic bytes / HBM peak, flops / P_eff), burst peaks
        # (the kernel is timed alone); P_eff = the split scheme's tensor rate / 3 products
        f16 = prof["tc_gemm"]["launches"] > 0
        p_eff = (peaks.get("bf16_tflops", 1590.0) if f16 else tf32["tf32_tflops"]) / 3.0
        t_hbm, t_tc = nbytes / (peaks.get("hbm_gbs") * 1e9), flops / (p_eff * 1e12)
        bound = "tensor" if t_tc > t_hbm else "hbm"
        roof = ({"bound": "tensor", "achieved": flops / dt / 1e12, "peak": p_eff, "unit": "TFLOP/s"} if bound == "tensor"
                else {"bound": "hbm", "achieved": nbytes / dt / 1e9, "peak": peaks.get("hbm_gbs"), "unit": "GB/s"})
        roof.update({"frac": max(t_hbm, t_tc) / dt, "traffic": None, "hbm_floor_ms": t_hbm * 1e3,
                     "tensor_floor_ms": t_tc * 1e3,
                     "scheme": "3xFP16 (bf16_tflops / 3)" if f16 else "3xTF32 (TF32 burst measured this run / 3)"})
        print(json.dumps({"metric": f"{case.name} contract+permute", "value": flops / dt / 1e12, "unit": "TFLOP/s",
                          "ms_per_step": dt * 1e3, "GB_per_s_algorithmic": nbytes / dt / 1e9,
                          "hbm_frac": nbytes / dt / 1e9 / peaks.get("hbm_gbs"), "roofline": roof, "shape_log2": [
                              m.bit_length() - 1, k.bit_length() - 1, n.bit_length() - 1],
                          "tf32_measured_this_run": tf32, "kernels": prof}),
              flush=True)
        del a, b, out, plan


def _profiled_traffic(workload: str):
    """DRAM bytes of the dominant tensor-core GEMM launch (the (15,15,14) C3
    step) from the latest committed ncu capture of this command
    (profiles/rNN_tc_traffic.json), with its own algorithmic bytes; None when
    not captured."""
    import glob

    paths = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                          "r*_tc_traffic.json")))
    if workload != "c3" or not paths:
        return None, None
    with open(paths[-1]) as f:
        d = json.load(f)
    dom = d.get("dominant")
    if dom is None:  # round-1 format: launches only
        launch = max(d["launches"], key=lambda x: x.get("gpu__time_duration.sum", 0))
        dom = {"dram_bytes": launch["dram__bytes_read.sum"] + launch["dram__bytes_write.sum"],
               "algorithmic_bytes_c64": 8 * (2 ** 30 + 2 ** 29 + 2 ** 29)}
        dom["traffic_over_algorithmic"] = dom["dram_bytes"] / dom["algorithmic_bytes_c64"]
    return dom["dram_bytes"], {"source": os.path.relpath(paths[-1], os.path.dirname(os.path.abspath(__file__))),
                               "dominant_launch": dom}


def _read_prof(lib) -> dict:
    import ctypes

    out = {}
    for kind, name in enumerate(["tc_gemm", "simt_gemm", "permute", "split_prep", "reduce", "absorb", "axpy", "stream", "tc_gather"]):
        n = ctypes.c_int64()
        ms, fl, by = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        lib.tnc_profile_read(kind, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(fl), ctypes.byref(by))
        out[name] = {"launches": n.value, "ms": ms.value, "flops": fl.value, "bytes": by.value}
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=["c3", "c4", "c2", "c1"])
    ap.add_argument("--slices-per-step", type=int, default=1)
    ap.add_argument("--variant", type=int, default=0, help="c1: force a kernel variant (tnc_variant)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-cap", type=int, default=25)
    ap.add_argument("--ref-cap", type=int, default=25)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reuse", type=int, default=0,
                    help="spindle reuse with this many nested sliced labels (0: slice-invariant reuse only)")
    ap.add_argument("--dry-run", action="store_true",
                    help="kernel-free multi-rank loop on CPU (gloo): launcher / deal / all-reduce check")
    args = ap.parse_args()
    import paper_2504_09186_b200._lib as _l  # noqa: F401  (fail fast if the package is broken)
    if args.impl == "reference":
        bench_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(launch_ranks(sys.argv[1:], args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if args.dry_run:
        bench_dry(args)
        return
    {"c3": bench_c3, "c4": bench_c3, "c2": bench_c2, "c1": bench_c1}[args.workload](args)


if __name__ == "__main__":
    main()
