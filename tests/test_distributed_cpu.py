"""Multi-rank slice partitioning + all-reduce on CPU (gloo, world_size 2).

The per-slice roots come from the reference's own golden per-slice outputs,
so this checks the host-side distribution logic (ownership, fold order,
collective) independently of the GPU kernels."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import arr, load_golden, rel_l2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, reproducible, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_09186_b200.distributed import partition, run_partitioned

    g = load_golden("sliced")
    roots = [torch.from_numpy(arr(it["data"]).astype(np.complex128)) for it in g["open_net"]["per_slice"]]
    seen = []

    def evaluate(sid):
        seen.append(sid)
        return roots[sid]

    total = run_partitioned(evaluate, len(roots), world, rank, reproducible=reproducible)
    out_q.put((rank, seen, total.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("reproducible", [False, True])
def test_two_rank_slice_sum_matches_reference_total(reproducible):
    g = load_golden("sliced")
    n = len(g["open_net"]["per_slice"])
    assert n == 2 ** len(g["open_net"]["slice_spec"])
    want = sum(arr(it["data"]).astype(np.complex128) for it in g["open_net"]["per_slice"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, reproducible, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    owned = {}
    for rank, seen, total in results:
        assert seen == list(range(rank, n, 2))  # round-robin ownership, slice order
        assert rel_l2(total, want) < 1e-12
        owned[rank] = seen
    assert sorted(owned[0] + owned[1]) == list(range(n))


def test_partition_covers_every_slice_once():
    from paper_2504_09186_b200.distributed import partition

    for world in (1, 2, 3, 8):
        got = sorted(s for r in range(world) for s in partition(37, world, r))
        assert got == list(range(37))
    with pytest.raises(ValueError):
        partition(4, 2, 2)


class _RootsExecutor:
    """Executor stand-in: unit i's root is the reference's golden slice root."""

    def __init__(self, roots):
        self.roots = roots
        self.n_units = len(roots)
        self.calls = []

    def run(self, ids, acc=None):
        for i in ids:
            self.calls.append(i)
            acc = self.roots[i].clone() if acc is None else acc + self.roots[i]
        return _Wrap(acc)

    def zeros(self):
        return _Wrap(torch.zeros_like(self.roots[0]))

    def finish(self, total):
        return total.data


class _Wrap:
    def __init__(self, data):
        self.data = data.data if isinstance(data, _Wrap) else data

    def __add__(self, other):
        return _Wrap(self.data + other)

    def clone(self):
        return _Wrap(self.data.clone())


def _worker_units(rank, world, port, n_units, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2504_09186_b200.distributed import run_slices_distributed

    g = load_golden("sliced")
    roots = [torch.from_numpy(arr(it["data"]).astype(np.complex128)) for it in g["open_net"]["per_slice"]]
    ex = _RootsExecutor(roots)
    total = run_slices_distributed(ex, world, rank, slice_ids=list(range(n_units)))
    out_q.put((rank, ex.calls, total.numpy()))
    dist.destroy_process_group()


def test_three_ranks_two_units_empty_rank_joins_with_zeros():
    """More ranks than units: rank 2 owns nothing, evaluates nothing and
    contributes zeros of the root's shape to the all-reduce."""
    g = load_golden("sliced")
    roots = [arr(it["data"]).astype(np.complex128) for it in g["open_net"]["per_slice"]]
    want = roots[0] + roots[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_units, args=(r, 3, port, 2, q)) for r in range(3)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [calls for _, calls, _ in results] == [[0], [1], []]
    for _, _, total in results:
        assert rel_l2(total, want) < 1e-12
