"""Multi-GPU slice partitioning with one all-reduce.

Slices are independent (reference ``execute.py:204-230``), so the only
exchange step is the final sum: slice id i (mixed radix over
``SliceSpec.entries``) goes to rank ``i % world``; every rank folds its
slices into a device-resident partial amplitude tensor in increasing slice-id
order and one ``all_reduce`` (NCCL over NVLink/NVSwitch; gloo in the CPU
tests) sums the partials.  The collective carries 2 x 64 floats at C3 and
2 x 1024 at C4 -- latency-bound, negligible next to the slice work.

The reference has no distributed path (its workers are threads over outer
slices, ``execute.py:353-362``); ``reproducible=True`` gathers the per-rank
partials and sums them in rank order on every rank instead of relying on the
collective's reduction order.
"""

from __future__ import annotations

from typing import Callable, Iterable, Sequence

import torch
import torch.distributed as dist


def partition(n_slices: int, world: int, rank: int) -> list[int]:
    """Round-robin slice ownership: slice i belongs to rank i % world."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    return list(range(rank, n_slices, world))


def _as_real(t: torch.Tensor) -> torch.Tensor:
    return torch.view_as_real(t) if t.is_complex() else t


def allreduce_partial(partial: torch.Tensor, group=None, reproducible: bool = False) -> torch.Tensor:
    """Sum a complex partial over all ranks (in place when not reproducible)."""
    if not dist.is_available() or not dist.is_initialized():
        return partial
    if not reproducible:
        dist.all_reduce(_as_real(partial), op=dist.ReduceOp.SUM, group=group)
        return partial
    world = dist.get_world_size(group)
    parts = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(parts, partial.contiguous(), group=group)
    total = parts[0].clone()
    for p in parts[1:]:
        total += p
    partial.copy_(total)
    return partial


def run_partitioned(evaluate: Callable[[int], torch.Tensor], n_slices: int, world: int, rank: int,
                    group=None, reproducible: bool = False,
                    zeros: Callable[[], torch.Tensor] | None = None) -> torch.Tensor:
    """Evaluate this rank's slices with ``evaluate(slice_id)`` (device tensor),
    fold them in slice order, then all-reduce.  Returns the global sum.  A
    rank that owns no slice joins the collective with ``zeros()``."""
    acc = None
    for sid in partition(n_slices, world, rank):
        part = evaluate(sid)
        acc = part.clone() if acc is None else acc.add_(part)
    if acc is None:
        if zeros is None:
            raise ValueError(f"rank {rank} owns no slice of {n_slices}: pass zeros= for the output shape")
        acc = zeros()
    return allreduce_partial(acc, group, reproducible)


def _world_rank(world, rank, group):
    if world is None:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    return world, rank


def accumulate_rank_units(executor, unit_ids: Sequence[int], world: int | None = None, rank: int | None = None,
                          acc=None, group=None):
    """This rank's share (round-robin, ``partition``) of ``unit_ids`` folded
    into ``acc`` on the device -- no collective.  A unit is a slice
    (:class:`SliceExecutor`) or a reuse program (:class:`ReuseRunner`).  Used
    by the bench, which accumulates several steps and all-reduces once."""
    world, rank = _world_rank(world, rank, group)
    ids = list(unit_ids)
    mine = [ids[i] for i in partition(len(ids), world, rank)]
    if mine:
        acc = executor.run(mine, acc)
    elif acc is None:
        acc = executor.zeros()
    return acc


def run_slices_distributed(executor, world: int | None = None, rank: int | None = None,
                           slice_ids: Sequence[int] | None = None, group=None, reproducible: bool = False):
    """Distributed sum of a :class:`~paper_2504_09186_b200.execute.SliceExecutor`
    (or ``ReuseRunner``) over all (or the given) units; returns the output
    tensor on every rank."""
    world, rank = _world_rank(world, rank, group)
    ids = list(range(executor.n_units)) if slice_ids is None else list(slice_ids)
    total = accumulate_rank_units(executor, ids, world, rank, None, group)
    allreduce_partial(total.data, group, reproducible)
    return executor.finish(total)
