"""Multi-GPU: the iteration space sharded over one process per GPU.

The GPU level reuses the reference's block rule (devicert.static_bounds,
devicert.py:110-115): rank r of G owns static_bounds(lb, ub, r, G); inside a
GPU the team and thread levels apply the schedule again (runtime.reduce).
Per-GPU partials are combined by one collective over NVLink/NVSwitch:

  * integer add/max/min: one NCCL all-reduce (bit-exact for any combine
    order; int64 SUM wraps mod 2^64 exactly like the reference's adds)
  * fp (or deterministic=True): all-gather of the G partials, then every rank
    folds them in rank order on its device (omprt_combine_partials), so all
    ranks hold the identical, run-to-run deterministic value.

The reference itself is single-device; there is no
reference collective to match.  torch.distributed is the plumbing (NCCL on
GPUs, gloo for the CPU tests of this host logic).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import runtime

_REDUCE_OPS = {"add": dist.ReduceOp.SUM, "max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN}


def shard(lb: int, ub: int, rank: int, world: int) -> tuple[int, int]:
    """Iterations [lo, hi] owned by `rank` (empty when lo > hi)."""
    return runtime.static_bounds(lb, ub, rank, world)


def gather_partials(partial: torch.Tensor, group=None) -> torch.Tensor:
    """All ranks' 1-element partials stacked in rank order."""
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(bufs, partial, group=group)
    return torch.cat(bufs)


def allreduce_partial(partial: torch.Tensor, op: str = "add", group=None) -> torch.Tensor:
    """One all-reduce of the per-GPU partial, in place."""
    dist.all_reduce(partial, op=_REDUCE_OPS[op], group=group)
    return partial


def identity(dtype: torch.dtype, op: str):
    if op == "add":
        return 0
    if dtype.is_floating_point:
        return float("-inf") if op == "max" else float("inf")
    info = torch.iinfo(dtype)
    return info.min if op == "max" else info.max


def reduce_sharded(x_shard: torch.Tensor, op: str = "add", *, out: torch.Tensor,
                   sched="static", chunk: int = 1, teams: int | None = None,
                   threads: int | None = None, deterministic: bool | None = None,
                   group=None) -> torch.Tensor:
    """Reduce this rank's shard on its GPU, then combine across ranks.

    x_shard holds this rank's iterations (shard() of the global space);
    `out` holds the initial value on entry (same on every rank) and the
    global result on return, on every rank."""
    partial = torch.full((1,), identity(x_shard.dtype, op), dtype=x_shard.dtype,
                         device=x_shard.device)
    if x_shard.numel():
        runtime.reduce(x_shard, op, sched=sched, chunk=chunk, teams=teams, threads=threads,
                       out=partial)
    if deterministic is None:
        deterministic = x_shard.dtype.is_floating_point
    if deterministic:
        parts = gather_partials(partial, group)
        runtime.combine_partials(parts, op, out=out)
    else:
        allreduce_partial(partial, op, group)
        runtime.combine_partials(partial, op, out=out)
    return out


def dot_sharded(x_shard: torch.Tensor, y_shard: torch.Tensor, *, out: torch.Tensor,
                sched="static", chunk: int = 1, teams: int | None = None,
                threads: int | None = None, deterministic: bool = False,
                group=None) -> torch.Tensor:
    """fp64 dot of this rank's shard, combined with one NCCL all-reduce
    (config 5), or rank-ordered when deterministic."""
    partial = torch.zeros(1, dtype=torch.float64, device=x_shard.device)
    if x_shard.numel():
        runtime.dot(x_shard, y_shard, sched=sched, chunk=chunk, teams=teams, threads=threads,
                    out=partial)
    if deterministic:
        runtime.combine_partials(gather_partials(partial, group), "add", out=out)
    else:
        allreduce_partial(partial, "add", group)
        runtime.combine_partials(partial, "add", out=out)
    return out
