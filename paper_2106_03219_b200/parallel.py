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

  * or fused into the reduction kernel (PeerExchange): the last team on
    each GPU stores its partial into every rank's mailbox over NVLink peer
    memory (CUDA IPC) and folds the world's partials in rank order — one
    kernel per step, no collective launch.

The reference itself is single-device; there is no
reference collective to match.  torch.distributed is the plumbing (NCCL on
GPUs, gloo for the CPU tests of this host logic).
"""

from __future__ import annotations

import ctypes as C
import os

import torch
import torch.distributed as dist

from . import _lib, runtime
from ._lib import check

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


def _splitmix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


class PeerExchange:
    """The multi-GPU combine fused into the reduction kernel
    (omprt_reduce_exchange, csrc/exchange.cuh): every rank owns a mailbox
    in its HBM, exported as a CUDA IPC handle and opened by every other rank
    (NVLink peer memory on an NVSwitch box); at each step the team that
    draws the last ticket on each GPU stores the GPU's partial into every
    rank's mailbox and folds the world's partials in rank order into the
    cell — one kernel, no collective launch, identical bits on every rank.
    torch.distributed only carries the one-time handle exchange."""

    def __init__(self, device: torch.device, group=None):
        L = _lib.load()
        self.L = L
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device
        hb = L.omprt_ipc_handle_bytes()
        handle = (C.c_char * hb)()
        mb = C.c_void_p()
        check(L.omprt_mailbox_create(self.world, C.byref(mb), handle), "omprt_mailbox_create")
        self.mailbox = mb
        handles: list = [None] * self.world
        dist.all_gather_object(handles, bytes(handle), group=group)
        self.opened: list[C.c_void_p] = []
        ptrs = []
        for r, h in enumerate(handles):
            if r == self.rank:
                ptrs.append(mb.value)
                continue
            p = C.c_void_p()
            buf = (C.c_char * hb).from_buffer_copy(h)
            check(L.omprt_mailbox_open(buf, C.byref(p)), "omprt_mailbox_open")
            self.opened.append(p)
            ptrs.append(p.value)
        self.peers = torch.tensor(ptrs, dtype=torch.int64, device=device)
        nonce = [int.from_bytes(os.urandom(8), "little") if self.rank == 0 else None]
        dist.broadcast_object_list(nonce, src=0, group=group)
        self.nonce = nonce[0]
        self.step = 0

    def reduce(self, x_shard: torch.Tensor, op: str = "add", *, out: torch.Tensor,
               sched="static", chunk: int = 1, teams: int | None = None,
               threads: int | None = None) -> torch.Tensor:
        """out = out OP (the world's shard reductions, in rank order), on
        every rank, in one kernel launch."""
        g = runtime.default_grid(x_shard.device)
        teams = teams or g.teams
        threads = threads or g.threads
        ws = runtime.reduce_workspace(x_shard.device, teams, threads, 0)
        key = _splitmix64(self.nonce + self.step) or 1
        n = x_shard.numel()
        check(self.L.omprt_reduce_exchange(
            C.c_void_p(x_shard.data_ptr()), 0, n - 1, runtime.dtype_code(x_shard.dtype),
            _lib.OP_NAMES[op], _lib.SCHED_NAMES[sched], chunk, teams, threads,
            C.c_void_p(ws.data_ptr()), C.c_void_p(out.data_ptr()),
            C.c_void_p(self.peers.data_ptr()), self.rank, self.world, key, self.step,
            C.c_void_p(runtime.stream_handle(x_shard.device))),
            "omprt_reduce_exchange")
        self.step += 1
        return out

    def close(self) -> None:
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)
        for p in self.opened:
            self.L.omprt_mailbox_close(p)
        self.opened = []
        dist.barrier(group=self.group)
        if self.mailbox is not None:
            self.L.omprt_mailbox_destroy(self.mailbox)
            self.mailbox = None
