"""Host logic of the multi-GPU path on CPU: world_size 2 over gloo.

The device kernels cannot run here; each rank computes its shard's partial
with the oracle (the CPU stand-in for runtime.reduce on its GPU), and the
product's sharding and collective plumbing (parallel.shard,
allreduce_partial, gather_partials) must combine them into exactly the
single-device reference result.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2106_03219_b200 import parallel


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank: int, world: int, port: int, q) -> None:
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        n = 1_000_003
        lo, hi = parallel.shard(0, n - 1, rank, world)
        res["shard"] = (lo, hi)
        # int64 sum: per-rank partial (oracle stand-in), one all-reduce
        part = O.reduce(None, lo, hi, O.I64, O.ADD, O.DISTRIBUTE, 1, 8, 64)
        t = torch.tensor([int(part)], dtype=torch.int64)
        parallel.allreduce_partial(t, "add")
        res["i64_sum"] = int(t.item())
        # int64 max
        pm = O.reduce(None, lo, hi, O.I64, O.MAX, O.DISTRIBUTE, 1, 8, 64,
                      np.iinfo(np.int64).min)
        t = torch.tensor([int(pm)], dtype=torch.int64)
        parallel.allreduce_partial(t, "max")
        res["i64_max"] = int(t.item())
        # fp64: rank-ordered gather (deterministic combine)
        pf = O.reduce(None, lo, hi, O.F64, O.ADD, O.DISTRIBUTE, 1, 8, 64)
        g = parallel.gather_partials(torch.tensor([float(pf)], dtype=torch.float64))
        res["f64_parts"] = g.tolist()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_reduction_combines_exactly(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 1_000_003
    # shards: the reference block rule over ranks, disjoint cover
    cover = []
    for r in range(world):
        lo, hi = out[r]["shard"]
        assert (lo, hi) == O.static_bounds(0, n - 1, r, world)
        cover.extend(range(lo, hi + 1))
    assert cover == list(range(n))
    want_sum = int(O.reduce_flat_gen(0, n - 1, O.I64, O.ADD))
    want_max = int(O.reduce_flat_gen(0, n - 1, O.I64, O.MAX, init=np.iinfo(np.int64).min))
    for r in range(world):
        assert out[r]["i64_sum"] == want_sum  # bit-exact for every world size
        assert out[r]["i64_max"] == want_max
        assert out[r]["f64_parts"] == out[0]["f64_parts"]  # identical on every rank
    total = sum(out[0]["f64_parts"])
    exact = O.exact_sum_gen(0, n - 1, O.F64)
    assert abs(total - exact) <= 1e-12 * exact


def test_shard_edges():
    # more ranks than iterations: trailing ranks get empty shards
    shards = [parallel.shard(0, 2, r, 8) for r in range(8)]
    assert shards[:3] == [(0, 0), (1, 1), (2, 2)]
    assert all(lo > hi or lo > 2 for lo, hi in shards[3:])
    assert parallel.identity(torch.int64, "max") == np.iinfo(np.int64).min
    assert parallel.identity(torch.float64, "min") == float("inf")
