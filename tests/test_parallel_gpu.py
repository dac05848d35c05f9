"""The multi-GPU path end to end on the device: 2 ranks (processes) sharing
cuda:0 over gloo run parallel.reduce_sharded / dot_sharded — each rank's
shard through the real kernels, then the collective and the rank-ordered
device combine — and must reproduce the single-launch result (integers:
bit-exact; fp64: the exact sum within 1e-6, identical bits on both ranks).
The 8-GPU NCCL run is the bench's; this checks the plumbing on one GPU.
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

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank: int, world: int, port: int, q) -> None:
    from paper_2106_03219_b200 import parallel, runtime

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        n = 3_000_017
        lo, hi = parallel.shard(0, n - 1, rank, world)
        res = {}
        xi = runtime.synthetic(hi - lo + 1, "i64", O.SEED, 0, offset=lo, device=dev)
        out = torch.zeros(1, dtype=torch.int64, device=dev)
        parallel.reduce_sharded(xi, "add", out=out, sched="distribute", teams=37, threads=256)
        res["i64_sum"] = int(out.item())
        outm = torch.full((1,), np.iinfo(np.int64).min, dtype=torch.int64, device=dev)
        parallel.reduce_sharded(xi, "max", out=outm, teams=16, threads=128)
        res["i64_max"] = int(outm.item())
        xf = runtime.synthetic(hi - lo + 1, "f64", O.SEED, 0, offset=lo, device=dev)
        of = torch.zeros(1, dtype=torch.float64, device=dev)
        parallel.reduce_sharded(xf, "add", out=of, sched="distribute", teams=64, threads=256)
        res["f64_sum"] = float(of.item())
        yf = runtime.synthetic(hi - lo + 1, "f64", O.SEED, 1, offset=lo, device=dev)
        od = torch.zeros(1, dtype=torch.float64, device=dev)
        parallel.dot_sharded(xf, yf, out=od, deterministic=True)
        res["dot"] = float(od.item())
        torch.cuda.synchronize()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_sharded_reduce_and_dot_two_ranks_one_gpu(cuda):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = 3_000_017
    want_sum = O.reduce_flat_gen(0, n - 1, O.I64, O.ADD)
    want_max = O.reduce_flat_gen(0, n - 1, O.I64, O.MAX, init=np.iinfo(np.int64).min)
    exact = O.exact_sum_gen(0, n - 1, O.F64)
    dot_truth = O.accurate_dot_gen(0, n - 1)
    for r in range(world):
        assert got[r]["i64_sum"] == int(want_sum)
        assert got[r]["i64_max"] == int(want_max)
        assert abs(got[r]["f64_sum"] - exact) <= 1e-6 * exact
        assert abs(got[r]["dot"] - dot_truth) <= 1e-6 * dot_truth
    # the deterministic (rank-ordered) combines leave identical bits on every rank
    assert got[0]["f64_sum"] == got[1]["f64_sum"]
    assert got[0]["dot"] == got[1]["dot"]


def test_c_abi_allreduce_over_a_one_rank_nccl_comm(cuda):
    # omprt_allreduce (the C-ABI combine of per-GPU partials) through a real
    # NCCL communicator: one rank on cuda:0, so the all-reduce is the
    # identity — exercises the dlopen'd ncclAllReduce, dtype/op mapping and
    # stream ordering; the 8-rank reduction is the bench's
    import ctypes as C

    from paper_2106_03219_b200 import _lib, runtime

    nccl = C.CDLL("libnccl.so.2")
    comm = C.c_void_p()
    devs = (C.c_int * 1)(0)
    assert nccl.ncclCommInitAll(C.byref(comm), 1, devs) == 0
    try:
        L = _lib.load()
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        for dt, vals, op in (("i64", [5, -7, 2**62, -(2**63)], 0), ("f64", [1.5, -2.25, 3.0], 0),
                             ("u32", [1, 2**32 - 1], 1), ("i32", [-3, 9], 2)):
            t = torch.tensor(vals, dtype=runtime.torch_dtype(runtime.dtype_code(dt)), device=cuda)
            before = t.clone()
            rc = L.omprt_allreduce(C.c_void_p(t.data_ptr()), t.numel(), runtime.dtype_code(dt),
                                   op, comm, stream)
            assert rc == 0, _lib.last_error()
            torch.cuda.synchronize()
            assert torch.equal(t.view(torch.uint8), before.view(torch.uint8)), dt
        assert L.omprt_allreduce(C.c_void_p(1), 0, 2, 0, comm, stream) == 0  # empty
    finally:
        nccl.ncclCommDestroy(comm)


def _xchg_worker(rank: int, world: int, port: int, q) -> None:
    from paper_2106_03219_b200 import parallel, runtime

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        n = 2_000_003
        lo, hi = parallel.shard(0, n - 1, rank, world)
        xi = runtime.synthetic(hi - lo + 1, "i64", O.SEED, 0, offset=lo, device=dev)
        xf = runtime.synthetic(hi - lo + 1, "f64", O.SEED, 0, offset=lo, device=dev)
        px = parallel.PeerExchange(dev)
        res = {"i64": [], "f64": [], "max": []}
        for _ in range(5):  # several steps: the mailbox banks alternate
            out = torch.zeros(1, dtype=torch.int64, device=dev)
            px.reduce(xi, "add", out=out, teams=16, threads=128)
            res["i64"].append(int(out.item()))
            of = torch.zeros(1, dtype=torch.float64, device=dev)
            px.reduce(xf, "add", out=of, sched="distribute", teams=8, threads=256)
            res["f64"].append(float(of.item()))
            om = torch.full((1,), np.iinfo(np.int64).min, dtype=torch.int64, device=dev)
            px.reduce(xi, "max", out=om, teams=4, threads=64)
            res["max"].append(int(om.item()))
        px.close()
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_fused_peer_exchange_two_ranks_one_gpu(cuda):
    # omprt_reduce_exchange: the combine inside the reduction kernel through
    # CUDA IPC mailboxes (two processes on one GPU map each other's buffers)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xchg_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = 2_000_003
    want = int(O.reduce_flat_gen(0, n - 1, O.I64, O.ADD))
    want_max = int(O.reduce_flat_gen(0, n - 1, O.I64, O.MAX, init=np.iinfo(np.int64).min))
    exact = O.exact_sum_gen(0, n - 1, O.F64)
    for r in range(world):
        assert got[r]["i64"] == [want] * 5
        assert got[r]["max"] == [want_max] * 5
        assert all(abs(v - exact) <= 1e-6 * exact for v in got[r]["f64"])
    assert got[0]["f64"] == got[1]["f64"]  # rank-ordered fold: the same bits everywhere


def test_reduce_exchange_single_rank_matches_reduce(cuda):
    # omprt_reduce_exchange with a world of one (the mailbox is the rank's
    # own): the exchange epilogue folds the lone GPU partial into the cell,
    # so the result equals the plain construct's, for every key/bank
    import ctypes as C

    from paper_2106_03219_b200 import _lib, runtime

    L = _lib.load()
    hb = L.omprt_ipc_handle_bytes()
    handle = (C.c_char * hb)()
    mb = C.c_void_p()
    assert L.omprt_mailbox_create(1, C.byref(mb), handle) == 0
    try:
        peers = torch.tensor([mb.value], dtype=torch.int64, device=cuda)
        x = runtime.synthetic(5_000_011, "i64", O.SEED, 3, device=cuda)
        want = int(runtime.reduce(x, "add", teams=148, threads=256).item())
        stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        ws = runtime.reduce_workspace(cuda, 148, 256, 0)
        for step in range(4):
            out = torch.zeros(1, dtype=torch.int64, device=cuda)
            rc = L.omprt_reduce_exchange(C.c_void_p(x.data_ptr()), 0, x.numel() - 1,
                                         runtime.dtype_code("i64"), 0, 0, 1, 148, 256,
                                         C.c_void_p(ws.data_ptr()), C.c_void_p(out.data_ptr()),
                                         C.c_void_p(peers.data_ptr()), 0, 1, 1000 + step, step,
                                         stream)
            assert rc == 0, _lib.last_error()
            assert int(out.item()) == want
        assert runtime.check_trap(cuda) is None
    finally:
        L.omprt_mailbox_destroy(mb)


def _nccl_worker(port: int, q) -> None:
    """One rank over a real NCCL process group: the bench's overlapped
    step (ShardedStep: the shard construct on the compute stream, the
    8-byte NCCL all-reduce + combine on a side stream, double-buffered
    partials), the integer all-reduce through parallel.reduce_sharded, a
    device-side barrier and the max-over-ranks timing reduction."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    import bench
    from paper_2106_03219_b200 import parallel, runtime

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        n = 1 << 22
        x = runtime.synthetic(n, "i64", O.SEED, 3, device=dev)
        out = torch.zeros(1, dtype=torch.int64, device=dev)
        stream = torch.cuda.current_stream(dev)
        step = bench.ShardedStep(lambda p: runtime.reduce(x, "add", out=p), out, 2, stream,
                                 overlap=True)  # G = 2: take the collective path with 1 rank
        for _ in range(5):
            step.step()
        step.drain()
        torch.cuda.synchronize()
        res = {"overlapped_5_steps": int(out.item())}
        o2 = torch.zeros(1, dtype=torch.int64, device=dev)
        parallel.reduce_sharded(x, "add", out=o2, deterministic=False)
        res["allreduce"] = int(o2.item())
        dist.barrier()
        res["max_over_ranks"] = bench.max_over_ranks(1.5, 2, dev)
        q.put(res)
    finally:
        dist.destroy_process_group()


def test_nccl_process_group_one_rank_overlapped_step(cuda):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    want = int(O.reduce(None, 0, (1 << 22) - 1, O.I64, O.ADD, O.STATIC, 1, 1, 1, k=3))
    wrap = lambda v: (v + (1 << 63)) % (1 << 64) - (1 << 63)  # noqa: E731
    assert res["overlapped_5_steps"] == wrap(5 * want)
    assert res["allreduce"] == want
    assert res["max_over_ranks"] == 1.5
