"""Config 5 at full size: fp64 dot over N = 2^33 (x, y: 64 GiB each), sharded
over the ranks with static_bounds and combined with one NCCL all-reduce.

    python tools/bench_dot33.py                      # 1 GPU: the whole 128 GiB on one B200
    torchrun --nproc-per-node G tools/bench_dot33.py # G GPUs (strong scaling)

Prints one JSON line on rank 0 (aggregate GB/s of algorithmic bytes).
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2106_03219_b200 import _lib, parallel, runtime  # noqa: E402

SEED = 0x210603219


def main():
    n = int(os.environ.get("DOT_N", str(1 << 33)))
    steps = int(os.environ.get("DOT_STEPS", "20"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.ensure_device(local)
    lo, hi = parallel.shard(0, n - 1, rank, world)
    m = hi - lo + 1
    x = runtime.synthetic(m, "f64", SEED, 0, offset=lo, device=dev)
    y = runtime.synthetic(m, "f64", SEED, 1, offset=lo, device=dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)

    def step():
        if world == 1:
            runtime.dot(x, y, out=out)
        else:
            parallel.dot_sharded(x, y, out=out)

    for _ in range(3):
        step()
    out.zero_()
    step()
    torch.cuda.synchronize()
    result = float(out.item())
    if world > 1:
        dist.barrier()
    s = torch.cuda.current_stream(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(steps):
        step()
    b.record(s)
    torch.cuda.synchronize()
    ms = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    if rank == 0:
        gbs = n * 16 / (float(ms.item()) / 1e3) / 1e9
        print(json.dumps({"config": "C5 fp64 dot N=2^33", "n": n, "gpus": world,
                          "ms_per_step": round(float(ms.item()), 4), "gbs": round(gbs, 1),
                          "gbs_per_gpu": round(gbs / world, 1), "result": result,
                          "scaling": "strong"}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
