"""ORDERED policy A/B under the bench's steady (power-capped) state: heat the
GPU with SPMD reductions, then alternate the default policy and variant 44
(no six-warp policy) in back-to-back blocks of 30 launches."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 30
x = runtime.synthetic(n, "f64", 0x210603219, 0, device=dev)
out = torch.zeros(1, dtype=torch.float64, device=dev)
for _ in range(3000):  # ~3.5 s of SPMD streaming
    runtime.reduce(x, "add", sched="distribute", teams=148, threads=384, out=out)
torch.cuda.synchronize()


def block(threads, var, reps=30):
    runtime.set_variant(var)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        runtime.reduce(x, "add", sched="distribute", teams=148, threads=threads, mode="ordered",
                       out=out)
    b.record()
    b.synchronize()
    runtime.set_variant(0)
    return n * 8 * reps / (a.elapsed_time(b) * 1e6)


y = runtime.synthetic(n // 2, "f64", 0x210603219, 1, device=dev)


def dot_block(threads, var, reps=30):
    runtime.set_variant(var)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        runtime.dot(x[: n // 2], y, sched="distribute", teams=148, threads=threads, mode="ordered",
                    out=out)
    b.record()
    b.synchronize()
    runtime.set_variant(0)
    return n * 8 * reps / (a.elapsed_time(b) * 1e6)


for kind, fn in (("sum", block), ("dot", dot_block)):
    for threads in (384, 1024, 768):
        r = {0: [], 44: []}
        for _ in range(4):
            for var in (0, 44):
                r[var].append(round(fn(threads, var), 1))
        print(json.dumps({"kernel": kind, "threads": threads, "policy": r[0], "no_six": r[44]}),
              flush=True)
