"""ORDERED fp sums / dot with the folder's exact 32-lane batch fold vs without,
and the literal walk (chunk < 16) with loads issued ahead of the fold vs one
round trip per element (A/B of two library builds: run once per library with
OMPRT_B200_LIB set).
Every result is checked bit-for-bit against the oracle's reference order.

    OMPRT_B200_LIB=... python tools/exact_fold_ab.py <tag>"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2106_03219_b200 import runtime  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("OMPRT_B200_LIB", "default")
dev = torch.device("cuda", 0)
S = 0x210603219
N = 1 << 30
x = runtime.synthetic(N, "f64", S, device=dev)
st = torch.cuda.current_stream(dev)


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / reps


for teams, threads in ((148, 256), (148, 384), (148, 1024)):
    out = torch.zeros(1, dtype=torch.float64, device=dev)

    def step():
        out.zero_()
        runtime.reduce(x, "add", sched="distribute", teams=teams, threads=threads,
                       mode="ordered", out=out)

    ms = timed(step)
    want = float(O.reduce(None, 0, N - 1, O.F64, O.ADD, O.DISTRIBUTE, 1, teams, threads, 0.0,
                          seed=S))
    print(json.dumps({"lib": tag, "what": "f64 sum ORDERED 2^30", "teams": teams,
                      "threads": threads, "ms": round(ms, 4),
                      "gbs": round(N * 8 / ms / 1e6, 1),
                      "bit_identical": float(out.item()) == want}), flush=True)

# the literal walk (chunk 1 is below the row kernels' minimum): its last team
# folds the P thread partials (fold_in_order_team)
for teams, threads in ((148, 384),):
    out = torch.zeros(1, dtype=torch.float64, device=dev)

    def lstep():
        out.zero_()
        runtime.reduce(x, "add", sched="static_chunked", chunk=1, teams=teams, threads=threads,
                       mode="ordered", out=out)

    ms = timed(lstep, reps=5)
    want = float(O.reduce(None, 0, N - 1, O.F64, O.ADD, O.STATIC_CHUNKED, 1, teams, threads,
                          0.0, seed=S))
    print(json.dumps({"lib": tag, "what": "f64 sum ORDERED 2^30 literal walk (static_chunked 1)",
                      "teams": teams, "threads": threads, "ms": round(ms, 4),
                      "gbs": round(N * 8 / ms / 1e6, 1),
                      "bit_identical": float(out.item()) == want}), flush=True)

del x
n = 1 << 28
xd = runtime.synthetic(n, "f64", S, 0, device=dev)
yd = runtime.synthetic(n, "f64", S, 1, device=dev)
for teams, threads in ((148, 384), (148, 1024)):
    out = torch.zeros(1, dtype=torch.float64, device=dev)

    def dstep():
        out.zero_()
        runtime.dot(xd, yd, sched="distribute", teams=teams, threads=threads, mode="ordered",
                    out=out)

    ms = timed(dstep)
    print(json.dumps({"lib": tag, "what": "f64 dot ORDERED 2^28", "teams": teams,
                      "threads": threads, "ms": round(ms, 4),
                      "gbs": round(n * 16 / ms / 1e6, 1)}), flush=True)
for teams, threads in ((148, 384),):
    out = torch.zeros(1, dtype=torch.float64, device=dev)

    def ldstep():
        out.zero_()
        runtime.dot(xd, yd, sched="static_chunked", chunk=1, teams=teams, threads=threads,
                    mode="ordered", out=out)

    ms = timed(ldstep, reps=5)
    print(json.dumps({"lib": tag, "what": "f64 dot ORDERED 2^28 literal walk (static_chunked 1)",
                      "teams": teams, "threads": threads, "ms": round(ms, 4),
                      "gbs": round(n * 16 / ms / 1e6, 1)}), flush=True)
del xd, yd
xf = runtime.synthetic(1 << 30, "f32", S, device=dev)
for teams, threads in ((148, 384),):
    out = torch.zeros(1, dtype=torch.float32, device=dev)

    def fstep():
        out.zero_()
        runtime.reduce(xf, "add", sched="distribute", teams=teams, threads=threads,
                       mode="ordered", out=out)

    ms = timed(fstep)
    print(json.dumps({"lib": tag, "what": "f32 sum ORDERED 2^30", "teams": teams,
                      "threads": threads, "ms": round(ms, 4),
                      "gbs": round((1 << 30) * 4 / ms / 1e6, 1)}), flush=True)
