"""ORDERED fp64 sum (row-group kernel, 2^30): 512-byte row windows on six
warps (variant 29; the default policy at these geometries) against 1 KiB
windows on three / two warps (variants 94 / 95, a temporary build: see
profiles/r2_ordered_window_1k.jsonl), alternating rounds, bits checked equal
on every launch."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.bench_configs import timeit  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 30
x = runtime.synthetic(n, "f64", 0x210603219, device=dev)
o = torch.zeros(1, dtype=torch.float64, device=dev)
VARS = tuple(int(v) for v in sys.argv[1:]) or (0, 29, 94, 95)
for sched, threads in (("distribute", 384), ("distribute", 1024), ("distribute", 256),
                       ("static", 512)):
    res = {v: [] for v in VARS}
    ref = None
    for rnd in range(8):
        for v in (VARS if rnd % 2 == 0 else VARS[::-1]):
            runtime.set_variant(v)
            try:
                o.zero_()
                runtime.reduce(x, sched=sched, teams=148, threads=threads, mode="ordered", out=o)
                b = o.view(torch.int64).item()
                ref = b if ref is None else ref
                assert b == ref, (sched, threads, v)
                ms = timeit(lambda: runtime.reduce(x, sched=sched, teams=148, threads=threads,
                                                   mode="ordered", out=o), 20, 3)
                res[v].append(round(n * 8 / ms / 1e6, 1))
            finally:
                runtime.set_variant(0)
    print(json.dumps({"sched": sched, "threads": threads,
                      **{str(v): statistics.median(res[v]) for v in VARS}, "bit_identical": True}),
          flush=True)
