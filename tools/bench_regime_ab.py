"""Ring shapes of the bench kernel A/B'd in the DRIVER's bench regime, not
the power-capped steady state: the round-end bench runs `--steps 20
--warmup 5`, so its timed region is 20 launches (~23 ms) right after 5
warm-up steps, 20 event-timed launches, 6 torch.sum calibration passes and a
0.1 s idle gap — SM clocks near max, the power cap barely engaged.

Each block replays exactly that sequence for one variant (0 = the library
default; 12 = 4 x 32 KiB, 19 = 3 x 64 KiB, 36 = 4 x 48 KiB, 37 = 2 x 96 KiB,
46 = 4 x 56 KiB, 40 = 3 x 72 KiB), variants in a rotated order every round.

    python tools/bench_regime_ab.py [rounds] [variants...] > gpurun_out/bench_regime_ab.jsonl
"""

from __future__ import annotations

import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 30
x = runtime.synthetic(n, "f64", 0x210603219, 0, device=dev)
out = torch.zeros(1, dtype=torch.float64, device=dev)
s = torch.cuda.current_stream(dev)
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 6
# "bN" entries: the default kernel on N-thread CTAs (omprt_set_spmd_block)
variants = [v if v.startswith("b") else int(v) for v in sys.argv[2:]] or [0, 12, 19, 36, 46]


def step():
    runtime.reduce(x, "add", sched="distribute", teams=148, threads=384, out=out)


def block() -> float:
    for _ in range(5):
        step()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(20)]
    for a, b in ev:
        a.record(s)
        step()
        b.record(s)
    for _ in range(6):
        torch.sum(x)
    torch.cuda.synchronize()
    time.sleep(0.1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(20):
        step()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 20


res: dict[int, list[float]] = {v: [] for v in variants}
for r in range(rounds):
    order = variants[r % len(variants):] + variants[:r % len(variants)]
    for v in order:
        if isinstance(v, str):
            runtime.set_spmd_block(int(v[1:]))
        else:
            runtime.set_variant(v)
        try:
            ms = block()
        finally:
            runtime.set_variant(0)
            runtime.set_spmd_block(0)
        res[v].append(round(n * 8 / ms / 1e6, 1))
        time.sleep(1.0)
for v in variants:
    print(json.dumps({"variant": v, "gbs": res[v], "median": statistics.median(res[v]),
                      "best": max(res[v])}), flush=True)
