"""Steady-state A/B of bench-kernel ring shapes (power-capped regime): heat
with 2,000 default launches, then alternate blocks of 150 back-to-back
launches per variant, 8 rounds.  Variants: 0 (4 x 32 KiB), 19 (3 x 64 KiB),
37 (2 x 96 KiB), 39 (2 x 112 KiB), 40 (3 x 72 KiB), 46 (4 x 56 KiB); earlier
runs also 36 (4 x 48 KiB) and 38 (2 x 64 KiB).

    python tools/ring_steady_r2.py > gpurun_out/ring_steady_r2.jsonl
"""

from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.bench_configs import SEED, timeit  # noqa: E402

VARIANTS = tuple(int(v) for v in sys.argv[1:]) or (0, 19, 37, 39, 40, 46)


def main():
    dev = torch.device("cuda", 0)
    n = 1 << 30
    x = runtime.synthetic(n, "f64", SEED, 0, device=dev)
    o = torch.zeros(1, dtype=torch.float64, device=dev)
    run = lambda: runtime.reduce(x, sched="distribute", teams=148, threads=384, out=o)  # noqa: E731
    timeit(run, 2000, 10)
    res = {v: [] for v in VARIANTS}
    for rnd in range(8):
        for v in VARIANTS:
            runtime.set_variant(v)
            ms = timeit(run, 150, 3)
            runtime.set_variant(0)
            res[v].append(n * 8 / ms / 1e6)
            print(json.dumps({"variant": v, "round": rnd, "gbs": round(res[v][-1], 1)}), flush=True)
    print(json.dumps({"summary": {v: round(statistics.median(g), 1) for v, g in res.items()}}))


if __name__ == "__main__":
    main()
