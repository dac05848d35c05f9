"""Steady-state A/B of the two-stream rings (C5 dot shard 2^30, C3 axpy
2^28): variant 0 (4 stages x 2 streams x 16 KiB), 47 (2 x 2 x 48 KiB), 48
(3 x 2 x 32 KiB); heat, then alternating blocks, 6 rounds.

    python tools/ring2_steady_r2.py > gpurun_out/ring2_steady_r2.jsonl
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

VARIANTS = (0, 47, 48)


def ab(name, run, nbytes, reps):
    timeit(run, reps * 5, 5)
    res = {v: [] for v in VARIANTS}
    for rnd in range(6):
        for v in VARIANTS:
            runtime.set_variant(v)
            ms = timeit(run, reps, 3)
            runtime.set_variant(0)
            res[v].append(nbytes / ms / 1e6)
    print(json.dumps({"what": name, "median_gbs": {v: round(statistics.median(g), 1)
                                                   for v, g in res.items()},
                      "all": {v: [round(x, 1) for x in g] for v, g in res.items()}}), flush=True)


def main():
    dev = torch.device("cuda", 0)
    n = 1 << 30
    x = runtime.synthetic(n, "f64", SEED, 0, device=dev)
    y = runtime.synthetic(n, "f64", SEED, 1, device=dev)
    o = torch.zeros(1, dtype=torch.float64, device=dev)
    ab("C5 dot 2^30 148x384", lambda: runtime.dot(x, y, teams=148, threads=384, out=o), n * 16, 80)
    del x, y
    torch.cuda.empty_cache()
    n = 1 << 28
    xs = runtime.synthetic(n, "f32", SEED, 0, device=dev)
    ys = runtime.synthetic(n, "f32", SEED, 1, device=dev)
    mx = torch.full((1,), float("-inf"), device=dev)
    mn = torch.full((1,), float("inf"), device=dev)
    ab("C3 axpy static_chunked 4096 148x384",
       lambda: runtime.axpy_minmax(1e-7, xs, ys, sched="static_chunked", chunk=4096, teams=148,
                                   threads=384, out_max=mx, out_min=mn), n * 12, 200)


if __name__ == "__main__":
    main()
