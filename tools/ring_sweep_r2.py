"""The C2 bench kernel's ring and CTA-to-address mapping, A/B in one process:
variant 0 (default 4 x 32 KiB ring, contiguous 1/148 per CTA), 18 (6 x 32 KiB),
19 (3 x 64 KiB), 33/34/35 (CTAs take interleaved 64 KiB / 512 KiB / 2 MiB
tiles), three rounds of 300 back-to-back launches each.

    python tools/ring_sweep_r2.py > gpurun_out/ring_sweep_r2.jsonl
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.bench_configs import SEED, timeit  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    n = 1 << 30
    x = runtime.synthetic(n, "f64", SEED, 0, device=dev)
    exact = O.exact_sum_gen(0, n - 1, O.F64)
    o = torch.zeros(1, dtype=torch.float64, device=dev)
    for rnd in range(3):
        for v in (0, 18, 19, 33, 34, 35):
            runtime.set_variant(v)
            o.zero_()
            runtime.reduce(x, sched="distribute", teams=148, threads=384, out=o)
            ok = abs(float(o.item()) - exact) <= 1e-6 * exact
            ms = timeit(lambda: runtime.reduce(x, sched="distribute", teams=148, threads=384,
                                               out=o), 300)
            runtime.set_variant(0)
            print(json.dumps({"variant": v, "round": rnd, "ms": round(ms, 5),
                              "gbs": round(n * 8 / ms / 1e6, 1), "parity": ok}), flush=True)


if __name__ == "__main__":
    main()
