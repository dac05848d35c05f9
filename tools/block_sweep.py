"""CTA size of the SPMD construct kernels (omprt_set_spmd_block) at the
BASELINE configs, OpenMP geometry fixed: C2 fp64 sum 2^30, C5 dot shard 2^30,
C3 axpy+max/min 2^28 — back to back, two rounds (the second in the
power-capped steady state).

    python tools/block_sweep.py [c2c5,c3] > gpurun_out/block_sweep.jsonl
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.bench_configs import SEED, timeit  # noqa: E402

BLOCKS = (0, 256, 384, 512, 640, 768, 1024)


def emit(what, omp, blk, ms, nbytes, rnd):
    print(json.dumps({"what": what, "omp_threads": omp, "cta_threads": blk or "policy",
                      "ms": round(ms, 5), "gbs": round(nbytes / ms / 1e6, 1), "round": rnd}),
          flush=True)


def main():
    secs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c2c5", "c3"]
    dev = torch.device("cuda", 0)
    if "c2c5" in secs:
        c2c5(dev)
    if "c3" in secs:
        c3(dev)


def c2c5(dev):
    n = 1 << 30
    x = runtime.synthetic(n, "f64", SEED, 0, device=dev)
    y = runtime.synthetic(n, "f64", SEED, 1, device=dev)
    o = torch.zeros(1, dtype=torch.float64, device=dev)
    for rnd in range(2):
        for omp in (384, 1024):
            for blk in BLOCKS:
                runtime.set_spmd_block(blk)
                ms = timeit(lambda: runtime.reduce(x, sched="distribute", teams=148, threads=omp,
                                                   out=o), 300)
                emit("C2 fp64 sum distribute 2^30", omp, blk, ms, n * 8, rnd)
        for blk in BLOCKS:
            runtime.set_spmd_block(blk)
            ms = timeit(lambda: runtime.dot(x, y, teams=148, threads=384, out=o), 100)
            emit("C5 dot 2^30 shard", 384, blk, ms, n * 16, rnd)
    runtime.set_spmd_block(0)
    del x, y
    torch.cuda.empty_cache()


def c3(dev):
    n = 1 << 28
    xs = runtime.synthetic(n, "f32", SEED, 0, device=dev)
    ys = runtime.synthetic(n, "f32", SEED, 1, device=dev)
    mx = torch.full((1,), float("-inf"), device=dev)
    mn = torch.full((1,), float("inf"), device=dev)
    for rnd in range(2):
        for sched, chunk in (("distribute_chunked", 64), ("static_chunked", 4096)):
            for omp in (384, 1024):
                for blk in BLOCKS:
                    runtime.set_spmd_block(blk)
                    ms = timeit(lambda: runtime.axpy_minmax(1e-7, xs, ys, sched=sched,
                                                            chunk=chunk, teams=148, threads=omp,
                                                            out_max=mx, out_min=mn), 300)
                    emit(f"C3 axpy {sched} {chunk} 2^28", omp, blk, ms, n * 12, rnd)
    runtime.set_spmd_block(0)


if __name__ == "__main__":
    main()
