"""Round-2 A/B of the library's default policies against the variant that
keeps the round-1 behaviour, same process, same buffers, back to back:

  C3 SPMD flat static_chunked  default (balanced contiguous CTA pieces)  vs variant 30 (team combs)
  C4 generic SPMD              default (one-wave 288x7 instance)         vs variant 45 (1.7 waves)

    python tools/r2_ab.py [--reps 100] > gpurun_out/r2_ab.jsonl
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.bench_configs import SEED, timeit  # noqa: E402


def emit(what, variant, ms, nbytes, **kw):
    rec = {"what": what, "variant": variant, "ms": round(ms, 5),
           "gbs": round(nbytes / ms / 1e6, 1)}
    rec.update(kw)
    print(json.dumps(rec), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--sections", default="c3,c4")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    sms = runtime.num_sms()
    n = 1 << 28
    xs = runtime.synthetic(n, "f32", SEED, 0, device=dev)
    ys = runtime.synthetic(n, "f32", SEED, 1, device=dev)
    mx = torch.full((1,), float("-inf"), device=dev)
    mn = torch.full((1,), float("inf"), device=dev)
    for rnd in range(2 if "c3" in a.sections else 0):
        for thr in (384, 1024):
            for chunk in (1, 64, 4096):
                for v in (0, 30):
                    runtime.set_variant(v)
                    ms = timeit(lambda: runtime.axpy_minmax(1e-7, xs, ys, sched="static_chunked",
                                                            chunk=chunk, teams=sms, threads=thr,
                                                            out_max=mx, out_min=mn), a.reps)
                    runtime.set_variant(0)
                    emit(f"C3 spmd static_chunked {sms}x{thr} chunk={chunk}", v, ms, n * 12,
                         round=rnd)
    del xs, ys
    torch.cuda.empty_cache()
    n = 1 << 26
    for dtype in (("i64", "f64") if "c4" in a.sections else ()):
        x = runtime.synthetic(n, dtype, SEED, 4, device=dev)
        o = torch.zeros(1, dtype=x.dtype, device=dev)
        for rnd in range(2):
            for v in (0, 45):
                runtime.set_variant(v)
                ms = timeit(lambda: runtime.generic_reduce(x, teams=1024, par_threads=256, out=o),
                            a.reps * 2)
                runtime.set_variant(0)
                emit(f"C4 generic {dtype} spmd 1024x(32+256)", v, ms, n * 8, round=rnd)
            for v in (0, 45):
                runtime.set_variant(v)
                ms = timeit(lambda: runtime.generic_reduce(x, teams=1024, par_threads=256,
                                                           ordered=True, out=o), a.reps * 2)
                runtime.set_variant(0)
                emit(f"C4 generic {dtype} ordered 1024x(32+256)", v, ms, n * 8, round=rnd)
            # the same bytes through the SPMD construct kernel (k_reduce_bulk,
            # 148 x 384): the size's streaming ceiling, launch ramp included
            ms = timeit(lambda: runtime.reduce(x, out=o), a.reps * 2)
            emit(f"C4-size ceiling: reduce {dtype} 148x384 N=2^26", 0, ms, n * 8, round=rnd)


if __name__ == "__main__":
    main()
