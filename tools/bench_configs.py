"""Throughput of every BASELINE.json config on one GPU (secondary lines; the
headline is bench.py).  Back-to-back CUDA-event timing after warm-up; GB/s of
algorithmic bytes; fraction of the measured copy peak and of nominal 8 TB/s.

    python tools/bench_configs.py [--reps 200] > profiles/<round>_configs.jsonl
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

SEED = 0x210603219
PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0


def timeit(fn, reps, warm=10):
    for _ in range(warm):
        fn()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / reps


def line(config, ms, nbytes, **kw):
    gbs = nbytes / ms / 1e6
    rec = {"config": config, "ms": round(ms, 5), "gbs": round(gbs, 1),
           "frac_measured_peak": round(gbs / PEAK, 4), "frac_nominal_8tbs": round(gbs / 8000, 4)}
    rec.update(kw)
    print(json.dumps(rec), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    sms = runtime.num_sms()

    # C1: static partition + int64 sum, 1 team x 128 threads, N = 2^20
    n = 1 << 20
    x = runtime.synthetic(n, "i64", SEED, device=dev)
    out = torch.zeros(1, dtype=torch.int64, device=dev)
    ms = timeit(lambda: runtime.reduce(x, teams=1, threads=128, out=out), a.reps)
    line("C1 int64 sum static 1x128 N=2^20", ms, n * 8,
         note="one OpenMP team split over 16 CTAs (team_set_cta); L2-resident after the first pass")
    ms = timeit(lambda: runtime.reduce(x, out=out), a.reps)
    line("C1 int64 sum N=2^20, default grid", ms, n * 8, teams=sms, threads=256,
         note="L2-resident after the first pass")
    del x

    # C2: fp64 sum 2^30 (the headline; ordered mode for reference)
    n = 1 << 30
    x = runtime.synthetic(n, "f64", SEED, device=dev)
    outf = torch.zeros(1, dtype=torch.float64, device=dev)
    ms = timeit(lambda: runtime.reduce(x, sched="distribute", out=outf), a.reps)
    line("C2 fp64 sum distribute SPMD N=2^30", ms, n * 8, teams=sms, threads=256)
    for sched in ("static", "distribute_chunked", "static_chunked"):
        ms = timeit(lambda: runtime.reduce(x, sched=sched, chunk=64, out=outf), a.reps // 4)
        line(f"C2 fp64 sum {sched} chunk=64 N=2^30", ms, n * 8, teams=sms, threads=256)
    xi = x.view(torch.int64)
    outi = torch.zeros(1, dtype=torch.int64, device=dev)
    ms = timeit(lambda: runtime.reduce(xi, "max", out=outi), a.reps // 4)
    line("C2-int int64 max N=2^30", ms, n * 8)
    for thr in (1024, 256):
        ms = timeit(lambda: runtime.reduce(x, mode="ordered", teams=sms, threads=thr, out=outf),
                    10, 1)
        line("C2 fp64 sum ORDERED (reference order, bit-exact) N=2^30", ms, n * 8,
             teams=sms, threads=thr)

    # C5 shard: fp64 dot over 2^30 (16 B / iteration)
    y = runtime.synthetic(n, "f64", SEED, 1, device=dev)
    ms = timeit(lambda: runtime.dot(x, y, out=outf), a.reps // 2)
    line("C5 fp64 dot N=2^30 per GPU shard", ms, n * 16, teams=sms, threads=256)
    del x, y, xi
    torch.cuda.empty_cache()

    # C3: chunked static axpy + fp32 max/min, N=2^28 (read x, read y, write y)
    n = 1 << 28
    xs = runtime.synthetic(n, "f32", SEED, 0, device=dev)
    ys = runtime.synthetic(n, "f32", SEED, 1, device=dev)
    mx = torch.full((1,), float("-inf"), device=dev)
    mn = torch.full((1,), float("inf"), device=dev)
    for sched in ("distribute_chunked", "static_chunked"):
        for chunk in (1, 64, 4096):
            ms = timeit(lambda: runtime.axpy_minmax(1e-7, xs, ys, sched=sched, chunk=chunk,
                                                    out_max=mx, out_min=mn), a.reps // 2)
            line(f"C3 axpy+max/min {sched} chunk={chunk} N=2^28", ms, n * 12)
    del xs, ys
    torch.cuda.empty_cache()

    # C4: generic mode, __kmpc_alloc_shared globalisation, 1024 teams, x[2^26]
    n = 1 << 26
    for dtype in ("i64", "f64"):
        x = runtime.synthetic(n, dtype, SEED, 4, device=dev)
        o = torch.zeros(1, dtype=x.dtype, device=dev)
        for ordered in (False, True):
            ms = timeit(lambda: runtime.generic_reduce(x, teams=1024, par_threads=256,
                                                       ordered=ordered, out=o), a.reps // 2)
            line(f"C4 generic {dtype} 1024 teams x (32+256) {'ordered' if ordered else 'spmd'}"
                 " N=2^26", ms, n * 8)
        del x
    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
