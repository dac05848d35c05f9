"""Throughput of every BASELINE.json config on one GPU (secondary lines; the
headline is bench.py).  Back-to-back CUDA-event timing after warm-up; GB/s of
algorithmic bytes; fraction of the measured copy peak and of nominal 8 TB/s.

    python tools/bench_configs.py [--reps 200] [--cpu] > profiles/<round>_configs.jsonl

--cpu times the CPU reference (the oracle's C restatement of the host
fallback's algorithm, all host cores, bounded in-memory samples) beside every
config: "cpu_reference" and "gpu_over_cpu" in each line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
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


CPU = {"on": False}


def cpu_ref(fn, nbytes, min_s=2.0):
    """The reference's CPU algorithm restated in C (oracle/, kind "port") on
    a bounded in-memory sample, all host cores: GB/s of the same
    algorithmic bytes.  Only timed with --cpu (test infrastructure as a
    baseline leg, never the measured product)."""
    if not CPU["on"]:
        return None
    fn()
    t0 = time.perf_counter()
    k = 0
    while k < 2 or time.perf_counter() - t0 < min_s:
        fn()
        k += 1
    dt = (time.perf_counter() - t0) / k
    return {"gbs": round(nbytes / dt / 1e9, 2), "ms": round(dt * 1e3, 3), "cores": CPU["cores"],
            "kind": "port", "sample_bytes": nbytes}


def line(config, ms, nbytes, cpu=None, **kw):
    gbs = nbytes / ms / 1e6
    rec = {"config": config, "ms": round(ms, 5), "gbs": round(gbs, 1),
           "frac_measured_peak": round(gbs / PEAK, 4), "frac_nominal_8tbs": round(gbs / 8000, 4)}
    rec.update(kw)
    if cpu is not None:
        rec["cpu_reference"] = cpu
        rec["gpu_over_cpu"] = round(gbs / cpu["gbs"], 1)
    print(json.dumps(rec), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--cpu", action="store_true",
                    help="time the CPU reference (oracle port, all host cores) beside each config")
    ap.add_argument("--sections", default="c1,c2,c5,c3,c4",
                    help="comma-separated subset of c1,c2,c5,c3,c4")
    a = ap.parse_args()
    want = set(a.sections.split(","))
    if a.cpu:
        from oracle import oracle as O

        CPU["on"] = True
        CPU["cores"] = len(os.sched_getaffinity(0))
        O.set_threads(CPU["cores"])
    dev = torch.device("cuda", 0)
    sms = runtime.num_sms()

    if "c1" in want:
        c1_lines(a, dev, sms)
    if "c2" in want or "c5" in want:
        c2_c5_lines(a, dev, sms, want)
    if "c3" in want:
        c3_lines(a, dev, sms)
    if "c4" in want:
        c4_lines(a, dev, sms)


def c1_lines(a, dev, sms):
    if CPU["on"]:
        from oracle import oracle as O
    # C1: static partition + int64 sum, 1 team x 128 threads, N = 2^20
    n = 1 << 20
    x = runtime.synthetic(n, "i64", SEED, device=dev)
    out = torch.zeros(1, dtype=torch.int64, device=dev)
    ms = timeit(lambda: runtime.reduce(x, teams=1, threads=128, out=out), a.reps)
    c1 = None
    if CPU["on"]:
        xh = O.fill(n, O.I64, SEED)
        c1 = cpu_ref(lambda: O.reduce(xh, 0, n - 1, O.I64, O.ADD, O.STATIC, 1, 1, 128), n * 8)
    line("C1 int64 sum static 1x128 N=2^20", ms, n * 8, cpu=c1,
         note="one OpenMP team split over 148 CTAs (team_set_cta); L2-resident after the first pass")
    ms = timeit(lambda: runtime.reduce(x, out=out), a.reps)
    line("C1 int64 sum N=2^20, default grid", ms, n * 8, teams=sms, threads=runtime.DEFAULT_THREADS,
         note="L2-resident after the first pass")
    del x


def c2_c5_lines(a, dev, sms, want):
    if CPU["on"]:
        from oracle import oracle as O
    # C2: fp64 sum 2^30 (the headline; ordered mode for reference)
    n = 1 << 30
    x = runtime.synthetic(n, "f64", SEED, device=dev)
    outf = torch.zeros(1, dtype=torch.float64, device=dev)
    ms = timeit(lambda: runtime.reduce(x, sched="distribute", out=outf), a.reps)
    c2 = None
    if CPU["on"]:
        ns = 1 << 26
        xh = O.fill(ns, O.F64, SEED)
        c2 = cpu_ref(lambda: O.reduce(xh, 0, ns - 1, O.F64, O.ADD, O.DISTRIBUTE, 1, sms,
                                     runtime.DEFAULT_THREADS),
                     ns * 8)
    line("C2 fp64 sum distribute SPMD N=2^30", ms, n * 8, cpu=c2, teams=sms,
         threads=runtime.DEFAULT_THREADS)
    for sched in ("static", "distribute_chunked", "static_chunked"):
        ms = timeit(lambda: runtime.reduce(x, sched=sched, chunk=64, out=outf), a.reps // 4)
        line(f"C2 fp64 sum {sched} chunk=64 N=2^30", ms, n * 8, teams=sms,
             threads=runtime.DEFAULT_THREADS)
    xi = x.view(torch.int64)
    outi = torch.zeros(1, dtype=torch.int64, device=dev)
    ms = timeit(lambda: runtime.reduce(xi, "max", out=outi), a.reps // 4)
    line("C2-int int64 max N=2^30", ms, n * 8)
    for thr in (1024, 384, 256):
        ms = timeit(lambda: runtime.reduce(x, mode="ordered", teams=sms, threads=thr, out=outf),
                    20, 5)
        line("C2 fp64 sum ORDERED (reference order, bit-exact) N=2^30", ms, n * 8,
             teams=sms, threads=thr)

    # C5 shard: fp64 dot over 2^30 (16 B / iteration)
    y = runtime.synthetic(n, "f64", SEED, 1, device=dev)
    ms = timeit(lambda: runtime.dot(x, y, out=outf), a.reps // 2)
    c5 = None
    if CPU["on"]:
        ns = 1 << 25
        xh, yh = O.fill(ns, O.F64, SEED, 0), O.fill(ns, O.F64, SEED, 1)
        c5 = cpu_ref(lambda: O.dot(xh, yh, 0, ns - 1, O.DISTRIBUTE, 1, sms,
                                     runtime.DEFAULT_THREADS), ns * 16)
    line("C5 fp64 dot N=2^30 per GPU shard", ms, n * 16, cpu=c5, teams=sms,
         threads=runtime.DEFAULT_THREADS)
    del x, y, xi
    torch.cuda.empty_cache()


def c3_lines(a, dev, sms):
    if CPU["on"]:
        from oracle import oracle as O
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
            c3 = None
            if CPU["on"]:
                ns = 1 << 26
                xh, yh = O.fill(ns, O.F32, SEED, 0), O.fill(ns, O.F32, SEED, 1)
                code = {"distribute_chunked": O.DISTRIBUTE_CHUNKED,
                        "static_chunked": O.STATIC_CHUNKED}[sched]
                c3 = cpu_ref(lambda: O.axpy_minmax(1e-7, xh, yh, 0, ns - 1, code, chunk, sms,
                                                   runtime.DEFAULT_THREADS,
                                                   float("-inf"), float("inf")), ns * 12)
            line(f"C3 axpy+max/min {sched} chunk={chunk} N=2^28", ms, n * 12, cpu=c3)
    # the same at 148 x 1024, and ORDERED mode (reference order of max/min)
    for chunk in (1, 64, 4096):
        ms = timeit(lambda: runtime.axpy_minmax(1e-7, xs, ys, sched="static_chunked", chunk=chunk,
                                                teams=sms, threads=1024, out_max=mx, out_min=mn),
                    a.reps // 2)
        line(f"C3 axpy+max/min static_chunked chunk={chunk} N=2^28", ms, n * 12, teams=sms,
             threads=1024)
    for thr in (384, 1024):
        for chunk in (64, 4096):
            ms = timeit(lambda: runtime.axpy_minmax(1e-7, xs, ys, sched="static_chunked",
                                                    chunk=chunk, teams=sms, threads=thr,
                                                    mode="ordered", out_max=mx, out_min=mn),
                        a.reps // 4, 5)
            line(f"C3 axpy+max/min static_chunked chunk={chunk} ORDERED N=2^28", ms, n * 12,
                 teams=sms, threads=thr,
                 note="two passes: axpy (12 B/elem) + the ORDERED max/min pass over y (4 B/elem); "
                      "GB/s counts the algorithmic 12 B/elem")
    del xs, ys
    torch.cuda.empty_cache()


def c4_lines(a, dev, sms):
    if CPU["on"]:
        from oracle import oracle as O
    # C4: generic mode, __kmpc_alloc_shared globalisation, 1024 teams, x[2^26]
    n = 1 << 26
    for dtype in ("i64", "f64"):
        x = runtime.synthetic(n, dtype, SEED, 4, device=dev)
        o = torch.zeros(1, dtype=x.dtype, device=dev)
        for ordered in (False, True):
            ms = timeit(lambda: runtime.generic_reduce(x, teams=1024, par_threads=256,
                                                       ordered=ordered, out=o), a.reps // 2)
            c4 = None
            if CPU["on"] and ordered:
                dt = O.I64 if dtype == "i64" else O.F64
                xh = O.fill(n, dt, SEED, 4)
                c4 = cpu_ref(lambda: O.generic_reduce(xh, 0, n - 1, dt, O.ADD, 1024, 256), n * 8)
            line(f"C4 generic {dtype} 1024 teams x (32+256) {'ordered' if ordered else 'spmd'}"
                 " N=2^26", ms, n * 8, cpu=c4)
        del x
    torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
