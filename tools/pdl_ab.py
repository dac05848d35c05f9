"""Programmatic dependent launch for back-to-back constructs: variant 0
(PDL, default) against 77 (plain launches), alternating rounds in one
process, back-to-back CUDA-event timing (tools/bench_configs.timeit) of the
launch-bound and short constructs (config 1, config 4) and the long ones
(config 2 / 3 / 5 shard), plus config 1 replayed from a CUDA graph.

    python tools/pdl_ab.py > gpurun_out/pdl_ab.jsonl
"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.bench_configs import timeit  # noqa: E402

SEED = 0x210603219
dev = torch.device("cuda", 0)
x1 = runtime.synthetic(1 << 20, "i64", SEED, device=dev)
x4 = runtime.synthetic(1 << 26, "f64", SEED, 4, device=dev)
x2 = runtime.synthetic(1 << 30, "f64", SEED, device=dev)
xs = runtime.synthetic(1 << 28, "f32", SEED, device=dev)
ys = runtime.synthetic(1 << 28, "f32", SEED, 1, device=dev)
o1 = torch.zeros(1, dtype=torch.int64, device=dev)
od = torch.zeros(1, dtype=torch.float64, device=dev)

cases = {
    "C1 int64 1x128 2^20": (lambda: runtime.reduce(x1, teams=1, threads=128, out=o1), 1 << 23, 500),
    "C4 f64 SPMD 1024x(32+256)": (lambda: runtime.generic_reduce(x4, teams=1024, par_threads=256,
                                                                  out=od), 1 << 29, 200),
    "C4 f64 ORDERED": (lambda: runtime.generic_reduce(x4, teams=1024, par_threads=256,
                                                       ordered=True, out=od), 1 << 29, 200),
    "C2 f64 2^30": (lambda: runtime.reduce(x2, sched="distribute", teams=148, threads=384,
                                           out=od), 1 << 33, 40),
    "C3 axpy 2^28 static_chunked 64": (lambda: runtime.axpy_minmax(1e-7, xs, ys,
                                                                  sched="static_chunked",
                                                                  chunk=64), 12 << 28, 60),
    "C5 dot 2^30 shard": (lambda: runtime.dot(x2, x2, out=od), 1 << 34, 30),
}


def graph_us() -> float:
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        runtime.reduce(x1, teams=1, threads=128, out=o1)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                runtime.reduce(x1, teams=1, threads=128, out=o1)
    torch.cuda.synchronize()
    t = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        t.append(a.elapsed_time(b) * 1e3 / 20)
    return statistics.median(t)


res = {(name, v): [] for name in list(cases) + ["C1 graph replay us"] for v in (0, 77)}
for rnd in range(4):
    for v in ((0, 77) if rnd % 2 == 0 else (77, 0)):
        runtime.set_variant(v)
        try:
            for name, (fn, nbytes, reps) in cases.items():
                ms = timeit(fn, reps)
                res[(name, v)].append(round(nbytes / ms / 1e6, 1))
            res[("C1 graph replay us", v)].append(round(graph_us(), 2))
        finally:
            runtime.set_variant(0)
for name in list(cases) + ["C1 graph replay us"]:
    print(json.dumps({"case": name, "pdl": statistics.median(res[(name, 0)]),
                      "plain": statistics.median(res[(name, 77)]),
                      "unit": "us per launch" if "graph" in name else "GB/s",
                      "all_pdl": res[(name, 0)], "all_plain": res[(name, 77)]}), flush=True)
