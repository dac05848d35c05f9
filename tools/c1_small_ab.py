"""Config 1 (int64 sum, 1 team x 128, 2^20, split over 148 CTAs): the small-piece
LDG path (default) vs the TMA ring (variant 78), alternating, from a CUDA
graph of 20 constructs and back to back from Python; results must agree."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.bench_configs import timeit  # noqa: E402

dev = torch.device("cuda", 0)
sizes = (1 << 17, 1 << 20, 1 << 22)
xs = {n: runtime.synthetic(n, "i64", 0x210603219, device=dev) for n in sizes}
out = torch.zeros(1, dtype=torch.int64, device=dev)


def graph_us(x) -> float:
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        runtime.reduce(x, teams=1, threads=128, out=out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                runtime.reduce(x, teams=1, threads=128, out=out)
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


for n, x in xs.items():
    res = {0: [], 78: []}
    py = {0: [], 78: []}
    vals = {}
    for rnd in range(4):
        for v in ((0, 78) if rnd % 2 == 0 else (78, 0)):
            runtime.set_variant(v)
            try:
                out.zero_()
                runtime.reduce(x, teams=1, threads=128, out=out)
                vals[v] = int(out.item())
                res[v].append(round(graph_us(x), 2))
                py[v].append(round(timeit(lambda: runtime.reduce(x, teams=1, threads=128, out=out),
                                          500) * 1e3, 2))
            finally:
                runtime.set_variant(0)
    print(json.dumps({"n": n, "bytes": n * 8, "graph_us_small_path": statistics.median(res[0]),
                      "graph_us_ring": statistics.median(res[78]),
                      "python_us_small_path": statistics.median(py[0]),
                      "python_us_ring": statistics.median(py[78]),
                      "same": vals[0] == vals[78]}), flush=True)
