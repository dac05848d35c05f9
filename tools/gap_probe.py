"""Inter-launch gap of the bench step: eager back-to-back launches vs the same
steps replayed from a CUDA graph (per-step ms, CUDA events)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 30
x = runtime.synthetic(n, "f64", 0x210603219, device=dev)
out = torch.zeros(1, dtype=torch.float64, device=dev)
s = torch.cuda.Stream()
K = 200


def step():
    runtime.reduce(x, "add", sched="distribute", teams=148, threads=256, out=out)


with torch.cuda.stream(s):
    for _ in range(10):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        step()
    b.record(s)
    torch.cuda.synchronize()
    eager = a.elapsed_time(b) / K
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            step()
    g.replay()
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(K // 20):
        g.replay()
    b.record(s)
    torch.cuda.synchronize()
    graph = a.elapsed_time(b) / K
print(json.dumps({"eager_ms_per_step": round(eager, 5), "graph_ms_per_step": round(graph, 5),
                  "eager_gbs": round(n * 8 / eager / 1e6, 1), "graph_gbs": round(n * 8 / graph / 1e6, 1)}))
