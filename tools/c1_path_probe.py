"""Config 1 (int64 sum, 1 team x 128 threads, 2^20, split over all SMs):
device time per launch replayed from a CUDA graph, for the TMA-ring path
(unroll 4, default) and the LDG walker (unroll 8 / 2), plus an L2-cold
variant (a 256 MiB scratch written between replays)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 20
x = runtime.synthetic(n, "i64", 0x210603219, device=dev)
out = torch.zeros(1, dtype=torch.int64, device=dev)
scratch = torch.empty(1 << 28, dtype=torch.uint8, device=dev)
K = 20


def graph_us(cold: bool) -> float:
    s = torch.cuda.Stream(dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s):
        runtime.reduce(x, teams=1, threads=128, out=out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(K):
                runtime.reduce(x, teams=1, threads=128, out=out)
    torch.cuda.synchronize()
    times = []
    for _ in range(30):
        if cold:
            scratch.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        times.append(a.elapsed_time(b) * 1e3 / K)
    times.sort()
    return round(times[len(times) // 2], 2)


res = {}
want = None
for unroll in (4, 8, 2):
    runtime.set_unroll(unroll)
    try:
        out.zero_()
        runtime.reduce(x, teams=1, threads=128, out=out)
        v = int(out.item())
        want = v if want is None else want
        res[f"unroll{unroll}"] = {"graph_us_per_launch": graph_us(False),
                                  "first_of_graph_l2_cold_us": graph_us(True), "same": v == want}
    finally:
        runtime.set_unroll(4)
print(json.dumps(res), flush=True)
