"""A/B in one process: default bulk ring vs the same ring with a
fence.proxy.async per stage (variant 17), steady state, alternating."""
import sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2106_03219_b200 import runtime
dev = torch.device("cuda", 0)
n = 1 << 30
x = runtime.synthetic(n, "f64", 0x210603219, device=dev)
out = torch.zeros(1, dtype=torch.float64, device=dev)
s = torch.cuda.current_stream()
def steady(v, K=500):
    runtime.set_variant(v)
    for _ in range(K):
        runtime.reduce(x, teams=148, threads=256, out=out)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(K):
        runtime.reduce(x, teams=148, threads=256, out=out)
    b.record(s); b.synchronize()
    runtime.set_variant(0)
    return n * 8 / (a.elapsed_time(b) / K) / 1e6
for rnd in range(3):
    for v in (0, 17):
        print(json.dumps({"round": rnd, "variant": v, "gbs": round(steady(v), 1)}), flush=True)
