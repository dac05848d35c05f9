"""C3 axpy + max/min in ORDERED mode (literal per-thread walk) vs SPMD, 2^28 fp32."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.bench_configs import timeit  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 28
xs = runtime.synthetic(n, "f32", 0x210603219, 0, device=dev)
ys = runtime.synthetic(n, "f32", 0x210603219, 1, device=dev)
mx = torch.full((1,), float("-inf"), device=dev)
mn = torch.full((1,), float("inf"), device=dev)
for sched, chunk in (("distribute_chunked", 4096), ("static_chunked", 64), ("distribute", 1)):
    for mode in ("spmd", "ordered"):
        ms = timeit(lambda: runtime.axpy_minmax(1e-7, xs, ys, sched=sched, chunk=chunk, mode=mode,
                                                out_max=mx, out_min=mn), 30)
        print(json.dumps({"sched": sched, "chunk": chunk, "mode": mode,
                          "gbs": round(n * 12 / ms / 1e6, 1)}), flush=True)
