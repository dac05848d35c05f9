"""C3 SPMD axpy + max/min at the default grid: GB/s per chunk/schedule."""
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
for rep in range(2):
    for sched in ("distribute_chunked", "static_chunked"):
        for chunk in (1, 64, 4096):
            ms = timeit(lambda: runtime.axpy_minmax(1e-7, xs, ys, sched=sched, chunk=chunk,
                                                    out_max=mx, out_min=mn), 50)
            print(json.dumps({"rep": rep, "sched": sched, "chunk": chunk,
                              "gbs": round(n * 12 / ms / 1e6, 1)}), flush=True)
