"""C3 comb (static_chunked) axpy: TMA bulk ring vs LDG walker per chunk."""
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
for sched in ("static_chunked",):
    for chunk in (1, 2, 4, 8, 16, 64):
        for unroll, name in ((4, "bulk"), (8, "ldg u8"), (2, "ldg u2")):
            runtime.set_unroll(unroll)
            for thr in (256, 1024):
                ms = timeit(lambda: runtime.axpy_minmax(1e-7, xs, ys, sched=sched, chunk=chunk,
                                                        threads=thr, out_max=mx, out_min=mn), 50)
                print(json.dumps({"sched": sched, "chunk": chunk, "path": name, "threads": thr,
                                  "gbs": round(n * 12 / ms / 1e6, 1)}), flush=True)
runtime.set_unroll(4)
x = runtime.synthetic(1 << 30, "f64", 0x210603219, 0, device=dev)
o = torch.zeros(1, dtype=torch.float64, device=dev)
for chunk in (1, 2, 4, 8):
    for unroll, name in ((4, "bulk"), (8, "ldg u8")):
        runtime.set_unroll(unroll)
        ms = timeit(lambda: runtime.reduce(x, sched="static_chunked", chunk=chunk, out=o), 30)
        print(json.dumps({"kernel": "reduce f64", "chunk": chunk, "path": name,
                          "gbs": round((1 << 30) * 8 / ms / 1e6, 1)}), flush=True)
runtime.set_unroll(4)
