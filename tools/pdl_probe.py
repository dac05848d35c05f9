"""Back-to-back fp64 sum steps with and without programmatic dependent launch (variant 40)."""
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
for rep in range(3):
    for var in (0, 40):
        runtime.set_variant(var)
        for _ in range(20):
            runtime.reduce(x, sched="distribute", teams=148, threads=384, out=out)
        torch.cuda.synchronize()
        out.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(500):
            runtime.reduce(x, sched="distribute", teams=148, threads=384, out=out)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / 500
        print(json.dumps({"rep": rep, "variant": var, "ms": round(ms, 5),
                          "gbs": round(n * 8 / ms / 1e6, 1), "sum": out.item()}), flush=True)
runtime.set_variant(0)
