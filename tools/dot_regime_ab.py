"""fp64 dot (the c5_dot leg's kernel) ring shapes in the bench's regime:
2 x 2 x 48 KiB (default) vs 3 x 2 x 32 KiB (variant 48), 2^31-element
shards (2 x 16 GiB), 20 launches per block after 3 warm-up, alternating."""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 31
x = runtime.synthetic(n, "f64", 0x210603219, 0, device=dev)
y = runtime.synthetic(n, "f64", 0x210603219, 1, device=dev)
o = torch.zeros(1, dtype=torch.float64, device=dev)
VARS = (0, 48)
res = {v: [] for v in VARS}
for rnd in range(6):
    for v in (VARS if rnd % 2 == 0 else VARS[::-1]):
        runtime.set_variant(v)
        try:
            for _ in range(3):
                runtime.dot(x, y, sched="distribute", teams=148, threads=384, out=o)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                runtime.dot(x, y, sched="distribute", teams=148, threads=384, out=o)
            b.record()
            b.synchronize()
            res[v].append(round(n * 16 * 20 / (a.elapsed_time(b) / 1e3) / 1e9, 1))
        finally:
            runtime.set_variant(0)
        time.sleep(1.0)
print(json.dumps({"dot_2x2x48": statistics.median(res[0]), "dot_3x2x32": statistics.median(res[48]),
                  "all": {str(k): v for k, v in res.items()}}))
