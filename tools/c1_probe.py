"""Config 1 (int64 sum, 1 team x 128 threads, 2^20) back-to-back time, team split on/off."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.bench_configs import timeit  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 20
x = runtime.synthetic(n, "i64", 0x210603219, device=dev)
out = torch.zeros(1, dtype=torch.int64, device=dev)
want = None
for rep in range(2):
    for var, name in ((30, "no split"), (0, "split over all SMs")):
        runtime.set_variant(var)
        ms = timeit(lambda: runtime.reduce(x, teams=1, threads=128, out=out), 300)
        out.zero_()
        runtime.reduce(x, teams=1, threads=128, out=out)
        v = int(out.item())
        want = v if want is None else want
        print(json.dumps({"rep": rep, "split": name, "us": round(ms * 1e3, 2),
                          "gbs": round(n * 8 / ms / 1e6, 1), "same": v == want}), flush=True)
runtime.set_variant(0)
