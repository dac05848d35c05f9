"""Config 4 (generic mode, 1024 teams x (32+256), 2^26) GB/s, i64/f64, spmd/ordered."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.bench_configs import timeit  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 26
for dtype in ("i64", "f64"):
    x = runtime.synthetic(n, dtype, 0x210603219, 4, device=dev)
    o = torch.zeros(1, dtype=x.dtype, device=dev)
    for ordered in (False, True):
        ms = timeit(lambda: runtime.generic_reduce(x, teams=1024, par_threads=256, ordered=ordered,
                                                   out=o), 100)
        o.zero_()
        runtime.generic_reduce(x, teams=1024, par_threads=256, ordered=ordered, out=o)
        bits = o.view(torch.int64).item()
        print(json.dumps({"dtype": dtype, "ordered": ordered, "gbs": round(n * 8 / ms / 1e6, 1),
                          "bits": hex(bits & (2**64 - 1))}), flush=True)
