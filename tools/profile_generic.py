"""Config 4 generic-mode reduction, fp64 ORDERED, for an ncu capture:
    ncu --set full -k regex:k_generic python tools/profile_generic.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 26
x = runtime.synthetic(n, sys.argv[1] if len(sys.argv) > 1 else "f64", 0x210603219, 4, device=dev)
o = torch.zeros(1, dtype=x.dtype, device=dev)
for _ in range(3):
    runtime.generic_reduce(x, teams=1024, par_threads=256, ordered=True, out=o)
torch.cuda.synchronize()
print(o.item())
