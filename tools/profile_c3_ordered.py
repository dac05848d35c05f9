"""C3 ORDERED at 148 x THREADS for an ncu capture of the max/min pass:
    ncu --set full -k regex:k_minmax_ordered_rows python tools/profile_c3_ordered.py 1024"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

dev = torch.device("cuda", 0)
m = 1 << 28
threads = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
xf = runtime.synthetic(m, "f32", 0x210603219, 2, device=dev)
yf = runtime.synthetic(m, "f32", 0x210603219, 3, device=dev)
for _ in range(3):
    runtime.axpy_minmax(0.75, xf, yf, sched="distribute", teams=148, threads=threads,
                        mode="ordered")
torch.cuda.synchronize()
