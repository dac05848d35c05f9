"""Launch each secondary construct kernel twice at its BASELINE config size
(for ncu --set full captures; see tools/gpu_profile2.sh)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2106_03219_b200 import runtime

dev = torch.device("cuda", 0)
SEED = 0x210603219
n = 1 << 28
xs = runtime.synthetic(n, "f32", SEED, 0, device=dev)
ys = runtime.synthetic(n, "f32", SEED, 1, device=dev)
for _ in range(2):
    runtime.axpy_minmax(1e-7, xs, ys, sched="distribute_chunked", chunk=64)
del xs, ys
n = 1 << 30
x = runtime.synthetic(n, "f64", SEED, 0, device=dev)
y = runtime.synthetic(n, "f64", SEED, 1, device=dev)
for _ in range(2):
    runtime.dot(x, y)
for _ in range(2):
    runtime.reduce(x, sched="static_chunked", chunk=64)
del y
xg = x[: 1 << 26]
for _ in range(2):
    runtime.generic_reduce(xg, teams=1024, par_threads=256)
torch.cuda.synchronize()
print("done")
