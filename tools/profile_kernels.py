"""Launch each secondary construct kernel twice at its BASELINE config size
(for ncu --set full captures; see tools/gpu_r2_profile.sh): C3 SPMD flat
static_chunked 4096 at 148x384 (balanced CTA pieces), C3 ORDERED at 148x1024
(one pass: the SPMD axpy with the leftmost-extremum max/min, leftext.cuh),
the fp64 max ORDERED over 2^30 (same technique), C5 dot shard, C4 generic
mode SPMD and ORDERED (fp64, 1024 teams x (32+256))."""
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
    runtime.axpy_minmax(1e-7, xs, ys, sched="static_chunked", chunk=4096, teams=148, threads=384)
for _ in range(2):
    runtime.axpy_minmax(1e-7, xs, ys, sched="static_chunked", chunk=64, teams=148, threads=1024,
                        mode="ordered")
del xs, ys
n = 1 << 30
x = runtime.synthetic(n, "f64", SEED, 0, device=dev)
y = runtime.synthetic(n, "f64", SEED, 1, device=dev)
for _ in range(2):
    runtime.dot(x, y)
del y
for _ in range(2):
    runtime.reduce(x, "max", sched="distribute", teams=148, threads=384, mode="ordered")
xg = x[: 1 << 26]
for _ in range(2):
    runtime.generic_reduce(xg, teams=1024, par_threads=256)
for _ in range(2):
    runtime.generic_reduce(xg, teams=1024, par_threads=256, ordered=True)
torch.cuda.synchronize()
print("done")
