import sys; sys.path.insert(0, ".")
import torch
from paper_2106_03219_b200 import runtime
dev = torch.device("cuda", 0)
n = 1 << 28
x = runtime.synthetic(n, "f32", 0x210603219, 0, device=dev)
y = runtime.synthetic(n, "f32", 0x210603219, 1, device=dev)
for sched, chunk in (("static_chunked", 4096), ("static_chunked", 64), ("distribute", 1)):
    for mode in ("spmd", "ordered"):
        runtime.axpy_minmax(0.5, x, y, sched=sched, chunk=chunk, teams=148, threads=384, mode=mode)
torch.cuda.synchronize()
print("done")
