import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2106_03219_b200 import runtime
dev = torch.device("cuda", 0)
x = runtime.synthetic(1 << 28, "f64", 0x210603219, device=dev)
for thr in (128, 256):
    runtime.reduce(x, sched="distribute", mode="ordered", teams=148, threads=thr)
torch.cuda.synchronize()
