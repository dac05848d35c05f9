"""ncu target: ORDERED fp64 sum at 2^30 with a chosen variant / geometry.
   python tools/profile_ordered.py VARIANT THREADS [SCHED]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2106_03219_b200 import runtime
dev = torch.device("cuda", 0)
var, thr = int(sys.argv[1]), int(sys.argv[2])
sched = sys.argv[3] if len(sys.argv) > 3 else "distribute"
x = runtime.synthetic(1 << 30, "f64", 0x210603219, device=dev)
runtime.set_variant(var)
runtime.reduce(x, sched=sched, mode="ordered", teams=148, threads=thr)
torch.cuda.synchronize()
