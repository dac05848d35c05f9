"""ncu target: config-4 generic mode (1024 teams x (32+256)), i64 then f64."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2106_03219_b200 import runtime
dev = torch.device("cuda", 0)
for dt in ("i64", "f64"):
    x = runtime.synthetic(1 << 26, dt, 0x210603219, 4, device=dev)
    for _ in range(2):
        runtime.generic_reduce(x, teams=1024, par_threads=256)
torch.cuda.synchronize()
