"""C3 ORDERED = SPMD axpy + one reference-order max/min pass: time each part
(the pass alone = ORDERED minus SPMD) at several thread counts."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.ordered_probe import timed, SEED  # noqa: E402

dev = torch.device("cuda", 0)
m = 1 << 28
xf = runtime.synthetic(m, "f32", SEED, 2, device=dev)
yf = runtime.synthetic(m, "f32", SEED, 3, device=dev)
for threads in (256, 384, 512, 768, 1024):
    r = {}
    for mode in ("spmd", "ordered"):
        best, _ = timed(lambda: runtime.axpy_minmax(0.75, xf, yf, sched="distribute", teams=148,
                                                    threads=threads, mode=mode), reps=8)
        r[mode] = best
    print(json.dumps({"threads": threads, "spmd_ms": round(r["spmd"], 4),
                      "ordered_ms": round(r["ordered"], 4),
                      "pass_ms": round(r["ordered"] - r["spmd"], 4),
                      "pass_gbs": round(m * 4 / (r["ordered"] - r["spmd"]) / 1e6, 1)}), flush=True)
