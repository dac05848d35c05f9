"""Steady-state (power-capped) per-launch time of fp64-sum variants:
run 2K launches back to back, time only the second K (CUDA events)."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2106_03219_b200 import runtime

dev = torch.device("cuda", 0)
n = 1 << 30
x = runtime.synthetic(n, "f64", 0x210603219, device=dev)
out = torch.zeros(1, dtype=torch.float64, device=dev)
sms = runtime.num_sms()
s = torch.cuda.current_stream()
K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000

def steady(variant, teams, threads, unroll=4):
    runtime.set_variant(variant)
    runtime.set_unroll(unroll)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(K):
        runtime.reduce(x, "add", sched="distribute", teams=teams, threads=threads, out=out)
    a.record(s)
    for _ in range(K):
        runtime.reduce(x, "add", sched="distribute", teams=teams, threads=threads, out=out)
    b.record(s)
    b.synchronize()
    ms = a.elapsed_time(b) / K
    runtime.set_variant(0); runtime.set_unroll(4)
    return {"variant": variant, "teams": teams, "threads": threads, "unroll": unroll,
            "ms": round(ms, 4), "gbs": round(n * 8 / ms / 1e6, 1)}

if len(sys.argv) > 2 and sys.argv[2] == "bulk":
    cfgs = []
    for v in (0, 10, 12, 13, 14, 15, 16):
        for thr in (160, 256, 512):
            for tpsm in (1, 2, 4, 8):
                cfgs.append((v, tpsm * sms, thr))
    for c in cfgs:
        print(json.dumps(steady(*c)), flush=True)
    sys.exit(0)
cfgs = [(0, sms, 1024), (0, sms, 512), (0, sms, 256), (0, 2 * sms, 256), (0, sms, 128),
        (8, 32 * sms, 512), (8, 16 * sms, 1024), (6, 32 * sms, 512), (7, 32 * sms, 512),
        (1, 32 * sms, 512), (0, 32 * sms, 512, 8), (12, 4 * sms, 512), (15, 16 * sms, 256),
        (0, sms, 1024)]
for c in cfgs:
    r = steady(*c)
    print(json.dumps(r), flush=True)
    time.sleep(1.0)
