"""ORDERED dot (fp64) and axpy + max/min (fp32) GB/s and result bits at five
geometries.  profiles/r1_ordered_six_dot.jsonl holds the A/B that chose the
six-warp policy for the dot (a temporary variant 43 forced it); run now it
prints the same numbers under both keys."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.ordered_probe import timed, SEED  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 29
x = runtime.synthetic(n, "f64", SEED, 0, device=dev)
y = runtime.synthetic(n, "f64", SEED, 1, device=dev)
m = 1 << 28
xf = runtime.synthetic(m, "f32", SEED, 2, device=dev)
yf0 = runtime.synthetic(m, "f32", SEED, 3, device=dev)
for sched, chunk, teams, threads in (("distribute", 1, 148, 384), ("distribute", 1, 148, 256),
                                     ("distribute", 1, 148, 1024), ("distribute_chunked", 4096, 148, 1024),
                                     ("static_chunked", 64, 148, 384)):
    res = {}
    for var in (0, 43):
        runtime.set_variant(var)
        f = lambda: runtime.dot(x, y, sched=sched, chunk=chunk, teams=teams, threads=threads,
                                mode="ordered")
        best, _ = timed(f)
        v = f().item()
        yf = yf0.clone()
        g = lambda: runtime.axpy_minmax(0.75, xf, yf, sched=sched, chunk=chunk, teams=teams,
                                        threads=threads, mode="ordered")
        bm, _ = timed(g, reps=5)
        yf.copy_(yf0)
        mx, mn = g()
        res[var] = {"dot_gbs": round(n * 16 / best / 1e6, 1), "dot": v,
                    "c3_gbs": round(m * 12 / bm / 1e6, 1), "mx": mx.item(), "mn": mn.item()}
    runtime.set_variant(0)
    same = all(res[0][k] == res[43][k] for k in ("dot", "mx", "mn"))
    print(json.dumps({"sched": sched, "chunk": chunk, "teams": teams, "threads": threads,
                      "default": {k: res[0][k] for k in ("dot_gbs", "c3_gbs")},
                      "six": {k: res[43][k] for k in ("dot_gbs", "c3_gbs")}, "same": same}),
          flush=True)
