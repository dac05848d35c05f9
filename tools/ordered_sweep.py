"""Sweep the ORDERED fp64-sum variants (omprt_set_variant 0, 20..29, 41) at 2^30.
    python tools/ordered_sweep.py [vars=0,22,29] [sched:chunk:teams:threads ...]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.ordered_probe import timed, SEED  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 30
x = runtime.synthetic(n, "f64", SEED, 0, device=dev)
GEOMS = (("distribute", 1, 148, 256), ("distribute", 1, 148, 1024),
         ("distribute", 1, 148, 128), ("distribute", 1, 296, 256),
         ("static_chunked", 64, 148, 256))
VARS = (20, 31, 0, 21, 22, 23, 24, 25, 26, 27, 28, 29, 41)
args = sys.argv[1:]
if args and args[0].startswith("vars="):  # e.g. vars=0,22,29
    VARS = tuple(int(v) for v in args.pop(0)[5:].split(","))
if args:  # e.g. distribute:1:148:384
    GEOMS = tuple((a, int(b), int(c), int(d)) for a, b, c, d in (g.split(":") for g in args))
for sched, chunk, teams, threads in GEOMS:
    ref = None
    for var in VARS:
        runtime.set_variant(var)
        out = torch.zeros(1, dtype=torch.float64, device=dev)

        def f():
            out.zero_()
            runtime.reduce(x, "add", sched=sched, chunk=chunk, teams=teams, threads=threads,
                           mode="ordered", out=out)
        try:
            best, med = timed(f)
        except RuntimeError as e:
            print(json.dumps({"variant": var, "sched": sched, "threads": threads, "err": str(e)[:200]}))
            continue
        f()
        v = out.item()
        ref = v if ref is None else ref
        print(json.dumps({"variant": var, "sched": sched, "chunk": chunk, "teams": teams,
                          "threads": threads, "best_ms": round(best, 4), "med_ms": round(med, 4),
                          "gbs": round(n * 8 / best / 1e6, 1), "same": v == ref}), flush=True)
runtime.set_variant(0)
