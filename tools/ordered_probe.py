"""ORDERED mode: staged (cp.async window) kernels vs the literal per-thread
walk — bit-identity and CUDA-event timing at full size.  One JSON line per
case on stdout.   python tools/ordered_probe.py [--n LOG2]"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402

SEED = 0x210603219


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    ms.sort()
    return ms[0], ms[len(ms) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=30)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    n = 1 << args.n
    x = runtime.synthetic(n, "f64", SEED, 0, device=dev)
    cases = [("distribute", 1, 148, 256), ("distribute", 1, 148, 384), ("distribute", 1, 148, 320),
             ("distribute", 1, 148, 1024), ("static", 1, 148, 1024),
             ("static", 1, 296, 512), ("distribute_chunked", 4096, 148, 1024),
             ("static_chunked", 64, 148, 256)]
    for sched, chunk, teams, threads in cases:
        res = {}
        for name, var in (("literal", 20), ("staged", 0)):
            runtime.set_variant(var)
            out = torch.zeros(1, dtype=torch.float64, device=dev)

            def f():
                out.zero_()
                runtime.reduce(x, "add", sched=sched, chunk=chunk, teams=teams, threads=threads,
                               mode="ordered", out=out)

            best, med = timed(f)
            f()
            torch.cuda.synchronize()
            res[name] = {"value": out.item(), "best_ms": round(best, 4), "med_ms": round(med, 4),
                         "gbs": round(n * 8 / best / 1e6, 1)}
        runtime.set_variant(0)
        print(json.dumps({"kernel": "reduce_f64_add", "sched": sched, "chunk": chunk,
                          "teams": teams, "threads": threads, "n": n,
                          "bit_identical": res["literal"]["value"] == res["staged"]["value"],
                          **res}), flush=True)
    # dot (C5 shard), ordered
    y = runtime.synthetic(n // 2, "f64", SEED, 1, device=dev)
    xs = x[: n // 2]
    for sched, chunk, teams, threads in (("distribute", 1, 148, 256), ("distribute", 1, 148, 1024)):
        res = {}
        for name, var in (("literal", 20), ("staged", 0)):
            runtime.set_variant(var)

            def f():
                return runtime.dot(xs, y, sched=sched, chunk=chunk, teams=teams, threads=threads,
                                   mode="ordered")

            best, med = timed(f)
            v = f().item()
            res[name] = {"value": v, "best_ms": round(best, 4), "med_ms": round(med, 4),
                         "gbs": round(n // 2 * 16 / best / 1e6, 1)}
        runtime.set_variant(0)
        print(json.dumps({"kernel": "dot_f64", "sched": sched, "teams": teams, "threads": threads,
                          "n": n // 2,
                          "bit_identical": res["literal"]["value"] == res["staged"]["value"],
                          **res}), flush=True)


if __name__ == "__main__":
    main()
