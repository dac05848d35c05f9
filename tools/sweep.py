"""Tuning sweep of the fp64 sum kernel variants / geometries on one GPU.

    python tools/sweep.py [--n 1073741824] [--reps 20]

Prints one JSON line per configuration: GB/s (median and best of `reps`
CUDA-event-timed launches after warm-up) and the relative difference of the
result to the default kernel's (a sanity check, not the parity test — that
lives in tests/).
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402


def timed(x, reps, **kw):
    out = torch.zeros(1, dtype=x.dtype, device=x.device)
    for _ in range(3):
        out.zero_()
        runtime.reduce(x, "add", out=out, **kw)
    torch.cuda.synchronize()
    out.zero_()
    runtime.reduce(x, "add", out=out, **kw)
    val = float(out.item())
    ms = []
    s = torch.cuda.current_stream()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        runtime.reduce(x, "add", out=out, **kw)
        b.record(s)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return val, statistics.median(ms), min(ms)


def b2b(x, launches, **kw):
    """Back-to-back launches (the bench's regime: power cap, no idle gaps)."""
    out = torch.zeros(1, dtype=x.dtype, device=x.device)
    for _ in range(5):
        runtime.reduce(x, "add", out=out, **kw)
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    for _ in range(launches):
        runtime.reduce(x, "add", out=out, **kw)
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / launches


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 30)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--b2b", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    x = runtime.synthetic(a.n, "f64", 0x210603219, device=dev)
    nbytes = a.n * 8
    sms = runtime.num_sms()
    runtime.set_variant(0)
    ref, _, _ = timed(x, 2, sched="distribute", teams=2 * sms, threads=1024)

    configs = []
    if a.b2b:
        cand = [(0, sms, 1024), (11, sms, 1024), (12, 2 * sms, 1024), (12, sms, 1024),
                (15, 2 * sms, 512), (8, 32 * sms, 512), (6, 32 * sms, 512), (10, 2 * sms, 1024),
                (12, 4 * sms, 512), (15, 4 * sms, 512), (11, 2 * sms, 512), (12, 8 * sms, 256),
                (15, 8 * sms, 256), (15, 16 * sms, 256), (12, 16 * sms, 512), (11, 8 * sms, 512)]
        for v, teams, thr in cand:
            runtime.set_variant(v)
            ms = b2b(x, 200, sched="distribute", teams=teams, threads=thr)
            print(json.dumps({"mode": "b2b", "variant": v, "teams": teams, "threads": thr,
                              "gbs": round(nbytes / ms / 1e6, 1), "ms": round(ms, 4)}),
                  flush=True)
        runtime.set_variant(0)
        return
    for v in (0, 1, 2, 3, 4, 5, 6, 7, 8, 9):
        configs.append((v, 2 * sms, 1024))
    for v in (10, 11, 12, 13, 14, 15, 16):
        for tpsm, thr in ((1, 1024), (2, 512), (2, 1024), (3, 512), (4, 256), (8, 256),
                          (16, 256), (8, 512)):
            configs.append((v, tpsm * sms, thr))
    if not a.quick:
        for v in (0, 6, 8):
            for teams in (sms, 2 * sms, 3 * sms, 4 * sms, 8 * sms, 16 * sms, 32 * sms):
                for thr in (256, 512, 1024):
                    configs.append((v, teams, thr))
    for v, teams, thr in configs:
        runtime.set_variant(v)
        try:
            val, med, best = timed(x, a.reps, sched="distribute", teams=teams, threads=thr)
        except Exception as err:  # noqa: BLE001
            print(json.dumps({"variant": v, "teams": teams, "threads": thr, "error": str(err)}))
            continue
        print(json.dumps({"variant": v, "teams": teams, "threads": thr,
                          "gbs_median": round(nbytes / med / 1e6, 1),
                          "gbs_best": round(nbytes / best / 1e6, 1),
                          "ms_median": round(med, 4), "rel_diff": abs(val - ref) / abs(ref)}),
              flush=True)
    runtime.set_variant(0)


if __name__ == "__main__":
    main()
