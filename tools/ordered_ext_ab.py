"""ORDERED max/min: the leftmost-extremum SPMD kernels (leftext.cuh, default)
against the row-group kernels (variant 76) and the literal walk (variant 20),
same process; every line checks that the three give identical bits.

C3: axpy + max/min, 2^28 fp32, static_chunked 64 / 4096 and distribute_chunked 1
at 148 x 384 and 148 x 1024; fp64 max / min ORDERED over 2^30 (distribute).

    python tools/ordered_ext_ab.py > gpurun_out/ordered_ext_ab.jsonl
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import runtime  # noqa: E402
from tools.bench_configs import timeit  # noqa: E402

SEED = 0x210603219
dev = torch.device("cuda", 0)
VARIANTS = {0: "leftmost-extremum SPMD", 76: "row-group kernels", 20: "literal walk"}


def bits(t: torch.Tensor) -> int:
    return int(t.view(torch.int32 if t.dtype == torch.float32 else torch.int64).item())


n3 = 1 << 28
x = runtime.synthetic(n3, "f32", SEED, 0, device=dev)
y0 = runtime.synthetic(n3, "f32", SEED, 1, device=dev)
y = y0.clone()
for sched, chunk in (("static_chunked", 64), ("static_chunked", 4096), ("distribute_chunked", 1)):
    for threads in (384, 1024):
        line = {"config": f"C3 axpy+max/min ORDERED {sched} {chunk} 148x{threads}"}
        ref = None
        for v, name in VARIANTS.items():
            runtime.set_variant(v)
            try:
                y.copy_(y0)
                mx, mn = runtime.axpy_minmax(2.5, x, y, sched=sched, chunk=chunk, teams=148,
                                             threads=threads, mode="ordered")
                got = (bits(mx), bits(mn), int(y.view(torch.int32)[::4097].sum().item()))
                ms = timeit(lambda: runtime.axpy_minmax(2.5, x, y, sched=sched, chunk=chunk,
                                                        teams=148, threads=threads,
                                                        mode="ordered"), 20 if v == 20 else 100)
            finally:
                runtime.set_variant(0)
            ref = ref or got
            line[name] = {"ms": round(ms, 4), "gbs": round(n3 * 12 / ms / 1e6, 1),
                          "same_bits": got == ref}
        print(json.dumps(line), flush=True)
del x, y, y0

n2 = 1 << 30
xd = runtime.synthetic(n2, "f64", SEED, 0, device=dev)
for op in ("max", "min"):
    line = {"config": f"C2-shape fp64 {op} ORDERED 2^30 distribute 148x384"}
    ref = None
    for v, name in VARIANTS.items():
        if v == 20:
            continue
        runtime.set_variant(v)
        try:
            o = runtime.reduce(xd, op, sched="distribute", teams=148, threads=384, mode="ordered")
            got = bits(o)
            ms = timeit(lambda: runtime.reduce(xd, op, sched="distribute", teams=148, threads=384,
                                               mode="ordered"), 50)
        finally:
            runtime.set_variant(0)
        ref = ref if ref is not None else got
        line[name] = {"ms": round(ms, 4), "gbs": round(n2 * 8 / ms / 1e6, 1), "same_bits": got == ref}
    print(json.dumps(line), flush=True)
