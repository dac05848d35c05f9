"""Randomised bit-exactness fuzz of every ORDERED path against the oracle's
reference order: fp32/fp64 sums and max/min (row-group kernels with static
and dynamic segments, literal walk), fp64 dot, axpy + max/min; plus SPMD
integer reductions (bit-exact: every bulk / LDG / team-split path), SPMD
fp64 sums and dots (within 1e-6) and SPMD axpy + max/min (y bit-exact,
max/min exact) at random CTA sizes (omprt_set_spmd_block).  Sizes are
chosen so that rows span many windows (dynamic segments > 1) as well as
single windows.  Prints one JSON summary line; exits 1 on any mismatch.

    python tools/ordered_fuzz.py [--cases 400] [--seed 2106]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2106_03219_b200 import runtime  # noqa: E402

SCHEDS = {"static": O.STATIC, "static_chunked": O.STATIC_CHUNKED,
          "distribute": O.DISTRIBUTE, "distribute_chunked": O.DISTRIBUTE_CHUNKED}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=400)
    ap.add_argument("--seed", type=int, default=2106)
    ap.add_argument("--variant", type=int, default=0,
                    help="omprt_set_variant for the ORDERED sum kinds (row-kernel A/B)")
    ap.add_argument("--kinds", default="", help="comma-separated subset of kinds")
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    dev = torch.device("cuda", 0)
    N = 6_000_011
    data = {dt: O.fill(N, dt, O.SEED, 5) for dt in (O.F32, O.F64, O.I64, O.U32)}
    dev_data = {dt: torch.from_numpy(v).to(dev) for dt, v in data.items()}
    # zero-heavy data for the ORDERED max/min tie rule: every extremal element
    # is a zero of random sign (plus NaNs), so the result's sign bit is decided
    # by the reference sequence's order (owner thread, iteration)
    zr = np.random.default_rng(a.seed + 1)
    zdata = {}
    for dt, npdt in ((O.F32, np.float32), (O.F64, np.float64)):
        z = (-1.0 - zr.random(N)).astype(npdt)
        idx = zr.choice(N, N // 8, replace=False)
        z[idx] = np.where(zr.random(idx.size) < 0.5, -0.0, 0.0).astype(npdt)
        z[zr.choice(N, 1000, replace=False)] = np.nan
        zdata[dt] = z
    zdev = {dt: torch.from_numpy(v).to(dev) for dt, v in zdata.items()}
    y64 = O.fill(N, O.F64, O.SEED, 6)
    y64d = torch.from_numpy(y64).to(dev)
    fails, kinds = [], {}
    for c in range(a.cases):
        sched = str(rng.choice(list(SCHEDS)))
        chunk = int(rng.choice([1, 7, 16, 64, 100, 512, 4096, int(rng.integers(1, 20000))]))
        teams = int(rng.choice([1, 3, 17, 148, 296, int(rng.integers(1, 600))]))
        threads = int(rng.choice([32, 64, 96, 128, 256, 1024, int(rng.integers(1, 1025))]))
        lb = int(rng.integers(0, 100))
        ub = int(rng.integers(lb - 2, N))
        kind = str(rng.choice(a.kinds.split(",") if a.kinds else
                              ["sum64", "sum32", "max64", "min32", "dot", "axpy",
                               "spmd_i64", "spmd_u32max", "spmd_f64", "spmd_dot", "spmd_axpy",
                               "zmax64", "zmax32", "zmin64", "zmin32"]))
        kinds[kind] = kinds.get(kind, 0) + 1
        # SPMD kinds also draw the CTA size (omprt_set_spmd_block; 0 = policy)
        blk = int(rng.choice([0, 0, 0, 64, 96, 256, 384, 1024])) if kind.startswith("spmd") else 0
        runtime.set_spmd_block(blk)
        if kind == "spmd_dot":
            want = O.dot(data[O.F64], y64, lb, ub, SCHEDS[sched], chunk, teams, threads)
            got = float(runtime.dot(dev_data[O.F64], y64d, lb=lb, ub=ub, sched=sched, chunk=chunk,
                                    teams=teams, threads=threads).item())
            ok = abs(got - want) <= 1e-6 * max(abs(want), 1e-30)
        elif kind == "spmd_axpy":
            n = min(N, 2_000_003)
            ub = min(ub, n - 1)
            x = data[O.F32][:n]
            y = O.fill(n, O.F32, O.SEED, 7)
            yo = y.copy()
            mx, mn = O.axpy_minmax(0.75, x, yo, lb, ub, SCHEDS[sched], chunk, teams, threads,
                                   -np.inf, np.inf)
            yd = torch.from_numpy(y).to(dev)
            gmx, gmn = runtime.axpy_minmax(0.75, dev_data[O.F32][:n], yd, lb=lb, ub=ub,
                                           sched=sched, chunk=chunk, teams=teams,
                                           threads=threads)
            ok = (float(gmx.item()) == float(mx) and float(gmn.item()) == float(mn)
                  and np.array_equal(yd.cpu().numpy().view(np.uint32), yo.view(np.uint32)))
        elif kind.startswith("spmd"):
            dt, op = {"spmd_i64": (O.I64, "add"), "spmd_u32max": (O.U32, "max"),
                      "spmd_f64": (O.F64, "add")}[kind]
            init = 0
            want = O.reduce(data[dt], lb, ub, dt, O.ADD if op == "add" else O.MAX,
                            SCHEDS[sched], chunk, teams, threads, init)
            out = torch.zeros(1, dtype=dev_data[dt].dtype, device=dev)
            runtime.reduce(dev_data[dt], op, lb=lb, ub=ub, sched=sched, chunk=chunk, teams=teams,
                           threads=threads, out=out)
            got = out.cpu().numpy()[0]
            if dt == O.F64:
                ex = O.accurate_sum_f64(data[dt][lb:ub + 1]) if ub >= lb else 0.0
                ok = abs(float(got) - ex) <= 1e-6 * max(abs(ex), 1e-30)
            else:
                ok = int(got) == int(want)
        elif kind in ("sum64", "sum32", "max64", "min32"):
            dt = O.F64 if kind.endswith("64") else O.F32
            op = {"sum": "add", "max": "max", "min": "min"}[kind[:3]]
            init = {"add": 0.0, "max": -np.inf, "min": np.inf}[op]
            want = O.reduce(data[dt], lb, ub, dt, {"add": O.ADD, "max": O.MAX, "min": O.MIN}[op],
                            SCHEDS[sched], chunk, teams, threads, init)
            out = torch.full((1,), init, dtype=dev_data[dt].dtype, device=dev)
            runtime.set_variant(a.variant if op == "add" else 0)
            try:
                runtime.reduce(dev_data[dt], op, lb=lb, ub=ub, sched=sched, chunk=chunk,
                               teams=teams, threads=threads, mode="ordered", out=out)
            finally:
                runtime.set_variant(0)
            got = out.cpu().numpy()[0]
            ok = np.array([got]).tobytes() == np.array([want], dtype=data[dt].dtype).tobytes()
        elif kind.startswith("z"):
            # ORDERED max/min on zero-heavy data (min: negated, the extreme is
            # again a zero); the cell starts at the identity, 0.0 or NaN
            dt = O.F64 if kind.endswith("64") else O.F32
            op = kind[1:4]
            xs = zdata[dt] if op == "max" else -zdata[dt]
            xd = zdev[dt] if op == "max" else -zdev[dt]
            init = float(rng.choice([-np.inf if op == "max" else np.inf, 0.0, np.nan]))
            want = O.reduce(xs, lb, ub, dt, O.MAX if op == "max" else O.MIN, SCHEDS[sched],
                            chunk, teams, threads, init)
            out = torch.full((1,), init, dtype=xd.dtype, device=dev)
            runtime.reduce(xd, op, lb=lb, ub=ub, sched=sched, chunk=chunk, teams=teams,
                           threads=threads, mode="ordered", out=out)
            got = out.cpu().numpy()[0]
            ok = np.array([got]).tobytes() == np.array([want], dtype=xs.dtype).tobytes()
        elif kind == "dot":
            want = O.dot(data[O.F64], y64, lb, ub, SCHEDS[sched], chunk, teams, threads)
            got = float(runtime.dot(dev_data[O.F64], y64d, lb=lb, ub=ub, sched=sched, chunk=chunk,
                                    teams=teams, threads=threads, mode="ordered").item())
            ok = got == want
        else:
            n = min(N, 2_000_003)
            ub = min(ub, n - 1)
            x = data[O.F32][:n]
            y = O.fill(n, O.F32, O.SEED, 7)
            yo = y.copy()
            mx, mn = O.axpy_minmax(0.75, x, yo, lb, ub, SCHEDS[sched], chunk, teams, threads,
                                   -np.inf, np.inf)
            yd = torch.from_numpy(y).to(dev)
            gmx, gmn = runtime.axpy_minmax(0.75, dev_data[O.F32][:n], yd, lb=lb, ub=ub,
                                           sched=sched, chunk=chunk, teams=teams,
                                           threads=threads, mode="ordered")
            ok = (np.float32(gmx.item()).tobytes() == np.float32(mx).tobytes()
                  and np.float32(gmn.item()).tobytes() == np.float32(mn).tobytes()
                  and np.array_equal(yd.cpu().numpy().view(np.uint32), yo.view(np.uint32)))
        runtime.set_spmd_block(0)
        if not ok:
            fails.append({"case": c, "kind": kind, "sched": sched, "chunk": chunk,
                          "teams": teams, "threads": threads, "lb": lb, "ub": ub, "cta": blk})
    print(json.dumps({"cases": a.cases, "kinds": kinds, "failures": len(fails),
                      "first_failures": fails[:5]}), flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
