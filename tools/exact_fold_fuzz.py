"""Adversarial fuzz of the ORDERED fp sums (row-group kernels + folder, literal
walk + its last-team combine), aimed at the exact 32-lane batch fold
(csrc/exactfold.cuh): random geometry, schedule, chunk, size, dtype and initial
cell value; data mixing half-ulp ties of a random binade, random exponents and
signs, zeros of both signs and occasional NaN / infinities.  Every result is
compared bit for bit with the oracle's reference order (host.py:567-582).

    python tools/exact_fold_fuzz.py [--cases N] [--seed S]"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2106_03219_b200 import runtime  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=500)
ap.add_argument("--seed", type=int, default=2106)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
dev = torch.device("cuda", 0)
SCHED = {"static": O.STATIC, "distribute": O.DISTRIBUTE, "static_chunked": O.STATIC_CHUNKED,
         "distribute_chunked": O.DISTRIBUTE_CHUNKED}
fails = []
kinds = {}
for case in range(a.cases):
    ftype = np.float64 if rng.random() < 0.7 else np.float32
    mant = 52 if ftype == np.float64 else 23
    teams = int(rng.integers(1, 300))
    threads = int(rng.integers(1, 1025))
    sched = str(rng.choice(list(SCHED)))
    chunk = int(rng.choice([1, 2, 7, 15, 16, 64, 1000]))
    n = int(rng.integers(1, 1 << 21))
    init = float(rng.choice([-1.0, 1.0]) * 2.0 ** rng.integers(-10, 40) * (1 + rng.random()))
    if rng.random() < 0.1:
        init = float(rng.choice([0.0, -0.0]))
    e = int(np.frexp(abs(init) or 1.0)[1]) - 1
    u = 2.0 ** (e - mant)
    kind = str(rng.choice(["uniform", "ties", "exps", "signs", "grid", "special"]))
    kinds[kind] = kinds.get(kind, 0) + 1
    if kind == "uniform":
        x = rng.random(n) * (abs(init) or 1.0) * 2.0 ** -16
    elif kind == "ties":
        x = (2 * rng.integers(0, 9, n) + 1) * (u / 2)
        m = rng.random(n) < 0.5
        x[m] = rng.random(int(m.sum())) * 3 * u
    elif kind == "exps":
        x = rng.choice([-1.0, 1.0], n, p=[0.2, 0.8]) * u * 2.0 ** rng.integers(-6, 12, n) * \
            (1 + rng.random(n))
    elif kind == "signs":
        x = (rng.random(n) - 0.5) * (abs(init) or 1.0) * 2.0 ** -8
    elif kind == "grid":
        x = rng.integers(-20, 20, n) * (u / 2)
    else:
        x = rng.random(n) * 10.0
        x[rng.random(n) < 0.01] = -0.0
        k = rng.random()
        if k < 0.3:
            x[int(rng.integers(0, n))] = np.nan
        elif k < 0.6:
            x[int(rng.integers(0, n))] = float(rng.choice([np.inf, -np.inf]))
    x = np.ascontiguousarray(x, dtype=ftype)
    dt = O.F64 if ftype == np.float64 else O.F32
    want = O.reduce(x, 0, n - 1, dt, O.ADD, SCHED[sched], chunk, teams, threads, init)
    xd = torch.from_numpy(x).to(dev)
    out = torch.full((1,), init, dtype=xd.dtype, device=dev)
    runtime.reduce(xd, "add", sched=sched, chunk=chunk, teams=teams, threads=threads,
                   mode="ordered", out=out)
    got = out.cpu().numpy()[0]
    w = np.array([want], dtype=ftype)
    ok = (np.isnan(w[0]) and np.isnan(got)) or np.array([got]).tobytes() == w.tobytes()
    if not ok:
        fails.append({"case": case, "dtype": str(ftype.__name__), "teams": teams,
                      "threads": threads, "sched": sched, "chunk": chunk, "n": n,
                      "init": init, "kind": kind, "got": float(got), "want": float(want)})
print(json.dumps({"cases": a.cases, "seed": a.seed, "kinds": kinds, "failures": len(fails),
                  "first_failures": fails[:5]}))
