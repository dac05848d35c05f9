"""The ORDERED folder's exact 32-lane batch fold (csrc/exactfold.cuh) against
the reference's one-add-at-a-time combine (host.py:567-582, restated in
oracle/omprt_oracle.c): bit-identical on inputs built to hit every way the
fast path can be wrong — ties at half an ulp, chains hovering at a binade's
ends, negative and sign-changing sums, cancellation, signed zeros, NaN and
infinities, subnormals — and on random chains with random exponents.

One element per OpenMP thread (static schedule, n = teams x threads) makes
every per-thread partial a chosen value (0 + x), so the folder sees exactly
the crafted sequence; a second geometry folds several elements per thread."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2106_03219_b200 import runtime

pytestmark = pytest.mark.gpu

GEOMS = [(148, 384), (7, 33), (3, 1000)]


SCHED = {"static": O.STATIC, "distribute": O.DISTRIBUTE, "static_chunked": O.STATIC_CHUNKED}


def _check(cuda, x: np.ndarray, init: float, teams: int, threads: int, sched="static"):
    """sched static / distribute: the row-group kernels and their folder warp;
    static_chunked (chunk 1, below the row kernels' minimum chunk): the literal
    walk, whose last team folds the thread partials (fold_in_order_team)."""
    dt = O.F64 if x.dtype == np.float64 else O.F32
    n = x.size
    want = O.reduce(x, 0, n - 1, dt, O.ADD, SCHED[sched], 1, teams, threads, init)
    xd = torch.from_numpy(x).to(cuda)
    out = torch.full((1,), init, dtype=xd.dtype, device=cuda)
    runtime.reduce(xd, "add", sched=sched, chunk=1, teams=teams, threads=threads,
                   mode="ordered", out=out)
    got = out.cpu().numpy()[0]
    w = np.array([want], dtype=x.dtype)
    if np.isnan(w[0]):
        assert np.isnan(got), (got, want)
    else:
        assert np.array([got]).tobytes() == w.tobytes(), (got, want, init)


def _ulp_exp(v: float, mant: int) -> int:
    return int(np.frexp(v)[1]) - 1 - mant  # ulp(v) = 2^(e - mant) for v in [2^e, 2^(e+1))


@pytest.mark.parametrize("ftype", [np.float64, np.float32])
def test_crafted_chains(cuda, ftype):
    mant = 52 if ftype == np.float64 else 23
    rng = np.random.default_rng(20261018)
    for teams, threads in GEOMS:
        P = teams * threads
        cases = []
        # C2-like: small positive partials growing the sum through binades
        cases.append((rng.random(P), 0.0))
        cases.append((rng.random(P) * 1e3, 12345.5))
        # ties everywhere (half an ulp of the start binade), and ties in half of the batches
        init = 3.0 * 2.0 ** (mant - 12)
        u = 2.0 ** _ulp_exp(init, mant)
        ties = (2 * rng.integers(0, 50, P) + 1) * (u / 2)
        cases.append((ties, init))
        mixed = ties.copy()
        blk = (np.arange(P) // 256) % 2 == 0
        mixed[blk] = rng.random(int(blk.sum())) * 7 * u
        cases.append((mixed, init))
        # hovering at the top and the bottom of a binade (crossing both ways)
        top = 2.0 ** (mant + 1) - 40.0  # u = 1 below 2^(mant+1), 2 above
        cases.append(((rng.random(P) - 0.5) * 6.0, top))
        cases.append(((rng.random(P) - 0.5) * 6.0, 2.0 ** mant + 3.0))
        # negative sums, sign changes, cancellation
        cases.append((-(rng.random(P) * 3.0), -(2.0 ** (mant - 5)) - 0.75))
        cases.append(((rng.random(P) - 0.5) * 4.0, 1.0))
        alt = np.where(np.arange(P) % 2 == 0, 1e6, -1e6) + rng.random(P)
        cases.append((alt, 0.5))
        # signed zeros, NaN, infinities, subnormals
        z = np.where(rng.random(P) < 0.5, -0.0, 0.0)
        cases.append((z, -0.0))
        cases.append((z, 0.0))
        tiny = np.finfo(ftype).tiny
        cases.append((rng.random(P) * tiny / 4, 0.0))
        cases.append((rng.random(P) * tiny * 4, tiny))
        for bad in (np.nan, np.inf, -np.inf):
            v = rng.random(P) * 100.0
            v[int(rng.integers(0, P))] = bad
            cases.append((v, 1.0e6))
        big = np.full(P, np.finfo(ftype).max / 4)
        cases.append((big, 0.0))  # overflows to +inf in the chain
        for x, init in cases:
            for sched in ("static", "static_chunked"):
                _check(cuda, np.ascontiguousarray(x, dtype=ftype), init, teams, threads, sched)


@pytest.mark.parametrize("ftype", [np.float64, np.float32])
def test_random_exponent_chains(cuda, ftype):
    """Partials with random signs and exponents around the running sum's,
    some exact half-ulp ties sprinkled in, several elements per thread."""
    mant = 52 if ftype == np.float64 else 23
    rng = np.random.default_rng(7)
    for trial in range(24):
        teams, threads = GEOMS[trial % len(GEOMS)]
        per = 1 + trial % 3
        n = teams * threads * per
        init = float(rng.choice([-1.0, 1.0]) * 2.0 ** rng.integers(-20, 40) *
                     (1 + rng.random()))
        rel = 2.0 ** rng.integers(-(mant + 4), -2, n).astype(np.float64)
        x = rng.choice([-1.0, 1.0], n, p=[0.3, 0.7]) * abs(init) * rel * (1 + rng.random(n))
        k = rng.random(n) < 0.05
        e = np.frexp(abs(init))[1] - 1 - mant
        x[k] = (2 * rng.integers(0, 8, int(k.sum())) + 1) * 2.0 ** (e - 1)
        sched = ("static", "distribute", "static_chunked")[(trial // 3) % 3]
        _check(cuda, np.ascontiguousarray(x, dtype=ftype), init, teams, threads, sched)


def _check_generic(cuda, x: np.ndarray, init: float, teams: int, P: int):
    dt = O.F64 if x.dtype == np.float64 else O.F32
    want = O.generic_reduce(x, 0, x.size - 1, dt, O.ADD, teams, P, init)
    xd = torch.from_numpy(x).to(cuda)
    out = torch.full((1,), init, dtype=xd.dtype, device=cuda)
    runtime.generic_reduce(xd, "add", teams=teams, par_threads=P, ordered=True, out=out)
    assert runtime.check_trap(xd.device) is None
    got = out.cpu().numpy()[0]
    w = np.array([want], dtype=x.dtype)
    if np.isnan(w[0]):
        assert np.isnan(got), (got, want)
    else:
        assert np.array([got]).tobytes() == w.tobytes(), (got, want, init, teams, P)


@pytest.mark.parametrize("ftype", [np.float64])
def test_generic_mode_chains(cuda, ftype):
    """Generic mode's two in-order folds (a team's P worker partials, then the
    team partials) on the same crafted and random chains (one element per
    worker makes every worker partial a chosen value; 1024 teams also
    exercise the folder team).  These folds stay one add at a time: the
    32-lane exact fold measured no gain there (profiles/r2_exact_fold_ab.jsonl)."""
    mant = 52 if ftype == np.float64 else 23
    rng = np.random.default_rng(11)
    for teams, P in ((1024, 256), (300, 64), (5, 992)):
        n = teams * P
        init = 3.0 * 2.0 ** (mant - 12)
        u = 2.0 ** _ulp_exp(init, mant)
        cases = [(rng.random(n), 0.0),
                 ((2 * rng.integers(0, 50, n) + 1) * (u / 2), init),
                 ((rng.random(n) - 0.5) * 6.0, 2.0 ** (mant + 1) - 40.0),
                 (-(rng.random(n) * 3.0), -(2.0 ** (mant - 5)) - 0.75),
                 (np.where(rng.random(n) < 0.5, -0.0, 0.0), -0.0)]
        v = rng.random(n)
        v[int(rng.integers(0, n))] = np.nan
        cases.append((v, 1.0))
        rel = 2.0 ** rng.integers(-(mant + 4), -2, n).astype(np.float64)
        cases.append((rng.choice([-1.0, 1.0], n, p=[0.3, 0.7]) * 1e4 * rel * (1 + rng.random(n)),
                      1e4 * (1 + rng.random())))
        # several elements per worker
        cases.append((rng.random(3 * n + 17) * 10.0, 5.0))
        for x, init in cases:
            _check_generic(cuda, np.ascontiguousarray(x, dtype=ftype), init, teams, P)
