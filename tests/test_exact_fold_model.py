"""CPU model check of the exact 32-lane batch fold (csrc/exactfold.cuh).

The device fast path claims: while the running sum s stays inside one binade,
RN(s + p) = s + u * rint(p / u) (u = ulp(s)) unless p/u is a tie, so a batch
of the reference's one-add-at-a-time chain (host.py:567-582) can be folded as
an int64 scan.  This restates exact_fold_batch step for step in numpy (same
exponent window, same tie test, same |S_j| bounds) and checks, on crafted
and random batches, that whenever the model takes the fast path its result
has exactly the bits of the sequential IEEE chain — fp64 and fp32 — and that
it does take the fast path on ordinary data (so the check is not vacuous)."""

from __future__ import annotations

import numpy as np
import pytest

PARAMS = {np.float64: (52, -900, 900), np.float32: (23, -100, 100)}


def model_fold(acc, v, ftype):
    """exact_fold_batch's decision and result: None (serial) or the new acc."""
    mant, emin, emax = PARAMS[ftype]
    acc = ftype(acc)
    if not np.isfinite(acc) or acc == 0:
        return None
    if abs(acc) < np.finfo(ftype).tiny:  # subnormal: the device's biased exponent is 0
        return None
    e = int(np.frexp(acc)[1]) - 1
    if e < emin or e > emax:
        return None
    inv = ftype(2.0 ** (mant - e))
    lim = ftype(2.0 ** (mant + 2))
    s0 = int(acc * inv)
    lo, hi = (1 << mant) + 1, (1 << (mant + 1)) - 1
    run = s0
    with np.errstate(over="ignore", invalid="ignore"):
        for p in v:
            y = ftype(p) * inv
            if not abs(y) <= lim:
                return None
            q = int(np.rint(y))
            if abs(y - ftype(q)) == ftype(0.5):
                return None
            run += q
            if not lo <= abs(run) <= hi:
                return None
    return ftype(run) * ftype(2.0 ** (e - mant))


def seq_fold(acc, v, ftype):
    s = ftype(acc)
    with np.errstate(over="ignore", invalid="ignore"):
        for p in v:
            s = ftype(s + ftype(p))
    return s


def _bits(x, ftype):
    return np.array([x], dtype=ftype).tobytes()


@pytest.mark.parametrize("ftype", [np.float64, np.float32])
def test_fast_path_is_the_sequential_chain(ftype):
    mant = PARAMS[ftype][0]
    rng = np.random.default_rng(2106)
    taken = 0
    total = 0
    for trial in range(3000):
        kind = trial % 6
        init = float(rng.choice([-1.0, 1.0]) * 2.0 ** rng.integers(-30, 60) * (1 + rng.random()))
        e = int(np.frexp(abs(init))[1]) - 1
        u = 2.0 ** (e - mant)
        n = 256
        if kind == 0:    # small positive partials (the C2 shape)
            v = rng.random(n) * abs(init) * 2.0 ** -12
        elif kind == 1:  # ties at half an ulp, mixed with ordinary values
            v = (2 * rng.integers(0, 9, n) + 1) * (u / 2)
            mask = rng.random(n) < 0.5
            v[mask] = rng.random(int(mask.sum())) * 5 * u
        elif kind == 2:  # around the binade's top and bottom, both signs
            init = float(np.sign(init) * (2.0 ** (e + 1) - u * rng.integers(1, 40)))
            v = (rng.random(n) - 0.5) * u * 6
        elif kind == 3:  # sign changes, cancellation
            v = (rng.random(n) - 0.5) * abs(init) * 2.0 ** rng.integers(-60, 2)
        elif kind == 4:  # random exponents around u
            v = rng.choice([-1.0, 1.0], n) * u * 2.0 ** rng.integers(-8, 8, n) * (1 + rng.random(n))
        else:            # values on the u/2 grid (ties and exact multiples)
            v = rng.integers(-40, 40, n) * (u / 2)
        v = v.astype(ftype)
        init_t = ftype(init)
        got = model_fold(init_t, v, ftype)
        total += 1
        if got is not None:
            taken += 1
            want = seq_fold(init_t, v, ftype)
            assert _bits(got, ftype) == _bits(want, ftype), (trial, kind, init_t, got, want)
    assert taken > total // 4, (taken, total)  # the fast path is exercised, not vacuous


@pytest.mark.parametrize("ftype", [np.float64, np.float32])
def test_fast_path_declines_special_values(ftype):
    v = np.ones(256, dtype=ftype)
    for bad in (np.nan, np.inf, -np.inf):
        w = v.copy()
        w[100] = bad
        assert model_fold(ftype(1e6), w, ftype) is None
    assert model_fold(ftype(0.0), v, ftype) is None
    assert model_fold(ftype(-0.0), v, ftype) is None
    assert model_fold(np.finfo(ftype).tiny / 4, v, ftype) is None
    assert model_fold(np.finfo(ftype).max, v, ftype) is None  # exponent outside the window
