"""ORDERED mode (fp: the row-group kernels of csrc/ordered.cuh; integers: the
SPMD kernels, whose wrapping/exact combine gives the same bits): every
OpenMP thread's in-order fold and the global-thread-order combine must be
bit-identical to the reference order (host.py:567-582) restated in
oracle/omprt_oracle.c — for fp too — on every geometry: threads not a
multiple of 32, groups straddling teams, windows touching lb/ub, chunked
schedules on both sides of the row-kernel threshold, misaligned pointers
(literal walk), and the full 2^30 C2 size."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2106_03219_b200 import runtime

pytestmark = pytest.mark.gpu

SCHEDS = {"static": O.STATIC, "static_chunked": O.STATIC_CHUNKED,
          "distribute": O.DISTRIBUTE, "distribute_chunked": O.DISTRIBUTE_CHUNKED}
DTS = {"f64": O.F64, "f32": O.F32, "i64": O.I64, "u32": O.U32}
LITERAL = 20  # omprt_set_variant: ORDERED through the literal per-thread walk


def _ordered(xd, op, sched, chunk, teams, threads, lb, ub, init):
    out = torch.zeros(1, dtype=xd.dtype, device=xd.device)
    out.fill_(init)
    runtime.reduce(xd, op, lb=lb, ub=ub, sched=sched, chunk=chunk, teams=teams,
                   threads=threads, mode="ordered", out=out)
    return out.cpu().numpy()[0]


@pytest.mark.parametrize("dtype", list(DTS))
def test_rows_kernel_bit_exact_random_geometries(cuda, dtype):
    dt = DTS[dtype]
    n = 400_009
    x = O.fill(n, dt, O.SEED, 3)
    xd = torch.from_numpy(x).to(cuda)
    rng = np.random.default_rng(2106)
    cases = [(3, 100, 0, n - 1, "static", 1), (148, 256, 1, n - 2, "distribute", 1),
             (7, 33, 5, n - 7, "distribute", 1), (1, 1, 0, n - 1, "static", 1),
             (2, 1000, 0, 12_345, "static", 1), (40, 64, 3, n - 1, "static_chunked", 16),
             (9, 96, 0, n - 1, "distribute_chunked", 300), (5, 64, 0, n - 1, "static_chunked", 15)]
    for _ in range(12):
        sched = str(rng.choice(list(SCHEDS)))
        lb = int(rng.integers(0, 50))
        cases.append((int(rng.integers(1, 200)), int(rng.integers(1, 1025)), lb,
                      int(rng.integers(lb - 3, n)), sched, int(rng.integers(1, 5000))))
    for op in ("add", "max"):
        init = 0 if op == "add" else (-np.inf if dt in (O.F32, O.F64)
                                      else np.iinfo(O.NP_DTYPE[dt]).min)
        for teams, threads, lb, ub, sched, chunk in cases:
            opc = O.ADD if op == "add" else O.MAX
            want = O.reduce(x, lb, ub, dt, opc, SCHEDS[sched], chunk, teams, threads, init)
            got = _ordered(xd, op, sched, chunk, teams, threads, lb, ub, init)
            assert np.array([got]).tobytes() == np.array([want], dtype=x.dtype).tobytes(), \
                (dtype, op, teams, threads, lb, ub, sched, chunk, got, want)


def test_rows_and_literal_agree(cuda):
    n = 1_000_003
    xd = runtime.synthetic(n, "f64", O.SEED, 4, device=cuda)
    try:
        for teams, threads, sched, chunk in ((148, 256, "distribute", 1), (13, 77, "static", 1),
                                             (64, 512, "static_chunked", 100)):
            rows = _ordered(xd, "add", sched, chunk, teams, threads, 0, n - 1, 0.0)
            runtime.set_variant(LITERAL)
            lit = _ordered(xd, "add", sched, chunk, teams, threads, 0, n - 1, 0.0)
            runtime.set_variant(0)
            assert rows == lit, (teams, threads, sched)
    finally:
        runtime.set_variant(0)


def test_misaligned_pointer_falls_back_to_literal(cuda):
    # an 8-byte offset view: the row kernels need 16-byte alignment, the
    # literal walk takes it — same bits
    n = 100_001
    x = O.fill(n + 1, O.F64, O.SEED, 6)
    base = torch.from_numpy(x).to(cuda)
    view = base[1:]
    assert view.data_ptr() % 16 == 8
    want = O.reduce(np.ascontiguousarray(x[1:]), 0, n - 1, O.F64, O.ADD, O.DISTRIBUTE, 1, 11, 64)
    assert _ordered(view, "add", "distribute", 1, 11, 64, 0, n - 1, 0.0) == want


def test_dot_ordered_rows_bit_exact(cuda):
    n = 700_001
    x, y = O.fill(n, O.F64, O.SEED, 0), O.fill(n, O.F64, O.SEED, 1)
    xd, yd = torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda)
    for teams, threads, lb, ub, sched, chunk in ((148, 256, 0, n - 1, "distribute", 1),
                                                 (9, 40, 3, n - 2, "static", 1),
                                                 (20, 128, 0, n - 1, "static_chunked", 64)):
        want = O.dot(x, y, lb, ub, SCHEDS[sched], chunk, teams, threads)
        got = float(runtime.dot(xd, yd, lb=lb, ub=ub, sched=sched, chunk=chunk, teams=teams,
                                threads=threads, mode="ordered").item())
        assert got == want, (teams, threads, sched)


def test_ordered_full_size_bit_exact(cuda):
    # C2 at full size: 2^30 fp64, the bench geometry and 1024-thread teams;
    # the oracle regenerates the data itself (reference order, C, all cores)
    n = 1 << 30
    x = runtime.synthetic(n, "f64", O.SEED, device=cuda)
    for teams, threads in ((148, 256), (148, 1024)):
        want = O.reduce(None, 0, n - 1, O.F64, O.ADD, O.DISTRIBUTE, 1, teams, threads, 0.0)
        got = _ordered(x, "add", "distribute", 1, teams, threads, 0, n - 1, 0.0)
        assert got == want, (teams, threads, got, want)
    del x
    torch.cuda.empty_cache()


def test_ordered_repeated_launches_reuse_workspace(cuda):
    # per-group ready flags carry a per-launch epoch: back-to-back launches
    # on one workspace must not see the previous launch's flags
    n = 3_000_017
    x = runtime.synthetic(n, "f64", O.SEED, 8, device=cuda)
    want = O.reduce(None, 0, n - 1, O.F64, O.ADD, O.STATIC, 1, 37, 192, 0.0, k=8)
    out = torch.zeros(1, dtype=torch.float64, device=cuda)
    vals = []
    for _ in range(50):
        out.zero_()
        runtime.reduce(x, "add", teams=37, threads=192, mode="ordered", out=out)
        vals.append(float(out.item()))
    assert set(vals) == {float(want)}


def test_ordered_ignores_stale_workspace_contents(cuda):
    # the workspace is shared with every kernel; ready flags must not be
    # fooled by whatever an earlier launch left there (small integers, old
    # flags, partials)
    n = 2_000_003
    x = runtime.synthetic(n, "f64", O.SEED, 9, device=cuda)
    want = O.reduce(None, 0, n - 1, O.F64, O.ADD, O.DISTRIBUTE, 1, 64, 320, 0.0, k=9)
    for pattern in ("ramp32", "ramp64", "ones"):
        ws = runtime.reduce_workspace(cuda, 64, 320, 2)
        w32 = ws.view(torch.int32) if ws.numel() % 4 == 0 else None
        if pattern == "ramp32" and w32 is not None:
            w32.copy_(torch.arange(w32.numel(), dtype=torch.int32, device=cuda))
        elif pattern == "ramp64" and ws.numel() % 8 == 0:
            w64 = ws.view(torch.int64)
            w64.copy_(torch.arange(w64.numel(), dtype=torch.int64, device=cuda))
        else:
            ws.fill_(1)
        ws.view(torch.uint32)[:64].zero_()  # the ticket word starts at 0
        got = _ordered(x, "add", "distribute", 1, 64, 320, 0, n - 1, 0.0)
        assert got == want, pattern
    runtime.reduce_workspace(cuda, 64, 320, 2).zero_()


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("op", ["max", "min"])
def test_ordered_maxmin_signed_zeros_and_nans(cuda, dtype, op):
    """The folder folds max/min partials as a left-biased tree (ord_folder):
    the reference step keeps the leftmost of tied values (-0 vs +0) and never
    takes a NaN element, and a NaN cell stays NaN — all bit-exact against the
    sequential order at geometries with many full folder batches."""
    dt = DTS[dtype]
    n = 1_000_003
    rng = np.random.default_rng(11)
    x = (-rng.random(n)).astype(np.float64 if dtype == "f64" else np.float32)
    if op == "min":
        x = -x
    # the extreme value is a zero of either sign, scattered; NaNs sprinkled
    zeros = rng.choice(n, 5000, replace=False)
    x[zeros] = np.where(rng.random(5000) < 0.5, -0.0, 0.0)
    x[rng.choice(n, 3000, replace=False)] = np.nan
    xd = torch.from_numpy(x).to(cuda)
    ident = -np.inf if op == "max" else np.inf
    opc = O.MAX if op == "max" else O.MIN
    cases = (("static", 1, 148, 256, 0), ("distribute", 1, 148, 384, 0),
             ("static_chunked", 64, 37, 1024, 0), ("static_chunked", 7, 148, 256, 0),
             ("distribute", 1, 148, 384, LITERAL), ("static", 1, 67, 1000, LITERAL))
    try:
        for sched, chunk, teams, threads, variant in cases:
            runtime.set_variant(variant)  # LITERAL: the literal walk's team combine
            for init in (ident, np.nan):
                want = O.reduce(x, 0, n - 1, dt, opc, SCHEDS[sched], chunk, teams, threads, init)
                got = _ordered(xd, op, sched, chunk, teams, threads, 0, n - 1, init)
                assert np.array([got]).tobytes() == np.array([want], dtype=x.dtype).tobytes(), \
                    (sched, chunk, teams, threads, variant, init, got, want)
    finally:
        runtime.set_variant(0)


def test_axpy_ordered_minmax_signed_zeros(cuda):
    """C3 in ORDERED mode: the max/min pass's float2 folder (tree over full
    batches) against the oracle when the extremes are signed zeros."""
    n = 600_001
    rng = np.random.default_rng(5)
    x = np.full(n, -0.0, dtype=np.float32)  # fmaf(a, -0, y) keeps y's sign
    y = np.where(rng.random(n) < 0.5, -0.0, 0.0).astype(np.float32)
    y[rng.choice(n, 100, replace=False)] = 0.0
    yo = y.copy()
    mx, mn = O.axpy_minmax(0.75, x, yo, 0, n - 1, O.DISTRIBUTE, 1, 148, 1024, -np.inf, np.inf)
    yd = torch.from_numpy(y).to(cuda)
    gmx, gmn = runtime.axpy_minmax(0.75, torch.from_numpy(x).to(cuda), yd, sched="distribute",
                                   teams=148, threads=1024, mode="ordered")
    assert np.float32(gmx.item()).tobytes() == np.float32(mx).tobytes()
    assert np.float32(gmn.item()).tobytes() == np.float32(mn).tobytes()
    # chunk 1: the literal walk (k_axpy_minmax_ordered) and its team combine
    yo = y.copy()
    mx, mn = O.axpy_minmax(0.75, x, yo, 0, n - 1, O.DISTRIBUTE_CHUNKED, 1, 148, 384, -np.inf,
                           np.inf)
    yd = torch.from_numpy(y).to(cuda)
    gmx, gmn = runtime.axpy_minmax(0.75, torch.from_numpy(x).to(cuda), yd,
                                   sched="distribute_chunked", chunk=1, teams=148, threads=384,
                                   mode="ordered")
    assert np.float32(gmx.item()).tobytes() == np.float32(mx).tobytes()
    assert np.float32(gmn.item()).tobytes() == np.float32(mn).tobytes()


ROWS_MINMAX = 76  # omprt_set_variant: ORDERED fp max/min through the row-group kernels


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("op", ["max", "min"])
def test_ordered_maxmin_leftmost_in_thread_order(cuda, dtype, op):
    """ORDERED fp max/min run as the SPMD construct keeping the extremum with
    the smallest position in the reference sequence (leftext.cuh).  Every
    extremal element is a zero of random sign, so the result's sign bit is
    decided by which zero the reference order meets first — (owner thread,
    iteration), which for the chunked schedules is NOT iteration order
    (chunk 1: consecutive iterations belong to consecutive threads, and the
    owner wraps around P).  Ragged lb/ub and a misaligned base (the LDG
    walker and scalar heads) included; the row-group kernels (variant 76)
    must agree."""
    dt = DTS[dtype]
    npdt = np.float64 if dtype == "f64" else np.float32
    n = 200_003
    rng = np.random.default_rng(2106)
    x = (-1.0 - rng.random(n)).astype(npdt)
    if op == "min":
        x = -x
    z = rng.choice(n, 20_000, replace=False)
    x[z] = np.where(rng.random(z.size) < 0.5, -0.0, 0.0).astype(npdt)
    x[rng.choice(n, 500, replace=False)] = np.nan
    ident = -np.inf if op == "max" else np.inf
    opc = O.MAX if op == "max" else O.MIN
    full = torch.from_numpy(x).to(cuda)
    cases = (("static_chunked", 1, 7, 96, 0, n - 1, 0), ("static_chunked", 3, 148, 384, 5, n - 3, 0),
             ("distribute_chunked", 1, 13, 64, 1, n - 1, 0),
             ("distribute_chunked", 5, 148, 1024, 0, n - 2, 0), ("static", 1, 3, 100, 2, n - 1, 0),
             ("distribute", 1, 148, 384, 0, n - 1, 0), ("static_chunked", 2, 9, 33, 0, n - 2, 1),
             ("distribute_chunked", 7, 5, 128, 3, n - 2, 1),
             ("static_chunked", 3, 148, 384, 5, n - 3, ROWS_MINMAX))
    try:
        for sched, chunk, teams, threads, lb, ub, tag in cases:
            variant = tag if tag == ROWS_MINMAX else 0
            off = 1 if tag == 1 else 0  # misaligned base pointer
            xs = x[off:]
            xd = full[off:]
            runtime.set_variant(variant)
            for init in (ident, 0.0, np.nan):
                want = O.reduce(xs, lb, ub - off, dt, opc, SCHEDS[sched], chunk, teams, threads,
                                init)
                got = _ordered(xd, op, sched, chunk, teams, threads, lb, ub - off, init)
                assert np.array([got]).tobytes() == np.array([want], dtype=npdt).tobytes(), \
                    (sched, chunk, teams, threads, lb, ub, tag, init, got, want)
    finally:
        runtime.set_variant(0)


@pytest.mark.gpu
def test_axpy_ordered_leftmost_in_thread_order(cuda):
    """C3 ORDERED in one pass (SPMD axpy + leftmost-extremum max/min): the
    extremes are zeros of random sign, every schedule and chunk; y must equal
    the oracle's elementwise and max/min must carry the reference order's
    sign bits."""
    n = 300_007
    rng = np.random.default_rng(7)
    x = np.where(rng.random(n) < 0.5, -0.0, 0.0).astype(np.float32)
    y0 = np.where(rng.random(n) < 0.5, -0.0, 0.0).astype(np.float32)
    y0[rng.choice(n, 1000, replace=False)] = np.float32(-3.0)
    y0[rng.choice(n, 1000, replace=False)] = np.float32(3.0)
    for sched, chunk, teams, threads in (("static_chunked", 1, 148, 384), ("static_chunked", 64, 37, 1000),
                                          ("distribute_chunked", 1, 148, 1024),
                                          ("distribute_chunked", 3, 11, 96), ("static", 1, 148, 384),
                                          ("distribute", 1, 64, 256)):
        for a in (0.75, -1.0):
            yo = y0.copy()
            mx, mn = O.axpy_minmax(a, x, yo, 0, n - 1, SCHEDS[sched], chunk, teams, threads,
                                   -np.inf, np.inf)
            yd = torch.from_numpy(y0.copy()).to(cuda)
            gmx, gmn = runtime.axpy_minmax(a, torch.from_numpy(x).to(cuda), yd, sched=sched,
                                           chunk=chunk, teams=teams, threads=threads,
                                           mode="ordered")
            assert yd.cpu().numpy().tobytes() == yo.tobytes(), (sched, chunk, a)
            assert np.float32(gmx.item()).tobytes() == np.float32(mx).tobytes(), (sched, chunk, a)
            assert np.float32(gmn.item()).tobytes() == np.float32(mn).tobytes(), (sched, chunk, a)
