"""Parity of the teams-distribute-parallel-for reduction kernels (GPU).

Bar (BASELINE north star): schedules and integer results bit-exact against
the CPU reference; fp64 within rel 1e-6 and fp32 within rel 1e-4 of the
exactly rounded sum; ORDERED mode bit-identical to the reference order even
for fp.  Oracle = oracle/omprt_oracle.c, pinned to forge by test_oracle.py.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2106_03219_b200 import runtime
from tests.helpers import DT, OPS

pytestmark = pytest.mark.gpu

SCHEDS = {"static": O.STATIC, "static_chunked": O.STATIC_CHUNKED,
          "distribute": O.DISTRIBUTE, "distribute_chunked": O.DISTRIBUTE_CHUNKED}
ALLDT = {"i32": O.I32, "u32": O.U32, "i64": O.I64, "u64": O.U64, "f32": O.F32, "f64": O.F64}
TOL = {O.F32: 1e-4, O.F64: 1e-6}


def dev_array(x: np.ndarray, cuda) -> torch.Tensor:
    return torch.from_numpy(x).to(cuda)


def run_reduce(cuda, x_np, dt, op, sched, chunk, teams, threads, lb, ub, mode="spmd", init=None):
    x = dev_array(x_np, cuda)
    out = torch.zeros(1, dtype=x.dtype, device=cuda)
    if init is not None:
        out.copy_(torch.from_numpy(np.array([init], dtype=x_np.dtype)))
    runtime.reduce(x, op, lb=lb, ub=ub, sched=sched, chunk=chunk, teams=teams, threads=threads,
                   mode=mode, out=out)
    return out.cpu().numpy()[0]


def init_for(dt, op):
    """A non-trivial initial cell: the identity of max/min, 0 for add."""
    if op == "add":
        return 0
    np_t = O.NP_DTYPE[dt]
    if dt in (O.F32, O.F64):
        return -np.inf if op == "max" else np.inf
    return np.iinfo(np_t).min if op == "max" else np.iinfo(np_t).max


def check(dt, got, want, exact=None):
    if dt in (O.F32, O.F64):
        if exact is None:
            exact = float(want)
        assert abs(float(got) - exact) <= TOL[dt] * max(abs(exact), 1e-30), (got, want, exact)
    else:
        assert int(got) == int(want), (got, want)


def test_bounds_dump_bit_exact(cuda, devicert_golden, fallback_golden):
    # every (team, thread) of the BASELINE geometries and random ones
    for rec in fallback_golden["vgpu_bounds"]:
        d = runtime.bounds_dump(rec["lb"], rec["ub"], "static", teams=rec["teams"],
                                threads=rec["threads"], device=cuda).cpu().numpy()
        assert d[:, :2].tolist() == rec["bounds"]
    rng = np.random.default_rng(11)
    for sched, code in SCHEDS.items():
        for _ in range(25):
            lb = int(rng.integers(-(2**40), 2**40))
            ub = lb + int(rng.integers(-40, 100000))
            teams, threads = int(rng.integers(1, 300)), int(rng.integers(1, 1025))
            chunk = int(rng.integers(1, 5000))
            got = runtime.bounds_dump(lb, ub, sched, chunk, teams=teams, threads=threads,
                                      device=cuda).cpu().numpy()
            assert np.array_equal(got, O.bounds_dump(lb, ub, code, chunk, teams, threads))
    # the full 2^30 geometries of SURVEY §A.3
    for teams in (592, 1024, 296):
        got = runtime.bounds_dump(0, 2**30 - 1, "static", teams=teams, threads=1024,
                                  device=cuda).cpu().numpy()
        assert np.array_equal(got, O.bounds_dump(0, 2**30 - 1, O.STATIC, 1, teams, 1024))
    got = runtime.bounds_dump(0, 2**30 - 1, "static", teams=592, threads=1024,
                              device=cuda).cpu().numpy()
    assert int((got[:, 0] > 2**30 - 1).sum()) == 258  # empty tail threads


def test_config1_int64_sum_matches_reference_fallback(cuda, fallback_golden):
    # static partition + int64 sum, 1 team x 128 threads, N = 2^20 (bit-exact)
    recs = [r for r in fallback_golden["reductions"] if r["threads"] == 128]
    assert recs
    for r in recs:
        x = runtime.synthetic(r["n"], "i64", r["seed"], r["k"], device=cuda)
        for mode in ("spmd", "ordered"):
            out = torch.full((1,), r["init"], dtype=torch.int64, device=cuda)
            runtime.reduce(x, "add", teams=r["teams"], threads=r["threads"], mode=mode, out=out)
            assert int(out.item()) == r["fallback"], (r["n"], mode)


def test_all_fallback_goldens(cuda, fallback_golden):
    for r in fallback_golden["reductions"]:
        x = O.fill(r["n"], DT[r["dtype"]], r["seed"], r["k"])
        for sched in ("static", "distribute"):
            got = run_reduce(cuda, x, DT[r["dtype"]], r["op"], sched, 1, r["teams"],
                             r["threads"], r["lb"], r["ub"], init=r["init"])
            assert int(got) == r["fallback"], r


def test_device_generator_matches_oracle(cuda):
    for name, dt in ALLDT.items():
        got = runtime.synthetic(10007, name, O.SEED, 2, 12345, device=cuda).cpu().numpy()
        assert np.array_equal(got, O.fill(10007, dt, O.SEED, 2, 12345)), name


@pytest.mark.parametrize("dtype", list(ALLDT))
@pytest.mark.parametrize("op", ["add", "max", "min"])
@pytest.mark.parametrize("sched", list(SCHEDS))
def test_reduce_matrix(cuda, dtype, op, sched):
    dt = ALLDT[dtype]
    n = 200_003
    init = init_for(dt, op)
    x = O.fill(n, dt, O.SEED, 7)
    for teams, threads, lb, ub, chunk in ((3, 96, 0, n - 1, 1), (17, 256, 5, n - 2, 64),
                                          (1, 33, 1, 4099, 7), (40, 1024, 3, n - 1, 4096),
                                          (8, 64, 0, 10, 3), (5, 7, 2, 1, 1)):
        want = O.reduce(x, lb, ub, dt, OPS[op], SCHEDS[sched], chunk, teams, threads, init)
        exact = None
        if dt in (O.F32, O.F64) and op == "add" and ub >= lb:
            exact = O.accurate_sum_f64(x[lb:ub + 1].astype(np.float64))
        for mode in ("spmd", "ordered"):
            got = run_reduce(cuda, x, dt, op, sched, chunk, teams, threads, lb, ub, mode,
                             init=init)
            if mode == "ordered" or dt not in (O.F32, O.F64) or op != "add":
                # integer results, max/min and the ORDERED fp path: bit-exact
                assert got.tobytes() == np.array([want]).astype(x.dtype).tobytes(), \
                    (dtype, op, sched, mode, teams, threads, lb, ub, got, want)
            else:
                check(dt, got, want, exact)


def test_misaligned_and_ragged(cuda):
    # the head/tail paths of the vector walk: every lb mod 4 and odd lengths
    x = O.fill(70_001, O.I32, O.SEED, 9)
    for lb in range(0, 9):
        for ub in (lb - 1, lb, lb + 1, lb + 5, 70_000 - lb):
            for teams, threads in ((1, 1), (2, 3), (7, 64), (64, 128)):
                want = O.reduce(x, lb, ub, O.I32, O.ADD, O.STATIC, 1, teams, threads, 13)
                got = run_reduce(cuda, x, O.I32, "add", "static", 1, teams, threads, lb, ub,
                                 init=13)
                assert int(got) == int(want), (lb, ub, teams, threads)


def test_empty_space_leaves_cell(cuda):
    x = O.fill(16, O.I64)
    for lb, ub in ((0, -1), (5, 2), (-3, -10)):
        got = run_reduce(cuda, x, O.I64, "add", "static", 1, 4, 32, max(lb, 0), ub, init=77)
        assert int(got) == 77


def test_more_teams_than_iterations(cuda):
    x = O.fill(5, O.U64, O.SEED, 1)
    for sched in SCHEDS:
        got = run_reduce(cuda, x, O.U64, "add", sched, 1, 1000, 1024, 0, 4, init=0)
        assert int(got) == int(x.astype(np.uint64).sum())


def test_deterministic_run_to_run(cuda):
    x = runtime.synthetic(1 << 24, "f64", O.SEED, device=cuda)
    vals = set()
    for _ in range(4):
        vals.add(float(runtime.reduce(x, teams=296, threads=1024).item()))
    assert len(vals) == 1


def test_ticket_self_resets_across_launches(cuda):
    # the last-team-finishes ticket must wrap to 0 after every launch
    x = runtime.synthetic(1 << 16, "i64", O.SEED, device=cuda)
    want = int(O.reduce(x.cpu().numpy(), 0, (1 << 16) - 1, O.I64, O.ADD, O.STATIC, 1, 1, 1))
    for teams in (1, 2, 3, 296, 1000, 7, 1):
        assert int(runtime.reduce(x, teams=teams, threads=256).item()) == want


def test_full_size_int64_and_fp64(cuda):
    # BASELINE config 2 size: 2^30 fp64 (8 GiB) — rel 1e-6 vs the exact sum;
    # the same size in int64 — bit-exact (wrapping) vs the oracle
    n = 1 << 30
    x = runtime.synthetic(n, "f64", O.SEED, device=cuda)
    exact = O.exact_sum_gen(0, n - 1, O.F64)
    for teams, threads in ((296, 1024), (592, 1024), (148, 512)):
        got = float(runtime.reduce(x, "add", sched="distribute", teams=teams,
                                   threads=threads).item())
        assert abs(got - exact) <= 1e-6 * exact
    del x
    torch.cuda.empty_cache()
    xi = runtime.synthetic(n, "i64", O.SEED, device=cuda)
    want = O.reduce_flat_gen(0, n - 1, O.I64, O.ADD)
    got = int(runtime.reduce(xi, "add", teams=296, threads=1024).item())
    assert got == int(want)
    want_max = O.reduce_flat_gen(0, n - 1, O.I64, O.MAX, init=np.iinfo(np.int64).min)
    got_max = int(runtime.reduce(xi, "max", teams=296, threads=1024,
                                 init=np.iinfo(np.int64).min).item())
    assert got_max == int(want_max)
    del xi
    torch.cuda.empty_cache()


def test_bulk_ring_stress(cuda):
    # many short rings: partial last stages, one-stage teams, teams with no
    # vector part, every stage count; the result must be exact every time
    # (variant 78 keeps small pieces on the ring instead of the LDG walker)
    x = runtime.synthetic(3_000_017, "i64", O.SEED, 11, device=cuda)
    xn = x.cpu().numpy()
    try:
        for variant in (0, 78):
            runtime.set_variant(variant)
            for lb, ub, teams, threads in ((0, 3_000_016, 148, 256), (7, 2_999_999, 1000, 64),
                                           (1, 40_000, 3, 96), (0, 4096 * 4 - 1, 4, 128)):
                want = int(O.reduce(xn, lb, ub, O.I64, O.ADD, O.STATIC, 1, 1, 1))
                out = torch.zeros(1, dtype=torch.int64, device=cuda)
                for _ in range(200):
                    runtime.reduce(x, lb=lb, ub=ub, sched="distribute", teams=teams,
                                   threads=threads, out=out)
                assert int(out.item()) == (want * 200 + 2**63) % 2**64 - 2**63, (variant, lb, ub)
    finally:
        runtime.set_variant(0)


@pytest.mark.parametrize("dtype", ["f64", "i32", "u64"])
def test_comb_bulk_plans(cuda, dtype):
    # flat schedule(static, c): teeth packed per stage (case B), cut into
    # stages (case A), clipped last teeth, aligned and misaligned starts
    dt = ALLDT[dtype]
    n = 1_000_003
    x = O.fill(n, dt, O.SEED, 5)
    xd = torch.from_numpy(x).to(cuda)
    V = 16 // x.itemsize
    for teams, threads, chunk, lb, ub in ((7, 128, 3, 0, n - 3), (5, 64, 1, 0, n - 1),
                                          (3, 256, 700, 0, n - 1), (9, 96, 64, V, n - 2),
                                          (148, 256, 1, 0, n - 1), (2, 64, 4096, 0, 70_000),
                                          (4, 128, 2, 1, n - 1)):
        want = O.reduce(x, lb, ub, dt, O.ADD, O.STATIC_CHUNKED, chunk, teams, threads, 0)
        # default: balanced contiguous CTA pieces; variant 30: each team's
        # literal comb of teeth through the comb bulk plans
        for variant in (0, 30):
            out = torch.zeros(1, dtype=xd.dtype, device=cuda)
            runtime.set_variant(variant)
            try:
                runtime.reduce(xd, lb=lb, ub=ub, sched="static_chunked", chunk=chunk,
                               teams=teams, threads=threads, out=out)
            finally:
                runtime.set_variant(0)
            got = out.cpu().numpy()[0]
            if dt == O.F64:
                exact = O.accurate_sum_f64(x[lb:ub + 1])
                assert abs(float(got) - exact) <= 1e-9 * exact
            else:
                assert int(got) == int(want), (teams, threads, chunk, lb, ub, variant)


@pytest.mark.parametrize("sched", list(SCHEDS))
def test_team_split_matches_one_cta_per_team(cuda, sched):
    # few teams: each team is split over several CTAs (team_set_cta); integer
    # results must equal the one-CTA-per-team launch (variant 30) and the
    # oracle bit for bit, for contiguous and comb team sets
    n = 1_500_007
    x = O.fill(n, O.I64, O.SEED, 12)
    xd = torch.from_numpy(x).to(cuda)
    try:
        for teams, threads, lb, ub, chunk in ((1, 128, 0, n - 1, 1), (1, 128, 3, n - 5, 64),
                                              (2, 256, 1, n - 1, 4096), (5, 96, 0, 700_000, 7),
                                              (9, 1024, 0, n - 1, 300), (3, 64, 10, 5000, 1)):
            want = O.reduce(x, lb, ub, O.I64, O.ADD, SCHEDS[sched], chunk, teams, threads, 0)
            got = run_reduce(cuda, x, O.I64, "add", sched, chunk, teams, threads, lb, ub)
            runtime.set_variant(30)
            one = run_reduce(cuda, x, O.I64, "add", sched, chunk, teams, threads, lb, ub)
            runtime.set_variant(0)
            assert int(got) == int(want) == int(one), (teams, threads, lb, ub, chunk)
            # fp64 through the split path stays within the SPMD tolerance
            xf = runtime.synthetic(n, "f64", O.SEED, 12, device=cuda)
            gf = float(runtime.reduce(xf, lb=lb, ub=ub, sched=sched, chunk=chunk, teams=teams,
                                      threads=threads).item())
            ex = O.exact_sum_gen(lb, ub, O.F64, k=12)
            assert abs(gf - ex) <= 1e-6 * ex
    finally:
        runtime.set_variant(0)


def test_spmd_cta_size_is_unobservable(cuda):
    # the OpenMP geometry defines every team's iteration set; the CTA that
    # runs a team may have another size (omprt_set_spmd_block): integer
    # results are identical for every CTA size, also for OpenMP thread
    # counts that are not a multiple of 32
    n = 1_000_003
    x = O.fill(n, O.I64, O.SEED, 13)
    xd = torch.from_numpy(x).to(cuda)
    try:
        for sched in SCHEDS:
            for teams, threads, chunk in ((148, 384, 64), (37, 100, 7), (3, 1000, 4096)):
                want = int(O.reduce(x, 0, n - 1, O.I64, O.ADD, SCHEDS[sched], chunk, teams,
                                    threads, 0))
                for blk in (0, 64, 96, 384, 1024):
                    runtime.set_spmd_block(blk)
                    got = run_reduce(cuda, x, O.I64, "add", sched, chunk, teams, threads, 0, n - 1)
                    assert int(got) == want, (sched, teams, threads, chunk, blk)
    finally:
        runtime.set_spmd_block(0)
    # axpy + max/min: y bit for bit, max/min exact
    xf = O.fill(n, O.F32, O.SEED, 0)
    yf = O.fill(n, O.F32, O.SEED, 1)
    yo = yf.copy()
    mx, mn = O.axpy_minmax(1.5, xf, yo, 0, n - 1, O.STATIC_CHUNKED, 64, 37, 100, -np.inf, np.inf)
    try:
        for blk in (64, 1024):
            runtime.set_spmd_block(blk)
            xd2, yd2 = torch.from_numpy(xf).to(cuda), torch.from_numpy(yf).to(cuda)
            gmx, gmn = runtime.axpy_minmax(1.5, xd2, yd2, sched="static_chunked", chunk=64,
                                           teams=37, threads=100)
            assert np.array_equal(yd2.cpu().numpy(), yo) and float(gmx.item()) == mx \
                and float(gmn.item()) == mn
    finally:
        runtime.set_spmd_block(0)


@pytest.mark.gpu
def test_constructs_capture_into_cuda_graphs(cuda):
    """Launch-bound callers (config 1) replay the constructs from a CUDA
    graph: every construct entry point must be capture-safe (no stream or
    device queries that invalidate a capture) and the replays must give the
    same results as direct launches (the ticket self-resets between them)."""
    n = 1 << 20
    xi = runtime.synthetic(n, "i64", O.SEED, device=cuda)
    xf = runtime.synthetic(n, "f64", O.SEED, device=cuda)
    ys = runtime.synthetic(n, "f32", O.SEED, 1, device=cuda)
    xs = runtime.synthetic(n, "f32", O.SEED, device=cuda)
    oi = torch.zeros(1, dtype=torch.int64, device=cuda)
    od = torch.zeros(1, dtype=torch.float64, device=cuda)
    omx = torch.full((1,), float("-inf"), dtype=torch.float32, device=cuda)
    omn = torch.full((1,), float("inf"), dtype=torch.float32, device=cuda)
    om = torch.full((1,), float("-inf"), dtype=torch.float64, device=cuda)

    def body():
        runtime.reduce(xi, sched="static", teams=1, threads=128, out=oi)  # config 1 (split CTAs)
        runtime.dot(xf, xf, out=od)
        runtime.axpy_minmax(0.0, xs, ys, sched="static_chunked", chunk=64, mode="ordered",
                            out_max=omx, out_min=omn)
        runtime.reduce(xf, "max", sched="distribute", mode="ordered", out=om)

    s = torch.cuda.Stream(cuda)
    s.wait_stream(torch.cuda.current_stream(cuda))
    with torch.cuda.stream(s):
        body()  # warm-up outside the capture (smem attributes, workspace)
        torch.cuda.synchronize()
        want = (oi.item(), od.item(), omx.item(), omn.item(), om.item())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            body()
    torch.cuda.synchronize()
    for _ in range(3):
        oi.zero_()
        od.zero_()
        omx.fill_(float("-inf"))
        omn.fill_(float("inf"))
        om.fill_(float("-inf"))
        g.replay()
        torch.cuda.synchronize()
        assert oi.item() == want[0]
        assert abs(od.item() - want[1]) <= 1e-12 * abs(want[1])
        assert (omx.item(), omn.item(), om.item()) == want[2:]


@pytest.mark.gpu
def test_concurrent_host_threads_and_streams(cuda):
    """A multi-threaded host program: four threads, each on its own stream
    (own cached workspace), launch constructs concurrently — tuning knobs are
    per thread, the ticket of each workspace self-resets — and every result
    is exact."""
    import threading

    n = 1 << 21
    xi = runtime.synthetic(n, "i64", O.SEED, 21, device=cuda)
    want = int(O.reduce(None, 0, n - 1, O.I64, O.ADD, O.STATIC, 1, 1, 1, k=21))
    errors = []

    def work(tid: int) -> None:
        try:
            s = torch.cuda.Stream(cuda)
            with torch.cuda.stream(s):
                runtime.set_spmd_block([0, 256, 512, 96][tid])  # per-thread knob
                out = torch.zeros(1, dtype=torch.int64, device=cuda)
                for _ in range(50):
                    runtime.reduce(xi, sched=["static", "distribute", "static_chunked",
                                              "distribute_chunked"][tid], chunk=64,
                                   teams=[148, 37, 1, 300][tid], threads=[384, 256, 128, 64][tid],
                                   out=out)
                s.synchronize()
                got = int(out.item())
                runtime.set_spmd_block(0)
            exp = (want * 50 + 2**63) % 2**64 - 2**63
            if got != exp:
                errors.append((tid, got, exp))
        except Exception as e:  # noqa: BLE001
            errors.append((tid, repr(e)))

    threads = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
