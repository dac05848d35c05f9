"""Config 3 (chunked static axpy + fp32 max/min) and config 5 (fp64 dot), GPU.

axpy: y is elementwise bit-exact against the CPU restatement (both use one
correctly rounded fused multiply-add, fmaf / __fmaf_rn), max/min bit-exact
(order-independent, no NaN/-0 in the inputs).  dot: rel 1e-6 of the
accurate sum in SPMD mode; bit-identical in ORDERED mode.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2106_03219_b200 import runtime

pytestmark = pytest.mark.gpu

SCHEDS = {"static": O.STATIC, "static_chunked": O.STATIC_CHUNKED,
          "distribute": O.DISTRIBUTE, "distribute_chunked": O.DISTRIBUTE_CHUNKED}


def axpy_case(cuda, n, a, sched, chunk, teams, threads, lb, ub, mode="spmd"):
    x = O.fill(n, O.F32, O.SEED, 0)
    y = O.fill(n, O.F32, O.SEED, 1)
    yo = y.copy()
    mx, mn = O.axpy_minmax(a, x, yo, lb, ub, SCHEDS[sched], chunk, teams, threads, -np.inf, np.inf)
    xd, yd = torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda)
    gmx, gmn = runtime.axpy_minmax(a, xd, yd, lb=lb, ub=ub, sched=sched, chunk=chunk, teams=teams,
                                   threads=threads, mode=mode)
    assert np.array_equal(yd.cpu().numpy(), yo), (sched, chunk, teams, threads, lb, ub)
    assert float(gmx.item()) == mx and float(gmn.item()) == mn


@pytest.mark.parametrize("chunk", [1, 64, 4096])
@pytest.mark.parametrize("sched", ["static_chunked", "distribute_chunked"])
@pytest.mark.parametrize("mode", ["spmd", "ordered"])
def test_axpy_chunked_schedules(cuda, chunk, sched, mode):
    n = 300_007
    for teams, threads, lb, ub in ((4, 128, 0, n - 1), (37, 256, 3, n - 5), (1, 96, 1, 9999),
                                    (148, 1024, 0, n - 1)):
        axpy_case(cuda, n, 2.5, sched, chunk, teams, threads, lb, ub, mode)


def test_axpy_block_schedules_and_misalignment(cuda):
    n = 70_001
    for sched in ("static", "distribute"):
        for lb in range(4):
            axpy_case(cuda, n, -1.75, sched, 1, 7, 64, lb, n - 1 - lb)


def test_axpy_config3_full_size(cuda):
    # N = 2^28 fp32 (1 GiB per array), chunk = 1, 64, 4096
    n = 1 << 28
    xd = runtime.synthetic(n, "f32", O.SEED, 0, device=cuda)
    x = xd.cpu().numpy()
    y0 = O.fill(n, O.F32, O.SEED, 1)
    for chunk in (1, 64, 4096):
        yd = torch.from_numpy(y0).to(cuda)
        yo = y0.copy()
        mx, mn = O.axpy_minmax(2.5, x, yo, 0, n - 1, O.DISTRIBUTE_CHUNKED, chunk, 148, 1024,
                               -np.inf, np.inf)
        gmx, gmn = runtime.axpy_minmax(2.5, xd, yd, sched="distribute_chunked", chunk=chunk,
                                       teams=148, threads=1024)
        assert float(gmx.item()) == mx and float(gmn.item()) == mn
        assert torch.equal(yd, torch.from_numpy(yo).to(cuda))
        del yd
    torch.cuda.empty_cache()


@pytest.mark.parametrize("teams,threads", [(148, 384), (148, 1024)])
def test_axpy_config3_flat_static_chunked_full_size(cuda, teams, threads):
    # config 3 as the bench runs it: flat schedule(static, c) at N = 2^28,
    # chunk 1/64/4096, in the bench geometry (148 x 384) and 148 x 1024;
    # y bit for bit, max/min exact against the oracle's chunk walk
    n = 1 << 28
    xd = runtime.synthetic(n, "f32", O.SEED, 0, device=cuda)
    x = xd.cpu().numpy()
    y0 = O.fill(n, O.F32, O.SEED, 1)
    for chunk in (1, 64, 4096):
        for mode in ("spmd", "ordered"):
            yd = torch.from_numpy(y0).to(cuda)
            yo = y0.copy()
            mx, mn = O.axpy_minmax(2.5, x, yo, 0, n - 1, O.STATIC_CHUNKED, chunk, teams, threads,
                                   -np.inf, np.inf)
            gmx, gmn = runtime.axpy_minmax(2.5, xd, yd, sched="static_chunked", chunk=chunk,
                                           teams=teams, threads=threads, mode=mode)
            assert float(gmx.item()) == mx and float(gmn.item()) == mn, (chunk, mode)
            assert torch.equal(yd, torch.from_numpy(yo).to(cuda)), (chunk, mode)
            del yd
    torch.cuda.empty_cache()


def test_axpy_spmd_signed_zero_rule(cuda):
    # SPMD max/min return the exact extreme; when +0 and -0 tie for it the
    # zero's sign is unspecified (include/omprt_b200.h, omprt_mode), so only
    # the value is checked here; y stays bit-exact (ORDERED pins the sign:
    # test_axpy_ordered_keeps_the_reference_order_of_signed_zeros)
    n = 1 << 20
    for base in (-1.0, 1.0):
        x = np.zeros(n, dtype=np.float32)
        y = np.full(n, base, dtype=np.float32)
        i = np.arange(n)
        x[(i % 997) == 5], y[(i % 997) == 5] = np.float32(-0.0), np.float32(-0.0)
        x[(i % 1009) == 3], y[(i % 1009) == 3] = np.float32(0.0), np.float32(0.0)
        yo = y.copy()
        mx, mn = O.axpy_minmax(1.0, x, yo, 0, n - 1, O.STATIC_CHUNKED, 64, 148, 384,
                               -np.inf, np.inf)
        xd, yd = torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda)
        gmx, gmn = runtime.axpy_minmax(1.0, xd, yd, sched="static_chunked", chunk=64, teams=148,
                                       threads=384)
        assert float(gmx.item()) == mx and float(gmn.item()) == mn  # -0 == +0
        assert (float(gmx.item()) == 0.0) == (base < 0) and (float(gmn.item()) == 0.0) == (base > 0)
        assert np.array_equal(yd.cpu().numpy().view(np.uint32), yo.view(np.uint32))


@pytest.mark.parametrize("sched", list(SCHEDS))
def test_dot_matches_oracle(cuda, sched):
    n = 500_003
    x, y = O.fill(n, O.F64, O.SEED, 0), O.fill(n, O.F64, O.SEED, 1)
    xd, yd = torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda)
    for teams, threads, lb, ub, chunk in ((5, 64, 0, n - 1, 1), (148, 256, 1, n - 2, 64),
                                          (1, 32, 3, 1000, 7)):
        truth = O.accurate_dot_gen(lb, ub)
        got = float(runtime.dot(xd, yd, lb=lb, ub=ub, sched=sched, chunk=chunk, teams=teams,
                                threads=threads).item())
        assert abs(got - truth) <= 1e-6 * truth
        want = O.dot(x, y, lb, ub, SCHEDS[sched], chunk, teams, threads)
        got_o = float(runtime.dot(xd, yd, lb=lb, ub=ub, sched=sched, chunk=chunk, teams=teams,
                                  threads=threads, mode="ordered").item())
        assert got_o == want  # reference order: bit-identical


def test_dot_full_shard(cuda):
    # one GPU's shard of config 5 at 2^30 (two 8 GiB arrays)
    n = 1 << 30
    x = runtime.synthetic(n, "f64", O.SEED, 0, device=cuda)
    y = runtime.synthetic(n, "f64", O.SEED, 1, device=cuda)
    got = float(runtime.dot(x, y).item())
    truth = O.accurate_dot_gen(0, n - 1)
    assert abs(got - truth) <= 1e-6 * truth
    del x, y
    torch.cuda.empty_cache()


@pytest.mark.parametrize("n,teams,threads,sched", [(1 << 20, 8, 64, "distribute"),
                                                   (1 << 24, 8, 64, "static"),
                                                   (300_001, 5, 96, "static_chunked")])
def test_axpy_ordered_keeps_the_reference_order_of_signed_zeros(cuda, n, teams, threads, sched):
    # max/min are exact but not order-free for +0/-0 (a < b is false both
    # ways): the ORDERED result's zero sign must be the reference order's
    chunk = 64
    for base in (-1.0, 1.0):  # max picks among zeros, then min does
        x = np.zeros(n, dtype=np.float32)
        y = np.full(n, base, dtype=np.float32)
        i = np.arange(n)
        neg = (i % 997) == 5
        pos = (i % 1009) == 3
        x[neg], y[neg] = np.float32(-0.0), np.float32(-0.0)  # 1*-0 + -0 = -0
        x[pos], y[pos] = np.float32(0.0), np.float32(0.0)    # 1*+0 + +0 = +0
        yo = y.copy()
        mx, mn = O.axpy_minmax(1.0, x, yo, 0, n - 1, SCHEDS[sched], chunk, teams, threads,
                               -np.inf, np.inf)
        xd, yd = torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda)
        gmx, gmn = runtime.axpy_minmax(1.0, xd, yd, sched=sched, chunk=chunk, teams=teams,
                                       threads=threads, mode="ordered")
        got = np.array([gmx.item(), gmn.item()], dtype=np.float32)
        want = np.array([mx, mn], dtype=np.float32)
        assert got.tobytes() == want.tobytes(), (base, sched, got, want)
        assert np.array_equal(yd.cpu().numpy().view(np.uint32), yo.view(np.uint32))
