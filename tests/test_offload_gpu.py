"""The forge-shaped launch boundary (tgt_target) on the B200 (GPU).

Arguments are passed exactly as the reference passes them: packed
little-endian bytearrays for buffers, ints for scalars, in sema's capture
order; results are written back into the bytearrays only on status 0
(host.py:255-296).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2106_03219_b200 import (
    ArgDescriptor,
    RegionKernel,
    TargetCall,
    kernel_name,
    reduce_host,
    tgt_target,
)

pytestmark = pytest.mark.gpu


def le(vals, dt):
    return bytearray(np.asarray(vals, dtype=dt).tobytes())


def partial_sums_call():
    # corpus.PARTIAL_SUMS with its x = i buffer made explicit: capture order
    # of `kernel(u32 *x, u32 *cell, i64 n)` as sema records it (n, x, cell)
    args = (ArgDescriptor("n", "scalar", "i64"), ArgDescriptor("x", "buffer", "u32"),
            ArgDescriptor("cell", "buffer", "u32"))
    call = TargetCall(0, kernel_name(0), args, grid=(2, 4))
    image = {"b200": {kernel_name(0): RegionKernel("reduce", {"x": "x", "cell": "cell", "n": "n"},
                                                    op="add", lb=1)}}
    return call, image


def test_partial_sums_region(cuda):
    call, image = partial_sums_call()
    x = le(range(101), np.uint32)
    cell = le([0], np.uint32)
    out = {}
    st = tgt_target(call.bind([100, x, cell]), image, "b200", out=out)
    assert st == 0
    assert np.frombuffer(cell, np.uint32)[0] == 5050  # corpus output, SURVEY §A.1
    # the NVIDIA arch name of the reference's target table runs here too
    cell2 = le([0], np.uint32)
    assert tgt_target(call.bind([100, x, cell2]), image, "nvptx64") == 0
    assert np.frombuffer(cell2, np.uint32)[0] == 5050


def test_config1_through_tgt_target(cuda, fallback_golden):
    r = next(r for r in fallback_golden["reductions"] if r["threads"] == 128)
    args = (ArgDescriptor("n", "scalar", "i64"), ArgDescriptor("x", "buffer", "i64"),
            ArgDescriptor("cell", "buffer", "i64"))
    call = TargetCall(0, kernel_name(0), args)
    image = {"b200": {kernel_name(0): RegionKernel("reduce", {"x": "x", "cell": "cell",
                                                              "n": "n"})}}
    x = bytearray(O.fill(r["n"], O.I64, r["seed"], r["k"]).tobytes())
    cell = le([r["init"]], np.int64)
    assert tgt_target(call.bind([r["n"], x, cell]), image, grid=(1, 128)) == 0
    assert np.frombuffer(cell, np.int64)[0] == r["fallback"]


def test_trap_leaves_buffers_untouched(cuda):
    args = (ArgDescriptor("n", "scalar", "i64"), ArgDescriptor("x", "buffer", "i64"),
            ArgDescriptor("cell", "buffer", "i64"))
    call = TargetCall(3, kernel_name(3), args)
    image = {"b200": {kernel_name(3): RegionKernel("generic_reduce", {"x": "x", "cell": "cell",
                                                                      "n": "n"},
                                                    pad_bytes=65536 - 64, par_threads=64)}}
    x = le(range(1000), np.int64)
    cell = le([42], np.int64)
    out = {}
    st = tgt_target(call.bind([1000, x, cell]), image, grid=(4, 96), out=out)
    assert st == 2
    assert out["trap"][0] == "SharedOverflow"
    assert np.frombuffer(cell, np.int64)[0] == 42
    # with the heap fallback the same region runs
    image["b200"][kernel_name(3)] = RegionKernel("generic_reduce",
                                                 {"x": "x", "cell": "cell", "n": "n"},
                                                 pad_bytes=65536 - 64, par_threads=64,
                                                 heap_fallback=True)
    assert tgt_target(call.bind([1000, x, cell]), image, grid=(4, 96)) == 0
    assert np.frombuffer(cell, np.int64)[0] == 42 + sum(range(1000))


def test_axpy_and_dot_regions(cuda):
    n = 10_000
    x = O.fill(n, O.F32, O.SEED, 0)
    y = O.fill(n, O.F32, O.SEED, 1)
    yo = y.copy()
    mx, mn = O.axpy_minmax(0.5, x, yo, 0, n - 1, O.DISTRIBUTE_CHUNKED, 64, 8, 64, -np.inf, np.inf)
    args = (ArgDescriptor("n", "scalar", "i64"), ArgDescriptor("y", "buffer", "f32"),
            ArgDescriptor("a", "scalar", "f32"), ArgDescriptor("x", "buffer", "f32"),
            ArgDescriptor("mx", "buffer", "f32"), ArgDescriptor("mn", "buffer", "f32"))
    call = TargetCall(1, kernel_name(1), args)
    image = {"b200": {kernel_name(1): RegionKernel(
        "axpy_minmax", {"a": "a", "x": "x", "y": "y", "max": "mx", "min": "mn", "n": "n"},
        sched="distribute_chunked", chunk=64)}}
    yb = bytearray(y.tobytes())
    mxb, mnb = le([-np.inf], np.float32), le([np.inf], np.float32)
    assert tgt_target(call.bind([n, yb, 0.5, bytearray(x.tobytes()), mxb, mnb]), image,
                      grid=(8, 64)) == 0
    assert np.array_equal(np.frombuffer(yb, np.float32), yo)
    assert np.frombuffer(mxb, np.float32)[0] == mx and np.frombuffer(mnb, np.float32)[0] == mn

    xd, yd = O.fill(n, O.F64, O.SEED, 0), O.fill(n, O.F64, O.SEED, 1)
    args = (ArgDescriptor("n", "scalar", "i64"), ArgDescriptor("x", "buffer", "f64"),
            ArgDescriptor("y", "buffer", "f64"), ArgDescriptor("c", "buffer", "f64"))
    call = TargetCall(2, kernel_name(2), args)
    image = {"b200": {kernel_name(2): RegionKernel("dot", {"x": "x", "y": "y", "cell": "c",
                                                           "n": "n"}, mode="ordered")}}
    c = le([0.0], np.float64)
    assert tgt_target(call.bind([n, xd, yd, c]), image, grid=(4, 32)) == 0
    assert np.frombuffer(c, np.float64)[0] == O.dot(xd, yd, 0, n - 1, O.STATIC, 1, 4, 32)


def test_bounds_region_matches_vgpu(cuda, fallback_golden):
    rec = fallback_golden["vgpu_bounds"][1]
    n = rec["teams"] * rec["threads"]
    args = (ArgDescriptor("out", "buffer", "i64"), ArgDescriptor("lb", "scalar", "i64"),
            ArgDescriptor("ub", "scalar", "i64"))
    call = TargetCall(4, kernel_name(4), args)
    image = {"b200": {kernel_name(4): RegionKernel("bounds", {"out": "out", "lb": "lb",
                                                              "ub": "ub"})}}
    out = le([0] * (4 * n), np.int64)
    assert tgt_target(call.bind([out, rec["lb"], rec["ub"]]), image,
                      grid=(rec["teams"], rec["threads"])) == 0
    got = np.frombuffer(out, np.int64).reshape(n, 4)[:, :2].tolist()
    assert got == rec["bounds"]


def test_reduce_host_entry(cuda):
    n = 1 << 22
    x = torch.from_numpy(O.fill(n, O.I64, O.SEED, 5)).pin_memory()
    cell = torch.tensor([7], dtype=torch.int64)
    reduce_host(x, cell, teams=148, threads=256)
    assert int(cell.item()) == 7 + int(O.reduce_flat_gen(0, n - 1, O.I64, O.ADD, k=5))
    xn = O.fill(n, O.F64, O.SEED, 6)  # pageable numpy memory
    c2 = np.zeros(1, np.float64)
    reduce_host(xn, c2, teams=148, threads=256, mode="ordered")
    assert c2[0] == O.reduce(xn, 0, n - 1, O.F64, O.ADD, O.STATIC, 1, 148, 256)


def test_reduce_host_pipelined(cuda):
    # above 512 MiB the input lands in 256 MiB pieces on a copy stream while
    # the previous piece is reduced (each launch accumulates into the cell):
    # integers bit-exact, fp64 SPMD within 1e-6; a ragged last piece
    n = (600 << 20) // 8 + 12345
    x = torch.from_numpy(O.fill(n, O.I64, O.SEED, 8)).pin_memory()
    cell = torch.tensor([-3], dtype=torch.int64)
    reduce_host(x, cell, sched="distribute", teams=148, threads=384)
    assert int(cell.item()) == O._signed(-3 + int(O.reduce_flat_gen(0, n - 1, O.I64, O.ADD, k=8)),
                                         64)
    cmax = torch.tensor([-(1 << 63)], dtype=torch.int64)
    reduce_host(x, cmax, op="max", teams=148, threads=384, mode="ordered")
    assert int(cmax.item()) == int(x.max().item())
    xf = torch.from_numpy(O.fill(n, O.F64, O.SEED, 8)).pin_memory()
    cf = torch.zeros(1, dtype=torch.float64)
    reduce_host(xf, cf, sched="distribute", teams=148, threads=384)
    ex = O.exact_sum_gen(0, n - 1, O.F64, k=8)
    assert abs(float(cf.item()) - ex) <= 1e-6 * ex
    del x, xf


def test_axpy_dot_generic_host_entries(cuda):
    """The host-buffer C entries for configs 3, 5 and 4: copy-in, launch,
    copy-out only on status 0 (host.py:276-295), bit-exact vs the oracle."""
    from paper_2106_03219_b200 import axpy_minmax_host, dot_host, generic_reduce_host

    n = (1 << 20) + 37
    x = O.fill(n, O.F32, O.SEED, 2)
    y = O.fill(n, O.F32, O.SEED, 3)
    yo = y.copy()
    mx, mn = O.axpy_minmax(2.5, x, yo, 0, n - 1, O.STATIC_CHUNKED, 64, 148, 384, -np.inf, np.inf)
    cells = np.array([-np.inf, np.inf], np.float32)
    yt = torch.from_numpy(y.copy()).pin_memory()
    axpy_minmax_host(2.5, torch.from_numpy(x).pin_memory(), yt, cells, sched="static_chunked",
                     chunk=64, teams=148, threads=384)
    assert np.array_equal(yt.numpy(), yo)
    assert cells[0] == mx and cells[1] == mn

    xd, yd = O.fill(n, O.F64, O.SEED, 0), O.fill(n, O.F64, O.SEED, 1)
    c = np.array([1.5], np.float64)
    dot_host(xd, yd, c, teams=148, threads=384, mode="ordered")
    assert c[0] == O.dot(xd, yd, 0, n - 1, O.STATIC, 1, 148, 384, 1.5)

    xi = O.fill(n, O.I64, O.SEED, 4)
    cell = np.array([9], np.int64)
    offs = np.full(64, -1, np.int64)
    assert generic_reduce_host(xi, cell, teams=64, par_threads=128, team_offsets=offs) == 0
    assert cell[0] == O.generic_reduce(xi, 0, n - 1, O.I64, O.ADD, 64, 128, 9)
    assert (offs == 0).all()  # parts is the team's first (and only) allocation
    # an arena overflow traps: status 2, cell and offsets untouched
    out = {}
    cell2 = np.array([9], np.int64)
    offs2 = np.full(64, -1, np.int64)
    assert generic_reduce_host(xi, cell2, teams=64, par_threads=128, pad_bytes=65536 - 64,
                               team_offsets=offs2, out=out) == 2
    assert out["trap"][0] == "SharedOverflow"
    assert cell2[0] == 9 and (offs2 == -1).all()


def test_iteration_space_escape_is_out_of_bounds(cuda):
    """A trip count larger than a buffer: the vgpu traps OutOfBounds (status 2,
    buffers untouched); the B200 boundary refuses before any launch."""
    from paper_2106_03219_b200 import runtime

    x = torch.zeros(100, dtype=torch.float32, device=cuda)
    y = torch.zeros(50, dtype=torch.float32, device=cuda)
    with pytest.raises(IndexError):
        runtime.axpy_minmax(1.0, x, y)  # ub = 99 escapes y[0:50]
    with pytest.raises(IndexError):
        runtime.dot(x.double(), y.double())
    with pytest.raises(IndexError):
        runtime.reduce(x, lb=-1, ub=10)
    with pytest.raises(IndexError):
        runtime.generic_reduce(x.double(), ub=100, teams=4, par_threads=32)
    runtime.dot(x.double(), y.double(), ub=-1)  # an empty space touches nothing

    args = (ArgDescriptor("n", "scalar", "i64"), ArgDescriptor("y", "buffer", "f32"),
            ArgDescriptor("a", "scalar", "f32"), ArgDescriptor("x", "buffer", "f32"),
            ArgDescriptor("mx", "buffer", "f32"), ArgDescriptor("mn", "buffer", "f32"))
    call = TargetCall(1, kernel_name(1), args)
    image = {"b200": {kernel_name(1): RegionKernel(
        "axpy_minmax", {"a": "a", "x": "x", "y": "y", "max": "mx", "min": "mn", "n": "n"})}}
    yb = le(range(50), np.float32)
    mxb = le([-1.0], np.float32)
    out = {}
    st = tgt_target(call.bind([100, yb, 2.0, le(range(100), np.float32), mxb,
                               le([1.0], np.float32)]), image, grid=(2, 32), out=out)
    assert st == 2 and out["trap"][0] == "OutOfBounds"
    assert np.array_equal(np.frombuffer(yb, np.float32), np.arange(50, dtype=np.float32))
    assert np.frombuffer(mxb, np.float32)[0] == -1.0
