"""Device-side entry points of the data-parallel core, over torch tensors.

Every function here launches a kernel of libomprt_b200.so on the tensors'
CUDA device and current stream; none has a CPU path.  Iteration spaces are
inclusive [lb, ub] and index the input arrays directly (x[i]), exactly like
the reference's `for_static_init(lb, ub, ...)` loops (runtime.mc:193-203).

Names follow the OpenMP device runtime the paper rewrites:
  bounds_dump        __kmpc_for_static_init / __kmpc_distribute_static_init
  reduce             target teams distribute parallel for reduction(op: cell)
  axpy_minmax        the same construct over y = a*x + y with max/min
  dot                fp64 dot product reduction
  generic_reduce     generic-mode region: __kmpc_alloc_shared + nested parallel reduce
  arena_replay       __kmpc_alloc_shared / __kmpc_free_shared scripts
  atomic_probe       the seq_cst atomic intrinsics on one cell
  atomic_apply       batched step_* semantics
"""

from __future__ import annotations

import ctypes as C
import functools
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check

_TORCH_DTYPE = {
    _lib.I32: torch.int32, _lib.U32: torch.uint32, _lib.I64: torch.int64,
    _lib.U64: torch.uint64, _lib.F32: torch.float32, _lib.F64: torch.float64,
}
_FROM_TORCH = {v: k for k, v in _TORCH_DTYPE.items()}


def dtype_code(dtype) -> int:
    if isinstance(dtype, int):
        return dtype
    if isinstance(dtype, str):
        return _lib.DTYPE_NAMES[dtype]
    return _FROM_TORCH[dtype]


def torch_dtype(code: int) -> torch.dtype:
    return _TORCH_DTYPE[code]


def _code(table: dict, v) -> int:
    return v if isinstance(v, int) else table[v]


# the current stream's raw handle without building a torch.cuda.Stream object
# (the wrapper is most of a small launch's host time: profiles/r1_c1_host.json)
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_handle(device: torch.device) -> int:
    """cudaStream_t of the current stream on `device`, as an int."""
    if _raw_stream is not None:
        idx = device.index if device.index is not None else torch.cuda.current_device()
        return _raw_stream(idx)
    return torch.cuda.current_stream(device).cuda_stream


def _stream(t: torch.Tensor) -> int:
    # a plain int: the bound argtypes (c_void_p) convert it, and building a
    # c_void_p per argument is a measurable part of a small launch's host time
    return stream_handle(t.device)


def _dev(t: torch.Tensor) -> torch.device:
    if not t.is_cuda:
        raise ValueError("tensors must live on a CUDA device (there is no CPU path)")
    _lib.ensure_device(t.device.index or 0)
    return t.device


def _check_range(lb: int, ub: int, *bufs: tuple[str, torch.Tensor]) -> None:
    """Every buffer the loop body touches must hold iterations [lb, ub] — the
    device kernels index x[i] without a size, so an escape here would read or
    write past the allocation; the vgpu traps OutOfBounds on the same access
    (vgpu.py:28-36).  An empty space (ub < lb) touches nothing."""
    if ub < lb:
        return
    for name, t in bufs:
        if lb < 0 or ub >= t.numel():
            raise IndexError(f"iteration space [{lb}, {ub}] escapes {name}[0:{t.numel()}]")


def _p(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


_sms: dict[int, int] = {}


def num_sms(index: int | None = None) -> int:
    """SM count of CUDA device `index` (default: the current one), cached."""
    dev = index if index is not None else (
        torch.cuda.current_device() if torch.cuda.is_available() else -1)
    n = _sms.get(dev)
    if n is None:
        if dev == torch.cuda.current_device():
            n = check(_lib.load().omprt_num_sms(), "omprt_num_sms")
        else:
            with torch.cuda.device(dev):
                n = check(_lib.load().omprt_num_sms(), "omprt_num_sms")
        _sms[dev] = n
    return n


def set_unroll(unroll: int) -> None:
    check(_lib.load().omprt_set_unroll(unroll), "omprt_set_unroll")


def set_spmd_block(threads: int) -> None:
    """Tuning: CUDA threads per CTA of the SPMD construct kernels for this
    thread (0 = the measured per-construct policy; see omprt_set_spmd_block)."""
    check(_lib.load().omprt_set_spmd_block(threads), "omprt_set_spmd_block")


def set_variant(variant: int) -> None:
    """Tuning: kernel variant of the fp64 sum (see omprt_set_variant)."""
    check(_lib.load().omprt_set_variant(variant), "omprt_set_variant")


@dataclass(frozen=True)
class Grid:
    """Launch geometry: num_teams x thread_limit (GridConfig, vgpu.py:50-61)."""

    teams: int
    threads: int


DEFAULT_THREADS = int(os.environ.get("OMPRT_DEFAULT_THREADS", "384"))


def default_grid(device: torch.device | None = None, threads: int | None = None,
                 teams_per_sm: int = 1) -> Grid:
    """A persistent grid: teams_per_sm resident teams on every SM (one team
    per SM holds the 3 x 48 KiB bulk-copy ring; 384 threads = 1 producer + 11
    consumer warps, which keep the ring drained when the power cap lowers
    the SM clock — profiles/r1_threads_sweep_256_384.txt)."""
    if device is not None:
        _lib.ensure_device(device.index or 0)
        return Grid(num_sms(device.index) * teams_per_sm, threads or DEFAULT_THREADS)
    return Grid(num_sms() * teams_per_sm, threads or DEFAULT_THREADS)


# ------------------------------------------------------------------ trap

@dataclass(frozen=True)
class DeviceTrap:
    kind: int
    code: int
    team: int
    thread: int


def check_trap(device: torch.device) -> DeviceTrap | None:
    """Synchronise the current stream and fetch/clear the device trap word."""
    _lib.ensure_device(device.index or 0)
    L = _lib.load()
    k, c, tm, th = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    st = check(L.omprt_check_trap(C.c_void_p(torch.cuda.current_stream(device).cuda_stream),
                                  C.byref(k), C.byref(c), C.byref(tm), C.byref(th)),
               "omprt_check_trap")
    if st == _lib.OK:
        return None
    return DeviceTrap(k.value, c.value, tm.value, th.value)


# ------------------------------------------------------------ worksharing

def static_bounds(lb: int, ub: int, tid: int, nthreads: int) -> tuple[int, int]:
    """for_static_init / devicert.static_bounds through the library's
    __host__ __device__ routine (the same code every device thread runs)."""
    a, b = C.c_int64(), C.c_int64()
    st = _lib.load().omprt_static_bounds(lb, ub, tid, nthreads, C.byref(a), C.byref(b))
    if st == _lib.TRAP:
        raise ZeroDivisionError("for_static_init: nthreads == 0 (DivideByZero trap)")
    check(st, "omprt_static_bounds")
    return a.value, b.value


def bounds_dump(lb: int, ub: int, sched="static", chunk: int = 1, *, teams: int, threads: int,
                device="cuda") -> torch.Tensor:
    """Every device thread's schedule init result: int64 [teams*threads, 4]
    (lower, upper, stride, last) — see include/omprt_b200.h."""
    out = torch.empty((teams * threads, 4), dtype=torch.int64, device=device)
    _dev(out)
    check(_lib.load().omprt_bounds_dump(lb, ub, _code(_lib.SCHED_NAMES, sched), chunk, teams,
                                        threads, _p(out), _stream(out)), "omprt_bounds_dump")
    return out


# ------------------------------------------------------------- NVTX ranges

_NVTX = os.environ.get("OMPRT_NVTX", "") not in ("", "0")


def _nvtx(name: str):
    """With OMPRT_NVTX=1 every construct launch is an NVTX range (for Nsight
    Systems timelines); otherwise the function is returned untouched."""
    def deco(fn):
        if not _NVTX:
            return fn

        @functools.wraps(fn)
        def wrapped(*a, **k):
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*a, **k)
            finally:
                torch.cuda.nvtx.range_pop()
        return wrapped
    return deco


# ------------------------------------------------------------- trace ring

TRACE_REC = np.dtype([("t_begin", "<u8"), ("t_end", "<u8"), ("cta", "<u4"), ("smid", "<u4"),
                      ("ticket", "<u4"), ("kind", "<u4")])
TRACE_KINDS = {1: "atomic.inc", 2: "combine", 3: "stream", 4: "fold"}


class Trace:
    """Per-team device trace of the constructs launched inside the block —
    the B200 analog of the vgpu's collect_trace (vgpu.py:351-353).  Every CTA
    of a construct records when it started, on which SM, when it took its
    last-team-finishes ticket and the ticket value its atom.inc returned; the
    last team records the ordered combine; ORDERED launches record each
    streaming warp and the folder.  `lines()` renders them like the vgpu's
    trace ("seq team thread kind detail"), ordered by completion time.
    One construct per Trace (records are indexed by CTA)."""

    def __init__(self, device: torch.device | None = None, capacity: int = 16384):
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.capacity = capacity
        self.buf = torch.zeros(capacity * TRACE_REC.itemsize // 8, dtype=torch.int64,
                               device=self.device)
        self.records = np.zeros(0, dtype=TRACE_REC)

    def __enter__(self):
        torch.cuda.synchronize(self.device)
        with torch.cuda.device(self.device):  # the ring symbol is per device
            check(_lib.load().omprt_set_trace(_p(self.buf), self.capacity), "omprt_set_trace")
        return self

    def __exit__(self, *exc):
        torch.cuda.synchronize(self.device)
        with torch.cuda.device(self.device):
            check(_lib.load().omprt_set_trace(None, 0), "omprt_set_trace")
        raw = self.buf.cpu().numpy().view(np.uint8).view(TRACE_REC)
        self.records = raw[raw["kind"] != 0].copy()
        return False

    def lines(self) -> list[str]:
        r = np.sort(self.records, order="t_end")
        if r.size == 0:
            return []
        t0 = int(r["t_begin"][r["t_begin"] > 0].min()) if (r["t_begin"] > 0).any() else 0
        out = []
        for seq, rec in enumerate(r):
            kind = TRACE_KINDS.get(int(rec["kind"]), f"kind{int(rec['kind'])}")
            b, e = int(rec["t_begin"]) - t0, int(rec["t_end"]) - t0
            if kind == "atomic.inc":
                detail = (f"ticket old={int(rec['ticket'])} sm={int(rec['smid'])} "
                          f"begin_ns={b} end_ns={e}")
            elif kind == "combine":
                detail = f"teams={int(rec['ticket']) + 1} begin_ns={b} end_ns={e}"
            elif kind == "stream":
                detail = f"groups={int(rec['ticket'])} sm={int(rec['smid'])} end_ns={e}"
            else:
                detail = f"batches={int(rec['ticket'])} end_ns={e}"
            out.append(f"{seq} {int(rec['cta'])} 0 {kind} {detail}")
        return out


# ------------------------------------------------------------- workspace

_ws_cache: dict[tuple, torch.Tensor] = {}


def workspace(device: torch.device, nbytes: int) -> torch.Tensor:
    """Zeroed device workspace, cached per (device, stream): the
    last-team-finishes ticket self-resets, so launches ordered on one stream
    may share it; concurrent streams each get their own."""
    key = (device.type, device.index or 0, stream_handle(device))
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros(max(nbytes, 1 << 16), dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws


_ws_bytes: dict[tuple, int] = {}


def reduce_workspace(device: torch.device, teams: int, threads: int, mode: int) -> torch.Tensor:
    key = (teams, threads, mode)
    nb = _ws_bytes.get(key)
    if nb is None:
        nb = _ws_bytes[key] = _lib.load().omprt_reduce_workspace_bytes(teams, threads, mode)
    return workspace(device, nb)


# ---------------------------------------------------------------- reduce

@_nvtx("omprt_reduce")
def reduce(x: torch.Tensor, op="add", *, lb: int = 0, ub: int | None = None, sched="static",
           chunk: int = 1, teams: int | None = None, threads: int | None = None, mode="spmd",
           out: torch.Tensor | None = None, init=None) -> torch.Tensor:
    """`#pragma omp target teams distribute parallel for reduction(op: cell)`
    over x[lb..ub].  Returns the 1-element device tensor `out`, updated in
    place as out = out OP reduce(x) (the original list item is combined in,
    like __atomic_add(cell, part) in corpus.py:219-247)."""
    dev = _dev(x)
    if not x.is_contiguous():
        raise ValueError("x must be contiguous")
    dt = dtype_code(x.dtype)
    opc = _code(_lib.OP_NAMES, op)
    m = _code(_lib.MODE_NAMES, mode)
    if ub is None:
        ub = lb + x.numel() - 1
    _check_range(lb, ub, ("x", x))
    if not (teams and threads):
        g = default_grid(dev)
        teams = teams or g.teams
        threads = threads or g.threads
    if out is None:
        out = torch.zeros(1, dtype=x.dtype, device=dev)
        if init is not None:
            out.fill_(init)
    ws = reduce_workspace(dev, teams, threads, m)
    check(_lib.load().omprt_reduce(_p(x), lb, ub, dt, opc, _code(_lib.SCHED_NAMES, sched), chunk,
                                   teams, threads, m, _p(ws), _p(out), _stream(x)),
          "omprt_reduce")
    return out


@_nvtx("omprt_axpy_minmax")
def axpy_minmax(a: float, x: torch.Tensor, y: torch.Tensor, *, lb: int = 0, ub: int | None = None,
                sched="distribute_chunked", chunk: int = 1, teams: int | None = None,
                threads: int | None = None, mode="spmd",
                out_max: torch.Tensor | None = None,
                out_min: torch.Tensor | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """y[i] = fmaf(a, x[i], y[i]) for i in [lb, ub], fused with max/min of y."""
    dev = _dev(x)
    if x.dtype != torch.float32 or y.dtype != torch.float32:
        raise TypeError("axpy_minmax is fp32")
    if not (x.is_contiguous() and y.is_contiguous()) or y.device != dev:
        raise ValueError("x and y must be contiguous and on one device")
    if ub is None:
        ub = lb + x.numel() - 1
    _check_range(lb, ub, ("x", x), ("y", y))
    g = default_grid(dev)
    teams = teams or g.teams
    threads = threads or g.threads
    m = _code(_lib.MODE_NAMES, mode)
    if out_max is None:
        out_max = torch.full((1,), float("-inf"), dtype=torch.float32, device=dev)
    if out_min is None:
        out_min = torch.full((1,), float("inf"), dtype=torch.float32, device=dev)
    ws = reduce_workspace(dev, teams, threads, m)
    check(_lib.load().omprt_axpy_minmax(C.c_float(a), _p(x), _p(y), lb, ub,
                                        _code(_lib.SCHED_NAMES, sched), chunk, teams, threads, m,
                                        _p(ws), _p(out_max), _p(out_min), _stream(x)),
          "omprt_axpy_minmax")
    return out_max, out_min


@_nvtx("omprt_dot")
def dot(x: torch.Tensor, y: torch.Tensor, *, lb: int = 0, ub: int | None = None,
        sched="static", chunk: int = 1, teams: int | None = None, threads: int | None = None,
        mode="spmd", out: torch.Tensor | None = None) -> torch.Tensor:
    """fp64 dot product reduction: out = out + sum fma(x[i], y[i], part)."""
    dev = _dev(x)
    if x.dtype != torch.float64 or y.dtype != torch.float64:
        raise TypeError("dot is fp64")
    if not (x.is_contiguous() and y.is_contiguous()) or y.device != dev:
        raise ValueError("x and y must be contiguous and on one device")
    if ub is None:
        ub = lb + x.numel() - 1
    _check_range(lb, ub, ("x", x), ("y", y))
    g = default_grid(dev)
    teams = teams or g.teams
    threads = threads or g.threads
    m = _code(_lib.MODE_NAMES, mode)
    if out is None:
        out = torch.zeros(1, dtype=torch.float64, device=dev)
    ws = reduce_workspace(dev, teams, threads, m)
    check(_lib.load().omprt_dot(_p(x), _p(y), lb, ub, _code(_lib.SCHED_NAMES, sched), chunk,
                                teams, threads, m, _p(ws), _p(out), _stream(x)), "omprt_dot")
    return out


def combine_partials(partials: torch.Tensor, op="add", out: torch.Tensor | None = None) -> torch.Tensor:
    """out = out OP p[0] OP p[1] ... in order (multi-GPU combine tail)."""
    dev = _dev(partials)
    if out is None:
        out = torch.zeros(1, dtype=partials.dtype, device=dev)
    check(_lib.load().omprt_combine_partials(_p(partials), partials.numel(),
                                             dtype_code(partials.dtype),
                                             _code(_lib.OP_NAMES, op), _p(out),
                                             _stream(partials)), "omprt_combine_partials")
    return out


# -------------------------------------------------------------- generic

@_nvtx("omprt_generic_reduce")
def generic_reduce(x: torch.Tensor, op="add", *, lb: int = 0, ub: int | None = None,
                   teams: int = 1024, par_threads: int = 256, ordered: bool = False,
                   pad_bytes: int = 0, heap_fallback: bool = False,
                   heap_bytes_per_team: int = 1 << 20, out: torch.Tensor | None = None,
                   team_offsets: torch.Tensor | None = None) -> torch.Tensor:
    """Generic-mode region with __kmpc_alloc_shared globalisation and a nested
    parallel reduce (config 4).  Does not synchronise; call check_trap()."""
    dev = _dev(x)
    if not x.is_contiguous():
        raise ValueError("x must be contiguous")
    if ub is None:
        ub = lb + x.numel() - 1
    _check_range(lb, ub, ("x", x))
    if team_offsets is not None and team_offsets.numel() < teams:
        raise IndexError(f"team_offsets holds {team_offsets.numel()} < {teams} teams")
    if out is None:
        out = torch.zeros(1, dtype=x.dtype, device=dev)
    L = _lib.load()
    nb = L.omprt_generic_workspace_bytes(teams, par_threads, int(heap_fallback),
                                         heap_bytes_per_team)
    ws = workspace(dev, nb)
    check(L.omprt_generic_reduce(_p(x), lb, ub, dtype_code(x.dtype), _code(_lib.OP_NAMES, op),
                                 teams, par_threads, int(ordered), pad_bytes, int(heap_fallback),
                                 heap_bytes_per_team, _p(ws), _p(out), _p(team_offsets),
                                 _stream(x)), "omprt_generic_reduce")
    return out


# -------------------------------------------------------- arena / atomics

def arena_replay(script, *, teams: int = 1, threads: int = 32, caller_tid: int = 0,
                 capacity: int = _lib.ARENA_CAPACITY, heap_fallback: bool = False,
                 heap_bytes_per_team: int = 0, check_uninit: bool = False,
                 device="cuda") -> tuple[torch.Tensor, DeviceTrap | None]:
    """Run an arena script ([(op, bytes, offset[, value]), ...], see
    omprt_arena_replay) on every team's device arena.  Returns
    (results [teams, nops] int64, trap or None)."""
    rows = [list(r) + [0] * (4 - len(r)) for r in script]
    s = torch.tensor(rows or [[0, 0, 0, 0]], dtype=torch.int64).reshape(-1, 4)[: len(rows)]
    s = s.to(device)
    dev = _dev(s)
    nops = s.shape[0]
    res = torch.zeros((teams, max(nops, 1)), dtype=torch.int64, device=dev)
    heap = None
    if heap_fallback:
        heap = torch.zeros(max(teams * heap_bytes_per_team, 16), dtype=torch.uint8, device=dev)
    st = _lib.load().omprt_arena_replay(_p(s), nops, teams, threads, caller_tid, capacity,
                                        int(heap_fallback), heap_bytes_per_team, _p(heap),
                                        int(check_uninit), _p(res), _stream(s))
    check(st, "omprt_arena_replay")
    trap = check_trap(dev) if st == _lib.TRAP else None
    return res[:, :nops], trap


def atomic_probe(kind: int, dtype, operands, desired=None, *, teams: int, threads: int,
                 init: int = 0, device="cuda") -> tuple[int, list[int]]:
    """Every thread g applies one seq_cst RMW with operands[g] to one cell.
    Returns (final cell, olds) as zero-extended words."""
    dt = dtype_code(dtype)
    n = teams * threads
    ops = torch.tensor([v & (2**64 - 1) for v in operands], dtype=torch.uint64, device=device)
    dev = _dev(ops)
    des = None
    if desired is not None:
        des = torch.tensor([v & (2**64 - 1) for v in desired], dtype=torch.uint64, device=dev)
    bits = 32 if dt in (_lib.I32, _lib.U32) else 64
    cell = torch.tensor([init & (2**bits - 1)], dtype=torch.uint32 if bits == 32 else torch.uint64,
                        device=dev)
    old = torch.zeros(n, dtype=torch.uint64, device=dev)
    check(_lib.load().omprt_atomic_probe(kind, dt, _p(ops), _p(des), _p(cell), _p(old), teams,
                                         threads, _stream(ops)), "omprt_atomic_probe")
    return int(cell.cpu().item()), [int(v) for v in old.cpu().tolist()]


def atomic_program(dtype, programs, *, teams: int, threads: int, init: int = 0,
                   device="cuda") -> tuple[int, list[list[int]]]:
    """programs[g] = [(kind, e, d), ...] for global thread g (corpus.probe_source
    shape).  Returns (final cell, olds per thread in program order)."""
    dt = dtype_code(dtype)
    n = teams * threads
    if len(programs) != n:
        raise ValueError("one program per thread is required")
    bits = 32 if dt in (_lib.I32, _lib.U32) else 64
    if any(k == _lib.ATOMIC_INC for p in programs for k, _, _ in p) and dt != _lib.U32:
        raise ValueError("atomic_inc is u32 only (runtime.mc:175-186)")
    flat = [op for p in programs for op in p]
    offs = [0]
    for p in programs:
        offs.append(offs[-1] + len(p))
    kinds = torch.tensor([k for k, _, _ in flat] or [0], dtype=torch.int32, device=device)
    dev = _dev(kinds)
    ops = torch.tensor([e & (2**64 - 1) for _, e, _ in flat] or [0], dtype=torch.uint64,
                       device=dev)
    des = torch.tensor([d & (2**64 - 1) for _, _, d in flat] or [0], dtype=torch.uint64,
                       device=dev)
    off = torch.tensor(offs, dtype=torch.int64, device=dev)
    cell = torch.tensor([init & (2**bits - 1)], dtype=torch.uint32 if bits == 32 else torch.uint64,
                        device=dev)
    old = torch.zeros(max(len(flat), 1), dtype=torch.uint64, device=dev)
    check(_lib.load().omprt_atomic_program(_p(kinds), _p(ops), _p(des), _p(off), len(flat), dt,
                                           _p(cell), _p(old), teams, threads, _stream(kinds)),
          "omprt_atomic_program")
    olds = [int(v) for v in old.cpu().tolist()]
    return int(cell.cpu().item()), [olds[offs[g]:offs[g + 1]] for g in range(n)]


def atomic_apply(kind: int, dtype, cells, operands, desired=None,
                 device="cuda") -> tuple[list[int], list[int]]:
    """Batched step semantics: returns (new cells, olds) as zero-extended words."""
    dt = dtype_code(dtype)
    bits = 32 if dt in (_lib.I32, _lib.U32) else 64
    m = 2**bits - 1
    ct = torch.tensor([v & m for v in cells], dtype=torch.uint32 if bits == 32 else torch.uint64,
                      device=device)
    dev = _dev(ct)
    ops = torch.tensor([v & (2**64 - 1) for v in operands], dtype=torch.uint64, device=dev)
    des = None
    if desired is not None:
        des = torch.tensor([v & (2**64 - 1) for v in desired], dtype=torch.uint64, device=dev)
    old = torch.zeros(len(cells), dtype=torch.uint64, device=dev)
    check(_lib.load().omprt_atomic_apply(kind, dt, _p(ct), _p(ops), _p(des), _p(old), len(cells),
                                         _stream(ct)), "omprt_atomic_apply")
    return [int(v) for v in ct.cpu().tolist()], [int(v) for v in old.cpu().tolist()]


# ------------------------------------------------------------------ data

def fill(x: torch.Tensor, seed: int, k: int = 0, offset: int = 0) -> torch.Tensor:
    """Counter-based synthetic data in place (see omprt_fill)."""
    _dev(x)
    check(_lib.load().omprt_fill(_p(x), x.numel(), dtype_code(x.dtype), seed, k, offset,
                                 _stream(x)), "omprt_fill")
    return x


def synthetic(n: int, dtype, seed: int, k: int = 0, offset: int = 0, device="cuda") -> torch.Tensor:
    x = torch.empty(n, dtype=torch_dtype(dtype_code(dtype)), device=device)
    return fill(x, seed, k, offset)
