"""The launch boundary: a B200 `tgt_target` with forge's calling convention.

Mirrors /root/reference/pkg/src/forge/host.py:91-130 (ArgDescriptor,
TargetCall), :255-296 (tgt_target) and vgpu.py:28-61 (TrapKind, TRAP_CODES,
GridConfig).  Where the reference interprets a vgpu IR image, the B200 image
is a table from kernel id (`__omp_offload_<region_id>`, codegen.py:59-63) to
a RegionKernel naming the hand-written construct kernel that implements the
region and which captured argument plays which role — or a compiled image
(`regionc.B200Image`, the region's own IR translated to sm_100a), in which
case every OpenMP thread runs the region literally (regions.launch).

Status codes are the reference's: 0 ran on the device (buffers hold the
results), 1 could not launch (force_fail, foreign arch, no image for the
kernel id — the reference's caller would then run its host fallback; this
package has none), 2 device trap (out["trap"] = (TrapKind.value, detail),
caller buffers untouched).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace
from enum import Enum

import numpy as np
import torch

from . import _lib, regionc, regions, runtime

#: Arch names this device answers to: its own, and the reference's NVIDIA
#: target whose intrinsic table (selectors.py:84-93) it implements.
ARCHS = ("b200", "nvptx64")


class TrapKind(Enum):
    SHARED_OVERFLOW = "SharedOverflow"
    NON_LIFO_FREE = "NonLIFOFree"
    NON_UNIFORM_ALLOC = "NonUniformAlloc"
    UNINITIALIZED_READ = "UninitializedRead"
    OUT_OF_BOUNDS = "OutOfBounds"
    DEADLOCK = "Deadlock"
    DIVIDE_BY_ZERO = "DivideByZero"
    ABORT = "Abort"


TRAP_CODES = {
    1: TrapKind.SHARED_OVERFLOW,
    2: TrapKind.NON_LIFO_FREE,
    3: TrapKind.NON_UNIFORM_ALLOC,
}

#: omprt_trap_kind -> TrapKind (include/omprt_b200.h)
KIND_OF = {1: TrapKind.SHARED_OVERFLOW, 2: TrapKind.NON_LIFO_FREE,
           3: TrapKind.NON_UNIFORM_ALLOC, 4: TrapKind.UNINITIALIZED_READ,
           5: TrapKind.OUT_OF_BOUNDS, 6: TrapKind.DEADLOCK, 7: TrapKind.DIVIDE_BY_ZERO,
           8: TrapKind.ABORT}


@dataclass
class GridConfig:
    """num_teams x threads_per_team, each 1..1024 (vgpu.py:50-61)."""

    num_teams: int = 1
    threads_per_team: int = 1
    sched_seed: int = 0

    def __post_init__(self) -> None:
        if not (1 <= self.num_teams <= 1024):
            raise ValueError("num_teams must lie in 1..1024")
        if not (1 <= self.threads_per_team <= 1024):
            raise ValueError("threads_per_team must lie in 1..1024")
        self.sched_seed &= (1 << 64) - 1


ELEM_BITS = {"i32": 32, "u32": 32, "i64": 64, "u64": 64, "f32": 32, "f64": 64}
NP_ELEM = {"i32": np.int32, "u32": np.uint32, "i64": np.int64, "u64": np.uint64,
           "f32": np.float32, "f64": np.float64}


@dataclass(frozen=True)
class ArgDescriptor:
    """One kernel argument: a named buffer or a scalar (host.py:91-104)."""

    name: str
    kind: str  # "buffer" | "scalar"
    elem: str  # "i32" | "u32" | "i64" | "u64" | "f32" | "f64"
    count: int | None = None

    @property
    def size(self) -> int | None:
        return None if self.count is None else self.count * ELEM_BITS[self.elem] // 8


def kernel_name(region_id: int) -> str:
    """Kernel naming convention of the offload bundle (codegen.py:59-63)."""
    return f"__omp_offload_{region_id}"


@dataclass(frozen=True)
class TargetCall:
    """One offload site (host.py:107-130).  `fallback` is carried for
    signature compatibility; this package never calls it."""

    region_id: int
    kernel_id: str
    args: tuple[ArgDescriptor, ...]
    fallback: object = None
    grid: tuple[int | None, int | None] = (None, None)
    values: tuple | None = None

    def bind(self, values) -> "TargetCall":
        vals = tuple(values)
        if len(vals) != len(self.args):
            raise ValueError(f"kernel {self.kernel_id} takes {len(self.args)} arguments, "
                             f"got {len(vals)}")
        return replace(self, values=vals)


@dataclass(frozen=True)
class RegionKernel:
    """What a region lowers to on the B200.

    construct   "reduce" | "axpy_minmax" | "dot" | "generic_reduce" | "bounds"
    roles       role -> captured argument name:
                  reduce          x (buffer), cell (buffer), n (scalar trip count)
                  axpy_minmax     a (scalar f32), x, y, max, min (buffers), n
                  dot             x, y, cell (buffers), n
                  generic_reduce  x, cell, offs (optional buffer), n
                  bounds          out (buffer int64 [threads*4]), lb, ub (scalars)
    lb          first iteration; the last is roles["n"] - 1 + lb
    """

    construct: str
    roles: dict = field(default_factory=dict)
    op: str = "add"
    sched: str = "static"
    chunk: int = 1
    mode: str = "spmd"
    lb: int = 0
    par_threads: int = 256
    pad_bytes: int = 0
    heap_fallback: bool = False


# ---------------------------------------------------------------- marshalling

def _host_array(desc: ArgDescriptor, v) -> np.ndarray:
    """A numpy view of a buffer argument (bytes / bytearray / ndarray / CPU tensor)."""
    dt = NP_ELEM[desc.elem]
    if isinstance(v, (bytes, bytearray, memoryview)):
        return np.frombuffer(v, dtype=dt)
    if isinstance(v, np.ndarray):
        return v.view(dt) if v.dtype != dt else v
    if isinstance(v, torch.Tensor):
        if v.is_cuda:
            raise TypeError(f"buffer '{desc.name}' is already on a device; pass host memory")
        return v.numpy().view(dt)
    raise TypeError(f"buffer argument '{desc.name}' needs bytes, a numpy array or a CPU tensor")


def _write_back(desc: ArgDescriptor, v, dev: torch.Tensor) -> None:
    host = dev.cpu().numpy()
    if isinstance(v, bytearray):
        v[:] = host.tobytes()
    elif isinstance(v, np.ndarray):
        v[...] = host.view(v.dtype).reshape(v.shape)
    elif isinstance(v, torch.Tensor):
        v.copy_(torch.from_numpy(host).view(v.dtype).reshape(v.shape))
    # bytes are immutable: nothing to write back (like the reference's _pack_arg copy)


def _scalar(desc: ArgDescriptor, v):
    if desc.elem in ("f32", "f64"):
        return float(v)
    m = (1 << ELEM_BITS[desc.elem]) - 1
    x = int(v) & m
    if desc.elem in ("i32", "i64") and x >> (ELEM_BITS[desc.elem] - 1):
        x -= 1 << ELEM_BITS[desc.elem]
    return x


def _image_for(bundle, arch: str):
    if bundle is None:
        return None
    if isinstance(bundle, dict):
        img = bundle.get(arch)
        if img is None and arch in ARCHS:
            for a in ARCHS:
                img = img or bundle.get(a)
        return img
    return None


def _trap_status(trap, out) -> int:
    kind = KIND_OF.get(trap.kind, TrapKind.ABORT)
    if out is not None:
        out["trap"] = (kind.value,
                       f"device trap code {trap.code} (team {trap.team} thread {trap.thread})")
    return 2


def tgt_target(call: TargetCall, bundle, device="b200", force_fail: bool = False, *,
               grid: tuple[int, int] | None = None, sched_seed: int = 0,
               check_uninit: bool = False, collect_trace: bool = False,
               out: dict | None = None) -> int:
    """Dispatch one offload: 0 ran on the device, 1 launch failed, 2 trapped.

    bundle: {"b200": {kernel_id: RegionKernel}}.  On 0 the buffer arguments
    hold the device results; on nonzero status they are untouched.
    sched_seed / check_uninit are accepted for signature compatibility: a
    construct kernel's result does not depend on the interleaving (its
    combine is the ticketed team-order fold).  Compiled regions
    (forge_bridge, regions.launch) honour both: sched_seed jitters every
    thread before its atomics and barriers (rt_jitter).  collect_trace=True
    records the construct's per-team device trace (runtime.Trace) into
    out["trace"] — team start/SM, the ticket each team's atom.inc took, the
    ordered combine — in the vgpu's "seq team thread kind detail" format.
    """
    if call.values is None:
        raise ValueError("TargetCall is not bound to argument values")
    arch = str(getattr(device, "arch", device))
    if force_fail or arch not in ARCHS:
        return 1
    image = _image_for(bundle, arch)
    if isinstance(image, (bytes, bytearray)) and bytes(image[:8]) == regionc.IMAGE_MAGIC:
        image = regionc.B200Image.from_bytes(image)
    if isinstance(image, regionc.B200Image):
        return _launch_compiled(image, call, grid, check_uninit, out)
    if image is None or call.kernel_id not in image:
        return 1
    rk: RegionKernel = image[call.kernel_id]
    teams, threads = grid if grid is not None else (call.grid[0] or 1, call.grid[1] or 1)
    GridConfig(teams, threads, sched_seed)  # same validation as the reference

    by_name = {d.name: (d, v) for d, v in zip(call.args, call.values)}
    dev = torch.device("cuda", torch.cuda.current_device())
    _lib.ensure_device(dev.index)

    # copy-in (host.py:276-281)
    dbufs: dict[str, torch.Tensor] = {}
    scal: dict[str, object] = {}
    for name, (d, v) in by_name.items():
        if d.kind == "scalar":
            scal[name] = _scalar(d, v)
        else:
            arr = np.ascontiguousarray(_host_array(d, v))
            dbufs[name] = torch.from_numpy(arr.copy()).to(dev, non_blocking=False)

    r = rk.roles
    c = rk.construct
    st = torch.cuda.current_stream(dev)
    tracer = runtime.Trace(dev) if (collect_trace and c != "bounds") else None
    if tracer is not None:
        tracer.__enter__()
    try:
        _launch_construct(rk, c, r, scal, dbufs, teams, threads, dev)
    except IndexError as err:
        # the loop would index a buffer outside its extent: the vgpu traps
        # OutOfBounds on that access (vgpu.py:28-36) -> status 2, the
        # caller's buffers untouched, nothing launched
        if out is not None:
            out["result"] = {"construct": c, "teams": teams, "threads": threads}
            out["trace"] = []
            out["trap"] = (TrapKind.OUT_OF_BOUNDS.value, str(err))
        return 2
    finally:
        if tracer is not None:
            tracer.__exit__(None, None, None)

    trap = runtime.check_trap(dev)  # synchronises the stream
    st.synchronize()
    if out is not None:
        out["result"] = {"construct": c, "teams": teams, "threads": threads}
        out["trace"] = tracer.lines() if tracer is not None else []
    if trap is not None:
        return _trap_status(trap, out)
    # copy-out only on status 0 (host.py:293-295)
    for name, (d, v) in by_name.items():
        if d.kind == "buffer":
            _write_back(d, v, dbufs[name])
    return 0


def _launch_construct(rk: RegionKernel, c: str, r: dict, scal: dict, dbufs: dict, teams: int,
                      threads: int, dev: torch.device) -> None:
    if c == "reduce":
        n = int(scal[r["n"]])
        runtime.reduce(dbufs[r["x"]], rk.op, lb=rk.lb, ub=rk.lb + n - 1, sched=rk.sched,
                       chunk=rk.chunk, teams=teams, threads=threads, mode=rk.mode,
                       out=dbufs[r["cell"]])
    elif c == "dot":
        n = int(scal[r["n"]])
        runtime.dot(dbufs[r["x"]], dbufs[r["y"]], lb=rk.lb, ub=rk.lb + n - 1, sched=rk.sched,
                    chunk=rk.chunk, teams=teams, threads=threads, mode=rk.mode,
                    out=dbufs[r["cell"]])
    elif c == "axpy_minmax":
        n = int(scal[r["n"]])
        runtime.axpy_minmax(float(scal[r["a"]]), dbufs[r["x"]], dbufs[r["y"]], lb=rk.lb,
                            ub=rk.lb + n - 1, sched=rk.sched, chunk=rk.chunk, teams=teams,
                            threads=threads, mode=rk.mode, out_max=dbufs[r["max"]],
                            out_min=dbufs[r["min"]])
    elif c == "generic_reduce":
        n = int(scal[r["n"]])
        offs = dbufs.get(r.get("offs", ""), None)
        runtime.generic_reduce(dbufs[r["x"]], rk.op, lb=rk.lb, ub=rk.lb + n - 1, teams=teams,
                               par_threads=rk.par_threads, ordered=rk.mode == "ordered",
                               pad_bytes=rk.pad_bytes, heap_fallback=rk.heap_fallback,
                               out=dbufs[r["cell"]], team_offsets=offs)
    elif c == "bounds":
        lb, ub = int(scal[r["lb"]]), int(scal[r["ub"]])
        res = runtime.bounds_dump(lb, ub, rk.sched, rk.chunk, teams=teams, threads=threads,
                                  device=dev)
        dbufs[r["out"]].copy_(res.reshape(-1)[: dbufs[r["out"]].numel()])
    else:
        raise ValueError(f"unknown construct '{c}'")


def _launch_compiled(image, call: TargetCall, grid, check_uninit: bool, out) -> int:
    """A compiled region (regionc.B200Image, from the reference's IR image):
    every OpenMP thread runs the region literally on the B200 (regions.launch)."""
    if call.kernel_id not in image.kernels:
        return 1
    teams, threads = grid if grid is not None else (call.grid[0] or 1, call.grid[1] or 1)
    packed = []
    for d, v in zip(call.args, call.values):
        if d.kind == "scalar":
            packed.append(int(v) & ((1 << ELEM_BITS[d.elem]) - 1))
        else:
            packed.append(bytearray(np.ascontiguousarray(_host_array(d, v)).tobytes()))
    res = regions.launch(image, call.kernel_id, (teams, threads), packed,
                         check_uninit=check_uninit)
    if out is not None:
        out["result"] = res
    if res.status == "trap":
        if out is not None:
            out["trap"] = (res.trap, res.trap_detail)
        return 2
    for d, v, raw in zip(call.args, call.values, res.buffers):
        if d.kind == "buffer":
            _write_back(d, v, torch.frombuffer(bytearray(raw), dtype=torch.uint8))
    return 0


# ------------------------------------------------------- host-buffer fast path

def reduce_host(x: np.ndarray | torch.Tensor, cell, *, op="add", sched="static", chunk: int = 1,
                teams: int, threads: int, mode="spmd") -> None:
    """The C-ABI host-buffer entry (omprt_reduce_host): copy-in of x (pinned
    or pageable host memory), device reduction, copy-out of the cell.  `cell`
    is a 1-element host array/tensor holding the initial value; updated in place."""
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            raise TypeError("reduce_host takes host memory")
        xp, n, dt = x.data_ptr(), x.numel(), runtime.dtype_code(x.dtype)
    else:
        xp, n = x.ctypes.data, x.size
        dt = runtime.dtype_code(torch.from_numpy(x[:0]).dtype)
    cp = cell.data_ptr() if isinstance(cell, torch.Tensor) else cell.ctypes.data
    _lib.ensure_device(torch.cuda.current_device())
    _lib.check(_lib.load().omprt_reduce_host(
        C.c_void_p(xp), n, dt, _lib.OP_NAMES[op] if isinstance(op, str) else op,
        _lib.SCHED_NAMES[sched] if isinstance(sched, str) else sched, chunk, teams, threads,
        _lib.MODE_NAMES[mode] if isinstance(mode, str) else mode, C.c_void_p(cp)),
        "omprt_reduce_host")


def _host_ptr(a, what: str):
    """(address, numel, dtype code) of a host array / CPU tensor."""
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            raise TypeError(f"{what} takes host memory")
        if not a.is_contiguous():
            raise ValueError(f"{what}: host tensors must be contiguous")
        return a.data_ptr(), a.numel(), runtime.dtype_code(a.dtype)
    a = np.asarray(a)
    if not a.flags.c_contiguous:
        raise ValueError(f"{what}: host arrays must be contiguous")
    return a.ctypes.data, a.size, runtime.dtype_code(torch.from_numpy(a[:0]).dtype)


def _code(table: dict, v) -> int:
    return table[v] if isinstance(v, str) else v


def axpy_minmax_host(a: float, x, y, cells, *, sched="distribute_chunked", chunk: int = 1,
                     teams: int, threads: int, mode="spmd") -> None:
    """omprt_axpy_minmax_host: copy-in of x and y, the fused axpy + max/min
    construct, copy-out of y and cells = [max, min] (host fp32 arrays holding
    the initial values) — only on status 0 (host.py:293-295)."""
    xp, n, dx = _host_ptr(x, "axpy_minmax_host")
    yp, ny, dy = _host_ptr(y, "axpy_minmax_host")
    cp, nc, dc = _host_ptr(cells, "axpy_minmax_host")
    if (dx, dy, dc) != (_lib.F32,) * 3 or ny < n or nc < 2:
        raise TypeError("axpy_minmax_host takes fp32 x, y (len(y) >= len(x)) and 2 cells")
    _lib.ensure_device(torch.cuda.current_device())
    f = C.POINTER(C.c_float)
    _lib.check(_lib.load().omprt_axpy_minmax_host(
        C.c_float(a), C.c_void_p(xp), C.c_void_p(yp), n, _code(_lib.SCHED_NAMES, sched), chunk,
        teams, threads, _code(_lib.MODE_NAMES, mode), C.cast(C.c_void_p(cp), f),
        C.cast(C.c_void_p(cp + 4), f)), "omprt_axpy_minmax_host")


def dot_host(x, y, cell, *, sched="static", chunk: int = 1, teams: int, threads: int,
             mode="spmd") -> None:
    """omprt_dot_host: copy-in of x and y, the fp64 dot construct, copy-out of
    the cell (a 1-element host fp64 array holding the initial value)."""
    xp, n, dx = _host_ptr(x, "dot_host")
    yp, ny, dy = _host_ptr(y, "dot_host")
    cp, _, dc = _host_ptr(cell, "dot_host")
    if (dx, dy, dc) != (_lib.F64,) * 3 or ny < n:
        raise TypeError("dot_host takes fp64 x, y (len(y) >= len(x)) and an fp64 cell")
    _lib.ensure_device(torch.cuda.current_device())
    _lib.check(_lib.load().omprt_dot_host(
        C.c_void_p(xp), C.c_void_p(yp), n, _code(_lib.SCHED_NAMES, sched), chunk, teams, threads,
        _code(_lib.MODE_NAMES, mode), C.c_void_p(cp)), "omprt_dot_host")


def generic_reduce_host(x, cell, *, op="add", teams: int = 1024, par_threads: int = 256,
                        ordered: bool = False, pad_bytes: int = 0, heap_fallback: bool = False,
                        heap_bytes_per_team: int = 1 << 20, team_offsets=None,
                        out: dict | None = None) -> int:
    """omprt_generic_reduce_host, with tgt_target's status: 0 ran (cell and
    team_offsets updated), 2 device trap (out["trap"] = (TrapKind.value,
    detail), host buffers untouched)."""
    xp, n, dt = _host_ptr(x, "generic_reduce_host")
    cp, _, dc = _host_ptr(cell, "generic_reduce_host")
    if dc != dt:
        raise TypeError("cell and x must have one element type")
    op_ = None
    if team_offsets is not None:
        op_, no, do = _host_ptr(team_offsets, "generic_reduce_host")
        if do != _lib.I64 or no < teams:
            raise TypeError("team_offsets must be an int64 array of >= teams entries")
    dev = torch.device("cuda", torch.cuda.current_device())
    _lib.ensure_device(dev.index)
    st = _lib.check(_lib.load().omprt_generic_reduce_host(
        C.c_void_p(xp), n, dt, _code(_lib.OP_NAMES, op), teams, par_threads, int(ordered),
        pad_bytes, int(heap_fallback), heap_bytes_per_team, C.c_void_p(cp),
        C.c_void_p(op_ or 0)), "omprt_generic_reduce_host")
    if st == _lib.TRAP:
        trap = runtime.check_trap(dev)
        if trap is not None:
            return _trap_status(trap, out)
        return 2
    return st
