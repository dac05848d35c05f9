"""TEST INFRASTRUCTURE ONLY — the CPU parity oracle.

ctypes front end of omprt_oracle.c (the C restatement of the reference's
semantics) plus pure-Python restatements for small cases.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / --impl reference leg
may import this module; the product package never does.

Pinned against the reference itself: tests/test_oracle.py replays the golden
vectors in tests/golden/ (made by oracle/gen_golden.py from
/root/reference/pkg/src/forge) through every function here.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liboracle.so"

SEED = 0x210603219

I32, U32, I64, U64, F32, F64 = range(6)
ADD, MAX, MIN = range(3)
STATIC, STATIC_CHUNKED, DISTRIBUTE, DISTRIBUTE_CHUNKED = range(4)
A_ADD, A_MAX, A_MIN, A_XCHG, A_CAS, A_INC = range(6)

NP_DTYPE = {I32: np.int32, U32: np.uint32, I64: np.int64, U64: np.uint64,
            F32: np.float32, F64: np.float64}
C_DTYPE = {I32: C.c_int32, U32: C.c_uint32, I64: C.c_int64, U64: C.c_uint64,
           F32: C.c_float, F64: C.c_double}

_lib = None


def build() -> Path:
    """Compile the restatement (make in oracle/); cheap when up to date."""
    src = HERE / "omprt_oracle.c"
    if LIB_PATH.exists() and LIB_PATH.stat().st_mtime >= src.stat().st_mtime:
        return LIB_PATH
    res = subprocess.run(["make", "-C", str(HERE)], capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{res.stdout}\n{res.stderr}")
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB_PATH))
        i64, u64, vp = C.c_int64, C.c_uint64, C.c_void_p
        L.oracle_static_bounds.argtypes = [i64, i64, i64, i64, C.POINTER(i64), C.POINTER(i64)]
        L.oracle_bounds_dump.argtypes = [i64, i64, C.c_int, i64, i64, i64, vp]
        L.oracle_bounds_dump.restype = None
        L.oracle_fill.argtypes = [vp, i64, C.c_int, u64, C.c_int, i64]
        L.oracle_fill.restype = None
        L.oracle_reduce.argtypes = [vp, i64, i64, C.c_int, C.c_int, C.c_int, i64, i64, i64, vp]
        L.oracle_reduce_gen.argtypes = [u64, C.c_int, i64, i64, C.c_int, C.c_int, C.c_int, i64,
                                        i64, i64, vp]
        L.oracle_reduce_gen_flat.argtypes = [u64, C.c_int, i64, i64, C.c_int, C.c_int, vp]
        L.oracle_exact_sum_gen.argtypes = [u64, C.c_int, i64, i64, C.c_int]
        L.oracle_exact_sum_gen.restype = C.c_double
        L.oracle_accurate_sum_f64.argtypes = [vp, i64]
        L.oracle_accurate_sum_f64.restype = C.c_double
        L.oracle_axpy_minmax.argtypes = [C.c_float, vp, vp, i64, i64, C.c_int, i64, i64, i64,
                                         C.POINTER(C.c_float), C.POINTER(C.c_float)]
        L.oracle_dot.argtypes = [vp, vp, u64, i64, i64, C.c_int, i64, i64, i64,
                                 C.POINTER(C.c_double)]
        L.oracle_accurate_dot_gen.argtypes = [u64, i64, i64]
        L.oracle_accurate_dot_gen.restype = C.c_double
        L.oracle_exact_dot_gen.argtypes = [u64, i64, i64]
        L.oracle_exact_dot_gen.restype = C.c_double
        L.oracle_generic_reduce.argtypes = [vp, u64, C.c_int, i64, i64, C.c_int, C.c_int, i64,
                                            i64, vp]
        L.oracle_arena_replay.argtypes = [vp, C.c_int, C.c_int, i64, C.c_int, i64, C.c_int, vp]
        L.oracle_atomic_step.argtypes = [C.c_int, C.c_int, u64, u64, u64, C.POINTER(u64),
                                         C.POINTER(u64)]
        L.oracle_set_threads.argtypes = [C.c_int]
        L.oracle_set_threads.restype = None
        _lib = L
    return _lib


def _ptr(a: np.ndarray | None):
    return None if a is None else C.c_void_p(a.ctypes.data)


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_threads(n: int) -> None:
    lib().oracle_set_threads(n)


# ---- worksharing

def static_bounds(lb: int, ub: int, tid: int, n: int) -> tuple[int, int]:
    """devicert.static_bounds (devicert.py:110-115); ZeroDivisionError for n == 0
    like the Python reference."""
    a, b = C.c_int64(), C.c_int64()
    if lib().oracle_static_bounds(lb, ub, tid, n, C.byref(a), C.byref(b)) != 0:
        raise ZeroDivisionError("integer division or modulo by zero")
    return a.value, b.value


def bounds_dump(lb: int, ub: int, sched: int, chunk: int, teams: int, threads: int) -> np.ndarray:
    out = np.empty((teams * threads, 4), dtype=np.int64)
    lib().oracle_bounds_dump(lb, ub, sched, chunk, teams, threads, _ptr(out))
    return out


# ---- data

def fill(n: int, dtype: int, seed: int = SEED, k: int = 0, offset: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=NP_DTYPE[dtype])
    lib().oracle_fill(_ptr(out), n, dtype, seed, k, offset)
    return out


# ---- reductions (reference order)

def reduce(x: np.ndarray | None, lb: int, ub: int, dtype: int, op: int, sched: int, chunk: int,
           teams: int, threads: int, init=0, *, seed: int = SEED, k: int = 0):
    """Reference-order reduction (host.py:567-582).  x None: generated data."""
    cell = np.array([init], dtype=NP_DTYPE[dtype])
    if x is None:
        rc = lib().oracle_reduce_gen(seed, k, lb, ub, dtype, op, sched, chunk, teams, threads,
                                     _ptr(cell))
    else:
        assert x.dtype == NP_DTYPE[dtype]
        rc = lib().oracle_reduce(_ptr(x), lb, ub, dtype, op, sched, chunk, teams, threads,
                                 _ptr(cell))
    if rc != 0:
        raise ValueError("oracle_reduce: bad arguments")
    return cell[0]


def reduce_flat_gen(lb: int, ub: int, dtype: int, op: int, init=0, *, seed: int = SEED,
                    k: int = 0):
    cell = np.array([init], dtype=NP_DTYPE[dtype])
    lib().oracle_reduce_gen_flat(seed, k, lb, ub, dtype, op, _ptr(cell))
    return cell[0]


def exact_sum_gen(lb: int, ub: int, dtype: int, *, seed: int = SEED, k: int = 0) -> float:
    return lib().oracle_exact_sum_gen(seed, k, lb, ub, dtype)


def accurate_sum_f64(x: np.ndarray) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    return lib().oracle_accurate_sum_f64(_ptr(x), x.size)


def axpy_minmax(a: float, x: np.ndarray, y: np.ndarray, lb: int, ub: int, sched: int, chunk: int,
                teams: int, threads: int, mx: float, mn: float):
    """Updates y in place; returns (max, min) in reference order."""
    cmx, cmn = C.c_float(mx), C.c_float(mn)
    rc = lib().oracle_axpy_minmax(a, _ptr(x), _ptr(y), lb, ub, sched, chunk, teams, threads,
                                  C.byref(cmx), C.byref(cmn))
    if rc:
        raise ValueError("oracle_axpy_minmax: bad arguments")
    return cmx.value, cmn.value


def dot(x, y, lb: int, ub: int, sched: int, chunk: int, teams: int, threads: int,
        init: float = 0.0, *, seed: int = SEED) -> float:
    cell = C.c_double(init)
    rc = lib().oracle_dot(_ptr(x), _ptr(y), seed, lb, ub, sched, chunk, teams, threads,
                          C.byref(cell))
    if rc:
        raise ValueError("oracle_dot: bad arguments")
    return cell.value


def accurate_dot_gen(lb: int, ub: int, *, seed: int = SEED) -> float:
    return lib().oracle_accurate_dot_gen(seed, lb, ub)


def exact_dot_gen(lb: int, ub: int, *, seed: int = SEED) -> float:
    """The generated dot accumulated exactly in 128-bit integer halves."""
    return lib().oracle_exact_dot_gen(seed, lb, ub)


def generic_reduce(x, lb: int, ub: int, dtype: int, op: int, teams: int, P: int, init=0, *,
                   seed: int = SEED, k: int = 0):
    cell = np.array([init], dtype=NP_DTYPE[dtype])
    rc = lib().oracle_generic_reduce(_ptr(x), seed, k, lb, ub, dtype, op, teams, P, _ptr(cell))
    if rc:
        raise ValueError("oracle_generic_reduce: bad arguments")
    return cell[0]


# ---- arena / atomics

def arena_replay(script, caller_tid: int = 0, capacity: int = 65536, heap_fallback: bool = False,
                 heap_cap: int = 0, check_uninit: bool = False) -> tuple[list[int], int]:
    """script rows: (op, bytes, offset[, value]); ops 0 alloc 1 free 2 write 3 read."""
    rows = [list(r) + [0] * (4 - len(r)) for r in script]
    s = np.ascontiguousarray(np.asarray(rows, dtype=np.int64).reshape(-1, 4))
    res = np.zeros(max(len(s), 1), dtype=np.int64)
    code = lib().oracle_arena_replay(_ptr(s), len(s), caller_tid, capacity, int(heap_fallback),
                                     heap_cap, int(check_uninit), _ptr(res))
    return [int(v) for v in res[:len(s)]], int(code)


def atomic_step(kind: int, dtype: int, x: int, e: int, d: int = 0) -> tuple[int, int]:
    """Returns (new, old) as zero-extended words."""
    nv, old = C.c_uint64(), C.c_uint64()
    rc = lib().oracle_atomic_step(kind, dtype, x & (2**64 - 1), e & (2**64 - 1), d & (2**64 - 1),
                                  C.byref(nv), C.byref(old))
    if rc:
        raise ValueError("atomic_step: bad kind/dtype")
    return nv.value, old.value


# ---- pure-Python restatements (small cases; used to cross-check the C code)

M64 = (1 << 64) - 1


def py_splitmix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def _signed(v: int, bits: int) -> int:
    return v - (1 << bits) if v >= (1 << (bits - 1)) else v


def py_gen(dtype: int, i: int, seed: int = SEED, k: int = 0):
    h = py_splitmix64(seed ^ (k << 56) ^ i)
    if dtype == I64:
        return _signed(h, 64) >> 24
    if dtype == U64:
        return h >> 24
    if dtype == I32:
        return _signed(h >> 32, 32) >> 8
    if dtype == U32:
        return h >> 40
    if dtype == F64:
        return (h >> 11) * 2.0 ** -53
    return float(np.float32((h >> 40) * 2.0 ** -24))


def py_static_bounds(lb: int, ub: int, tid: int, n: int) -> tuple[int, int]:
    chunk = (ub - lb + 1 + n - 1) // n
    my_lb = lb + tid * chunk
    return my_lb, min(my_lb + chunk - 1, ub)
