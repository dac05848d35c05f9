"""ctypes binding of libomprt_b200.so (the C ABI in include/omprt_b200.h).

There is no CPU fallback anywhere in this package: if the shared library is
missing or cannot be loaded, importing a compute entry point raises
OmprtUnavailable.  Build it with `python -m paper_2106_03219_b200._build`
(or __graft_entry__.build()).
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from . import _build

# ---- enums (mirror include/omprt_b200.h)
I32, U32, I64, U64, F32, F64 = range(6)
OP_ADD, OP_MAX, OP_MIN = range(3)
SCHED_STATIC, SCHED_STATIC_CHUNKED, SCHED_DISTRIBUTE, SCHED_DISTRIBUTE_CHUNKED = range(4)
MODE_SPMD, MODE_ORDERED = range(2)
ATOMIC_ADD, ATOMIC_MAX, ATOMIC_MIN, ATOMIC_XCHG, ATOMIC_CAS, ATOMIC_INC = range(6)
ARENA_ALLOC, ARENA_FREE, ARENA_WRITE, ARENA_READ = range(4)
OK, FALLBACK, TRAP = 0, 1, 2
EINVAL, ECUDA, ENOMEM, EUNAVAILABLE = -1, -2, -3, -4
ARENA_CAPACITY = 65536
ARENA_ALIGN = 8

DTYPE_NAMES = {"i32": I32, "u32": U32, "i64": I64, "u64": U64, "f32": F32, "f64": F64}
OP_NAMES = {"add": OP_ADD, "sum": OP_ADD, "+": OP_ADD, "max": OP_MAX, "min": OP_MIN}
SCHED_NAMES = {
    "static": SCHED_STATIC,
    "static_chunked": SCHED_STATIC_CHUNKED,
    "distribute": SCHED_DISTRIBUTE,
    "distribute_chunked": SCHED_DISTRIBUTE_CHUNKED,
}
MODE_NAMES = {"spmd": MODE_SPMD, "ordered": MODE_ORDERED}


class OmprtUnavailable(RuntimeError):
    """The native library is not built or not loadable: no fallback exists."""


class OmprtError(RuntimeError):
    def __init__(self, status: int, message: str) -> None:
        super().__init__(f"omprt status {status}: {message}")
        self.status = status


_lock = threading.Lock()
_lib = None
_inited_devices: set[int] = set()

_SIGS = {
    "omprt_version": ([], C.c_char_p),
    "omprt_last_error": ([], C.c_char_p),
    "omprt_device_init": ([C.c_int], C.c_int),
    "omprt_set_unroll": ([C.c_int], C.c_int),
    "omprt_set_variant": ([C.c_int], C.c_int),
    "omprt_set_spmd_block": ([C.c_int], C.c_int),
    "omprt_set_trace": ([C.c_void_p, C.c_int64], C.c_int),
    "omprt_ipc_handle_bytes": ([], C.c_size_t),
    "omprt_mailbox_create": ([C.c_int, C.POINTER(C.c_void_p), C.c_void_p], C.c_int),
    "omprt_mailbox_open": ([C.c_void_p, C.POINTER(C.c_void_p)], C.c_int),
    "omprt_mailbox_close": ([C.c_void_p], C.c_int),
    "omprt_mailbox_destroy": ([C.c_void_p], C.c_int),
    "omprt_reduce_exchange": ([C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                               C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                               C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_void_p], C.c_int),
    "omprt_allreduce": ([C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, C.c_void_p],
                        C.c_int),
    "omprt_num_sms": ([], C.c_int),
    "omprt_check_trap": ([C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                          C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
    "omprt_static_bounds": ([C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                             C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
    "omprt_bounds_dump": ([C.c_int64, C.c_int64, C.c_int, C.c_int64, C.c_int, C.c_int,
                           C.c_void_p, C.c_void_p], C.c_int),
    "omprt_reduce_workspace_bytes": ([C.c_int, C.c_int, C.c_int], C.c_size_t),
    "omprt_reduce": ([C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int64,
                      C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "omprt_axpy_minmax": ([C.c_float, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int,
                           C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                           C.c_void_p, C.c_void_p], C.c_int),
    "omprt_dot": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int64, C.c_int,
                   C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "omprt_combine_partials": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p],
                               C.c_int),
    "omprt_generic_workspace_bytes": ([C.c_int, C.c_int, C.c_int, C.c_int64], C.c_size_t),
    "omprt_generic_reduce": ([C.c_void_p, C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_int,
                              C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int64, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "omprt_arena_replay": ([C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int,
                            C.c_int64, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "omprt_atomic_probe": ([C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                            C.c_int, C.c_int, C.c_void_p], C.c_int),
    "omprt_atomic_program": ([C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                              C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p],
                             C.c_int),
    "omprt_atomic_apply": ([C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                            C.c_int64, C.c_void_p], C.c_int),
    "omprt_fill": ([C.c_void_p, C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_int64, C.c_void_p],
                   C.c_int),
    "omprt_reduce_host": ([C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_int,
                           C.c_int, C.c_int, C.c_void_p], C.c_int),
    "omprt_axpy_minmax_host": ([C.c_float, C.c_void_p, C.c_void_p, C.c_int64, C.c_int,
                                C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p],
                               C.c_int),
    "omprt_dot_host": ([C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int64, C.c_int, C.c_int,
                        C.c_int, C.c_void_p], C.c_int),
    "omprt_generic_reduce_host": ([C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                   C.c_int, C.c_int64, C.c_int, C.c_int64, C.c_void_p,
                                   C.c_void_p], C.c_int),
    "omprt_release_host_cache": ([], C.c_int),
    "omprt_image_load": ([C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)], C.c_int),
    "omprt_image_unload": ([C.c_void_p], C.c_int),
    "omprt_image_launch": ([C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.c_size_t, C.c_void_p,
                            C.c_size_t, C.c_void_p], C.c_int),
}

EXPORTED = tuple(_SIGS)


def lib_path() -> Path:
    return Path(os.environ.get("OMPRT_B200_LIB", _build.LIB))


def load(build_if_missing: bool = False):
    """Load (and bind) the shared library; never falls back to Python."""
    global _lib
    if _lib is not None:  # bound once; the lock only guards the first load
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = lib_path()
        if not path.exists() and build_if_missing:
            _build.build()
        if not path.exists():
            raise OmprtUnavailable(
                f"{path} is not built; run `python -m paper_2106_03219_b200._build` "
                "(there is no CPU fallback)")
        try:
            L = C.CDLL(str(path))
        except OSError as err:
            raise OmprtUnavailable(f"cannot load {path}: {err}") from err
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return L


def last_error() -> str:
    return load().omprt_last_error().decode()


def check(status: int, what: str = "") -> int:
    if status < 0:
        raise OmprtError(status, f"{what}: {last_error()}")
    return status


def ensure_device(device_index: int) -> None:
    """Bind the library to the CUDA device (clears its trap word once)."""
    if device_index in _inited_devices:
        return
    check(load().omprt_device_init(device_index), "omprt_device_init")
    _inited_devices.add(device_index)
