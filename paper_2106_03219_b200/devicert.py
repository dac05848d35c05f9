"""Drop-in for forge.devicert (/root/reference/pkg/src/forge/devicert.py),
executed by the B200.

Same names, argument meaning and errors as the reference module:
  RUNTIME_API, ARENA_CAPACITY, ARENA_ALIGN, U32_MASK, mask, to_signed
                       constants and bit helpers (devicert.py:10-55)
  step_add/max/min/exchange/cas/inc
                       one seq_cst device atomic on a u32 cell per call
                       (devicert.py:84-107 -> omprt_atomic_apply)
  static_bounds        the for_static_init block rule (devicert.py:110-115),
                       run by the library's __host__ __device__ routine — the
                       same compiled code every device thread executes
  Arena / ArenaError   the team-shared bump allocator (devicert.py:124-148);
                       each alloc/free replays the arena's script on a fresh
                       device arena (shared memory of one team, like a fresh
                       vgpu launch) and raises ArenaError(code) on a trap
"""

from __future__ import annotations

import torch

from . import _lib, runtime

U32_MASK = 0xFFFFFFFF
ARENA_CAPACITY = _lib.ARENA_CAPACITY
ARENA_ALIGN = _lib.ARENA_ALIGN

#: The runtime routines the reference exports to user code
#: (devicert.RUNTIME_API, devicert.py:24-52) and what implements each here.
RUNTIME_API: dict[str, str] = {
    "omp_thread_id": "omprt::omp_thread_id (%tid.x)",
    "omp_team_id": "omprt::omp_team_id (%ctaid.x)",
    "omp_num_threads": "omprt::omp_num_threads (%ntid.x)",
    "omp_num_teams": "omprt::omp_num_teams (%nctaid.x)",
    "__kmpc_alloc_shared": "omprt::kmpc_alloc_shared (shared-memory smart stack)",
    "__kmpc_free_shared": "omprt::kmpc_free_shared",
    "__kmpc_flush": "omprt::kmpc_flush (fence.sc.gpu)",
    "__kmpc_barrier": "omprt::kmpc_barrier (bar.sync 0)",
    "atomic_add": "omprt::atomic_rmw ADD (seq_cst, gpu scope)",
    "atomic_max": "omprt::atomic_rmw MAX",
    "atomic_min": "omprt::atomic_rmw MIN",
    "atomic_exchange": "omprt::atomic_rmw XCHG",
    "atomic_cas": "omprt::atomic_rmw CAS",
    "atomic_inc": "omprt::atomic_inc_acq_rel_gpu (atom.inc.u32)",
    "for_static_init": "omprt::static_bounds / schedule_init",
}


def mask(bits: int) -> int:
    return (1 << bits) - 1


def to_signed(v: int, bits: int) -> int:
    return v - (1 << bits) if v >= (1 << (bits - 1)) else v


def _device() -> torch.device:
    return torch.device("cuda", torch.cuda.current_device())


# ---- reference semantics, on the device

Step = tuple[int, int]


def _step(kind: int, x: int, e: int, d: int | None = None) -> Step:
    new, old = runtime.atomic_apply(kind, _lib.U32, [x], [e], None if d is None else [d],
                                    device=_device())
    return new[0], old[0]


def step_add(x: int, e: int) -> Step:
    """(new, old); wraps at 32 bits (devicert.py:84-86)."""
    return _step(_lib.ATOMIC_ADD, x, e)


def step_max(x: int, e: int) -> Step:
    return _step(_lib.ATOMIC_MAX, x, e)


def step_min(x: int, e: int) -> Step:
    return _step(_lib.ATOMIC_MIN, x, e)


def step_exchange(x: int, e: int) -> Step:
    return _step(_lib.ATOMIC_XCHG, x, e)


def step_cas(x: int, e: int, d: int) -> Step:
    return _step(_lib.ATOMIC_CAS, x, e, d)


def step_inc(x: int, e: int) -> Step:
    """Wrapping increment: reset to zero once the value reaches the bound."""
    return _step(_lib.ATOMIC_INC, x, e)


def static_bounds(lb: int, ub: int, tid: int, nthreads: int) -> tuple[int, int]:
    """Block partition of inclusive [lb, ub]; a pair with my_lb > ub is empty.
    Raises ZeroDivisionError for nthreads == 0 like the reference."""
    return runtime.static_bounds(lb, ub, tid, nthreads)


class ArenaError(Exception):
    def __init__(self, code: int, message: str) -> None:
        super().__init__(message)
        self.code = code


_MESSAGES = {1: "shared arena overflow", 2: "non-LIFO shared free",
             3: "shared allocation outside thread 0"}


class Arena:
    """The team-shared bump allocator, backed by a device team's arena.

    Offsets are byte offsets into the team's shared-memory arena, 8-byte
    aligned; frees must undo the most recent live allocation.  Trap codes:
    1 overflow, 2 non-LIFO free (3 = caller not thread 0 on the device).
    """

    def __init__(self, capacity: int = ARENA_CAPACITY) -> None:
        if capacity > ARENA_CAPACITY:
            raise ValueError(f"device arena capacity is at most {ARENA_CAPACITY} bytes")
        self.capacity = capacity
        self._script: list[tuple[int, int, int]] = []
        self.cursor = 0

    def _run(self, op: tuple[int, int, int]) -> int:
        script = self._script + [op]
        # device smem arena sizes are multiples of 16; the semantic capacity
        # is enforced exactly by replaying with the requested capacity
        res, trap = runtime.arena_replay(script, teams=1, threads=32,
                                         capacity=self._phys_capacity(), device=_device())
        last = int(res[0, -1].item())
        if trap is not None or last < 0:
            code = -last if last < 0 else trap.code
            raise ArenaError(code, _MESSAGES.get(code, f"trap code {code}"))
        self._script = script
        return last

    def _phys_capacity(self) -> int:
        if self.capacity % 16:
            raise ValueError("device arena capacity must be a multiple of 16")
        return self.capacity

    def alloc(self, bytes_: int) -> int:
        off = self._run((_lib.ARENA_ALLOC, bytes_, 0))
        self.cursor = off + (bytes_ + ARENA_ALIGN - 1) // ARENA_ALIGN * ARENA_ALIGN
        return off

    def free(self, off: int, bytes_: int) -> None:
        self._run((_lib.ARENA_FREE, bytes_, off))
        self.cursor = off
