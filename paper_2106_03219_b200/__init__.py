"""B200-native data-parallel core of the OpenMP device runtime (arXiv 2106.03219).

The drop-in for the reference package `forge`'s hot path
(/root/reference/pkg/src/forge): the `target teams distribute parallel for
reduction` lowering — worksharing (for_static_init and its chunked /
distribute forms), warp-shuffle + shared-memory + last-team-finishes
reductions, the __kmpc_alloc_shared smart stack, named barriers and scoped
atomics for SPMD and generic mode — as hand-written sm_100a kernels in
libomprt_b200.so behind a C ABI (include/omprt_b200.h), with forge's entry
points on top:

  devicert        static_bounds, Arena/ArenaError, step_*  (forge.devicert)
  offload         tgt_target, TargetCall, ArgDescriptor, GridConfig,
                  TrapKind, TRAP_CODES, kernel_name        (forge.host / forge.vgpu)
  runtime         tensor-level kernels: reduce, axpy_minmax, dot,
                  generic_reduce, bounds_dump, arena_replay, atomics
  parallel        sharding over GPUs + one NCCL collective

There is no CPU fallback: without the built library every compute entry
point raises OmprtUnavailable.
"""

from __future__ import annotations

from ._lib import OmprtError, OmprtUnavailable, load
from .offload import (
    ARCHS,
    TRAP_CODES,
    ArgDescriptor,
    GridConfig,
    RegionKernel,
    TargetCall,
    TrapKind,
    axpy_minmax_host,
    dot_host,
    generic_reduce_host,
    kernel_name,
    reduce_host,
    tgt_target,
)

__version__ = "0.1.0"

__all__ = [
    "ARCHS",
    "ArgDescriptor",
    "GridConfig",
    "OmprtError",
    "OmprtUnavailable",
    "RegionKernel",
    "TRAP_CODES",
    "TargetCall",
    "TrapKind",
    "axpy_minmax_host",
    "dot_host",
    "generic_reduce_host",
    "kernel_name",
    "load",
    "reduce_host",
    "tgt_target",
    "__version__",
]
