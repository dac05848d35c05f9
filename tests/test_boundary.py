"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/omprt_b200.h declares, its enums match the Python mirror, the host
routine shared with the device reproduces devicert.static_bounds, and the
product fails loudly instead of falling back to the CPU."""

from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import pytest
import torch

from paper_2106_03219_b200 import _build, _lib, devicert, offload, runtime

ROOT = Path(__file__).resolve().parents[1]
HEADER = (ROOT / "include" / "omprt_b200.h").read_text()


def declared_functions() -> set[str]:
    return set(re.findall(r"^\s*(?:const char \*|int|size_t)\s*(omprt_\w+)\(", HEADER, re.M))


def test_library_builds_and_loads():
    _build.build()
    L = _lib.load()
    assert L.omprt_version().decode().startswith("omprt_b200")


def test_every_declared_symbol_is_exported_and_bound():
    L = _lib.load()
    decl = declared_functions()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(L, name), name
    assert decl == set(_lib.EXPORTED)


def test_header_enums_match_python_mirror():
    def enum(name):
        m = re.search(r"\b" + name + r"\s*=\s*(-?\d+)", HEADER)
        return int(m.group(1))

    assert [enum(f"OMPRT_{t}") for t in ("I32", "U32", "I64", "U64", "F32", "F64")] == \
        [_lib.I32, _lib.U32, _lib.I64, _lib.U64, _lib.F32, _lib.F64]
    assert enum("OMPRT_SCHED_DISTRIBUTE_CHUNKED") == _lib.SCHED_DISTRIBUTE_CHUNKED
    assert enum("OMPRT_MODE_ORDERED") == _lib.MODE_ORDERED
    assert enum("OMPRT_ATOMIC_INC") == _lib.ATOMIC_INC
    assert enum("OMPRT_TRAP") == _lib.TRAP
    assert "#define OMPRT_ARENA_CAPACITY 65536" in HEADER


def test_header_compiles_as_c():
    import subprocess
    import tempfile

    src = '#include "omprt_b200.h"\nint main(void){return OMPRT_OK;}\n'
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "t.c"
        p.write_text(src)
        r = subprocess.run(["/usr/bin/gcc", "-std=c99", "-Wall", "-Werror", "-I",
                            str(ROOT / "include"), "-c", str(p), "-o", str(Path(d) / "t.o")],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr


def test_host_static_bounds_matches_reference(devicert_golden):
    for lb, ub, tid, n, lo, hi in devicert_golden["static_bounds"]:
        assert devicert.static_bounds(lb, ub, tid, n) == (lo, hi)
    with pytest.raises(ZeroDivisionError):
        devicert.static_bounds(0, 9, 0, 0)


def test_argument_validation_without_gpu():
    L = _lib.load()
    # bad grid / schedule are rejected before any launch
    assert L.omprt_bounds_dump(0, 9, 0, 1, 0, 32, C.c_void_p(1), None) == _lib.EINVAL
    assert L.omprt_bounds_dump(0, 9, 7, 1, 1, 32, C.c_void_p(1), None) == _lib.EINVAL
    assert L.omprt_reduce(C.c_void_p(1), 0, 9, 5, 0, 1, 0, 1, 32, 0, C.c_void_p(1),
                          C.c_void_p(1), None) == _lib.EINVAL  # chunk 0 for chunked
    assert "chunk" in _lib.last_error()
    assert L.omprt_reduce(C.c_void_p(1), 0, 9, 9, 0, 0, 1, 1, 32, 0, C.c_void_p(1),
                          C.c_void_p(1), None) == _lib.EINVAL  # dtype
    assert L.omprt_generic_reduce(C.c_void_p(1), 0, 9, 2, 0, 4, 48, 0, 0, 0, 0, C.c_void_p(1),
                                  C.c_void_p(1), None, None) == _lib.EINVAL  # P % 32
    assert L.omprt_atomic_apply(5, 2, None, None, None, None, 1, None) == _lib.EINVAL  # inc i64
    assert L.omprt_reduce_workspace_bytes(296, 1024, 1) >= 296 * 1024 * 8


def test_allreduce_argument_checks():
    # validated before NCCL is ever loaded (no GPU needed)
    L = _lib.load()
    assert L.omprt_allreduce(None, 1, 2, 0, C.c_void_p(1), None) == _lib.EINVAL  # null buffer
    assert L.omprt_allreduce(C.c_void_p(1), 1, 9, 0, C.c_void_p(1), None) == _lib.EINVAL  # dtype
    assert L.omprt_allreduce(C.c_void_p(1), 1, 2, 7, C.c_void_p(1), None) == _lib.EINVAL  # op
    assert L.omprt_allreduce(C.c_void_p(1), 1, 2, 0, None, None) == _lib.EINVAL  # no comm


def test_workspace_layout_covers_split_teams_and_ordered_flags():
    # SPMD launches may split a few teams over up to SMs CTAs: the team
    # partial slots (4 per CTA, 8 bytes: ORDERED max/min keep a (value, order
    # key) pair for max and for min) never shrink below 256 CTAs; ORDERED
    # keeps P partials plus one 8-byte ready flag per group of 32 threads
    L = _lib.load()
    for teams, threads in ((1, 128), (3, 64), (148, 256), (1024, 1024), (7, 33)):
        spmd = L.omprt_reduce_workspace_bytes(teams, threads, 0)
        ordered = L.omprt_reduce_workspace_bytes(teams, threads, 1)
        P = teams * threads
        assert spmd >= 256 + max(teams, 256) * 8 * 4
        assert ordered >= spmd + P * 8 + ((P + 31) // 32) * 8


def test_no_cpu_fallback():
    x = torch.arange(10, dtype=torch.int64)
    with pytest.raises(ValueError, match="CUDA"):
        runtime.reduce(x)
    call = offload.TargetCall(0, offload.kernel_name(0),
                              (offload.ArgDescriptor("x", "buffer", "i64"),))
    # a foreign arch or a missing image is status 1, as in the reference
    assert offload.tgt_target(call.bind([b"\0" * 8]), {}, "vgpu") == 1
    assert offload.tgt_target(call.bind([b"\0" * 8]), {}, "b200") == 1
    assert offload.tgt_target(call.bind([b"\0" * 8]), {"b200": {}}, "b200",
                              force_fail=True) == 1


def test_missing_library_raises(monkeypatch, tmp_path):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setenv("OMPRT_B200_LIB", str(tmp_path / "nope.so"))
    with pytest.raises(_lib.OmprtUnavailable):
        _lib.load()


def test_grid_config_validation():
    with pytest.raises(ValueError):
        offload.GridConfig(2048, 32)
    with pytest.raises(ValueError):
        offload.GridConfig(1, 0)
    g = offload.GridConfig(4, 8, -1)
    assert g.sched_seed == 2**64 - 1
    assert offload.kernel_name(3) == "__omp_offload_3"


def test_runtime_api_names_cover_reference():
    ref_names = {"omp_thread_id", "omp_team_id", "omp_num_threads", "omp_num_teams",
                 "__kmpc_alloc_shared", "__kmpc_free_shared", "__kmpc_flush", "__kmpc_barrier",
                 "atomic_add", "atomic_max", "atomic_min", "atomic_exchange", "atomic_cas",
                 "atomic_inc", "for_static_init"}  # devicert.RUNTIME_API, devicert.py:24-52
    assert set(devicert.RUNTIME_API) == ref_names
