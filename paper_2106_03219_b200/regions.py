"""Launch compiled target regions (B200 images) — the device half of tgt_target.

`launch(image, kernel_id, grid, args)` is VirtualGPU.launch (vgpu.py:254-347)
for a `regionc.B200Image`: it builds the same memory picture the vgpu builds
(global-space globals at their vgpu offsets, initialised / zeroed /
0xAA-poisoned; buffer arguments after them, 8-aligned; team-shared data per
team; the init shadow under check_uninit), launches the kernel through the C
ABI (omprt_image_launch) with one CTA per team, reads the launch's trap
record and, when the launch trapped, renders the vgpu's own message for it.
Buffers are returned for write-back only when the launch did not trap
(tgt_target, host.py:289-295).

There is no host fallback: without the native library or a CUDA device this
raises (OmprtUnavailable / RuntimeError).
"""

from __future__ import annotations

import ctypes as C
import struct
import threading
from dataclasses import dataclass, field

import torch

from . import _lib
from .regionc import ARGV_HEADER, SHARED_CAPACITY, B200Image, _align

# TrapKind values (vgpu.py:28-36) by omprt_trap_kind code
TRAP_NAMES = {1: "SharedOverflow", 2: "NonLIFOFree", 3: "NonUniformAlloc",
              4: "UninitializedRead", 5: "OutOfBounds", 6: "Deadlock", 7: "DivideByZero",
              8: "Abort"}
_SIZES = {"i32": 4, "u32": 4, "i64": 8, "u64": 8}
POISON = 0xAA


@dataclass
class RegionResult:
    """The fields of vgpu.ExecResult a host needs (vgpu.py:100-113)."""

    status: str                      # "ok" | "trap"
    trap: str | None = None          # TrapKind value
    trap_detail: str = ""
    buffers: list = field(default_factory=list)   # bytes per buffer arg (None: scalar)
    globals: dict = field(default_factory=dict)   # global-space globals after the launch
    instruction_count: int = 0       # IR instructions executed by all threads (vgpu.py:390)


_handles: dict[tuple[str, int], int] = {}
_hlock = threading.Lock()


def _handle(image: B200Image, device: int) -> int:
    key = (image.manifest.get("ir_sha256") or str(id(image)), device)
    with _hlock:
        h = _handles.get(key)
        if h is None:
            L = _lib.load()
            _lib.ensure_device(device)
            out = C.c_void_p()
            buf = C.create_string_buffer(image.cubin, len(image.cubin))
            _lib.check(L.omprt_image_load(buf, len(image.cubin), C.byref(out)), "omprt_image_load")
            h = out.value
            _handles[key] = h
        return h


def _label(image: B200Image, aux3: int) -> str:
    space, lab = aux3 >> 32, aux3 & 0xFFFFFFFF
    if space == 0:
        return "global"
    if space == 1:
        return f"shared:{lab}"
    labels = image.manifest["slot_labels"]
    return labels[lab] if lab < len(labels) else f"slot:{lab}"


def render_trap(image: B200Image, rec: bytes, waitmask, teams: int, threads: int) -> tuple[str, str]:
    """Trap record -> (TrapKind value, vgpu detail message)."""
    _flag, kind, site, team, thread, _pad = struct.unpack_from("<6I", rec, 0)
    aux = struct.unpack_from("<4Q", rec, 24)
    name = TRAP_NAMES.get(kind, "Abort")
    s = image.manifest["sites"][site] if site < len(image.manifest["sites"]) else {}
    sk = s.get("kind")
    if sk == "elem":
        detail = f"element {aux[0]} escapes {_label(image, aux[3])}[{aux[1]}:{aux[2]}]"
    elif sk == "access" and kind == 4:
        detail = f"{s['what']} at {_label(image, aux[3])}+{aux[1]} reads {POISON:#x} poison"
    elif sk == "access":
        detail = f"{s['what']} of {aux[0]} bytes at {_label(image, aux[3])}+{aux[1]}"
    elif sk == "div":
        detail = s["detail"]
    elif sk == "trap":
        detail = f"device trap code {aux[0]} in @{s['func']} (team {team} thread {thread})"
    elif sk == "deadlock":
        blocked = []
        wm = waitmask.tolist()
        for t in range(teams):
            for i in range(threads):
                if (wm[t * 32 + (i >> 5)] >> (i & 31)) & 1:
                    blocked.append(f"team {t} thread {i}")
        detail = "barrier can never release: " + "; ".join(blocked)
    else:
        detail = f"device trap kind {kind} at site {site} (team {team} thread {thread})"
    return name, detail


def _global_blob(image: B200Image, check_uninit: bool) -> tuple[bytearray, bytearray | None]:
    gb = image.manifest["global_bytes"]
    blob = bytearray(max(gb, 8))
    shadow = bytearray(b"\x01" * max(gb, 8)) if check_uninit else None
    for g in image.manifest["globals"]:
        if g["space"] != "global":
            continue
        off, n, w = g["off"], g["bytes"], _SIZES[g["ty"]]
        if g["init"] == "none":
            blob[off:off + n] = bytes([POISON]) * n
            if shadow is not None:
                shadow[off:off + n] = bytes(n)
        elif g["init"] != "zero":
            blob[off:off + w] = (int(g["init"]) & ((1 << (8 * w)) - 1)).to_bytes(w, "little")
    return blob, shadow


def launch(image: B200Image, kernel: str, grid: tuple[int, int], args: list,
           *, check_uninit: bool = False, device: torch.device | None = None,
           sched_seed: int = 0) -> RegionResult:
    """Run `kernel` of `image` on (teams x threads) with vgpu-packed args
    (bytes/bytearray per buffer, int per scalar; vgpu.launch's contract).
    `instruction_count` is the IR instructions every thread executed (exact
    for launches that complete; the vgpu's count, vgpu.py:390); a nonzero
    `sched_seed` perturbs the interleaving at atomics and barriers
    (rt_jitter, csrc/region_rt.cuh)."""
    info = image.kernels.get(kernel)
    if info is None:
        raise ValueError(f"no function '{kernel}' in the image")
    params = info["params"]
    if len(args) != len(params):
        raise ValueError(f"'{kernel}' takes {len(params)} arguments, got {len(args)}")
    teams, threads = int(grid[0]), int(grid[1])
    if not (1 <= teams <= 1024):
        raise ValueError("num_teams must lie in 1..1024")
    if not (1 <= threads <= 1024):
        raise ValueError("threads_per_team must lie in 1..1024")
    shared = image.manifest["shared_bytes"]
    if shared > SHARED_CAPACITY:
        return RegionResult("trap", "SharedOverflow",
                            f"static team-shared data needs {shared} bytes, "
                            f"capacity is {SHARED_CAPACITY}",
                            [None] * len(args))
    if not torch.cuda.is_available():
        raise RuntimeError("compiled regions need a CUDA device (there is no host fallback)")
    dev = device or torch.device("cuda", torch.cuda.current_device())
    h = _handle(image, dev.index)

    blob, gshadow = _global_blob(image, check_uninit)
    d_blob = torch.frombuffer(blob, dtype=torch.uint8).to(dev)
    d_gsh = torch.frombuffer(gshadow, dtype=torch.uint8).to(dev) if gshadow is not None else None
    d_ssh = (torch.zeros(max(teams * shared, 1), dtype=torch.uint8, device=dev)
             if check_uninit and shared else None)
    # launch record: the trap (56 B), the instruction counter, the seed
    rec0 = bytearray(128)
    struct.pack_into("<Q", rec0, 64, int(sched_seed) & ((1 << 64) - 1))
    d_trap = torch.frombuffer(rec0, dtype=torch.uint8).to(dev)
    d_wait = torch.zeros(teams * 32, dtype=torch.int32, device=dev)

    words = [d_trap.data_ptr(), d_blob.data_ptr(), d_gsh.data_ptr() if d_gsh is not None else 0,
             d_ssh.data_ptr() if d_ssh is not None else 0, d_wait.data_ptr()]
    assert len(words) == ARGV_HEADER
    size = image.manifest["global_bytes"]
    bufs: list = []
    for (pname, pty), a in zip(params, args):
        if pty.startswith("ptr<"):
            if not isinstance(a, (bytes, bytearray)):
                raise ValueError(f"parameter {pname} needs a buffer")
            size = _align(size)
            raw = bytearray(a)
            t = (torch.frombuffer(raw, dtype=torch.uint8).to(dev) if len(raw)
                 else torch.empty(0, dtype=torch.uint8, device=dev))
            bufs.append(t)
            words += [t.data_ptr() if len(raw) else 0, len(raw), size]
            size += len(raw)
        else:
            if isinstance(a, (bytes, bytearray)):
                raise ValueError(f"parameter {pname} is not a buffer")
            bufs.append(None)
            words.append(int(a) & ((1 << 64) - 1))
    if len(words) != info["argv_slots"]:
        raise ValueError(f"argument block has {len(words)} words, the image expects "
                         f"{info['argv_slots']}")
    argv = C.create_string_buffer(struct.pack(f"<{len(words)}Q", *words), 8 * len(words))
    stream = torch.cuda.current_stream(dev)
    L = _lib.load()
    _lib.check(L.omprt_image_launch(h, kernel.encode(), teams, threads, shared, argv,
                                    8 * len(words), C.c_void_p(stream.cuda_stream)),
               "omprt_image_launch")
    rec = bytes(d_trap.cpu().numpy())  # synchronises the stream
    count = struct.unpack_from("<Q", rec, 56)[0]
    if struct.unpack_from("<I", rec, 0)[0]:
        # (the count of a trapped launch covers the threads that finished)
        name, detail = render_trap(image, rec[:56], d_wait.cpu(), teams, threads)
        return RegionResult("trap", name, detail, [None] * len(args), instruction_count=count)
    out = [bytes(t.cpu().numpy()) if t is not None else None for t in bufs]
    gvals = {}
    host_blob = bytes(d_blob.cpu().numpy())
    for g in image.manifest["globals"]:
        if g["space"] != "global":
            continue
        w = _SIZES[g["ty"]]
        vals = [int.from_bytes(host_blob[g["off"] + i * w:g["off"] + (i + 1) * w], "little")
                for i in range(g["count"])]
        gvals[g["name"]] = vals[0] if g["count"] == 1 else vals
    return RegionResult("ok", None, "", out, gvals, instruction_count=count)
