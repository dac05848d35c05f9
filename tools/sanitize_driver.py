"""Small launches of every kernel family for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2106_03219_b200 import _lib, runtime

dev = torch.device("cuda", 0)
S = 0x210603219
x = runtime.synthetic(100_003, "f64", S, device=dev)
xi = runtime.synthetic(100_003, "i64", S, device=dev)
xf = runtime.synthetic(100_003, "f32", S, device=dev)
yf = runtime.synthetic(100_003, "f32", S, 1, device=dev)
for sched in ("static", "static_chunked", "distribute", "distribute_chunked"):
    for mode in ("spmd", "ordered"):
        runtime.reduce(x, sched=sched, chunk=64, teams=8, threads=256, mode=mode)
        runtime.reduce(xi, "max", lb=3, ub=99_000, sched=sched, chunk=7, teams=5, threads=96, mode=mode)
        runtime.axpy_minmax(0.5, xf, yf, sched=sched, chunk=64, teams=8, threads=256, mode=mode)
        runtime.dot(x, x, sched=sched, chunk=64, teams=8, threads=256, mode=mode)
# ORDERED row-group kernels: windows touching lb/ub (element-checked copies),
# OpenMP thread counts that are not multiples of 32, the folder's partial batch
runtime.reduce(x, lb=1, ub=100_001, sched="static", teams=7, threads=33, mode="ordered")
runtime.reduce(xf, lb=3, ub=100_000, sched="distribute", teams=3, threads=100, mode="ordered")
runtime.dot(x, x, lb=5, ub=99_999, sched="static_chunked", chunk=40, teams=9, threads=64,
            mode="ordered")
runtime.set_variant(20)
runtime.reduce(x, sched="distribute", teams=8, threads=256, mode="ordered")
# the literal walk's max/min team combine (left-biased tree, thread count not a multiple of 32)
runtime.reduce(x, "max", sched="static", teams=5, threads=100, mode="ordered",
               out=torch.full((1,), float("-inf"), dtype=torch.float64, device=dev))
runtime.set_variant(0)
# six-warp window policy (6 groups of 32 OpenMP threads per SM) for the sum and
# the dot; max/min folders over full 256-partial batches as trees
runtime.reduce(x, sched="distribute", teams=148, threads=192, mode="ordered")
runtime.dot(x, x, sched="distribute", teams=148, threads=192, mode="ordered")
runtime.reduce(xf, "min", sched="static", teams=148, threads=192, mode="ordered",
               out=torch.full((1,), float("inf"), dtype=torch.float32, device=dev))
runtime.axpy_minmax(0.5, xf, yf, sched="distribute", teams=148, threads=192, mode="ordered")
# few-team SPMD launches split over CTAs (team_set_cta)
runtime.reduce(xi, sched="static", teams=1, threads=128)
runtime.reduce(x, sched="static_chunked", chunk=5, teams=3, threads=64)
# the fused exchange epilogue with a world of one (own mailbox)
import ctypes as C  # noqa: E402
L = _lib.load()
_h = (C.c_char * L.omprt_ipc_handle_bytes())()
_mb = C.c_void_p()
L.omprt_mailbox_create(1, C.byref(_mb), _h)
_peers = torch.tensor([_mb.value], dtype=torch.int64, device=dev)
_ws = runtime.reduce_workspace(dev, 8, 256, 0)
_out = torch.zeros(1, dtype=torch.float64, device=dev)
for _k in range(2):
    L.omprt_reduce_exchange(C.c_void_p(x.data_ptr()), 0, x.numel() - 1, 5, 0, 2, 1, 8, 256,
                            C.c_void_p(_ws.data_ptr()), C.c_void_p(_out.data_ptr()),
                            C.c_void_p(_peers.data_ptr()), 0, 1, 77 + _k, _k,
                            C.c_void_p(torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
L.omprt_mailbox_destroy(_mb)
# trace ring installed around a construct
with runtime.Trace(dev):
    runtime.reduce(x, teams=8, threads=256)
runtime.set_unroll(8)
runtime.reduce(x, teams=8, threads=256)
runtime.set_unroll(4)
# round 2: SPMD construct CTAs decoupled from the OpenMP team size (odd sizes,
# per-thread override), balanced flat chunked pieces, the C3 ORDERED max/min
# group trees at 1024-thread teams, the 2 x 96 KiB bench ring geometry
runtime.reduce(x, sched="static_chunked", chunk=4096, teams=148, threads=1024)
runtime.reduce(x, sched="distribute", teams=148, threads=384)
runtime.set_spmd_block(160)
runtime.reduce(x, sched="static", teams=9, threads=1000)
runtime.dot(x, x, sched="static_chunked", chunk=1, teams=7, threads=300)
runtime.axpy_minmax(0.5, xf, yf, sched="static_chunked", chunk=64, teams=5, threads=96)
runtime.set_spmd_block(0)
runtime.axpy_minmax(0.5, xf, yf, sched="distribute", teams=148, threads=1024, mode="ordered")
runtime.generic_reduce(x, teams=64, par_threads=256)
runtime.generic_reduce(x, teams=64, par_threads=256, ordered=True)
# >= 256 teams: the ORDERED folder team folds the partials as they are published
runtime.generic_reduce(x, teams=300, par_threads=64, ordered=True)
runtime.bounds_dump(0, 99_999, "static_chunked", 3, teams=4, threads=64, device=dev)
runtime.generic_reduce(xi, teams=16, par_threads=64)
runtime.generic_reduce(xi, teams=16, par_threads=64, ordered=True)
runtime.generic_reduce(xi, teams=4, par_threads=64, pad_bytes=65000, heap_fallback=True, heap_bytes_per_team=4096)
runtime.check_trap(dev)
runtime.arena_replay([[0, 100, 0], [0, 2000, 0], [1, 2000, 104], [1, 100, 0]], teams=2, threads=64, device=dev)
runtime.atomic_probe(_lib.ATOMIC_ADD, "u32", list(range(64)), teams=2, threads=32, device=dev)
runtime.atomic_apply(_lib.ATOMIC_CAS, "i64", [1, 2, 3], [1, 0, 3], [9, 9, 9], device=dev)
torch.cuda.synchronize()
print("sanitize driver done")
