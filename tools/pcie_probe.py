"""PCIe host->device paths for the e2e leg: copy-engine memcpy (1 and 4
streams) vs the reduction kernel reading pinned (UVA-mapped) host memory
directly.  One JSON line per path."""
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import _lib, runtime  # noqa: E402

n = 1 << 30
dev = torch.device("cuda", 0)
hx = torch.empty(n, dtype=torch.float64, pin_memory=True)
hx.copy_(runtime.synthetic(n, "f64", 0x210603219, device=dev).cpu())
dx = torch.empty(n, dtype=torch.float64, device=dev)
B = n * 8


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


t = timed(lambda: dx.copy_(hx, non_blocking=True))
print(json.dumps({"path": "memcpy 1 stream", "gbs": round(B / t / 1e9, 2)}), flush=True)
streams = [torch.cuda.Stream() for _ in range(4)]


def four():
    q = n // 4
    for i, s in enumerate(streams):
        with torch.cuda.stream(s):
            dx[i * q:(i + 1) * q].copy_(hx[i * q:(i + 1) * q], non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)


t = timed(four)
print(json.dumps({"path": "memcpy 4 streams", "gbs": round(B / t / 1e9, 2)}), flush=True)

# the reduction kernel reading the pinned host buffer in place (zero-copy)
L = _lib.load()
out = torch.zeros(1, dtype=torch.float64, device=dev)
ws = runtime.reduce_workspace(dev, 148, 256, 0)
stream = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for var, name in ((0, "zero-copy TMA bulk ring (default)"), (6, "zero-copy LDG.128 L2::256B"),
                  (4, "zero-copy LDG.128 unroll 8")):
    runtime.set_variant(var)
    for teams, threads in ((148, 256), (296, 1024)):
        ws = runtime.reduce_workspace(dev, teams, threads, 0)

        def zc():
            rc = L.omprt_reduce(C.c_void_p(hx.data_ptr()), 0, n - 1, runtime.dtype_code(hx.dtype),
                                0, 2, 1, teams, threads, 0, C.c_void_p(ws.data_ptr()),
                                C.c_void_p(out.data_ptr()), stream)
            assert rc == 0, rc

        try:
            t = timed(zc, 2)
            print(json.dumps({"path": name, "teams": teams, "threads": threads,
                              "gbs": round(B / t / 1e9, 2)}), flush=True)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"path": name, "err": str(e)[:200]}), flush=True)
runtime.set_variant(0)
