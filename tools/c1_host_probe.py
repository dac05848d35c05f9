"""Config 1: how much of a back-to-back runtime.reduce call is host overhead?
Python loop vs the same launch replayed from a CUDA graph (device time only)."""
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2106_03219_b200 import _lib, runtime  # noqa: E402

dev = torch.device("cuda", 0)
n = 1 << 20
x = runtime.synthetic(n, "i64", 0x210603219, device=dev)
out = torch.zeros(1, dtype=torch.int64, device=dev)
R = 2000


def ev_loop(fn, reps=R):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    t1 = time.perf_counter()
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / reps, (t1 - t0) * 1e6 / reps


res = {}
us, host = ev_loop(lambda: runtime.reduce(x, teams=1, threads=128, out=out))
res["python_runtime_reduce"] = {"us_per_call": round(us, 2), "host_us_per_call": round(host, 2)}

L = _lib.load()
ws = runtime.reduce_workspace(dev, 1, 128, 0)
st = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
px, pw, po = C.c_void_p(x.data_ptr()), C.c_void_p(ws.data_ptr()), C.c_void_p(out.data_ptr())
sched = _lib.SCHED_NAMES["static"]
us, host = ev_loop(lambda: L.omprt_reduce(px, 0, n - 1, runtime.dtype_code(x.dtype), 0, sched, 1, 1, 128, 0, pw, po, st))
res["ctypes_omprt_reduce"] = {"us_per_call": round(us, 2), "host_us_per_call": round(host, 2)}

s = torch.cuda.Stream(dev)
s.wait_stream(torch.cuda.current_stream(dev))
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    runtime.reduce(x, teams=1, threads=128, out=out)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            runtime.reduce(x, teams=1, threads=128, out=out)
torch.cuda.synchronize()
us, host = ev_loop(lambda: g.replay(), R // 20)
res["cuda_graph_20_launches"] = {"us_per_launch": round(us / 20, 2)}
out.zero_()
runtime.reduce(x, teams=1, threads=128, out=out)
res["value"] = int(out.item())
print(json.dumps(res), flush=True)
