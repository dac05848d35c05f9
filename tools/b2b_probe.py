"""Probe: per-launch time of back-to-back fp64 sums vs run length and NVML polling."""
import sys, threading, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2106_03219_b200 import runtime

dev = torch.device("cuda", 0)
n = 1 << 30
x = runtime.synthetic(n, "f64", 0x210603219, device=dev)
out = torch.zeros(1, dtype=torch.float64, device=dev)
sms = runtime.num_sms()
s = torch.cuda.current_stream()

def run(k, teams=sms, threads=1024, sched="distribute", direct=False):
    for _ in range(5):
        runtime.reduce(x, "add", sched=sched, teams=teams, threads=threads, out=out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(s)
    for _ in range(k):
        runtime.reduce(x, "add", sched=sched, teams=teams, threads=threads, out=out)
    t1 = time.perf_counter()
    b.record(s)
    b.synchronize()
    ms = a.elapsed_time(b) / k
    return {"k": k, "ms": round(ms, 4), "gbs": round(n * 8 / ms / 1e6, 1),
            "cpu_enqueue_us_per_launch": round((t1 - t0) / k * 1e6, 1)}

for k in (50, 200, 1000, 3000):
    print(json.dumps(run(k)), flush=True)
stop = threading.Event()
def poll():
    import pynvml
    pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop.is_set():
        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        time.sleep(0.02)
t = threading.Thread(target=poll, daemon=True); t.start()
for k in (200, 1000):
    r = run(k); r["nvml_polling"] = True; print(json.dumps(r), flush=True)
stop.set(); t.join()
time.sleep(2)
for k in (1000,):
    print(json.dumps(run(k)), flush=True)
