#!/usr/bin/env python
"""Benchmark: teams-distribute-parallel-for fp64 sum reduction, N = 2^30 per GPU.

BASELINE.json metric "reduction GB/s (frac of HBM peak) at N=2^30, 1/2/4/8
B200 vs CPU ref" on configs[1] ("teams distribute parallel for fp64 sum
reduction, N=2^30, SPMD mode, 1 B200").  One step = one pass of the hot path
over the resident 8 GiB fp64 array: omprt_reduce (schedule distribute,
SPMD, last-team-finishes) and, for N > 1 GPUs, the one NCCL all-reduce of the
per-GPU partial plus the ordered combine.  `value` is weak-scaled: every rank
owns a 2^30-element shard (static_bounds over ranks of a G*2^30 global space).

Two more legs ride on the same JSON line:
  strong_c2   the same construct over N = 2^30 GLOBAL elements sharded over
              the G ranks (strong scaling; efficiency = T(1 GPU) / (G T(G)))
  c5_dot      BASELINE configs[4]: fp64 dot over N = 2^33 global elements
              (x, y: 64 GiB each) sharded with static_bounds, partials
              combined with one NCCL all-reduce; efficiency = aggregate GB/s
              / (G x one GPU's GB/s on the same shard without the collective)

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`--gpus N > 1` without torchrun re-launches itself under
torch.distributed.run (one rank per GPU, 127.0.0.1 rendezvous).  Prints ONE
JSON line on rank 0.  `--impl reference` times the CPU restatement of the
reference's own host-fallback algorithm (oracle/, "port") on this host's
cores over the SAME 2^30-element workload and geometry, plus forge's own
Python host fallback (TargetCall.fallback, host.py:536-585, from
baseline/_ref) on the C1 kernel and the C2 shape at bounded N.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "reduction GB/s (frac of HBM peak) at N=2^30, 1/2/4/8 B200 vs CPU ref"
N_PER_GPU = 1 << 30
ELEM = 8  # fp64
SEED = 0x210603219
BENCH_KERNEL = "k_reduce_bulk<double, 0, 3, 49152, 0>"


def workload_config(n: int, G: int, sched: str, teams: int, threads: int) -> dict:
    """The `config` both arms print (identical dicts, so the driver can match
    them): the C2 workload at G GPUs, n elements per GPU."""
    return {"workload": "C2 teams distribute parallel for fp64 sum reduction, SPMD",
            "n_per_gpu": n, "n_global": G * n, "schedule": sched, "teams": teams,
            "threads": threads, "mode": "spmd", "parallelism": f"dp{G}",
            "l2": "input 8 GiB per GPU >> 126 MB L2; no flush needed"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1000)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--teams", type=int, default=0, help="0: one team per SM")
    p.add_argument("--threads", type=int, default=384)
    p.add_argument("--sched", default="distribute")
    p.add_argument("--unroll", type=int, default=0)
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--ordered-steps", type=int, default=50,
                   help="steps of the ORDERED-mode (reference-order, bit-identical) leg")
    p.add_argument("--n-per-gpu", "--n", dest="n", type=int, default=N_PER_GPU,
                   help="elements per GPU (weak leg)")
    p.add_argument("--strong-n", type=int, default=1 << 30,
                   help="global elements of the strong-scaled C2 leg")
    p.add_argument("--c5-n", type=int, default=1 << 33,
                   help="global elements of the config-5 fp64 dot leg")
    p.add_argument("--leg-steps", type=int, default=20,
                   help="timed steps of the strong_c2 and c5_dot legs")
    p.add_argument("--no-legs", action="store_true", help="skip strong_c2 and c5_dot")
    p.add_argument("--exchange", choices=["nccl", "p2p"], default="nccl",
                   help="N > 1: combine the per-GPU partials with NCCL (overlapped with the "
                        "next step) or inside the reduction kernel over NVLink peer memory")
    p.add_argument("--no-overlap", action="store_true",
                   help="N > 1: run each step's all-reduce on the compute stream (no overlap)")
    p.add_argument("--backend", default="nccl",
                   help="torch.distributed backend for N > 1 (gloo: debug the multi-rank "
                        "flow with several ranks sharing one GPU)")
    p.add_argument("--ref-python-n1", type=int, default=1 << 20,
                   help="reference arm: N of forge's own fallback on the C1 kernel (1x128)")
    p.add_argument("--ref-python-n2", type=int, default=1 << 16,
                   help="reference arm: N of forge's own fallback on the C2 shape (148x384)")
    p.add_argument("--no-ref-python", action="store_true")
    return p.parse_args()


def spawn_ranks(args) -> int:
    """`--gpus N > 1` run as a plain process: re-launch this command under
    torch.distributed.run, one rank per GPU, rendezvous on 127.0.0.1."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    # torch.distributed.run's parser would take an abbreviation of its own
    # options out of the script's arguments ("--n" matches "--nnodes", ...)
    argv = ["--n-per-gpu" + a[3:] if a == "--n" or a.startswith("--n=") else a
            for a in sys.argv[1:]]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(ROOT / "bench.py"), *argv]
    print(f"bench: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def peaks() -> dict:
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def src_sha16() -> str:
    """Fingerprint of the library's sources + build flags (_build.source_sha16)."""
    from paper_2106_03219_b200 import _build

    return _build.source_sha16()


def ncu_capture(teams: int, threads: int, split: int) -> dict:
    """The committed `ncu --set full` capture of the bench kernel
    (profiles/ncu_bench_kernel.json): DRAM bytes per launch and ncu's DRAM
    throughput fraction — used only when the capture is of THIS launch (same
    kernel instance, grid and block); anything else is reported stale and
    its numbers are dropped, loudly, instead of decorating the line."""
    f = ROOT / "profiles" / "ncu_bench_kernel.json"
    if not f.exists():
        return {"status": "missing", "traffic": None, "frac_ncu_dram": None}
    d = json.loads(f.read_text())
    rec = d["launches"][0]
    want = {"kernel": BENCH_KERNEL, "grid": teams * split, "block": threads}
    got = {"kernel": rec.get("kernel", ""), "grid": int(rec.get("launch__grid_size", -1)),
           "block": int(rec.get("launch__block_size", -1))}
    info = {"captured_at": d.get("captured_at"), "capture_src_sha16": d.get("src_sha16"),
            "capture_kernel": got["kernel"], "capture_grid": got["grid"],
            "capture_block": got["block"]}
    if want["kernel"] not in got["kernel"] or want["grid"] != got["grid"] or \
            want["block"] != got["block"]:
        msg = f"stale ncu capture: captured {got}, timed {want}"
        print(f"bench: WARNING {msg}; roofline.traffic dropped", file=sys.stderr, flush=True)
        return {"status": msg, "traffic": None, "frac_ncu_dram": None, **info}
    sha = src_sha16()
    status = "current (captured from these library sources)" if sha == d.get("src_sha16") else \
        f"kernel geometry matches; library sources changed since the capture (now {sha})"
    return {"status": status, "traffic": d.get("dram_bytes_per_launch"),
            "frac_ncu_dram": round(rec["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
                                   / 100.0, 4), **info}


class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML while running."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples: list[tuple[float, int]] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thr = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((time.perf_counter(), mhz))
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.02)

    def start(self):
        if self.nv is not None:
            self._thr = threading.Thread(target=self._run, daemon=True)
            self._thr.start()

    def stop(self) -> dict:
        self._stop.set()
        if self._thr is not None:
            self._thr.join()
        mhz = [m for _, m in self.samples]
        return {"sm_mhz": statistics.median(mhz) if mhz else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(mhz)}


# --------------------------------------------------------------------- CPU arm

def cpu_reference(n_sample: int, steps: int, warmup: int, teams: int, threads: int,
                  min_seconds: float = 0.0, x=None) -> dict:
    """The reference's CPU path, restated in C (oracle/, kind "port"): the
    host fallback's algorithm (host.py:567-582) — every OpenMP thread folds its
    for_static_init block in order, partials combined in global-id order —
    parallelised over the forge threads on all host cores, over an in-memory
    fp64 array of n_sample elements."""
    from oracle import oracle as O

    # every host core this process may run on (torchrun sets OMP_NUM_THREADS=1)
    O.set_threads(len(os.sched_getaffinity(0)))
    if x is None:
        x = O.fill(n_sample, O.F64, SEED, 0)
    res = None
    for _ in range(warmup):
        res = O.reduce(x, 0, n_sample - 1, O.F64, O.ADD, O.DISTRIBUTE, 1, teams, threads)
    t0 = time.perf_counter()
    done = 0
    while done < steps or (time.perf_counter() - t0) < min_seconds:
        res = O.reduce(x, 0, n_sample - 1, O.F64, O.ADD, O.DISTRIBUTE, 1, teams, threads)
        done += 1
    dt = time.perf_counter() - t0
    return {"seconds": dt, "steps": done, "gbs": n_sample * ELEM * done / dt / 1e9,
            "cores": O.num_threads(), "n": n_sample, "result": float(res)}


# forge's own hot path, in forge's mini-language (the PARTIAL_SUMS idiom,
# corpus.py:219-247, over a for_static_init block per global thread id):
# the region the B200 construct replaces.  forge has no float type
# (parser.py:23-24), so the reference's own CPU path is timed on int64.
FORGE_REDUCE_SRC = """\
void kernel(i64 *x, i64 *cell, i64 n) {
  #pragma omp target
  {
    i64 bounds[2];
    i64 i;
    i64 g;
    i64 part;
    i64 old;
    g = (i64) (omp_team_id() * omp_num_threads() + omp_thread_id());
    for_static_init(0, n - 1, g, (i64) (omp_num_teams() * omp_num_threads()), bounds);
    if (bounds[0] <= bounds[1]) {
      i = bounds[0];
      part = x[i];
      i = i + 1;
      while (i <= bounds[1]) {
        part = part + x[i];
        i = i + 1;
      }
      old = __atomic_add(cell, part);
    }
  }
}
"""


def reference_python(n1: int, n2: int) -> dict:
    """forge's own CPU implementation of the path — TargetCall.fallback
    (host.py:536-585): teams and threads run one after another in the
    interpreter, so it uses exactly 1 host core — from the installed
    reference (baseline/_ref), on the C1 kernel (1 team x 128 threads) and
    the C2 geometry (148 teams x 384 threads).  Results are checked bit-exact
    against the oracle."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "forge").is_dir():
        return {"unavailable": "baseline/_ref (the reference install) is absent"}
    sys.path.insert(0, str(ref))
    try:
        from forge.host import HostProgram
        from forge.parser import parse_module
    except Exception as err:  # noqa: BLE001
        return {"unavailable": f"cannot import forge from baseline/_ref: {err!r}"}
    import numpy as np

    from oracle import oracle as O

    prog = HostProgram(parse_module(FORGE_REDUCE_SRC))
    call = prog.target_calls[0]
    out = {}
    for name, n, teams, threads in (("c1", n1, 1, 128), ("c2_shape", n2, 148, 384)):
        if n <= 0:
            continue
        x = O.fill(n, O.I64, SEED, 0)
        cell = bytearray(np.zeros(1, np.int64).tobytes())
        named = {"x": bytearray(x.tobytes()), "cell": cell, "n": n}
        vals = [named[a.name] for a in call.args]
        t0 = time.perf_counter()
        call.fallback(vals, teams, threads)
        dt = time.perf_counter() - t0
        got = int(np.frombuffer(cell, np.int64)[0])
        want = int(O.reduce(x, 0, n - 1, O.I64, O.ADD, O.STATIC, 1, teams, threads))
        out[name] = {"n": n, "teams": teams, "threads": threads, "dtype": "i64",
                     "seconds": round(dt, 3), "elem_per_s": round(n / dt, 1),
                     "gbs": round(n * 8 / dt / 1e9, 6), "bit_exact_vs_oracle": got == want,
                     "cores": 1, "of_cores": len(os.sched_getaffinity(0))}
    out["what"] = ("forge TargetCall.fallback (host.py:536-585) from baseline/_ref: the "
                   "reference's own CPU path, one interpreter thread (1 core)")
    return out


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the SAME workload as our arm's headline: 2^30 fp64 in host memory,
    # the distribute schedule over 148 x 384 OpenMP threads
    n = args.n
    teams = args.teams or 148  # our arm's default geometry: one team per B200 SM
    r = cpu_reference(n, args.steps, args.warmup, teams, args.threads)
    from oracle import oracle as O

    exact = O.exact_sum_gen(0, n - 1, O.F64, seed=SEED)
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(r["gbs"], 3),
        "unit": "GB/s",
        "n_gpus": args.gpus,
        "steps": r["steps"],
        "warmup": args.warmup,
        "ms_per_step": round(r["seconds"] / r["steps"] * 1e3, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (splitmix64 counter-based fp64 in [0,1), in host memory)",
        "config": workload_config(n, args.gpus, args.sched, teams, args.threads),
        "cpu_baseline": {"value": round(r["gbs"], 3), "unit": "GB/s", "cores": r["cores"],
                         "kind": "port",
                         "sample": (f"the full workload: {n}" if args.gpus == 1 else
                                    f"one GPU's share of the {args.gpus}-GPU workload: {n}") +
                                   f" fp64 elements ({n * 8 >> 20} MiB) "
                                   f"per step, host fallback order (host.py:567-582) over "
                                   f"{teams}x{args.threads} OpenMP threads, parallel over "
                                   "host cores"},
        "e2e": {"value": round(r["gbs"], 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "parity": {"rel_err_vs_exact": abs(r["result"] - exact) / exact, "tolerance": 1e-6},
    }
    if not args.no_ref_python:
        line["reference_python"] = reference_python(args.ref_python_n1, args.ref_python_n2)
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- GPU arm

class ShardedStep:
    """One step of a sharded construct on this rank: `local(p)` runs the
    rank's shard construct into the 1-element partial p; for G > 1 the
    partials are combined by one collective.  With NCCL the collective of
    step k (one 8-byte all-reduce + the combine into the cell) runs on a
    side stream, overlapping step k+1's shard (double-buffered partials; the
    NCCL kernel fits beside the one-CTA-per-SM construct kernel)."""

    def __init__(self, local, out, G: int, stream, overlap: bool):
        import torch

        self.local, self.out, self.G, self.stream = local, out, G, stream
        dev = out.device
        self.comm = torch.cuda.Stream(dev) if (G > 1 and overlap) else None
        self.partials = [torch.zeros(1, dtype=out.dtype, device=dev) for _ in range(2)]
        self.freed = [torch.cuda.Event(), torch.cuda.Event()]
        self.n = 0

    def step(self):
        import torch

        from paper_2106_03219_b200 import parallel, runtime

        if self.G == 1:
            self.local(self.out)  # the whole hot path: one construct launch into the cell
            return
        if self.comm is None:
            p = self.partials[0]
            p.zero_()
            self.local(p)
            parallel.allreduce_partial(p, "add")
            runtime.combine_partials(p, "add", out=self.out)
            return
        i = self.n % 2
        self.n += 1
        p = self.partials[i]
        self.stream.wait_event(self.freed[i])  # step k-2's collective is done with p
        p.zero_()
        self.local(p)
        self.comm.wait_stream(self.stream)
        with torch.cuda.stream(self.comm):
            parallel.allreduce_partial(p, "add")
            runtime.combine_partials(p, "add", out=self.out)
            self.freed[i].record(self.comm)

    def drain(self):
        if self.comm is not None:
            self.stream.wait_stream(self.comm)


def max_over_ranks(v: float, G: int, dev) -> float:
    import torch
    import torch.distributed as dist

    if G == 1:
        return v
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed_ms(step, drain, steps: int, stream, G: int, dev) -> float:
    """ms for `steps` steps on the device (CUDA events on the launching
    stream, barrier + synchronize on both sides), max over ranks."""
    import torch
    import torch.distributed as dist

    if G > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        step()
    drain()
    e1.record(stream)
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    return max_over_ranks(e0.elapsed_time(e1), G, dev)


def kernel_ms(launch, reps: int, stream, G: int, dev) -> float:
    """Average device time of one launch (events around each), max over ranks."""
    import torch

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for a, b in ev:
        a.record(stream)
        launch()
        b.record(stream)
    torch.cuda.synchronize()
    return max_over_ranks(sum(a.elapsed_time(b) for a, b in ev) / reps, G, dev)


def parse_cpulist(text: str) -> set[int]:
    """sysfs cpulist ("0-15,32-47\n") -> {0, ..., 15, 32, ..., 47}."""
    cpus: set[int] = set()
    for part in text.strip().split(","):
        if part:
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
    return cpus


def bind_numa(index: int) -> dict:
    """Pin this rank's host threads to the NUMA node its GPU hangs off (sysfs
    numa_node of the GPU's PCI function), so the pinned e2e buffer it
    allocates next is node-local and the copy-in does not cross the socket
    interconnect.  N > 1 only: at N = 1 the CPU-baseline leg keeps every core."""
    import torch

    p = torch.cuda.get_device_properties(index)
    bdf = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    info = {"gpu_pci": bdf, "numa_node": None, "cpus": None}
    try:
        node = int(Path(f"/sys/bus/pci/devices/{bdf}/numa_node").read_text())
        if node < 0:
            return info
        cpus = parse_cpulist(Path(f"/sys/devices/system/node/node{node}/cpulist").read_text())
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            info.update(numa_node=node, cpus=len(cpus))
    except (OSError, ValueError):
        pass
    return info


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2106_03219_b200 import _lib, offload, parallel, runtime

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    numa = bind_numa(local) if world > 1 else None
    if world > 1:
        if args.backend == "nccl":
            # NCCL's INIT log (rank count, NVLS/P2P transport) stays reachable,
            # on stderr so stdout keeps the one JSON line
            if "NCCL_DEBUG" not in os.environ:
                os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT",
                                  NCCL_DEBUG_FILE="/dev/stderr")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.backend)
    _lib.ensure_device(local)
    if args.unroll:
        runtime.set_unroll(args.unroll)

    n = args.n
    G = world
    glb, gub = 0, G * n - 1
    lo, hi = parallel.shard(glb, gub, rank, G)
    nloc = hi - lo + 1
    sms = runtime.num_sms()
    teams = args.teams or sms
    threads = args.threads
    x = runtime.synthetic(nloc, "f64", SEED, 0, offset=lo, device=dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    scratch = torch.zeros(1, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def reducer(xs):
        return lambda p: runtime.reduce(xs, "add", sched=args.sched, teams=teams,
                                        threads=threads, out=p)

    px = parallel.PeerExchange(dev) if (G > 1 and args.exchange == "p2p") else None
    weak = ShardedStep(reducer(x), out, G, stream, overlap=not args.no_overlap)
    if px is not None:
        # one kernel: shard reduction + the peer-memory exchange + the
        # rank-ordered fold into the cell
        weak.step = lambda: px.reduce(x, "add", out=out, sched=args.sched, teams=teams,
                                      threads=threads)

    out.zero_()
    weak.step()
    weak.drain()
    torch.cuda.synchronize()
    got = float(out.item())

    for _ in range(args.warmup):
        weak.step()
    weak.drain()
    # kernel-only timing of the bench kernel (CUDA events on the launching stream)
    k_avg_ms = kernel_ms(lambda: runtime.reduce(x, "add", sched=args.sched, teams=teams,
                                                threads=threads, out=scratch),
                         min(args.steps, 200), stream, G, dev)

    # in-run read-only calibration: the library reduction (torch.sum) over
    # the same resident array, best of 5 (SURVEY §8(d) peak iii)
    cal_ms = []
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        torch.sum(x)
        b.record(stream)
        b.synchronize()
        cal_ms.append(a.elapsed_time(b))
    cal_gbs = nloc * ELEM / (min(cal_ms[1:]) / 1e3) / 1e9

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.1)
    ms_max = timed_ms(weak.step, weak.drain, args.steps, stream, G, dev)
    clocks = sampler.stop()
    total_bytes = G * n * ELEM
    gbs = total_bytes * args.steps / (ms_max / 1e3) / 1e9
    launches = args.steps * (1 if (G == 1 or px is not None) else 2)

    # ORDERED mode on the same array and geometry: every OpenMP thread folds
    # its block in order, partials combined in global thread order — the
    # reference's own combine order (host.py:567-582), bit-identical to the
    # CPU reference arm's result (checked against the oracle below)
    ordered = None
    if G == 1 and args.ordered_steps > 0:
        o_out = torch.zeros(1, dtype=torch.float64, device=dev)

        def o_step():
            o_out.zero_()
            runtime.reduce(x, "add", sched=args.sched, teams=teams, threads=threads,
                           mode="ordered", out=o_out)

        for _ in range(3):
            o_step()
        torch.cuda.synchronize()
        got_ordered = float(o_out.item())
        o_ms = timed_ms(o_step, lambda: None, args.ordered_steps, stream, G, dev) / \
            args.ordered_steps
        ordered = {"value": round(nloc * ELEM / (o_ms / 1e3) / 1e9, 3), "unit": "GB/s",
                   "ms_per_step": round(o_ms, 5), "steps": args.ordered_steps,
                   "kernel": "omprt::k_reduce_ordered_rows (row-group cp.async windows + "
                             "folder warp, exact 32-lane batch fold of the partials)",
                   "result": got_ordered}

    # end to end through the C-ABI host-buffer call (pinned host -> HBM each
    # step), on every rank at once (each GPU copies its shard over its own link)
    e2e = None
    got_e2e = None
    if args.e2e_steps > 0:
        # every rank pins its whole shard; never ask the host for more than
        # ~half its free memory across the node's ranks (an 8-rank node pins
        # 8 x 8 GiB): beyond that each rank moves a bounded prefix and says so
        n_e2e = nloc
        try:
            import psutil

            avail = psutil.virtual_memory().available
            local_ranks = int(os.environ.get("LOCAL_WORLD_SIZE", str(G)))
            cap = int(avail * 0.5 / max(local_ranks, 1) / ELEM)
            if cap < n_e2e:
                n_e2e = max(cap - cap % 4096, 1 << 20)
        except Exception:  # noqa: BLE001
            pass
        hx = torch.empty(n_e2e, dtype=torch.float64, pin_memory=True)
        hx.copy_(x[:n_e2e])
        cell = torch.zeros(1, dtype=torch.float64)
        offload.reduce_host(hx, cell, op="add", sched=args.sched, teams=teams, threads=threads)
        got_e2e = float(cell.item())
        if G > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            cell.zero_()
            offload.reduce_host(hx, cell, op="add", sched=args.sched, teams=teams,
                                threads=threads)
        el = max_over_ranks(time.perf_counter() - t0, G, dev)
        e2e = {"value": round(G * n_e2e * ELEM * args.e2e_steps / el / 1e9, 3),
               "unit": "GB/s", "h2d_bytes_per_step": n_e2e * ELEM + ELEM,
               "d2h_bytes_per_step": ELEM,
               "path": "omprt_reduce_host (C ABI, pinned host buffer, copy-in + reduce + "
                       "copy-out per step), all ranks at once",
               "elements_per_rank": n_e2e,
               "host_numa": numa,
               "bound": "PCIe host->device copy of the 8 GiB input (Gen5 x16, 64 GB/s raw "
                        "per GPU)"}
        del hx
    launches_total = launches

    # ---- strong_c2 and c5_dot legs
    legs = {}
    if not args.no_legs:
        legs, leg_launches = run_legs(args, x, k_avg_ms, G, rank, dev, stream, teams, threads)
        launches_total += leg_launches
    del x
    torch.cuda.empty_cache()

    cpu = None
    parity = None
    if rank == 0 and not args.no_cpu_baseline:
        # the oracle is the checker of the device results (exact sums of the
        # generated data) and, at N=1, the timed CPU reference path
        from oracle import oracle as O

        exact = O.exact_sum_gen(glb, gub, O.F64, seed=SEED)
        parity = {"rel_err_vs_exact": abs(got - exact) / exact, "tolerance": 1e-6,
                  "n_global": G * n}
        if got_e2e is not None and e2e["elements_per_rank"] == nloc and G == 1:
            parity["e2e_rel_err_vs_exact"] = abs(got_e2e - exact) / exact
        if parity["rel_err_vs_exact"] > 1e-6:
            raise SystemExit(f"parity failure: {got} vs exact {exact}")
        for name, leg in legs.items():
            if "result" not in leg:
                continue
            want = (O.exact_dot_gen(0, leg["n_global"] - 1, seed=SEED) if name == "c5_dot"
                    else O.exact_sum_gen(0, leg["n_global"] - 1, O.F64, seed=SEED))
            leg["parity"] = {"rel_err_vs_exact": abs(leg["result"] - want) / want,
                             "tolerance": 1e-6}
            if leg["parity"]["rel_err_vs_exact"] > 1e-6:
                raise SystemExit(f"{name} parity failure: {leg['result']} vs {want}")
        if ordered is not None:
            # the reference order's exact bits (oracle: the host fallback's
            # algorithm in C, data regenerated on the host)
            want = float(O.reduce(None, glb, gub, O.F64, O.ADD,
                                  {"static": O.STATIC, "distribute": O.DISTRIBUTE}.get(
                                      args.sched, O.DISTRIBUTE), 1, teams, threads, 0.0))
            ordered["bit_identical_to_reference_order"] = ordered["result"] == want
            if not ordered["bit_identical_to_reference_order"]:
                raise SystemExit(f"ORDERED parity failure: {ordered['result']!r} vs {want!r}")
        if G == 1:
            r = cpu_reference(1 << 26, 3, 1, teams, threads, min_seconds=10.0)
            cpu = {"value": round(r["gbs"], 3), "unit": "GB/s", "cores": r["cores"],
                   "kind": "port",
                   "sample": f"{r['n']} fp64 elements (512 MiB, in host memory) x "
                             f"{r['steps']} passes ({r['seconds']:.1f} s), host fallback order "
                             f"(host.py:567-582) over {teams}x{threads} OpenMP threads"}
    if rank == 0:
        pk = peaks()
        achieved = n * ELEM / (k_avg_ms / 1e3) / 1e9
        split = 1  # teams <= SMs/2 would split teams over CTAs; the bench grid never does
        cap = ncu_capture(teams, threads, split)
        line = {
            "metric": METRIC,
            "value": round(gbs, 3),
            "unit": "GB/s",
            "n_gpus": G,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": round(ms_max / args.steps, 5),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (splitmix64 counter-based fp64 in [0,1), generated on device)",
            "config": workload_config(n, G, args.sched, teams, threads),
            "combine": (f"static_bounds shards + partials exchanged inside the reduction kernel "
                        "over NVLink peer memory" if px is not None else
                        f"static_bounds shards + {args.backend.upper()} all-reduce" +
                        (", overlapped with the next step's shard"
                         if (G > 1 and not args.no_overlap) else "")) if G > 1 else "none (one GPU)",
            "frac_of_hbm_peak": round(gbs / G / pk["hbm_gbs"], 4),
            "frac_of_nominal_8tbs": round(gbs / G / 8000.0, 4),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2),
                         "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": round(achieved / pk["hbm_gbs"], 4),
                         "traffic": cap["traffic"],
                         "frac_ncu_dram": cap["frac_ncu_dram"],
                         "ncu_capture": {k: v for k, v in cap.items()
                                         if k not in ("traffic", "frac_ncu_dram")},
                         "peak_source": pk["source"] + "; a read+write copy, so a read-only "
                                        "kernel can exceed 1.0 — frac_ncu_dram is ncu's "
                                        "DRAM-throughput fraction of this kernel",
                         "kernel": "omprt::k_reduce_bulk<double,ADD,3,49152> (TMA bulk-copy ring, 3 x 48 KiB stages)",
                         "kernel_avg_ms": round(k_avg_ms, 5),
                         "read_calibration": {"gbs": round(cal_gbs, 1),
                                              "what": "torch.sum over the same 8 GiB, best of 5",
                                              "frac": round(achieved / cal_gbs, 4)},
                         "frac_of_nominal_8tbs": round(achieved / 8000.0, 4),
                         "algorithmic_bytes_per_launch": n * ELEM},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "ordered": ordered,
            "strong_c2": legs.get("strong_c2"),
            "c5_dot": legs.get("c5_dot"),
            "gpu_launches": launches_total,
            "gpu_launches_headline": launches,
            "clocks": clocks,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if px is not None:
        px.close()
    if G > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_legs(args, x_weak, k1_ms: float, G: int, rank: int, dev, stream, teams: int,
             threads: int):
    """strong_c2 (2^30 global) and c5_dot (2^33 global) over the G ranks."""
    import torch

    from paper_2106_03219_b200 import parallel, runtime

    legs = {}
    launches = 0
    steps = args.leg_steps
    per_step = 1 if G == 1 else 2  # the construct (+ the combine kernel; NCCL's is not ours)

    # strong C2: the 2^30 global array sharded over the ranks
    ns = args.strong_n
    lo, hi = parallel.shard(0, ns - 1, rank, G)
    if G == 1 and ns == x_weak.numel():
        xs = x_weak  # the same elements: global [0, 2^30) on the one GPU
    else:
        xs = runtime.synthetic(hi - lo + 1, "f64", SEED, 0, offset=lo, device=dev)
    out = torch.zeros(1, dtype=torch.float64, device=dev)
    st = ShardedStep(lambda p: runtime.reduce(xs, "add", sched=args.sched, teams=teams,
                                              threads=threads, out=p),
                     out, G, stream, overlap=not args.no_overlap)
    st.step()
    st.drain()
    torch.cuda.synchronize()
    result = float(out.item())
    for _ in range(3):
        st.step()
    st.drain()
    ms = timed_ms(st.step, st.drain, steps, stream, G, dev) / steps
    launches += steps * per_step
    # efficiency = T(one GPU, the whole 2^30) / (G x T(G GPUs)); the one-GPU
    # time is the bench kernel on 2^30 elements (k1_ms, max over ranks)
    t1 = k1_ms * ns / x_weak.numel()
    agg = ns * ELEM / (ms / 1e3) / 1e9
    legs["strong_c2"] = {"value": round(agg, 3), "unit": "GB/s", "n_global": ns,
                         "n_per_gpu_max": (ns + G - 1) // G, "ms_per_step": round(ms, 5),
                         "steps": steps, "gbs_per_gpu": round(agg / G, 3),
                         "efficiency": round(t1 / (G * ms), 4) if G > 1 else 1.0,
                         "scaling": "strong", "result": result}
    if xs is not x_weak:
        del xs

    # C5: fp64 dot over 2^33 global elements (x, y: 64 GiB each at G = 1)
    nc = args.c5_n
    lo, hi = parallel.shard(0, nc - 1, rank, G)
    m = hi - lo + 1
    # never drive the GPU out of memory: every rank computes how many shard
    # elements fit its free HBM (ranks sharing one GPU split it), the
    # smallest over the ranks decides (a collective every rank executes)
    free, _ = torch.cuda.mem_get_info(dev)
    share = max(1, int(os.environ.get("LOCAL_WORLD_SIZE", "1")) // max(torch.cuda.device_count(), 1))
    cap = int((free / share - (2 << 30)) // (2 * ELEM))
    cap = -int(max_over_ranks(-cap, G, dev))
    note = None
    if cap < m:
        fit = max(cap - cap % 4096, 1 << 20)
        nc = fit * G
        lo, hi = parallel.shard(0, nc - 1, rank, G)
        m = hi - lo + 1
        note = f"global N reduced from {args.c5_n} to {nc} to fit free HBM"
    xc = runtime.synthetic(m, "f64", SEED, 0, offset=lo, device=dev)
    yc = runtime.synthetic(m, "f64", SEED, 1, offset=lo, device=dev)
    outc = torch.zeros(1, dtype=torch.float64, device=dev)
    scratch = torch.zeros(1, dtype=torch.float64, device=dev)
    sc = ShardedStep(lambda p: runtime.dot(xc, yc, teams=teams, threads=threads, out=p),
                     outc, G, stream, overlap=not args.no_overlap)
    sc.step()
    sc.drain()
    torch.cuda.synchronize()
    result_c = float(outc.item())
    for _ in range(3):
        sc.step()
    sc.drain()
    ms_c = timed_ms(sc.step, sc.drain, steps, stream, G, dev) / steps
    k_c = kernel_ms(lambda: runtime.dot(xc, yc, teams=teams, threads=threads, out=scratch),
                    min(steps, 10), stream, G, dev)
    launches += steps * per_step
    agg_c = nc * 16 / (ms_c / 1e3) / 1e9
    one_gpu = m * 16 / (k_c / 1e3) / 1e9  # this shard on one GPU, no collective
    legs["c5_dot"] = {"value": round(agg_c, 3), "unit": "GB/s", "n_global": nc,
                      "n_per_gpu_max": m, "ms_per_step": round(ms_c, 5), "steps": steps,
                      "gbs_per_gpu": round(agg_c / G, 3),
                      "one_gpu_gbs_same_shard": round(one_gpu, 3),
                      "efficiency": round(agg_c / (G * one_gpu), 4),
                      "frac_of_hbm_peak_per_gpu": round(agg_c / G / peaks()["hbm_gbs"], 4),
                      "scaling": "strong", "kernel": "omprt::k_dot_bulk (TMA bulk-copy ring)",
                      "combine": "one NCCL all-reduce of the 8-byte partial" if G > 1 else
                                 "none (one GPU)",
                      "result": result_c}
    if note:
        legs["c5_dot"]["note"] = note
    del xc, yc
    return legs, launches


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args))
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
