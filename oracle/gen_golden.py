"""Generate tests/golden/*.json by running the REFERENCE itself.

TEST INFRASTRUCTURE.  Run in the build container, where the read-only
reference is mounted (it does not exist on the GPU box; the JSON files it
writes are committed and travel instead):

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden.py

What it records (every value computed by forge code, never by ours):
  devicert_vectors.json   devicert.static_bounds / step_* / Arena on the
                          cases of test_devicert.py plus seeded random ones
  fallback_runs.json      hot-path kernels written in forge's mini-language,
                          executed by the host fallback (TargetCall.fallback,
                          host.py:536-585) and the simulated device
                          (tgt_target -> VirtualGPU, host.py:255-296) on
                          splitmix64-generated inputs; the for_static_init
                          bounds every vgpu thread computes; the generic-mode
                          arena globalisation pattern on vgpu;
                          atomic probes (corpus.probe_source) and the CORPUS
                          programs' outputs.
"""

from __future__ import annotations

import copy
import json
import random
import sys
import time
from pathlib import Path

REF = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"

sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

from forge import corpus, devicert  # noqa: E402
from forge.codegen import compile_device_image  # noqa: E402
from forge.host import HostProgram, run_source, tgt_target  # noqa: E402
from forge.lowering import lower_atomics  # noqa: E402
from forge.parser import parse_module  # noqa: E402

from oracle.oracle import SEED, py_gen  # noqa: E402  (generator only)

DT = {"i32": 0, "u32": 1, "i64": 2, "u64": 3}
BITS = {"i32": 32, "u32": 32, "i64": 64, "u64": 64}


def le_bytes(vals, ty):
    w = BITS[ty] // 8
    m = (1 << BITS[ty]) - 1
    return bytearray(b"".join((v & m).to_bytes(w, "little") for v in vals))


def from_le(raw, ty, signed=None):
    w = BITS[ty] // 8
    out = []
    for i in range(len(raw) // w):
        v = int.from_bytes(raw[i * w:(i + 1) * w], "little")
        if ty in ("i32", "i64"):
            v = devicert.to_signed(v, BITS[ty])
        out.append(v)
    return out


# --------------------------------------------------------------- devicert

def devicert_vectors() -> dict:
    rng = random.Random(0x2106)
    sb = []

    def rec(lb, ub, tid, n):
        lo, hi = devicert.static_bounds(lb, ub, tid, n)
        sb.append([lb, ub, tid, n, lo, hi])

    rec(0, 99, 1, 4)  # test_devicert.py:89-90
    for n in range(1, 33):  # test_devicert.py:93-96
        for span in (1, 2, 3, 5, 31, 32, 33, 100, 999, 1000):
            for tid in range(n):
                rec(0, span - 1, tid, n)
    for lb in (-7, 1, 13):  # test_devicert.py:99-102
        for n in (1, 3, 8, 32):
            for tid in range(n):
                rec(lb, lb + 99, tid, n)
    for tid in range(4):  # test_devicert.py:105-111
        rec(0, 1, tid, 4)
    # BASELINE geometries: 1x128 over 2^20; 592x1024 and 1024x1024 over 2^30
    for tid in (0, 1, 63, 127):
        rec(0, 2**20 - 1, tid, 128)
    for n in (592 * 1024, 1024 * 1024, 296 * 1024, 148 * 1024):
        for tid in (0, 1, 605_000, n - 259, n - 258, n - 1):
            if tid < n:
                rec(0, 2**30 - 1, tid, n)
    # seeded random, including empty (ub < lb) spaces and negative bounds
    for _ in range(3000):
        lb = rng.randint(-(2**40), 2**40)
        ub = lb + rng.randint(-50, 2**20)
        n = rng.randint(1, 4096)
        rec(lb, ub, rng.randint(0, n - 1), n)

    steps = {k: [] for k in ("add", "max", "min", "exchange", "cas", "inc")}
    edge = [0, 1, 2, 5, 7, 0x7FFFFFFF, 0x80000000, 0xFFFFFFFE, 0xFFFFFFFF]
    pairs = [(a, b) for a in edge for b in edge]
    pairs += [(rng.getrandbits(32), rng.getrandbits(32)) for _ in range(300)]
    for x, e in pairs:
        steps["add"].append([x, e, *devicert.step_add(x, e)])
        steps["max"].append([x, e, *devicert.step_max(x, e)])
        steps["min"].append([x, e, *devicert.step_min(x, e)])
        steps["exchange"].append([x, e, *devicert.step_exchange(x, e)])
        steps["inc"].append([x, e, *devicert.step_inc(x, e)])
        d = rng.getrandbits(32)
        steps["cas"].append([x, e, d, *devicert.step_cas(x, e, d)])
        steps["cas"].append([x, x, d, *devicert.step_cas(x, x, d)])

    inc_seq = []
    for e in range(1, 8):  # test_devicert.py:55-64
        x, seq = 0, []
        for _ in range(51):
            seq.append(x)
            x, _old = devicert.step_inc(x, e)
        inc_seq.append([e, seq])

    traces = []

    def replay(ops, capacity=devicert.ARENA_CAPACITY):
        arena = devicert.Arena(capacity)
        script, results, code = [], [], 0
        for kind, size, off in ops:
            script.append([0 if kind == "alloc" else 1, size, off])
            if code:
                results.append(-0x7FFF)
                continue
            try:
                if kind == "alloc":
                    results.append(arena.alloc(size))
                else:
                    arena.free(off, size)
                    results.append(0)
            except devicert.ArenaError as err:
                code = err.code
                results.append(-code)
        traces.append({"capacity": capacity, "script": script, "results": results,
                       "code": code})

    rng2 = random.Random(20240817)  # the seed of test_devicert.py:141
    for _ in range(50):
        arena = devicert.Arena()
        live, ops = [], []
        for _ in range(rng2.randint(1, 40)):
            if live and rng2.random() < 0.4:
                off, size = live.pop()
                ops.append(("free", size, off))
                arena.free(off, size)
            else:
                size = rng2.randint(1, 512)
                off = arena.alloc(size)
                ops.append(("alloc", size, 0))
                live.append((off, size))
        replay(ops)
    replay([("alloc", 1, 0), ("alloc", 1, 0)])  # alignment, test_devicert.py:172-177
    replay([("alloc", 32, 0), ("alloc", 64, 0)], 64)  # overflow code 1, :180-185
    replay([("alloc", 65, 0)], 64)  # oversized, :188-192
    replay([("alloc", 16, 0), ("alloc", 16, 0), ("free", 16, 0)])  # non-LIFO code 2, :195-201
    replay([("alloc", 32, 0), ("free", 32, 0), ("alloc", 32, 0)], 32)  # reuse, :204-208
    replay([("alloc", 12, 0), ("alloc", 1, 0), ("free", 1, 16), ("alloc", 64, 0)])
    replay([("alloc", 16, 0), ("alloc", 65530, 0)])  # overflow at 64 KiB, §A.6
    replay([("alloc", 65536, 0), ("free", 65536, 0), ("alloc", 65537, 0)])
    # random stacks that run into the 64 KiB capacity
    for _ in range(20):
        live, ops, arena = [], [], devicert.Arena()
        for _ in range(rng2.randint(5, 60)):
            if live and rng2.random() < 0.3:
                off, size = live.pop()
                ops.append(("free", size, off))
                arena.free(off, size)
            else:
                size = rng2.randint(1, 9000)
                ops.append(("alloc", size, 0))
                try:
                    live.append((arena.alloc(size), size))
                except devicert.ArenaError:
                    break
        replay(ops)
    return {
        "arena_capacity": devicert.ARENA_CAPACITY,
        "arena_align": devicert.ARENA_ALIGN,
        "static_bounds": sb,
        "steps": steps,
        "inc_sequences": inc_seq,
        "arena_traces": traces,
    }


# ------------------------------------------------------------- kernels

REDUCE_SRC = """\
void kernel({T} *x, {T} *cell, i64 n) {{
  #pragma omp target
  {{
    i64 bounds[2];
    i64 i;
    i64 g;
    {T} part;
    {T} old;
    g = (i64) (omp_team_id() * omp_num_threads() + omp_thread_id());
    for_static_init(0, n - 1, g, (i64) (omp_num_teams() * omp_num_threads()), bounds);
    if (bounds[0] <= bounds[1]) {{
      i = bounds[0];
      part = x[i];
      i = i + 1;
      while (i <= bounds[1]) {{
        {BODY}
        i = i + 1;
      }}
      old = {ATOMIC}(cell, part);
    }}
  }}
}}
"""

BODIES = {
    "add": ("part = part + x[i];", "__atomic_add"),
    "max": ("if (part < x[i]) {{ part = x[i]; }}", "__atomic_max"),
    "min": ("if (part > x[i]) {{ part = x[i]; }}", "__atomic_min"),
}

BOUNDS_SRC = """\
void kernel(i64 *out, i64 lb, i64 ub) {
  #pragma omp target
  {
    i64 bounds[2];
    i64 g;
    g = (i64) (omp_team_id() * omp_num_threads() + omp_thread_id());
    for_static_init(lb, ub, g, (i64) (omp_num_teams() * omp_num_threads()), bounds);
    out[2 * g] = bounds[0];
    out[2 * g + 1] = bounds[1];
  }
}
"""

# tid 0 allocates (pad, then the globalised parts array + one
# slot), publishes the offset through a pteam global, barrier, every thread
# folds its for_static_init share of the team's distribute block into the
# arena, barrier, tid 0 folds the parts in order, atomically adds, frees LIFO.
GENERIC_SRC = """\
#pragma omp begin declare target
i64 parts_off;
#pragma omp allocate(parts_off) allocator(omp_pteam_mem_alloc)
extern u64 __shared_arena[8192];
#pragma omp end declare target

void kernel(i64 *x, i64 *cell, i64 *offs, i64 n, i64 pad) {
  #pragma omp target
  {
    i64 tb[2];
    i64 mb[2];
    i64 i;
    i64 w;
    i64 v;
    i64 part;
    i64 old;
    i64 tid;
    i64 nt;
    u64 poff;
    tid = (i64) omp_thread_id();
    nt = (i64) omp_num_threads();
    for_static_init(0, n - 1, (i64) omp_team_id(), (i64) omp_num_teams(), tb);
    if (tid == 0) {
      if (pad > 0) {
        poff = __kmpc_alloc_shared((u64) pad);
      }
      parts_off = (i64) __kmpc_alloc_shared((u64) ((nt + 1) * 8));
      offs[omp_team_id()] = parts_off;
    }
    __kmpc_barrier(0);
    part = 0;
    if (tb[0] <= tb[1]) {
      for_static_init(tb[0], tb[1], tid, nt, mb);
      i = mb[0];
      while (i <= mb[1]) {
        part = part + x[i];
        i = i + 1;
      }
    }
    __shared_arena[parts_off / 8 + tid] = (u64) part;
    __kmpc_barrier(0);
    if (tid == 0) {
      v = 0;
      w = 0;
      while (w < nt) {
        v = v + (i64) __shared_arena[parts_off / 8 + w];
        w = w + 1;
      }
      old = __atomic_add(cell, v);
      __kmpc_free_shared((u64) parts_off, (u64) ((nt + 1) * 8));
      if (pad > 0) {
        __kmpc_free_shared(poff, (u64) pad);
      }
    }
  }
}
"""


def _prog(src):
    mod = parse_module(src)
    prog = HostProgram(mod)
    img = compile_device_image(lower_atomics(copy.deepcopy(mod)), "vgpu")
    return prog, prog.target_calls[0], img


def _bind(call, named):
    return [named[a.name] for a in call.args]


def run_reduce(ty, op, n, teams, threads, init, k, vgpu: bool, fallback: bool = True):
    body, atomic = BODIES[op]
    src = REDUCE_SRC.format(T=ty, BODY=body.replace("{{", "{").replace("}}", "}"), ATOMIC=atomic)
    prog, call, img = _prog(src)
    xs = [py_gen(DT[ty], i, SEED, k) for i in range(n)]
    rec = {"dtype": ty, "op": op, "n": n, "lb": 0, "ub": n - 1, "teams": teams,
           "threads": threads, "seed": SEED, "k": k, "init": init,
           "sched": "static (for_static_init over flat ids)"}
    if fallback:
        cell = le_bytes([init], ty)
        t0 = time.perf_counter()
        call.fallback(_bind(call, {"x": le_bytes(xs, ty), "cell": cell, "n": n}), teams, threads)
        rec["fallback_seconds"] = round(time.perf_counter() - t0, 3)
        rec["fallback"] = from_le(cell, ty)[0]
    if vgpu:
        cell = le_bytes([init], ty)
        out = {}
        t0 = time.perf_counter()
        st = tgt_target(call.bind(_bind(call, {"x": le_bytes(xs, ty), "cell": cell, "n": n})),
                        {"vgpu": img}, "vgpu", grid=(teams, threads), sched_seed=7, out=out)
        rec["vgpu_seconds"] = round(time.perf_counter() - t0, 3)
        assert st == 0, st
        rec["vgpu"] = from_le(cell, ty)[0]
        rec["vgpu_instructions"] = out["result"].instruction_count
    return rec


def run_bounds(lb, ub, teams, threads):
    prog, call, img = _prog(BOUNDS_SRC)
    n = teams * threads
    out = le_bytes([0] * (2 * n), "i64")
    st = tgt_target(call.bind(_bind(call, {"out": out, "lb": lb, "ub": ub})), {"vgpu": img},
                    "vgpu", grid=(teams, threads), sched_seed=1)
    assert st == 0
    vals = from_le(out, "i64")
    return {"lb": lb, "ub": ub, "teams": teams, "threads": threads,
            "bounds": [[vals[2 * g], vals[2 * g + 1]] for g in range(n)]}


def run_generic(n, teams, threads, pad, k):
    prog, call, img = _prog(GENERIC_SRC)
    xs = [py_gen(DT["i64"], i, SEED, k) for i in range(n)]
    cell = le_bytes([0], "i64")
    offs = le_bytes([-1] * teams, "i64")
    out = {}
    t0 = time.perf_counter()
    st = tgt_target(call.bind(_bind(call, {"x": le_bytes(xs, "i64"), "cell": cell, "offs": offs,
                                           "n": n, "pad": pad})),
                    {"vgpu": img}, "vgpu", grid=(teams, threads), sched_seed=5,
                    check_uninit=True, out=out)
    rec = {"n": n, "teams": teams, "threads": threads, "pad": pad, "seed": SEED, "k": k,
           "status": st, "vgpu_seconds": round(time.perf_counter() - t0, 3)}
    if st == 0:
        rec["cell"] = from_le(cell, "i64")[0]
        rec["offsets"] = from_le(offs, "i64")
    else:
        rec["trap"] = list(out["trap"])
    return rec


def run_probes():
    rng = random.Random(0xA70)
    probes = []
    for kind in ("add", "max", "xchg", "cas", "inc"):
        for teams, threads in ((1, 8), (2, 4), (4, 8)):
            n = teams * threads
            progs = []
            for g in range(n):
                e = rng.randint(0, 50) if kind != "inc" else 7
                d = rng.randint(0, 50)
                if kind == "cas":
                    e = rng.choice([0, 0, 3, rng.randint(0, 50)])
                progs.append([(kind, e, d)])
            src = corpus.probe_source(teams, threads, progs)
            for seed in (0, 1, 2):
                mod = parse_module(src)
                prog = HostProgram(mod)
                img = compile_device_image(lower_atomics(copy.deepcopy(mod)), "vgpu")
                call = prog.target_calls[0]
                cell = le_bytes([0], "u32")
                olds = le_bytes([0] * n, "u32")
                st = tgt_target(call.bind(_bind(call, {"c": cell, "olds": olds})), {"vgpu": img},
                                "vgpu", grid=(teams, threads), sched_seed=seed)
                assert st == 0
                probes.append({"kind": kind, "teams": teams, "threads": threads,
                               "ops": [[p[0][1], p[0][2]] for p in progs], "sched_seed": seed,
                               "cell": from_le(cell, "u32")[0], "olds": from_le(olds, "u32")})
    return probes


UNINIT_SRC = """\
#pragma omp begin declare target
extern u64 __shared_arena[8192];
#pragma omp end declare target

void kernel(u64 *out, i64 w, i64 r, u64 v, i64 pad) {
  #pragma omp target
  {
    u64 off;
    u64 poff;
    if (omp_thread_id() == 0) {
      if (pad > 0) {
        poff = __kmpc_alloc_shared((u64) pad);
      }
      off = __kmpc_alloc_shared(64);
      __shared_arena[off / 8 + (u64) w] = v;
      out[0] = __shared_arena[off / 8 + (u64) r];
      out[1] = off;
      __kmpc_free_shared(off, 64);
      if (pad > 0) {
        __kmpc_free_shared(poff, (u64) pad);
      }
    }
  }
}
"""


def run_uninit():
    """The arena's data on vgpu: loader_uninitialized poison and check_uninit
    (vgpu.py:64-77, 365-369)."""
    prog, call, img = _prog(UNINIT_SRC)
    out = []
    for w, r, pad in ((0, 0, 0), (1, 3, 0), (2, 2, 24), (7, 6, 8), (5, 5, 0)):
        for check in (True, False):
            buf = le_bytes([0, 0], "u64")
            sink = {}
            st = tgt_target(call.bind(_bind(call, {"out": buf, "w": w, "r": r,
                                                   "v": 0x1234567890ABCDEF, "pad": pad})),
                            {"vgpu": img}, "vgpu", grid=(2, 4), sched_seed=1, check_uninit=check,
                            out=sink)
            rec = {"w": w, "r": r, "pad": pad, "value": 0x1234567890ABCDEF, "check": check,
                   "status": st}
            if st == 0:
                rec["read"], rec["off"] = from_le(buf, "u64")
            else:
                rec["trap"] = sink["trap"][0]
            out.append(rec)
    return out


def run_program_probes():
    """Multi-op per-thread programs (corpus.probe_source) on vgpu, several seeds."""
    rng = random.Random(0xA71)
    out = []
    kinds = ("add", "max", "xchg", "cas", "inc")
    for mix in ("add", "max", "inc", "mixed", "mixed"):
        for teams, threads in ((1, 4), (2, 4), (2, 3)):
            progs = []
            for _ in range(teams * threads):
                ops = []
                for _ in range(rng.randint(1, 3)):
                    kind = rng.choice(kinds) if mix == "mixed" else mix
                    e = 7 if kind == "inc" else rng.randint(0, 40)
                    d = rng.randint(0, 40)
                    if kind == "cas":
                        e = rng.choice([0, 0, rng.randint(0, 40)])
                    ops.append((kind, e, d))
                progs.append(ops)
            src = corpus.probe_source(teams, threads, progs)
            mod = parse_module(src)
            prog = HostProgram(mod)
            img = compile_device_image(lower_atomics(copy.deepcopy(mod)), "vgpu")
            call = prog.target_calls[0]
            total = sum(len(p) for p in progs)
            for seed in (0, 5, 11):
                cell = le_bytes([0], "u32")
                olds = le_bytes([0] * total, "u32")
                st = tgt_target(call.bind(_bind(call, {"c": cell, "olds": olds})), {"vgpu": img},
                                "vgpu", grid=(teams, threads), sched_seed=seed)
                assert st == 0
                flat = from_le(olds, "u32")
                per, k = [], 0
                for p in progs:
                    per.append(flat[k:k + len(p)])
                    k += len(p)
                out.append({"mix": mix, "teams": teams, "threads": threads,
                            "programs": [[list(op) for op in p] for p in progs],
                            "sched_seed": seed, "cell": from_le(cell, "u32")[0], "olds": per})
    return out


def run_corpus():
    res = {}
    for name, src in corpus.CORPUS:
        a = run_source(src, device="vgpu", sched_seed=3)
        b = run_source(src, device="vgpu", force_offload_fail=True)
        assert a.stdout == b.stdout, name
        res[name] = {"stdout": a.stdout.split(), "fallback_stdout": b.stdout.split()}
    return res


def fallback_runs(quick: bool) -> dict:
    reds = []
    # config 1: int64 static-sum, 1 team x 128 threads, N = 2^20
    n1 = 2**14 if quick else 2**20
    reds.append(run_reduce("i64", "add", n1, 1, 128, 0, 0, vgpu=False))
    # same kernel small enough for the simulated device
    reds.append(run_reduce("i64", "add", 4096, 1, 128, 0, 0, vgpu=True))
    for ty in ("i32", "u32", "i64", "u64"):
        for op in ("add", "max", "min"):
            for (teams, threads, n) in ((2, 4, 100), (3, 5, 1000), (4, 32, 3000), (1, 1, 257)):
                init = {"add": 11, "max": -5 if ty[0] == "i" else 3, "min": 1 << 20}[op]
                reds.append(run_reduce(ty, op, n, teams, threads, init, 1,
                                       vgpu=(n <= 1000 and teams * threads <= 16)))
    # empty tails: more threads than iterations
    reds.append(run_reduce("i64", "add", 7, 2, 8, 0, 2, vgpu=True))
    # wrap-around of u32/i32 sums
    reds.append(run_reduce("u32", "add", 5000, 8, 16, 0xFFFFFF00, 3, vgpu=False))
    reds.append(run_reduce("i32", "add", 5000, 8, 16, 0x7FFFFF00, 3, vgpu=False))

    bounds = [run_bounds(0, 2**20 - 1, 1, 128), run_bounds(0, 99, 2, 4),
              run_bounds(-7, 92, 3, 5), run_bounds(0, 1, 1, 4), run_bounds(5, 1000, 4, 32)]

    generic = [run_generic(512, 4, 8, 0, 4), run_generic(2048, 16, 8, 24, 4),
               run_generic(100, 8, 4, 0, 5), run_generic(2**13, 256, 4, 40, 7),
               run_generic(64, 2, 4, 65536 - 8, 6)]  # pad + parts overflows -> trap 1
    return {"seed": SEED, "reductions": reds, "vgpu_bounds": bounds, "generic": generic,
            "probes": run_probes(), "program_probes": run_program_probes(),
            "uninit": run_uninit(),
            "corpus": run_corpus()}


def main():
    quick = "--quick" in sys.argv
    OUT.mkdir(parents=True, exist_ok=True)
    t0 = time.time()
    (OUT / "devicert_vectors.json").write_text(json.dumps(devicert_vectors()))
    print(f"devicert vectors: {time.time() - t0:.1f}s")
    t0 = time.time()
    (OUT / "fallback_runs.json").write_text(json.dumps(fallback_runs(quick), indent=0))
    print(f"fallback/vgpu runs: {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
