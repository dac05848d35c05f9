"""Golden vectors for compiled target regions (B200 images), from the reference.

TEST INFRASTRUCTURE — runs the unmodified reference (forge, /root/reference or
baseline/_ref) in this container and writes tests/golden/region_programs.json:
for every program below, forge's `run_source(src, device="vgpu", ...)`
(host.py:959-975) — stdout, stderr (trap kind and the vgpu's detail message),
exit status and per-offload statuses.  tests/test_regions_gpu.py runs the same
sources through forge's own host program with device "b200" (the region
compiled to sm_100a) and requires identical results.

The programs cover what the vgpu defines beyond the CORPUS: the ALU's
wrapping/signed semantics, every trap kind with its message (OutOfBounds on
elem.addr, DivideByZero, Deadlock, __trap codes 1/2/3 from the arena and an
Abort code, UninitializedRead under check_uninit), team-shared globals with
initialisers and loader_uninitialized poison, nested device functions, and
the generic-mode arena pattern.  Every trapping program has exactly one
trapping thread, so the message does not depend on the interleaving.

    python oracle/gen_region_golden.py
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
for cand in (Path("/root/reference/pkg/src"), ROOT / "baseline" / "_ref"):
    if (cand / "forge" / "__init__.py").exists():
        sys.path.insert(0, str(cand))
        break

ALU = """\
i64 out[24];

#pragma omp begin declare target
i64 twice(i64 v) {
  return v + v;
}
#pragma omp end declare target

void kernel(i64 *out, i64 a, i64 b, i32 c, u32 d, u64 e) {
  #pragma omp target num_teams(1) thread_limit(1)
  {
    out[0] = a / b;
    out[1] = a % b;
    out[2] = a >> 3;
    out[3] = (i64) ((u64) a >> 3);
    out[4] = a << 62;
    out[5] = (i64) c;
    out[6] = (i64) d;
    out[7] = (i64) (c * c * c);
    out[8] = (i64) (d - 5);
    out[9] = -a;
    out[10] = (i64) (c / -3);
    out[11] = (i64) (c % -3);
    out[12] = (i64) (d / 7);
    out[13] = (i64) (d % 7);
    out[14] = (i64) (e >> 60);
    out[15] = (i64) (a < b);
    out[16] = (i64) ((u64) a < e);
    out[17] = (i64) (c >> 1);
    out[18] = (i64) (d << 31);
    out[19] = (i64) ((a & 255) ^ (b | 3));
    out[20] = twice(twice(a));
    out[21] = (i64) (u32) a;
    out[22] = (i64) (i32) e;
    out[23] = (i64) !(a == b);
  }
}

void main() {
  u32 i;
  kernel(out, -1000000007, 13, -7, 4000000000, 18446744073709551615);
  i = 0;
  while (i < 24) {
    print(out[i]);
    i = i + 1;
  }
}
"""

# sdiv of INT64_MIN by -1 wraps (vgpu.py:547-556)
ALU_WRAP = """\
i64 out[4];

void kernel(i64 *out, i64 a, i64 b) {
  #pragma omp target num_teams(1) thread_limit(1)
  {
    out[0] = a / b;
    out[1] = a % b;
    out[2] = a * b;
    out[3] = a - 1;
  }
}

void main() {
  kernel(out, -9223372036854775807 - 1, -1);
  print(out[0]);
  print(out[1]);
  print(out[2]);
  print(out[3]);
}
"""

GRID_MAP = """\
u32 out[96];

void kernel(u32 *out) {
  #pragma omp target num_teams(3) thread_limit(32)
  {
    i64 bounds[2];
    i64 i;
    u32 g;
    g = omp_team_id() * omp_num_threads() + omp_thread_id();
    for_static_init(0, 95, (i64) g, (i64) (omp_num_teams() * omp_num_threads()), bounds);
    i = bounds[0];
    while (i <= bounds[1]) {
      out[i] = (u32) (i * i + (i64) omp_team_id());
      i = i + 1;
    }
  }
}

void main() {
  u32 i;
  kernel(out);
  i = 0;
  while (i < 96) {
    print(out[i]);
    i = i + 1;
  }
}
"""

OOB_STORE = """\
u32 out[4];

void kernel(u32 *out) {
  #pragma omp target num_teams(2) thread_limit(4)
  {
    u32 g;
    g = omp_team_id() * omp_num_threads() + omp_thread_id();
    if (g == 5) {
      out[g + 10] = 1;
    }
  }
}

void main() {
  kernel(out);
  print(out[0]);
}
"""

OOB_LOAD = """\
u64 x[8];
u64 y[1];

void kernel(u64 *x, u64 *y, i64 n) {
  #pragma omp target num_teams(1) thread_limit(4)
  {
    if (omp_thread_id() == 2) {
      y[0] = x[n];
    }
  }
}

void main() {
  kernel(x, y, 9);
  print(y[0]);
}
"""

DIV_ZERO = """\
u32 out[1];

void kernel(u32 *out, u32 z) {
  #pragma omp target num_teams(1) thread_limit(4)
  {
    if (omp_thread_id() == 1) {
      out[0] = 7 / z;
    }
  }
}

void main() {
  kernel(out, 0);
  print(out[0]);
}
"""

DEADLOCK = """\
u32 out[1];

void kernel(u32 *out) {
  #pragma omp target num_teams(2) thread_limit(4)
  {
    if (omp_team_id() == 1) {
      if (omp_thread_id() < 2) {
        __kmpc_barrier(0);
      }
    }
  }
}

void main() {
  kernel(out);
  print(out[0]);
}
"""

BARRIER_OK = """\
u64 out[8];

void kernel(u64 *out) {
  #pragma omp target num_teams(2) thread_limit(4)
  {
    u32 t;
    u32 w;
    u64 off;
    t = omp_thread_id();
    if (t == 0) {
      off = __kmpc_alloc_shared(32);
      out[omp_team_id() * 4] = off;
    }
    __kmpc_barrier(0);
    __kmpc_barrier(0);
    w = 0;
    while (w < 3) {
      __kmpc_barrier(0);
      w = w + 1;
    }
    if (t == 0) {
      __kmpc_free_shared(off, 32);
    }
  }
}

void main() {
  kernel(out);
  print(out[0]);
  print(out[4]);
}
"""

TRAP_ABORT = """\
u32 out[1];

void kernel(u32 *out) {
  #pragma omp target num_teams(1) thread_limit(4)
  {
    if (omp_thread_id() == 3) {
      __trap(9);
    }
  }
}

void main() {
  kernel(out);
  print(out[0]);
}
"""

ARENA_OVERFLOW = """\
u64 out[1];

void kernel(u64 *out, u64 bytes) {
  #pragma omp target num_teams(1) thread_limit(2)
  {
    u64 off;
    if (omp_thread_id() == 0) {
      off = __kmpc_alloc_shared(bytes);
      out[0] = off;
    }
  }
}

void main() {
  kernel(out, 70000);
  print(out[0]);
}
"""

ARENA_NON_LIFO = """\
u64 out[2];

void kernel(u64 *out) {
  #pragma omp target num_teams(1) thread_limit(2)
  {
    u64 a;
    u64 b;
    if (omp_thread_id() == 0) {
      a = __kmpc_alloc_shared(16);
      b = __kmpc_alloc_shared(24);
      out[0] = a;
      out[1] = b;
      __kmpc_free_shared(a, 16);
    }
  }
}

void main() {
  kernel(out);
  print(out[1]);
}
"""

ARENA_NON_UNIFORM = """\
u64 out[1];

void kernel(u64 *out) {
  #pragma omp target num_teams(1) thread_limit(4)
  {
    if (omp_thread_id() == 1) {
      out[0] = __kmpc_alloc_shared(8);
    }
  }
}

void main() {
  kernel(out);
  print(out[0]);
}
"""

TEAM_SHARED = """\
#pragma omp begin declare target
u64 base = 5;
#pragma omp allocate(base) allocator(omp_pteam_mem_alloc)
u64 counter[1];
#pragma omp allocate(counter) allocator(omp_pteam_mem_alloc)
u64 scratch[4] [[loader_uninitialized]];
#pragma omp allocate(scratch) allocator(omp_pteam_mem_alloc)
u64 zeros[3];
#pragma omp allocate(zeros) allocator(omp_pteam_mem_alloc)
#pragma omp end declare target

u64 out[12];

void kernel(u64 *out, i64 r) {
  #pragma omp target num_teams(3) thread_limit(4)
  {
    u64 old;
    old = __atomic_add(counter, (u64) omp_thread_id() + base);
    __kmpc_barrier(0);
    if (omp_thread_id() == 0) {
      scratch[0] = 77;
      out[omp_team_id() * 4] = counter[0];
      out[omp_team_id() * 4 + 1] = scratch[r];
      out[omp_team_id() * 4 + 2] = zeros[2];
      out[omp_team_id() * 4 + 3] = scratch[0];
    }
  }
}

void main() {
  u32 i;
  kernel(out, 1);
  i = 0;
  while (i < 12) {
    print(out[i]);
    i = i + 1;
  }
}
"""

GLOBAL_DEVICE_DATA = """\
#pragma omp begin declare target
u32 table[4] [[loader_uninitialized]];
u32 seed = 3;
#pragma omp end declare target

u32 out[2];

void kernel(u32 *out, i64 r) {
  #pragma omp target num_teams(1) thread_limit(1)
  {
    table[0] = seed * 7;
    out[0] = table[0];
    out[1] = table[r];
  }
}

void main() {
  kernel(out, 2);
  print(out[0]);
  print(out[1]);
}
"""

UNINIT_SHARED = TEAM_SHARED.replace("num_teams(3)", "num_teams(1)")

# (name, source, run_source kwargs)
PROGRAMS = [
    ("alu", ALU, {}),
    ("alu_wrap", ALU_WRAP, {}),
    ("grid_map", GRID_MAP, {}),
    ("oob_store", OOB_STORE, {}),
    ("oob_load", OOB_LOAD, {}),
    ("div_zero", DIV_ZERO, {}),
    ("deadlock", DEADLOCK, {}),
    ("barrier_ok", BARRIER_OK, {}),
    ("trap_abort", TRAP_ABORT, {}),
    ("arena_overflow", ARENA_OVERFLOW, {}),
    ("arena_non_lifo", ARENA_NON_LIFO, {}),
    ("arena_non_uniform", ARENA_NON_UNIFORM, {}),
    ("team_shared", TEAM_SHARED, {}),
    ("team_shared_uninit_check", UNINIT_SHARED, {"check_uninit": True}),
    ("global_device_data", GLOBAL_DEVICE_DATA, {}),
    ("global_device_data_check", GLOBAL_DEVICE_DATA, {"check_uninit": True}),
]


def main() -> None:
    from forge import corpus
    from forge.host import run_source

    progs = list(PROGRAMS) + [(f"corpus_{n}", s, {}) for n, s in corpus.CORPUS]
    out = {"generator": "oracle/gen_region_golden.py",
           "reference": "forge.host.run_source(device='vgpu') (host.py:959-975)",
           "programs": []}
    for name, src, kw in progs:
        seeds = (0, 3)
        runs = [run_source(src, device="vgpu", sched_seed=s, **kw) for s in seeds]
        r = runs[0]
        for o in runs[1:]:
            assert (o.stdout, o.stderr, o.exit_status) == (r.stdout, r.stderr, r.exit_status), name
        rec = {"name": name, "source": src, "kwargs": kw,
               "stdout": r.stdout, "stderr": r.stderr,
               "exit_status": r.exit_status,
               "offloads": [list(x) for x in r.offloads]}
        if r.exit_status == 0:
            # executed IR instructions per region (host.py:524-528): the sum
            # over threads, the same under every seed when nothing traps
            for o in runs[1:]:
                assert o.device_instructions == r.device_instructions, name
            rec["device_instructions"] = [list(x) for x in r.device_instructions]
        out["programs"].append(rec)
        print(f"{name:28s} exit={r.exit_status} {r.stderr.strip()[:90]}")
    dst = ROOT / "tests" / "golden" / "region_programs.json"
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", dst)


if __name__ == "__main__":
    main()
