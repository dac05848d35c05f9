// region_rt.cuh — device runtime for compiled target regions (B200 images).
//
// regionc.py translates a forge device image (the nvptx64 IR the reference
// emits, codegen.py / ir.py) into CUDA C++ that runs every OpenMP thread of
// the region as a real sm_100a thread: team = CTA, thread = CTA thread.  This
// header is prepended to that translation and compiled by NVRTC, so it is
// self-contained (no includes).  It supplies what the IR's instructions mean
// on the vgpu (vgpu.py:384-625), restated for the hardware:
//
//   * fat pointers carrying their allocation bounds, so elem.addr / ld / st
//     trap OutOfBounds exactly where the vgpu does (vgpu.py:352-363, 446-456);
//   * team-shared globals in dynamic shared memory, poisoned with 0xAA unless
//     initialised (loader_uninitialized, vgpu.py:234-250), with the optional
//     per-byte init shadow of check_uninit (vgpu.py:64-77, 365-369);
//   * seq_cst atomics at device scope (fence.sc.gpu around the RMW; vgpu.py:586-625),
//     atom.inc for __nvvm_atom_inc_gen_ui (devicert.step_inc);
//   * the team barrier as a non-.aligned `barrier.red.or.pred` whose predicate
//     says "this thread has finished": a barrier that meets a finished thread
//     can never release on the vgpu and traps Deadlock (vgpu.py:289-298);
//   * traps: the first trapping thread records {kind, site, team, thread, aux}
//     in the launch's trap record and every trapping thread exits (PTX `exit`
//     signals barriers waiting only on exited threads; `trap` would poison the
//     context).  Loops poll the record so a trapped launch drains quickly.
#pragma once

typedef unsigned int u32;
typedef int i32;
typedef unsigned long long u64;
typedef long long i64;
typedef unsigned char u8;

#define RT_D __device__ __forceinline__

enum : u32 {  // omprt_trap_kind (include/omprt_b200.h) == vgpu TrapKind order
  RT_SHARED_OVERFLOW = 1,
  RT_NON_LIFO_FREE = 2,
  RT_NON_UNIFORM_ALLOC = 3,
  RT_UNINITIALIZED_READ = 4,
  RT_OUT_OF_BOUNDS = 5,
  RT_DEADLOCK = 6,
  RT_DIVIDE_BY_ZERO = 7,
  RT_ABORT = 8
};

enum : u32 { RT_GLOBAL = 0, RT_SHARED = 1, RT_SLOT = 2 };

// Per-launch trap record (host reads it after the launch; omprt_region_launch).
struct RtTrap {
  u32 flag;    // 0 none, 1 being written, 2 complete
  u32 kind;
  u32 site;    // trap site id (the image manifest maps it to the vgpu message)
  u32 team;
  u32 thread;
  u32 pad;
  u64 aux[4];
};

// A pointer value: vgpu's Ptr(space, off, lo, hi) (vgpu.py:79-89).
struct P {
  u8 *p;    // current address
  u8 *lo;   // allocation start
  u8 *hi;   // allocation end (exclusive)
  u8 *sh;   // init shadow of `lo` (check_uninit), or null: always initialised
  u64 vlo;  // vgpu offset of `lo` inside its space (messages only)
  u32 space;
  u32 label;  // RT_SHARED: team; RT_SLOT: slot name id
};

struct RtCtx {
  RtTrap *trap;
  u8 *globals;      // global-space globals, vgpu layout (vgpu.py:171-207)
  u8 *gshadow;      // their init shadow (check_uninit) or null
  u8 *sshadow;      // this team's team-shared init shadow or null
  u32 *waitmask;    // per team 32 words: threads caught in a dead barrier
  u64 seed;         // sched_seed (0: the hardware's own interleaving)
};

// The launch record after the trap (regions.launch allocates 128 bytes):
// byte 56 the executed-IR-instruction counter (vgpu ExecResult
// .instruction_count, vgpu.py:390), byte 64 the sched_seed.
constexpr u32 kRtCountOff = 56, kRtSeedOff = 64;

__shared__ RtCtx rt_ctx;

RT_D u64 rt_mask(u64 v, int bits) { return bits == 32 ? (v & 0xffffffffull) : v; }
RT_D i64 rt_sext(u64 v, int bits) { return bits == 32 ? (i64)(i32)(u32)v : (i64)v; }

__device__ __noinline__ void rt_trap(u32 kind, u32 site, u64 a0, u64 a1, u64 a2, u64 a3) {
  RtTrap *t = rt_ctx.trap;
  if (atomicCAS(&t->flag, 0u, 1u) == 0u) {
    t->kind = kind;
    t->site = site;
    t->team = blockIdx.x;
    t->thread = threadIdx.x;
    t->aux[0] = a0;
    t->aux[1] = a1;
    t->aux[2] = a2;
    t->aux[3] = a3;
    __threadfence();
    atomicExch(&t->flag, 2u);
  }
  asm volatile("exit;");
  __builtin_unreachable();
}

// Loop back-edges: leave once any thread of the launch trapped.
RT_D void rt_poll() {
  if (*(volatile u32 *)&rt_ctx.trap->flag) asm volatile("exit;");
}

RT_D u32 rt_bar_or(u32 pred) {
  u32 r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "barrier.red.or.pred q, 0, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(pred)
      : "memory");
  return r;
}

// __nvvm_barrier0 / vgpu.barrier (vgpu.py:490-495, 627-631)
__device__ __noinline__ void rt_barrier(u32 site) {
  if (rt_bar_or(0u)) {
    atomicOr(&rt_ctx.waitmask[blockIdx.x * 32u + (threadIdx.x >> 5)], 1u << (threadIdx.x & 31u));
    rt_trap(RT_DEADLOCK, site, 0, 0, 0, 0);
  }
}

// the end of the region for this thread: a finished thread
RT_D void rt_finish() { (void)rt_bar_or(1u); }

// This thread's executed IR instructions (every basic block adds its length
// on entry, as the vgpu counts one per _step) into the launch's counter.
RT_D void rt_count(u64 n) {
  atomicAdd((unsigned long long *)((u8 *)rt_ctx.trap + kRtCountOff), (unsigned long long)n);
}

// Seeded interleaving (the vgpu's sched_seed, vgpu.py:285-306): with a
// nonzero seed every thread sleeps before each atomic and barrier for a
// splitmix64-drawn time keyed by (seed, team, warp, instructions executed so
// far) — 0..4095 ns, the same for the whole warp, so warps really do arrive
// in different orders (a per-lane draw made every warp wait for its slowest
// lane, ~2 us, and two warps then raced as without a seed) — plus a per-lane
// 0..255 ns.  A seed perturbs which thread reaches a racing operation first
// and different seeds explore different orders; the hardware still decides
// the final order, so a seed does not replay a schedule bit for bit; seed 0
// keeps the hardware's own interleaving.
RT_D u64 rt_mix(u64 z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
RT_D void rt_jitter(u64 k) {
  const u64 seed = rt_ctx.seed;
  if (seed == 0) return;
  const u64 base = seed ^ ((u64)blockIdx.x << 40) ^ (k * 0x9e3779b97f4a7c15ull);
  const u64 zw = rt_mix(base ^ ((u64)(threadIdx.x >> 5) << 24));
  const u64 zl = rt_mix(base ^ ((u64)threadIdx.x << 20) ^ 0x5bd1e995ull);
  __nanosleep((u32)(zw & 4095u) + (u32)(zl & 255u));
}

RT_D u64 rt_label(const P &p) { return ((u64)p.space << 32) | p.label; }

// elem.addr.T base, idx (vgpu.py:446-456): idx is the operand's masked value
RT_D P rt_elem(P b, u64 idx, u32 w, u32 site) {
  const u64 avail = (u64)(b.hi - b.p);
  if (b.p < b.lo || idx > avail / w || idx * w + w > avail)
    rt_trap(RT_OUT_OF_BOUNDS, site, idx, b.vlo, b.vlo + (u64)(b.hi - b.lo), rt_label(b));
  b.p += idx * w;
  return b;
}

RT_D u64 rt_off(const P &p) { return p.vlo + (u64)(p.p - p.lo); }

RT_D void rt_check(const P &p, u32 w, u32 site) {
  if (p.p < p.lo || p.p + w > p.hi) rt_trap(RT_OUT_OF_BOUNDS, site, w, rt_off(p), 0, rt_label(p));
  if (p.sh) {  // shadow present only under check_uninit
    const u8 *s = p.sh + (p.p - p.lo);
    for (u32 i = 0; i < w; ++i)
      if (!((volatile const u8 *)s)[i]) rt_trap(RT_UNINITIALIZED_READ, site, w, rt_off(p), 0, rt_label(p));
  }
}

RT_D void rt_mark(const P &p, u32 w) {
  if (p.sh) {
    u8 *s = p.sh + (p.p - p.lo);
    for (u32 i = 0; i < w; ++i) ((volatile u8 *)s)[i] = 1;
  }
}

RT_D u64 rt_raw_ld(const P &p, u32 w) {
  if (((unsigned long long)p.p & (w - 1)) == 0)
    return w == 4 ? (u64)*(volatile const u32 *)p.p : *(volatile const u64 *)p.p;
  u64 v = 0;
  for (u32 i = 0; i < w; ++i) v |= (u64)((volatile const u8 *)p.p)[i] << (8 * i);
  return v;
}

RT_D void rt_raw_st(const P &p, u32 w, u64 v) {
  if (((unsigned long long)p.p & (w - 1)) == 0) {
    if (w == 4)
      *(volatile u32 *)p.p = (u32)v;
    else
      *(volatile u64 *)p.p = v;
    return;
  }
  for (u32 i = 0; i < w; ++i) ((volatile u8 *)p.p)[i] = (u8)(v >> (8 * i));
}

// ld.T (vgpu.py:457-462, _load 352-363)
RT_D u64 rt_ld(const P &p, u32 w, u32 site) {
  rt_check(p, w, site);
  return rt_raw_ld(p, w);
}

// st.T (vgpu.py:463-468, _store 365-371)
RT_D void rt_st(const P &p, u32 w, u64 v, u32 site) {
  if (p.p < p.lo || p.p + w > p.hi) rt_trap(RT_OUT_OF_BOUNDS, site, w, rt_off(p), 0, rt_label(p));
  rt_raw_st(p, w, v);
  rt_mark(p, w);
}

// atomic.<kind>.seq_cst.<ty> (vgpu.py:586-625).  Private slots are
// thread-local, so their RMW is a plain load/store; global and team-shared
// cells use the hardware atomics bracketed by fence.sc.gpu.
enum : u32 { RT_A_ADD = 0, RT_A_MAX = 1, RT_A_MIN = 2, RT_A_XCHG = 3, RT_A_CAS = 4, RT_A_INC = 5 };

RT_D u64 rt_rmw_value(u32 kind, bool sgn, int bits, u64 old, u64 e, u64 d) {
  switch (kind) {
    case RT_A_ADD: return rt_mask(old + e, bits);
    case RT_A_XCHG: return e;
    case RT_A_MAX:
      if (sgn) return rt_sext(old, bits) < rt_sext(e, bits) ? e : old;
      return old < e ? e : old;
    case RT_A_MIN:
      if (sgn) return rt_sext(old, bits) > rt_sext(e, bits) ? e : old;
      return old > e ? e : old;
    case RT_A_CAS: return old == e ? d : old;
    default: return old >= e ? 0 : old + 1;  // RT_A_INC: devicert.step_inc
  }
}

// 128-bit compare-and-swap (atom.cas.b128, sm_90+; generic address: global
// or shared).  Returns the previous 16 bytes.
RT_D unsigned __int128 rt_cas128(void *a, unsigned __int128 e, unsigned __int128 d) {
  u64 olo, ohi;
  asm volatile(
      "{\n\t.reg .b128 e, d, o;\n\t"
      "mov.b128 e, {%2, %3};\n\t"
      "mov.b128 d, {%4, %5};\n\t"
      "atom.cas.b128 o, [%6], e, d;\n\t"
      "mov.b128 {%0, %1}, o;\n\t}"
      : "=l"(olo), "=l"(ohi)
      : "l"((u64)e), "l"((u64)(e >> 64)), "l"((u64)d), "l"((u64)(d >> 64)), "l"(a)
      : "memory");
  return ((unsigned __int128)ohi << 64) | olo;
}

// A cell that is not naturally aligned (the vgpu's RMW is atomic at any byte
// offset, vgpu.py:586-625): compare-and-swap loop on the enclosing aligned
// 8-byte word, or 16-byte line (atom.cas.b128) when the cell straddles two
// words; a cell straddling a 16-byte line cannot be updated by one hardware
// RMW and traps Abort instead of losing updates.
__device__ __noinline__ u64 rt_atomic_unaligned(const P &p, u32 kind, bool sgn, u32 w, u64 e,
                                                u64 d, u32 site) {
  const int bits = (int)w * 8;
  const u64 m = bits == 32 ? 0xffffffffull : ~0ull;
  const unsigned long long addr = (unsigned long long)p.p;
  if ((addr & 7) + w <= 8) {
    unsigned long long *word = (unsigned long long *)(addr & ~7ull);
    const int sh = (int)(addr & 7) * 8;
    unsigned long long cur = *(volatile unsigned long long *)word;
    for (;;) {
      const u64 old = (cur >> sh) & m;
      const u64 nv = rt_rmw_value(kind, sgn, bits, old, e, d) & m;
      const unsigned long long nxt = (cur & ~(m << sh)) | (nv << sh);
      const unsigned long long prev = atomicCAS(word, cur, nxt);
      if (prev == cur) return old;
      cur = prev;
    }
  }
  if ((addr & 15) + w <= 16) {
    void *line = (void *)(addr & ~15ull);
    const int sh = (int)(addr & 15) * 8;
    const unsigned __int128 mm = (unsigned __int128)m << sh;
    unsigned __int128 cur = ((unsigned __int128)((volatile u64 *)line)[1] << 64) |
                            ((volatile u64 *)line)[0];
    for (;;) {
      const u64 old = (u64)(cur >> sh) & m;
      const u64 nv = rt_rmw_value(kind, sgn, bits, old, e, d) & m;
      const unsigned __int128 nxt = (cur & ~mm) | ((unsigned __int128)nv << sh);
      const unsigned __int128 prev = rt_cas128(line, cur, nxt);
      if (prev == cur) return old;
      cur = prev;
    }
  }
  rt_trap(RT_ABORT, site, w, rt_off(p), 0, rt_label(p));
  return 0;
}

__device__ __noinline__ u64 rt_atomic(const P &p, u32 kind, bool sgn, u32 w, u64 e, u64 d,
                                      u32 site_ld, u32 site_st) {
  rt_check(p, w, site_ld);
  if (p.p + w > p.hi) rt_trap(RT_OUT_OF_BOUNDS, site_st, w, rt_off(p), 0, rt_label(p));
  const int bits = (int)w * 8;
  u64 old;
  if (p.space == RT_SLOT) {
    old = rt_raw_ld(p, w);
    rt_raw_st(p, w, rt_rmw_value(kind, sgn, bits, old, e, d));
  } else if (((unsigned long long)p.p & (w - 1)) != 0) {
    __threadfence();
    old = rt_atomic_unaligned(p, kind, sgn, w, e, d, site_st);
    __threadfence();
  } else {
    __threadfence();
    if (w == 4) {
      u32 *a = (u32 *)p.p;
      switch (kind) {
        case RT_A_ADD: old = atomicAdd(a, (u32)e); break;
        case RT_A_XCHG: old = atomicExch(a, (u32)e); break;
        case RT_A_MAX: old = sgn ? (u32)atomicMax((int *)a, (int)(u32)e) : atomicMax(a, (u32)e); break;
        case RT_A_MIN: old = sgn ? (u32)atomicMin((int *)a, (int)(u32)e) : atomicMin(a, (u32)e); break;
        case RT_A_CAS: old = atomicCAS(a, (u32)e, (u32)d); break;
        default: old = atomicInc(a, (u32)e); break;
      }
    } else {
      unsigned long long *a = (unsigned long long *)p.p;
      switch (kind) {
        case RT_A_ADD: old = atomicAdd(a, e); break;
        case RT_A_XCHG: old = atomicExch(a, e); break;
        case RT_A_MAX:
          old = sgn ? (u64)atomicMax((long long *)a, (long long)e) : atomicMax(a, e);
          break;
        case RT_A_MIN:
          old = sgn ? (u64)atomicMin((long long *)a, (long long)e) : atomicMin(a, e);
          break;
        case RT_A_CAS: old = atomicCAS(a, e, d); break;
        default: old = 0; break;  // INC is u32-only (codegen.py:70-71)
      }
    }
    __threadfence();
  }
  rt_mark(p, w);
  return rt_mask(old, bits);
}

// ALU (vgpu.py:528-565): values are kept masked to their width.
RT_D u64 rt_shl(u64 a, u64 b, int bits) { return rt_mask(a << (b % (u64)bits), bits); }
RT_D u64 rt_lshr(u64 a, u64 b, int bits) { return a >> (b % (u64)bits); }
RT_D u64 rt_ashr(u64 a, u64 b, int bits) { return rt_mask((u64)(rt_sext(a, bits) >> (b % (u64)bits)), bits); }

RT_D u64 rt_div(u32 op, u64 a, u64 b, int bits, u32 site) {
  if (b == 0) rt_trap(RT_DIVIDE_BY_ZERO, site, 0, 0, 0, 0);
  if (op == 0) return a / b;  // udiv
  if (op == 1) return a % b;  // urem
  const i64 sa = rt_sext(a, bits), sb = rt_sext(b, bits);
  if (sb == -1) return op == 2 ? rt_mask((u64)0 - a, bits) : 0;  // wraps like the vgpu
  return op == 2 ? rt_mask((u64)(sa / sb), bits) : rt_mask((u64)(sa % sb), bits);
}

RT_D u64 rt_cast(u64 v, int src_bits, bool src_signed, int dst_bits) {
  const u64 w = src_signed ? (u64)rt_sext(v, src_bits) : v;
  return rt_mask(w, dst_bits);
}

RT_D P rt_slot_ptr(void *base, u32 bytes, u32 label) {
  P r;
  r.p = r.lo = (u8 *)base;
  r.hi = r.lo + bytes;
  r.sh = nullptr;
  r.vlo = 0;
  r.space = RT_SLOT;
  r.label = label;
  return r;
}

RT_D P rt_global_ptr(u64 off, u32 bytes) {
  P r;
  r.p = r.lo = rt_ctx.globals + off;
  r.hi = r.lo + bytes;
  r.sh = rt_ctx.gshadow ? rt_ctx.gshadow + off : nullptr;
  r.vlo = off;
  r.space = RT_GLOBAL;
  r.label = 0;
  return r;
}

extern __shared__ __align__(16) u8 rt_team_shared[];

RT_D P rt_shared_ptr(u64 off, u32 bytes) {
  P r;
  r.p = r.lo = rt_team_shared + off;
  r.hi = r.lo + bytes;
  r.sh = rt_ctx.sshadow ? rt_ctx.sshadow + off : nullptr;
  r.vlo = off;
  r.space = RT_SHARED;
  r.label = blockIdx.x;
  return r;
}

// a buffer argument: device pointer, byte length, vgpu offset
RT_D P rt_arg_ptr(u64 ptr, u64 bytes, u64 voff) {
  P r;
  r.p = r.lo = (u8 *)ptr;
  r.hi = r.lo + bytes;
  r.sh = nullptr;
  r.vlo = voff;
  r.space = RT_GLOBAL;
  r.label = 0;
  return r;
}

// Kernel prologue: the launch context, then the team-shared space built like
// vgpu._build_shared (vgpu.py:234-250): poison everything, zero the globals
// that are not loader_uninitialized, write an initialiser into element 0.
RT_D void rt_prologue(const u64 *v, u32 shared_bytes) {
  if (threadIdx.x == 0) {
    rt_ctx.trap = (RtTrap *)v[0];
    rt_ctx.globals = (u8 *)v[1];
    rt_ctx.gshadow = (u8 *)v[2];
    rt_ctx.sshadow = v[3] ? (u8 *)v[3] + (u64)blockIdx.x * shared_bytes : nullptr;
    rt_ctx.waitmask = (u32 *)v[4];
    rt_ctx.seed = *(const u64 *)((const u8 *)v[0] + kRtSeedOff);
  }
  for (u32 i = threadIdx.x; i < shared_bytes; i += blockDim.x) rt_team_shared[i] = 0xAA;
  __syncthreads();
}

RT_D void rt_shared_init(u64 off, u32 bytes, int init_kind, u64 value, u32 width) {
  // init_kind: 0 "zero", 1 integer initialiser, 2 "none" (stays poison)
  if (init_kind == 2) return;
  for (u32 i = threadIdx.x; i < bytes; i += blockDim.x) {
    u8 b = 0;
    if (init_kind == 1 && i < width) b = (u8)(value >> (8 * i));
    rt_team_shared[off + i] = b;
    if (rt_ctx.sshadow) rt_ctx.sshadow[off + i] = 1;
  }
}
