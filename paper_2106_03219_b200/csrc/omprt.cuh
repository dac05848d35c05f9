// omprt.cuh — the device runtime: the sm_100a restatement of the reference's
// portable runtime (/root/reference/pkg/src/forge/runtime.mc) plus the pieces
// the combined `target teams distribute parallel for reduction` construct
// lowers to in LLVM's device runtime (__kmpc_for_static_init,
// __kmpc_distribute_static_init, __kmpc_nvptx_{parallel,teams}_reduce_nowait_v2).
//
// Everything here is header-only and is compiled into the single translation
// unit omprt_b200.cu, so the trap word below is one symbol per device.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/omprt_b200.h"

#define OMPRT_HD __host__ __device__ __forceinline__
#define OMPRT_D __device__ __forceinline__

namespace omprt {

// ---------------------------------------------------------------------------
// thread and team queries (runtime.mc:9-59; nvptx64 intrinsic names
// selectors.py:89-92 -> %tid.x, %ctaid.x, %ntid.x, %nctaid.x)
// ---------------------------------------------------------------------------
OMPRT_D uint32_t omp_thread_id() { return threadIdx.x; }
OMPRT_D uint32_t omp_team_id() { return blockIdx.x; }
OMPRT_D uint32_t omp_num_threads() { return blockDim.x; }
OMPRT_D uint32_t omp_num_teams() { return gridDim.x; }
OMPRT_D uint32_t lane_id() { return threadIdx.x & 31u; }
OMPRT_D uint32_t warp_id() { return threadIdx.x >> 5; }

// ---------------------------------------------------------------------------
// worksharing
// ---------------------------------------------------------------------------

// Python floor division (devicert.static_bounds uses `//`, devicert.py:110-115).
// It differs from the IR's truncating sdiv.i64 only when ub < lb.
OMPRT_HD int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

// for_static_init / devicert.static_bounds: block partition of inclusive
// [lb, ub] over n threads; a result with my_lb > ub is empty.
// (runtime.mc:193-203; devicert.py:110-115; fallback host.py:872-883)
OMPRT_HD void static_bounds(int64_t lb, int64_t ub, int64_t tid, int64_t n, int64_t &my_lb,
                            int64_t &my_ub) {
  const int64_t chunk = floordiv(ub - lb + 1 + n - 1, n);
  my_lb = lb + tid * chunk;
  my_ub = my_lb + chunk - 1;
  if (my_ub > ub) my_ub = ub;
}

// What __kmpc_for_static_init hands back to a thread: its first chunk, the
// distance to its next chunk, and whether it executes the last iteration.
struct Bounds {
  int64_t lower;
  int64_t upper;
  int64_t stride;
  int64_t last;
  int64_t limit;  // inclusive upper limit of this thread's chunk loop
};

// kmp_sch_static (unchunked): one block per thread, the reference rule.
OMPRT_HD Bounds block_init(int64_t lb, int64_t ub, int64_t tid, int64_t n) {
  Bounds b;
  static_bounds(lb, ub, tid, n, b.lower, b.upper);
  b.stride = (ub >= lb) ? (ub - lb + 1) : 1;
  b.last = (ub >= lb && b.lower <= ub && b.upper >= ub) ? 1 : 0;
  b.limit = ub;
  return b;
}

// kmp_sch_static_chunked: chunk k (iterations lb+k*c .. lb+k*c+c-1) goes to
// thread k mod n (round robin).  Extension: the reference has no chunk
// parameter; this is OpenMP schedule(static, c).
OMPRT_HD Bounds chunked_init(int64_t lb, int64_t ub, int64_t tid, int64_t n, int64_t c) {
  Bounds b;
  b.lower = lb + tid * c;
  b.upper = b.lower + c - 1;
  if (b.upper > ub) b.upper = ub;
  b.stride = n * c;
  b.last = 0;
  b.limit = ub;
  if (ub >= lb) {
    const int64_t last_chunk = (ub - lb) / c;  // span >= 0, so plain division
    b.last = (last_chunk % n == tid) ? 1 : 0;
  }
  return b;
}

// Nested partition: __kmpc_distribute_static_init gives the team a block of
// [lb, ub] (the reference rule applied over teams), then the team's threads
// partition that block (block rule or chunked).  An empty team block yields
// an empty thread range (lower > upper, lower > ub).
OMPRT_HD Bounds team_block(int64_t lb, int64_t ub, int64_t team, int64_t teams) {
  return block_init(lb, ub, team, teams);
}

OMPRT_HD Bounds schedule_init(int sched, int64_t lb, int64_t ub, int64_t chunk, int64_t team,
                              int64_t teams, int64_t tid, int64_t threads) {
  switch (sched) {
    case OMPRT_SCHED_STATIC:
      return block_init(lb, ub, team * threads + tid, teams * threads);
    case OMPRT_SCHED_STATIC_CHUNKED:
      return chunked_init(lb, ub, team * threads + tid, teams * threads, chunk);
    default: {
      const Bounds tb = team_block(lb, ub, team, teams);
      if (tb.lower > tb.upper) {
        Bounds e;
        e.lower = tb.lower;
        e.upper = tb.upper;
        e.stride = 1;
        e.last = 0;
        e.limit = tb.upper;
        return e;
      }
      Bounds b = (sched == OMPRT_SCHED_DISTRIBUTE)
                     ? block_init(tb.lower, tb.upper, tid, threads)
                     : chunked_init(tb.lower, tb.upper, tid, threads, chunk);
      b.last = (b.last && tb.last) ? 1 : 0;
      return b;
    }
  }
}

// The set of iterations a whole team owns, as `nseg` segments of `seg_len`
// consecutive iterations starting at `first`, `seg_stride` apart, the last
// one clipped to ub.  Contiguous (nseg <= 1) for every schedule except the
// flat chunked one, whose team set is a comb of threads*chunk-wide teeth.
// This is what lets the lanes of a team cover its iterations coalesced while
// every OpenMP thread's iteration set stays exactly what schedule_init says.
struct TeamSet {
  int64_t first;
  int64_t seg_len;
  int64_t seg_stride;
  int64_t nseg;
  int64_t ub;
};

OMPRT_HD TeamSet team_set(int sched, int64_t lb, int64_t ub, int64_t chunk, int64_t team,
                          int64_t teams, int64_t threads) {
  TeamSet s;
  s.ub = ub;
  s.seg_stride = 0;
  if (sched == OMPRT_SCHED_STATIC) {
    // union of the blocks of g = team*threads .. team*threads+threads-1
    const int64_t n = teams * threads;
    const int64_t c = floordiv(ub - lb + 1 + n - 1, n);
    s.first = lb + team * threads * c;
    int64_t last = s.first + threads * c - 1;
    if (last > ub) last = ub;
    s.seg_len = last - s.first + 1;
    s.nseg = (s.seg_len > 0 && s.first <= ub) ? 1 : 0;
    if (s.nseg == 0) s.seg_len = 0;
  } else if (sched == OMPRT_SCHED_STATIC_CHUNKED) {
    const int64_t n = teams * threads;
    s.first = lb + team * threads * chunk;
    s.seg_len = threads * chunk;
    s.seg_stride = n * chunk;
    s.nseg = (ub >= s.first) ? ((ub - s.first) / s.seg_stride + 1) : 0;
  } else {
    const Bounds tb = team_block(lb, ub, team, teams);
    s.first = tb.lower;
    s.seg_len = (tb.upper >= tb.lower) ? (tb.upper - tb.lower + 1) : 0;
    s.nseg = s.seg_len > 0 ? 1 : 0;
  }
  return s;
}

// ---------------------------------------------------------------------------
// reduction operators (the combine of __atomic_add/max/min: step_add/max/min
// devicert.py:84-95; signed compares for i32/i64 vgpu.py:608-617)
// ---------------------------------------------------------------------------
template <class T> struct Limits;
template <> struct Limits<int32_t> {
  static OMPRT_HD int32_t lowest() { return INT32_MIN; }
  static OMPRT_HD int32_t highest() { return INT32_MAX; }
};
template <> struct Limits<uint32_t> {
  static OMPRT_HD uint32_t lowest() { return 0u; }
  static OMPRT_HD uint32_t highest() { return 0xffffffffu; }
};
template <> struct Limits<int64_t> {
  static OMPRT_HD int64_t lowest() { return INT64_MIN; }
  static OMPRT_HD int64_t highest() { return INT64_MAX; }
};
template <> struct Limits<uint64_t> {
  static OMPRT_HD uint64_t lowest() { return 0ull; }
  static OMPRT_HD uint64_t highest() { return ~0ull; }
};
template <> struct Limits<float> {
  static OMPRT_HD float lowest() { return -__builtin_inff(); }
  static OMPRT_HD float highest() { return __builtin_inff(); }
};
template <> struct Limits<double> {
  static OMPRT_HD double lowest() { return -__builtin_inf(); }
  static OMPRT_HD double highest() { return __builtin_inf(); }
};

// Wrapping add (mod 2^bits) without signed-overflow UB.
template <class T> OMPRT_HD T wrap_add(T a, T b) { return a + b; }
template <> OMPRT_HD int32_t wrap_add<int32_t>(int32_t a, int32_t b) {
  return (int32_t)((uint32_t)a + (uint32_t)b);
}
template <> OMPRT_HD int64_t wrap_add<int64_t>(int64_t a, int64_t b) {
  return (int64_t)((uint64_t)a + (uint64_t)b);
}

template <int OP, class T> struct Red;
template <class T> struct Red<OMPRT_OP_ADD, T> {
  static OMPRT_HD T identity() { return T(0); }
  static OMPRT_HD T apply(T acc, T e) { return wrap_add<T>(acc, e); }
};
template <class T> struct Red<OMPRT_OP_MAX, T> {
  static OMPRT_HD T identity() { return Limits<T>::lowest(); }
  // step_max: new = e if x < e else x
  static OMPRT_HD T apply(T acc, T e) { return acc < e ? e : acc; }
};
template <class T> struct Red<OMPRT_OP_MIN, T> {
  static OMPRT_HD T identity() { return Limits<T>::highest(); }
  // step_min: new = e if x > e else x
  static OMPRT_HD T apply(T acc, T e) { return acc > e ? e : acc; }
};

// ---------------------------------------------------------------------------
// memory access primitives
// ---------------------------------------------------------------------------

// 128-bit streaming load through the non-coherent path, no L1 allocation,
// 256-byte L2 sector promotion (the whole input is read exactly once).
OMPRT_D uint4 ld_stream_v4(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Load-policy variants of the streaming load (tuning; kLoadDefault is what
// every kernel uses unless a tuned variant is selected).
enum LoadPolicy : int {
  kLoadNcL2_256B = 0,  // ld.global.nc.L1::no_allocate.L2::256B
  kLoadNc = 1,         // ld.global.nc.L1::no_allocate
  kLoadEvictFirst = 2, // ld.global.nc.L1::no_allocate.L2::evict_first
  kLoadPlain = 3,      // ld.global.nc (LDG.CONSTANT, L1 allocating)
  kLoadDefault = kLoadNcL2_256B
};

template <int LP> OMPRT_D uint4 ld_v4(const void *p) {
  uint4 r;
  if constexpr (LP == kLoadNcL2_256B) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  } else if constexpr (LP == kLoadNc) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  } else {
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
  }
  return r;
}

// 256-bit loads (sm_100: LDG.E.256): 32 bytes per lane per instruction.
struct U8x32 {
  uint4 lo, hi;
};

template <int LP> OMPRT_D U8x32 ld_v8(const void *p) {
  U8x32 r;
  if constexpr (LP == kLoadNcL2_256B) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.lo.x), "=r"(r.lo.y), "=r"(r.lo.z), "=r"(r.lo.w), "=r"(r.hi.x),
                   "=r"(r.hi.y), "=r"(r.hi.z), "=r"(r.hi.w)
                 : "l"(p));
  } else if constexpr (LP == kLoadEvictFirst) {
    asm volatile(
        "ld.global.nc.L1::no_allocate.L2::evict_first.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
        : "=r"(r.lo.x), "=r"(r.lo.y), "=r"(r.lo.z), "=r"(r.lo.w), "=r"(r.hi.x), "=r"(r.hi.y),
          "=r"(r.hi.z), "=r"(r.hi.w)
        : "l"(p));
  } else {
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.lo.x), "=r"(r.lo.y), "=r"(r.lo.z), "=r"(r.lo.w), "=r"(r.hi.x),
                   "=r"(r.hi.y), "=r"(r.hi.z), "=r"(r.hi.w)
                 : "l"(p));
  }
  return r;
}

// 128-bit load of data that this kernel also writes (y in axpy): coherent path.
OMPRT_D uint4 ld_rw_v4(const void *p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

OMPRT_D void st_stream_v4(void *p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// L2-coherent scalar load (bypasses a possibly stale L1 line) for data other
// teams published before a fence.
template <class T> OMPRT_D T ld_cg(const T *p) { return __ldcg(p); }

// ---------------------------------------------------------------------------
// fences, barriers, scoped atomics (runtime.mc:95-186; nvptx64 names
// __nvvm_membar_gl, __nvvm_barrier0, __nvvm_atom_inc_gen_ui, selectors.py:84-93)
// ---------------------------------------------------------------------------

// __kmpc_flush / __kmpc_impl_threadfence: device-scope sequentially
// consistent fence (fence.sc.gpu).
OMPRT_D void kmpc_flush() { asm volatile("fence.sc.gpu;" ::: "memory"); }
OMPRT_D void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
OMPRT_D void fence_acq_rel_cta() { asm volatile("fence.acq_rel.cta;" ::: "memory"); }

// __kmpc_barrier / __kmpc_impl_syncthreads: barrier 0 over the whole team.
OMPRT_D void kmpc_barrier() { __syncthreads(); }

// Named barriers: barrier.sync / barrier.arrive id, n (the non-.aligned
// forms: each thread arrives on its own, so a warp need not be converged);
// n counts threads and is a multiple of the warp size here.
OMPRT_D void named_barrier_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
OMPRT_D void named_barrier_arrive(uint32_t id, uint32_t nthreads) {
  asm volatile("barrier.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// atomic_inc (runtime.mc:175-186; step_inc devicert.py:105-107):
// old >= e ? 0 : old + 1, acquire-release at device scope.
OMPRT_D uint32_t atomic_inc_acq_rel_gpu(uint32_t *p, uint32_t e) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;"
               : "=r"(old)
               : "l"(p), "r"(e)
               : "memory");
  return old;
}

// ---------------------------------------------------------------------------
// trap word: a cooperative replacement for __trap(code) (intrinsics.py:46).
// PTX `trap` would poison the CUDA context, so the first trapping thread wins
// a CAS, records {kind, code, team, thread}, and the kernel unwinds; the host
// maps it to status 2 (host.py:289-292).
// ---------------------------------------------------------------------------
struct TrapWord {
  int kind;
  int code;
  int team;
  int thread;
};

// Defined here: the library is one translation unit (omprt_b200.cu).
__device__ TrapWord g_trap;

OMPRT_D void raise_trap(int kind, int code) {
  if (atomicCAS(&g_trap.kind, 0, kind) == 0) {
    g_trap.code = code;
    g_trap.team = (int)blockIdx.x;
    g_trap.thread = (int)threadIdx.x;
  }
  __threadfence();
}

OMPRT_D bool trap_raised() { return *(volatile int *)&g_trap.kind != 0; }

// ---------------------------------------------------------------------------
// per-team trace ring (the B200 analog of the vgpu's collect_trace,
// vgpu.py:351-353): when a buffer is installed (omprt_set_trace), thread 0 of
// every CTA of a construct records when the team started, on which SM, when
// it took its ticket and which ticket value the atom.inc returned; the last
// team adds a record for the ordered combine.  One record per CTA, indexed by
// blockIdx.x (+ gridDim.x for the combine); nothing is written when the
// buffer is absent (one global load per CTA).
// ---------------------------------------------------------------------------
struct TraceRec {
  uint64_t t_begin, t_end;  // %globaltimer, ns
  uint32_t cta, smid, ticket, kind;
};
enum : uint32_t { kTraceTeam = 1, kTraceCombine = 2, kTraceGroup = 3, kTraceFolder = 4 };
struct TraceRing {
  TraceRec *recs;
  uint32_t cap;
};
// constant bank: every CTA reads it at start and end, so it must cost nothing
// when no ring is installed (a global would put an L2 round trip on each
// short team's critical path)
__constant__ TraceRing g_trace;

OMPRT_D uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
OMPRT_D uint32_t smid() {
  uint32_t v;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
  return v;
}
OMPRT_D uint64_t &trace_t0() {
  __shared__ uint64_t t0;
  return t0;
}
// thread 0, at the top of a construct kernel
// Programmatic dependent launch: a construct launched with the PDL launch
// attribute may start while the previous kernel of its stream drains; it
// waits for that kernel's completion (and memory) before touching global
// memory, and lets its own dependents launch at once (they wait the same
// way, and only launch once every CTA of this grid has started).  Both are
// no-ops for a kernel launched without the attribute.
OMPRT_D void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

OMPRT_D void trace_begin() {
  pdl_begin();
  if (threadIdx.x == 0 && g_trace.recs) trace_t0() = globaltimer();
}
// thread 0: record slot `slot` (CTA index, or gridDim.x + k for extras)
OMPRT_D void trace_record(uint32_t slot, uint32_t kind, uint32_t ticket, uint64_t t0) {
  const TraceRing r = g_trace;
  if (r.recs && slot < r.cap) {
    TraceRec rec;
    rec.t_begin = t0;
    rec.t_end = globaltimer();
    rec.cta = blockIdx.x;
    rec.smid = smid();
    rec.ticket = ticket;
    rec.kind = kind;
    r.recs[slot] = rec;
  }
}

// ---------------------------------------------------------------------------
// team reductions: warp __shfl_xor_sync tree, then a shared-memory tree over
// the warps (__kmpc_nvptx_parallel_reduce_nowait_v2).  Handles a partial last
// warp (threads not a multiple of 32).  The result is valid in thread 0.
// `scratch` needs 32 slots and is free again after the call returns.
// ---------------------------------------------------------------------------
template <class T> OMPRT_D T shfl_xor(T v, int m, unsigned mask) {
  return __shfl_xor_sync(mask, v, m);
}

template <int OP, class T> OMPRT_D T warp_reduce(T v, uint32_t nact) {
  const uint32_t lane = lane_id();
  if (nact >= 32) {
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v = Red<OP, T>::apply(v, shfl_xor(v, m, 0xffffffffu));
  } else {
    const unsigned mask = (nact == 0) ? 0u : ((1u << nact) - 1u);
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      const T o = shfl_xor(v, m, mask);
      if ((lane ^ (uint32_t)m) < nact) v = Red<OP, T>::apply(v, o);
    }
  }
  return v;
}

// Reduce `v` over the first `nthreads` threads of the block (all of them must
// call).  Uses `scratch[0..31]`; ends with a barrier so scratch can be reused.
template <int OP, class T>
OMPRT_D T block_reduce(T v, T *scratch, uint32_t nthreads) {
  const uint32_t lane = lane_id(), warp = warp_id();
  const uint32_t nwarps = (nthreads + 31) >> 5;
  const uint32_t nact = (warp == nwarps - 1) ? (nthreads - warp * 32) : 32;
  v = warp_reduce<OP, T>(v, nact);
  if (nwarps == 1) return v;
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  if (warp == 0) {
    T w = (lane < nwarps) ? scratch[lane] : Red<OP, T>::identity();
    v = warp_reduce<OP, T>(w, 32);
  }
  __syncthreads();
  return v;
}

// The same over a subset of warps synchronised with a named barrier
// (generic-mode parallel regions exclude the main warp).  `first_warp` is the
// first hardware warp of the subset; nthreads a multiple of 32.
template <int OP, class T>
OMPRT_D T warps_reduce_named(T v, volatile T *scratch, uint32_t first_warp, uint32_t nthreads,
                             uint32_t bar_id) {
  const uint32_t lane = lane_id();
  const uint32_t w = warp_id() - first_warp;
  const uint32_t nwarps = nthreads >> 5;
  v = warp_reduce<OP, T>(v, 32);
  if (lane == 0) scratch[w] = v;
  named_barrier_sync(bar_id, nthreads);
  if (w == 0) {
    T x = (lane < nwarps) ? scratch[lane] : Red<OP, T>::identity();
    v = warp_reduce<OP, T>(x, 32);
  }
  return v;
}

// ---------------------------------------------------------------------------
// splitmix64 counter-based synthetic data (shared with the oracle's
// restatement).
// ---------------------------------------------------------------------------
OMPRT_HD uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

OMPRT_HD uint64_t gen_bits(uint64_t seed, int k, uint64_t i) {
  return splitmix64(seed ^ ((uint64_t)k << 56) ^ i);
}

template <class T> OMPRT_HD T gen_value(uint64_t h);
template <> OMPRT_HD int64_t gen_value<int64_t>(uint64_t h) { return ((int64_t)h) >> 24; }
template <> OMPRT_HD uint64_t gen_value<uint64_t>(uint64_t h) { return h >> 24; }
template <> OMPRT_HD int32_t gen_value<int32_t>(uint64_t h) {
  return ((int32_t)(uint32_t)(h >> 32)) >> 8;
}
template <> OMPRT_HD uint32_t gen_value<uint32_t>(uint64_t h) { return (uint32_t)(h >> 40); }
template <> OMPRT_HD double gen_value<double>(uint64_t h) {
  return (double)(h >> 11) * 0x1.0p-53;
}
template <> OMPRT_HD float gen_value<float>(uint64_t h) { return (float)(h >> 40) * 0x1.0p-24f; }

}  // namespace omprt
