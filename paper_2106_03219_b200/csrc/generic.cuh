// generic.cuh — the team-shared smart stack (__kmpc_alloc_shared /
// __kmpc_free_shared), generic-mode execution on named barriers, and the
// scoped-atomic probe.
//
// Reference: runtime.mc:67-91 (arena), devicert.Arena devicert.py:124-148
// (semantics and trap codes 1/2/3), vgpu.py:171-250 (team-shared layout,
// poison 0xAA for loader_uninitialized), runtime.mc:136-186 (atomics).
#pragma once

#include <cuda/atomic>

#include "kernels.cuh"

namespace omprt {

// ------------------------------------------------------------------ arena
//
// Offsets are byte offsets, as the reference returns (runtime.mc:73-84).
// [0, capacity) lives in this team's shared memory.  With heap_fallback the
// arena continues into a per-team slice of global memory: offsets
// >= capacity address heap byte (off - capacity).  Once an allocation spills,
// later allocations also go to the heap until the heap stack empties again,
// so the whole arena stays one LIFO stack and non-LIFO frees still trap.
struct ArenaState {
  uint64_t cursor;       // __arena_cursor (runtime.mc:67-68), zero-initialised per team
  uint64_t heap_cursor;  // bytes live in the heap part
  uint64_t capacity;     // shared-memory capacity (ARENA_CAPACITY by default)
  uint64_t heap_cap;     // heap bytes available to this team
  unsigned char *smem;
  unsigned char *heap;
  int heap_fallback;
};

OMPRT_D uint64_t arena_align(uint64_t b) {
  return (b + OMPRT_ARENA_ALIGN - 1) / OMPRT_ARENA_ALIGN * OMPRT_ARENA_ALIGN;
}

// Returns the offset, or -code (1 overflow, 3 not thread 0) — the caller
// turns a negative result into a trap.
OMPRT_D int64_t kmpc_alloc_shared(ArenaState &a, uint64_t bytes, uint32_t caller_tid) {
  if (caller_tid != 0) return -OMPRT_TRAP_NON_UNIFORM_ALLOC;
  const uint64_t need = arena_align(bytes);
  if (a.heap_cursor == 0) {
    if (bytes <= a.capacity && a.cursor + need <= a.capacity) {
      const uint64_t off = a.cursor;
      a.cursor += need;
      return (int64_t)off;
    }
    if (!a.heap_fallback) return -OMPRT_TRAP_SHARED_OVERFLOW;
  }
  if (need > a.heap_cap - a.heap_cursor) return -OMPRT_TRAP_SHARED_OVERFLOW;
  const uint64_t off = a.capacity + a.heap_cursor;
  a.heap_cursor += need;
  return (int64_t)off;
}

// Returns 0 or -code (2 non-LIFO, 3 not thread 0).
OMPRT_D int64_t kmpc_free_shared(ArenaState &a, uint64_t off, uint64_t bytes,
                                 uint32_t caller_tid) {
  if (caller_tid != 0) return -OMPRT_TRAP_NON_UNIFORM_ALLOC;
  const uint64_t need = arena_align(bytes);
  if (a.heap_fallback && off >= a.capacity) {
    if (off + need - a.capacity != a.heap_cursor) return -OMPRT_TRAP_NON_LIFO_FREE;
    a.heap_cursor = off - a.capacity;
    return 0;
  }
  if (a.heap_cursor != 0) return -OMPRT_TRAP_NON_LIFO_FREE;
  if (off + need != a.cursor) return -OMPRT_TRAP_NON_LIFO_FREE;
  a.cursor = off;
  return 0;
}

OMPRT_D unsigned char *arena_ptr(const ArenaState &a, uint64_t off) {
  return off < a.capacity ? a.smem + off : a.heap + (off - a.capacity);
}

struct ArenaCfg {
  int64_t capacity;
  int64_t heap_per_team;
  unsigned char *heap;  // teams * heap_per_team bytes (may be null without fallback)
  int heap_fallback;
};

OMPRT_D void arena_init(ArenaState &a, const ArenaCfg &c, unsigned char *smem) {
  a.cursor = 0;
  a.heap_cursor = 0;
  a.capacity = (uint64_t)c.capacity;
  a.heap_cap = c.heap_fallback ? (uint64_t)c.heap_per_team : 0;
  a.smem = smem;
  a.heap = c.heap_fallback ? c.heap + (int64_t)blockIdx.x * c.heap_per_team : nullptr;
  a.heap_fallback = c.heap_fallback;
}

// Replay an arena script (devicert.Arena parity; test_devicert.py:114-208).
// Script ops, 4 x int64 {opcode, bytes, offset, value}:
//   ALLOC bytes                 -> the offset
//   FREE  bytes, offset         -> 0
//   WRITE bytes, offset, value  -> 0; the team stores `value` (little-endian
//                                  u64, repeated) over [offset, offset+bytes)
//   READ  bytes(=8), offset     -> the u64 at offset (int64 bits)
// -code at the trapping op, kArenaSkipped after it.  The arena starts as
// loader_uninitialized poison (0xAA, vgpu.py:64-77).  With check_uninit a
// shadow bit per arena byte tracks WRITEs, and a READ touching an unwritten
// byte traps UninitializedRead (kind 4, vgpu.py:365-369).  Heap-spilled
// offsets (heap_fallback) are not shadowed.
constexpr int64_t kArenaSkipped = -0x7fff;

__global__ void k_arena_replay(const int64_t *__restrict__ script, int nops, int caller_tid,
                               ArenaCfg cfg, int check_uninit, int64_t *__restrict__ results) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ ArenaState st;
  __shared__ int64_t s_res;
  __shared__ int s_trapped;
  __shared__ uint32_t shadow[OMPRT_ARENA_CAPACITY / 32];
  for (int64_t i = threadIdx.x; i < cfg.capacity; i += blockDim.x) dsm[i] = 0xAA;
  for (int i = threadIdx.x; i < OMPRT_ARENA_CAPACITY / 32; i += blockDim.x) shadow[i] = 0;
  if (threadIdx.x == 0) {
    arena_init(st, cfg, dsm);
    s_trapped = 0;
  }
  __syncthreads();
  int64_t *res = results + (int64_t)blockIdx.x * nops;
  for (int op = 0; op < nops; ++op) {
    const int64_t *o = script + 4 * op;
    const int64_t kind = o[0], bytes = o[1], foff = o[2], value = o[3];
    if (kind == OMPRT_ARENA_WRITE) {
      // every thread of the team stores part of the range
      unsigned char *p = arena_ptr(st, (uint64_t)foff);
      for (int64_t j = threadIdx.x; j < bytes; j += blockDim.x) {
        p[j] = (unsigned char)(((uint64_t)value >> (8 * ((foff + j) & 7))) & 0xffu);
        const int64_t b = foff + j;
        if (b < (int64_t)st.capacity) atomicOr(&shadow[b >> 5], 1u << (b & 31));
      }
      __syncthreads();
      if (threadIdx.x == 0) res[op] = 0;
      continue;
    }
    if (kind == OMPRT_ARENA_READ) {
      if (threadIdx.x == (uint32_t)caller_tid) {
        const unsigned char *p = arena_ptr(st, (uint64_t)foff);
        uint64_t v = 0;
        bool init = true;
        for (int j = 0; j < 8 && j < bytes; ++j) {
          v |= (uint64_t)p[j] << (8 * j);
          const int64_t b = foff + j;
          if (b < (int64_t)st.capacity && !((shadow[b >> 5] >> (b & 31)) & 1u)) init = false;
        }
        s_res = (int64_t)v;
        if (check_uninit && !init) {
          s_res = -OMPRT_TRAP_UNINITIALIZED_READ;
          s_trapped = 1;
          raise_trap(OMPRT_TRAP_UNINITIALIZED_READ, 0);
        }
      }
    } else if (threadIdx.x == (uint32_t)caller_tid) {
      // the calling thread runs the runtime routine with its own thread id
      s_res = (kind == OMPRT_ARENA_ALLOC)
                  ? kmpc_alloc_shared(st, (uint64_t)bytes, threadIdx.x)
                  : kmpc_free_shared(st, (uint64_t)foff, (uint64_t)bytes, threadIdx.x);
      if (s_res < 0) {
        s_trapped = 1;
        raise_trap((int)-s_res, (int)-s_res);
      }
    }
    __syncthreads();
    const int64_t r = s_res;
    const int trapped = s_trapped;
    __syncthreads();  // every thread has read s_res before the next op rewrites it
    if (threadIdx.x == 0) res[op] = r;
    if (trapped) {
      if (threadIdx.x == 0)
        for (int k = op + 1; k < nops; ++k) res[k] = kArenaSkipped;
      return;
    }
    if (kind == OMPRT_ARENA_ALLOC && bytes > 0) {
      // data path: the team writes a tag through the returned offset and
      // reads it back with another thread->byte mapping, one blockDim-sized
      // window at a time, restoring the window's previous bytes afterwards
      // (an allocation does not initialise memory)
      unsigned char *p = arena_ptr(st, (uint64_t)r);
      const unsigned tag = (unsigned)(blockIdx.x * 131u + op * 17u);
      for (int64_t w = 0; w < bytes; w += blockDim.x) {
        const int64_t j = w + threadIdx.x;
        unsigned char orig = 0;
        if (j < bytes) {
          orig = p[j];
          p[j] = (unsigned char)((tag + (unsigned)j) & 0xffu);
        }
        __syncthreads();
        const int64_t k = w + (int64_t)blockDim.x - 1 - threadIdx.x;
        if (k < bytes && p[k] != (unsigned char)((tag + (unsigned)k) & 0xffu))
          raise_trap(OMPRT_TRAP_ABORT, 0);
        __syncthreads();
        if (j < bytes) p[j] = orig;
        __syncthreads();
      }
    }
  }
}

// ------------------------------------------------------------ generic mode
//
// One CTA = one team = 1 main warp + P/32 worker warps.  Named barriers:
//   1  fork       main warp + all workers (bar.sync)
//   2  in-region  workers only            (the parallel region's barrier)
//   3  join       workers bar.arrive, main warp bar.sync
// Lane 0 of the main warp is the team's initial thread (omp thread 0 in the
// sequential part): it owns the arena (tid-0 contract, runtime.mc:76, 87).
enum : int { kWorkExit = 0, kWorkRegion = 1 };

constexpr uint32_t kBarFork = 1, kBarRegion = 2, kBarJoin = 3;
constexpr int kGenericOrdDepth = 4;  // ORDERED workers: 32-byte loads in flight per lane

// The team partials folded into acc strictly in team order (the fallback's
// combine order, host.py:567-582) by one warp: the lanes stage up to `cap`
// partials at a time into shared memory with coalesced loads (one L2 round
// trip per block), then lane 0 adds them in order out of shared memory, the
// loads issued eight ahead so the chain is one dependent add per partial
// (8.2 cycles for fp64, profiles/r1_micro_latency.json).  Round 1 walked
// them through register shuffles instead: every step waited on a shuffle,
// ~30 cycles per partial — 16.3 us of C4's ORDERED launch at 1024 teams
// (tools/trace_generic.py).  All 32 lanes call; the result is returned in
// every lane.
// Stage m partials of src into shared memory with 16-byte cp.async copies
// (L2 only, no registers; all of a lane's in flight at once, so one L2 round
// trip), the unaligned remainder with ld.cg.  All 32 lanes call.
template <class T> OMPRT_D void warp_stage(T *buf, const T *src, int m) {
  constexpr int V = 16 / (int)sizeof(T);
  const uint32_t lane = lane_id();
  const int nv = (((uintptr_t)src & 15u) == 0) ? m / V : 0;
  for (int i = (int)lane; i < nv; i += 32)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(buf + (size_t)i * V)),
                 "l"(src + (size_t)i * V)
                 : "memory");
  asm volatile("cp.async.wait_all;" ::: "memory");
  for (int i = nv * V + (int)lane; i < m; i += 32) buf[i] = ld_cg(src + i);
  __syncwarp();
}

template <int OP, class T>
OMPRT_D T warp_fold_in_order(T acc, const T *p, int64_t n, T *buf, int cap) {
  const uint32_t lane = lane_id();
  for (int64_t b = 0; b < n; b += cap) {
    const int m = (int)(n - b < cap ? n - b : cap);
    warp_stage(buf, p + b, m);
    if (lane == 0) {
      // the next eight are read while the current eight are added
      int k = 0;
      T cur[8];
      if (m >= 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) cur[u] = buf[u];
      }
      for (; k + 8 <= m; k += 8) {
        T nxt[8];
        const bool more = k + 16 <= m;
#pragma unroll
        for (int u = 0; u < 8; ++u) nxt[u] = more ? buf[k + 8 + u] : cur[u];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = Red<OP, T>::apply(acc, cur[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) cur[u] = nxt[u];
      }
      for (; k < m; ++k) acc = Red<OP, T>::apply(acc, buf[k]);
    }
    __syncwarp();
  }
  return __shfl_sync(0xffffffffu, acc, 0);
}

// SPMD team combine by one warp: lane l folds partials l, l+32, ... (staged
// through shared memory, so one L2 round trip instead of one per 32), then
// the warp tree.  cap must be a multiple of 32 (the per-lane order is that
// of a plain strided walk over all n).
template <int OP, class T> OMPRT_D T warp_combine(const T *p, int64_t n, T *buf, int cap) {
  const uint32_t lane = lane_id();
  T v = Red<OP, T>::identity();
  for (int64_t b = 0; b < n; b += cap) {
    const int m = (int)(n - b < cap ? n - b : cap);
    warp_stage(buf, p + b, m);
#pragma unroll 8
    for (int i = (int)lane; i < m; i += 32) v = Red<OP, T>::apply(v, buf[i]);
    __syncwarp();
  }
  return warp_reduce<OP, T>(v, 32);
}

constexpr int kGenericFoldBytes = 8192;  // shared staging of the ORDERED team-partial fold

// ORDERED generic mode: the team that draws this ticket becomes the folder
// of the team partials (in team order, as they are published), from about
// half-way through the launch; below 256 teams the last team folds them all
// (UINT32_MAX: no folder).
OMPRT_HD uint32_t gen_fold_ticket(uint32_t teams) {
  return teams >= 256 ? teams / 2 : 0xffffffffu;
}

OMPRT_D void st_release_gpu_u64(uint64_t *p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
OMPRT_D uint64_t ld_acquire_gpu_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// ORD: the ORDERED instance (its in-order worker loop needs more registers;
// keeping it out of the SPMD instance keeps that one at 4 teams per SM).
// TRACE: the instance with the trace-ring hooks, launched only while a ring
// is installed (the hooks cost this kernel's short teams 4-6 % otherwise,
// profiles/README.md).
// MAXT / MINB: the launch bound.  The default instance takes any P; the
// one-wave instance (MAXT 288, MINB 7: at most 32 registers) is for teams of
// 32 + P <= 288 threads, where seven teams fit per SM and C4's 1024 teams
// (148 x 7 = 1036 slots) all run in a single wave instead of 1.7.
template <class T, int OP, int U, bool ORD = false, bool TRACE = false, int MAXT = kMaxThreads,
          int MINB = 1>
__global__ void __launch_bounds__(MAXT, MINB)
    k_generic(const T *__restrict__ x, int64_t lb, int64_t ub, int P, int ordered, int64_t pad,
              ArenaCfg cfg, Workspace ws, T *out, int64_t *team_offsets, uint64_t epoch) {
  extern __shared__ __align__(16) unsigned char dsm[];
  __shared__ ArenaState st;
  __shared__ volatile int s_work;
  __shared__ int64_t s_tlb, s_tub;
  __shared__ uint64_t s_off;
  const uint32_t nall = 32u + (uint32_t)P;
  const uint32_t lane = lane_id();
  if constexpr (TRACE) trace_begin();
  else pdl_begin();

  if (warp_id() == 0) {
    // ------------------------------------------------ main warp (sequential part)
    T team_val = Red<OP, T>::identity();
    if (lane == 0) {
      arena_init(st, cfg, dsm);
      const Bounds tb = team_block(lb, ub, blockIdx.x, gridDim.x);  // distribute
      s_tlb = tb.lower;
      s_tub = tb.upper;
      // an optional earlier allocation (pad) and then the globalised
      // `parts[P]` + the team reduction variable, stacked LIFO
      int64_t r = 0;
      if (pad > 0) r = kmpc_alloc_shared(st, (uint64_t)pad, 0);
      if (r >= 0) r = kmpc_alloc_shared(st, (uint64_t)(P + 1) * sizeof(T), 0);
      if (r < 0) {
        raise_trap((int)-r, (int)-r);
        s_work = kWorkExit;
      } else {
        s_off = (uint64_t)r;
        s_work = kWorkRegion;
        if (team_offsets) team_offsets[blockIdx.x] = r;
      }
    }
    __syncwarp();
    named_barrier_sync(kBarFork, nall);  // fork (or release to exit on trap)
    if (s_work == kWorkRegion) {
      named_barrier_sync(kBarJoin, nall);  // join: wait for the workers
      if (lane == 0) {
        T *parts = (T *)arena_ptr(st, s_off);
        T v = Red<OP, T>::identity();
        if constexpr (ORD) {
          for (int w = 0; w < P; ++w) v = Red<OP, T>::apply(v, parts[w]);
        } else {
          v = parts[P];
        }
        team_val = v;
        int64_t r = kmpc_free_shared(st, s_off, (uint64_t)(P + 1) * sizeof(T), 0);
        if (r == 0 && pad > 0) r = kmpc_free_shared(st, 0, (uint64_t)pad, 0);
        if (r < 0) raise_trap((int)-r, (int)-r);
        s_work = kWorkExit;
      }
      __syncwarp();
      named_barrier_sync(kBarFork, nall);  // release the workers to exit
    }
    // -------------------------------------- teams reduction within the main warps
    T *partials = (T *)ws.team_partials;
    if constexpr (ORD) {
      // ORDERED: the team partials are folded strictly in team order.  Most
      // of that chain need not wait for the last team: the team that draws
      // ticket teams/2 stays on as the folder and folds the partials as they
      // are published (ready flags carry the launch's epoch), overlapping
      // the chain with the teams still streaming.
      uint64_t *flags = (uint64_t *)(ws.team_partials + (size_t)partial_slots(gridDim.x) * 8);
      uint32_t t = 0;
      if (lane == 0) {
        partials[blockIdx.x] = team_val;
        st_release_gpu_u64(flags + blockIdx.x, epoch);
        fence_acq_rel_gpu();
        t = atomic_inc_acq_rel_gpu(ws.ticket, gridDim.x - 1);
        if constexpr (TRACE) {
          trace_record(blockIdx.x, kTraceTeam, t, trace_t0());
          if (t == gridDim.x - 1) trace_t0() = globaltimer();
        }
      }
      t = __shfl_sync(0xffffffffu, t, 0);
      __shared__ __align__(16) T s_fold[kGenericFoldBytes / sizeof(T)];
      constexpr int cap = (int)(kGenericFoldBytes / sizeof(T));
      const uint32_t tfold = gen_fold_ticket(gridDim.x);
      if (t == tfold) {
        // the folder: extends the folded prefix as the teams publish, so at
        // the end only the last few partials remain
        if constexpr (TRACE) {
          if (lane == 0) trace_t0() = globaltimer();
        }
        T acc = *out;
        int64_t K = 0;
        while (K < (int64_t)gridDim.x) {
          int64_t R = K;  // the ready frontier, 32 flags a step, at most one staging block
          for (;;) {
            const int64_t i = R + lane;
            const bool ready = i < (int64_t)gridDim.x && ld_acquire_gpu_u64(flags + i) == epoch;
            const uint32_t m = __ballot_sync(0xffffffffu, ready);
            const int k = m == 0xffffffffu ? 32 : __ffs(~m) - 1;
            R += k;
            if (k < 32 || R - K >= cap) break;
          }
          if (R == K) {
            __nanosleep(256);
            continue;
          }
          fence_acq_rel_gpu();  // every lane's acquire before any lane's partial loads
          acc = warp_fold_in_order<OP, T>(acc, partials + K, R - K, s_fold, cap);
          K = R;
        }
        if (lane == 0 && !trap_raised()) *out = acc;
        if constexpr (TRACE) trace_combine();
      } else if (tfold >= gridDim.x && t == gridDim.x - 1) {
        // few teams: the last one folds them all
        fence_acq_rel_gpu();
        const T v = warp_fold_in_order<OP, T>(*out, partials, (int64_t)gridDim.x, s_fold, cap);
        if (lane == 0 && !trap_raised()) *out = v;
        if constexpr (TRACE) trace_combine();
      }
    } else {
      int last = 0;
      if (lane == 0) {
        partials[blockIdx.x] = team_val;
        fence_acq_rel_gpu();
        const uint32_t t = atomic_inc_acq_rel_gpu(ws.ticket, gridDim.x - 1);
        last = t == gridDim.x - 1;
        if constexpr (TRACE) {
          trace_record(blockIdx.x, kTraceTeam, t, trace_t0());
          if (last) trace_t0() = globaltimer();
        }
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        fence_acq_rel_gpu();
        __shared__ __align__(16) T s_comb[kGenericFoldBytes / sizeof(T)];
        const T v = warp_combine<OP, T>(partials, (int64_t)gridDim.x, s_comb,
                                        (int)(kGenericFoldBytes / sizeof(T)));
        if (lane == 0 && !trap_raised()) *out = Red<OP, T>::apply(*out, v);
        if constexpr (TRACE) trace_combine();
      }
    }
  } else {
    // ------------------------------------------------ worker state machine
    const uint32_t wt = threadIdx.x - 32;  // omp thread id inside the parallel region
    for (;;) {
      named_barrier_sync(kBarFork, nall);
      if (s_work == kWorkExit) break;
      T *parts = (T *)arena_ptr(st, s_off);
      const int64_t tlb = s_tlb, tub = s_tub;
      if constexpr (ORD) {
        // for_static_init over the team block, literal sequential chunk
        int64_t mlb, mub;
        static_bounds(tlb, tub, wt, P, mlb, mub);
        parts[wt] = fold_row_in_order<OP, T, kGenericOrdDepth>(x, mlb, mub, Red<OP, T>::identity());
      } else {
        // 256-bit streaming loads: the worker warps share the SM with other
        // teams, so each lane keeps U x 32 bytes in flight
        ReduceBody<T, OP, kLoadNc, 32> body(x);
        if (tub >= tlb) run_contiguous<U>(body, tlb, tub - tlb + 1, wt, (uint32_t)P);
        // nested parallel reduce across the workers, scratch in the
        // globalised arena block, synchronised on the workers-only barrier
        const T v = warps_reduce_named<OP, T>(body.total(), (volatile T *)parts, 1, (uint32_t)P,
                                              kBarRegion);
        if (wt == 0) parts[P] = Red<OP, T>::apply(Red<OP, T>::identity(), v);
      }
      named_barrier_arrive(kBarJoin, nall);
    }
  }
}

// ------------------------------------------------------------ atomics probe
//
// seq_cst RMWs at device scope (the reference's constructs are seq_cst,
// runtime.mc:131-134; IR atomic.<kind>.seq_cst.<ty>, selectors.py:40-46).
template <class T> OMPRT_D T atomic_rmw(int kind, T *cell, T e, T d) {
  cuda::atomic_ref<T, cuda::thread_scope_device> ref(*cell);
  switch (kind) {
    case OMPRT_ATOMIC_ADD:
      return ref.fetch_add(e, cuda::std::memory_order_seq_cst);
    case OMPRT_ATOMIC_MAX:
      return ref.fetch_max(e, cuda::std::memory_order_seq_cst);
    case OMPRT_ATOMIC_MIN:
      return ref.fetch_min(e, cuda::std::memory_order_seq_cst);
    case OMPRT_ATOMIC_XCHG:
      return ref.exchange(e, cuda::std::memory_order_seq_cst);
    case OMPRT_ATOMIC_CAS: {
      T expected = e;
      ref.compare_exchange_strong(expected, d, cuda::std::memory_order_seq_cst);
      return expected;  // the observed value either way
    }
    default:  // INC: u32 only (validated on the host)
      kmpc_flush();
      return (T)atomic_inc_acq_rel_gpu((uint32_t *)cell, (uint32_t)e);
  }
}

template <class T> OMPRT_D uint64_t as_word(T v) {
  return (uint64_t)(typename std::make_unsigned<T>::type)v;
}

// Every thread of the grid applies one RMW to the single shared cell.
template <class T>
__global__ void k_atomic_probe(int kind, const uint64_t *__restrict__ ops,
                               const uint64_t *__restrict__ desired, T *cell,
                               uint64_t *__restrict__ old_out) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const T d = desired ? (T)desired[g] : T(0);
  old_out[g] = as_word<T>(atomic_rmw<T>(kind, cell, (T)ops[g], d));
}

// Every thread runs its own program of RMWs on the single shared cell, in
// program order (corpus.probe_source, corpus.py:374-408): thread g executes
// ops [offsets[g], offsets[g+1]) and records each old value in its slot.
template <class T>
__global__ void k_atomic_program(const int32_t *__restrict__ kinds,
                                 const uint64_t *__restrict__ ops,
                                 const uint64_t *__restrict__ desired,
                                 const int64_t *__restrict__ offsets, T *cell,
                                 uint64_t *__restrict__ old_out) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t k = offsets[g]; k < offsets[g + 1]; ++k) {
    const T d = desired ? (T)desired[k] : T(0);
    old_out[k] = as_word<T>(atomic_rmw<T>(kinds[k], cell, (T)ops[k], d));
  }
}

// Thread g applies one RMW to its own cell g (batched step_* semantics).
template <class T>
__global__ void k_atomic_apply(int kind, T *cells, const uint64_t *__restrict__ ops,
                               const uint64_t *__restrict__ desired,
                               uint64_t *__restrict__ old_out, int64_t n) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  const T d = desired ? (T)desired[g] : T(0);
  old_out[g] = as_word<T>(atomic_rmw<T>(kind, cells + g, (T)ops[g], d));
}

}  // namespace omprt
