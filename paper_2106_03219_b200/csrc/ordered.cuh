// ordered.cuh — ORDERED mode at streaming speed.  Every OpenMP thread still
// folds exactly its own schedule chunks in iteration order (the host
// fallback's per-thread loop, host.py:567-582) and the per-thread partials
// are combined in global thread order, so fp results are bit-identical to
// the reference order; only the way the bytes reach the fold changes.
//
// Why not the literal walk (k_reduce_ordered, kernels.cuh): its lane l reads
// row l (its own block) one element at a time, so DRAM sees thousands of
// rows advancing in 32-byte sectors; and staging 32 rows × W elements for
// every resident warp runs out of shared memory before the row pieces get
// long enough for HBM (measured: 128-byte pieces 3.4 TB/s, 256-byte pieces
// 4.3 TB/s — profiles/r1_ordered_sweep.jsonl).
//
// Row-group design: the CUDA grid is decoupled from the OpenMP geometry.  The
// P = teams × threads OpenMP threads are cut into groups of 32 consecutive
// global thread ids; each CUDA warp takes groups round-robin, one lane per
// OpenMP thread (lane l plays thread g·32+l: its (team, tid) gives its
// schedule_init bounds).  Per group the warp streams W-element windows of
// its 32 rows through a ring of STAGES shared-memory tiles with 16-byte
// cp.async copies (SASS LDGSTS.128; each warp instruction moves 32 × 16 B
// of row pieces W·sizeof(T) bytes long), and lane l folds row l of each tile
// in order out of shared memory (row stride = U+1 16-byte units, an odd
// number, so the lanes' 16-byte reads are bank-conflict-free).  Only NW × 32
// rows per SM are in flight, so pieces can be ≥ 512 B while the ring still
// fits in shared memory.  Windows are aligned to 16 bytes in the address
// space and never cross a schedule chunk; window elements outside the row
// are copied (outside [lb, ub]: skipped) but never folded.  All P
// partials are combined in global thread order.  The folding of the partials (a strictly
// sequential chain) is done by one extra "folder" warp that follows the
// streaming warps group by group (per-group ready flags), overlapping it with
// the stream.
#pragma once

#include "exactfold.cuh"
#include "kernels.cuh"

namespace omprt {

constexpr int kOrdSmemBudget = 216 * 1024;  // dynamic smem of a CTA's streaming warps

// No "memory" clobber on the copies themselves (the commit/wait carry it):
// that lets the compiler batch the window-table loads ahead of the copies.
OMPRT_D void cp_async_16(void *smem_dst, const void *gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc));
}

template <int BYTES> OMPRT_D void cp_async_small(void *smem_dst, const void *gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
  if (BYTES == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gsrc));
}

OMPRT_D void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// wait until at most `pending` groups of this thread are outstanding
OMPRT_D void cp_async_wait(int pending) {
  switch (pending) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
  }
}

OMPRT_D void st_release_gpu(uint64_t *p, uint64_t v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

OMPRT_D uint64_t ld_relaxed_gpu(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

OMPRT_D uint64_t ld_acquire_gpu(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

constexpr int kOrdMaxStages = 6;

// One OpenMP thread's walk over its schedule chunks (run_thread_chunks,
// loops.cuh), in W-element windows aligned to V elements (16 bytes).
template <int W, int V> struct OrdRow {
  int64_t p;   // next element to fold (current chunk)
  int64_t hi;  // current chunk end (inclusive)
  int64_t a;   // current window start (V-aligned, a <= p)
  int64_t clo, stride, limit, chunk;
  int64_t left;  // windows this cursor may still take (segmented walks)
  bool chunked;

  OMPRT_D void init(const LoopArgs &la, int64_t g, int64_t teams, int64_t threads) {
    left = INT64_MAX;
    chunked = (la.sched == OMPRT_SCHED_STATIC_CHUNKED ||
               la.sched == OMPRT_SCHED_DISTRIBUTE_CHUNKED);
    if (g >= teams * threads) {  // lane past the last OpenMP thread: dead row
      p = 1;
      hi = 0;
      a = 0;
      chunked = false;
      return;
    }
    const Bounds bd = schedule_init(la.sched, la.lb, la.ub, la.chunk, g / threads, teams,
                                    g % threads, threads);
    stride = bd.stride;
    limit = bd.limit;
    chunk = la.chunk;
    clo = bd.lower;
    p = bd.lower;
    if (chunked) {
      hi = (bd.lower <= bd.limit) ? bd.lower + chunk - 1 : bd.lower - 1;
      if (hi > bd.limit) hi = bd.limit;
    } else {
      hi = bd.upper;
    }
    a = p & ~(int64_t)(V - 1);
  }
  OMPRT_D bool live() const { return p <= hi && left > 0; }
  // Windows of the row, and positioning at window w0 with a budget of n
  // windows (segment s of a row is windows [s*K, s*K + K)).  Chunked rows
  // (the host only asks when chunk and stride are multiples of V, so every
  // chunk of the row has the same 16-byte offset `off`) have wc windows per
  // full chunk.  Call right after init().
  OMPRT_D int64_t windows() const {
    if (p > hi) return 0;
    if (!chunked) return (hi - a) / W + 1;
    const int64_t off = p - a;
    const int64_t nch = (limit - clo) / stride + 1;
    const int64_t wc = (chunk + off + W - 1) / W;
    const int64_t lo_last = clo + (nch - 1) * stride;
    int64_t cl = limit - lo_last + 1;
    if (cl > chunk) cl = chunk;
    return (nch - 1) * wc + (cl + off + W - 1) / W;
  }
  OMPRT_D void seek(int64_t w0, int64_t n) {
    if (w0 > 0) {
      if (!chunked) {
        a += w0 * W;
        p = a;
      } else {
        const int64_t off = p - a;
        const int64_t wc = (chunk + off + W - 1) / W;
        const int64_t k = w0 / wc, j = w0 - k * wc;
        clo += k * stride;
        hi = clo + chunk - 1;
        if (hi > limit) hi = limit;
        a = clo - off + j * W;
        p = j == 0 ? clo : a;
      }
    }
    left = n;
  }
  // the current window's fold range as offsets from a: [s, e]
  OMPRT_D int s() const { return (int)(p - a); }
  OMPRT_D int e() const { return (int)((hi - a) < (W - 1) ? (hi - a) : (W - 1)); }
  OMPRT_D void advance() {
    a += W;
    p = a;
    --left;
    if (p > hi && chunked) {
      clo += stride;
      if (clo <= limit) {
        p = clo;
        hi = clo + chunk - 1;
        if (hi > limit) hi = limit;
        a = p & ~(int64_t)(V - 1);
      }
    }
  }
};

// Shared-memory picture of one warp: table[32] {a, e or -1 if the row is
// done} of the window being issued | STAGES × NS tiles of 32 rows ×
// (U+1) 16-byte units.
template <class T, int W, int NS> struct OrdSmem {
  static constexpr int V = 16 / (int)sizeof(T);
  static constexpr int U = W / V;         // 16-byte units per row window
  static constexpr int RS = (U + 1) * V;  // row stride in elements (odd # of units)
  static constexpr size_t kTile = (size_t)32 * RS * sizeof(T);
  static constexpr size_t kTable = 32 * sizeof(longlong2);
  OMPRT_HD static size_t warp_bytes(int stages) { return kTable + (size_t)stages * NS * kTile; }
  // stages for nw warps per CTA within the budget (0 = does not fit)
  OMPRT_HD static int stages_for(int nw) {
    for (int s = kOrdMaxStages; s >= 2; --s)
      if ((size_t)nw * warp_bytes(s) <= (size_t)kOrdSmemBudget) return s;
    return 0;
  }
};

// Issue the cp.async copies of every live row's current window of this
// warp's group into stage `st` (one commit group), then advance this lane's
// load cursor.  All 32 lanes call it.  Copy f = i·32 + lane of the window
// is unit j = f % U of row r = f / U (U a power of two: shifts), so each
// warp instruction covers whole 16-byte-aligned row pieces.  Windows that
// touch lb or ub (the first/last of the iteration space) take the
// element-checked path; everything else is one table read + one LDGSTS.128.
template <class T, int W, int NS>
OMPRT_D void ord_issue(OrdRow<W, 16 / sizeof(T)> &row, const T *const (&src)[NS], int64_t lb,
                       int64_t ub, longlong2 *table, T *tiles, int st, uint32_t lane) {
  using L = OrdSmem<T, W, NS>;
  constexpr int V = L::V, U = L::U;
  static_assert((U & (U - 1)) == 0 && U <= 32, "units per window: a power of two <= 32");
  constexpr int RPI = 32 / U;  // rows per copy instruction; j = lane % U is lane-constant
  const bool live = row.live();
  const bool inside = !live || (row.a >= lb && row.a + W - 1 <= ub);
  const bool fast = __all_sync(0xffffffffu, inside);
  T *tile0 = tiles + (size_t)st * NS * (L::kTile / sizeof(T));
  const int j = (int)(lane % U), rsub = (int)(lane / U);
  if (fast) {
    // table: the window's byte address in stream 0 and its unit count
    table[lane] = make_longlong2((long long)(uintptr_t)(src[0] + row.a),
                                 live ? (long long)(row.e() / V + 1) : 0ll);
    __syncwarp();
    T *dlane = tile0 + rsub * L::RS + j * V;
#pragma unroll
    for (int i = 0; i < U; ++i) {
      const longlong2 en = table[i * RPI + rsub];
      if (j < (int)en.y) {
        const char *g = (const char *)(uintptr_t)en.x + j * 16;
#pragma unroll
        for (int s = 0; s < NS; ++s)
          cp_async_16(dlane + (size_t)s * (L::kTile / sizeof(T)) + i * RPI * L::RS,
                      g + ((const char *)src[s] - (const char *)src[0]));
      }
    }
  } else {
    // windows touching lb or ub: element-checked copies
    table[lane] = make_longlong2(row.a, live ? (long long)row.e() : -1ll);
    __syncwarp();
    for (int i = 0; i < U; ++i) {
      const int r = i * RPI + rsub;
      const longlong2 en = table[r];
      if (j * V <= (int)en.y) {
        const int64_t e0 = en.x + (int64_t)j * V;
        for (int s = 0; s < NS; ++s) {
          T *dst = tile0 + (size_t)s * (L::kTile / sizeof(T)) + r * L::RS + j * V;
          if (e0 >= lb && e0 + V - 1 <= ub) {
            cp_async_16(dst, src[s] + e0);
          } else {
            for (int k = 0; k < V; ++k)
              if (e0 + k >= lb && e0 + k <= ub)
                cp_async_small<sizeof(T)>(dst + k, src[s] + e0 + k);
          }
        }
      }
    }
  }
  cp_async_commit();
  __syncwarp();
  if (live) row.advance();
}

template <class T> OMPRT_D T shfl_any(T v, int src_or_delta, bool down) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "4- or 8-byte partials");
  if constexpr (sizeof(T) == 8) {
    unsigned long long u;
    memcpy(&u, &v, 8);
    u = down ? __shfl_down_sync(0xffffffffu, u, src_or_delta) : __shfl_sync(0xffffffffu, u, src_or_delta);
    memcpy(&v, &u, 8);
  } else {
    unsigned u;
    memcpy(&u, &v, 4);
    u = down ? __shfl_down_sync(0xffffffffu, u, src_or_delta) : __shfl_sync(0xffffffffu, u, src_or_delta);
    memcpy(&v, &u, 4);
  }
  return v;
}

// Stream this warp's work through the ring; fold(rows, s, e) consumes this
// lane's row offsets s..e of the current tile in order, fold.publish(g)
// stores OpenMP thread g's running partial (fold.resume(g) reloads it).
//
// seg == 0 (static): warp w takes groups w, w + all warps, ... whole, then
// flags[grp] = epoch announces the group's 32 final partials to the folder.
// seg > 0 (dynamic, block schedules): the work is seg × ngroups units
// (segment s of group g = windows [s*K, s*K+K) of its rows), claimed in
// segment-major order from a self-resetting atom.inc counter (the ticket
// word), so SMs that stream faster take more units.  Unit (g, s) waits for
// flags[g] == epoch + s (segment s-1 done), resumes the 32 running partials,
// and leaves flags[g] = epoch + s + 1; the folder waits for epoch + seg.
// The dependency always points at an earlier-claimed unit held by a running
// warp, so the chain terminates at s = 0 (no deadlock).
template <class T, int W, int NS, class Fold>
OMPRT_D void ord_groups(const LoopArgs &la, int64_t teams, int64_t threads,
                        const T *const (&src)[NS], int stages, Fold &fold, uint64_t *flags,
                        uint64_t epoch, int seg, uint32_t *counter) {
  using L = OrdSmem<T, W, NS>;
  constexpr int V = L::V;
  extern __shared__ __align__(16) unsigned char ord_smem[];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t nwarps = (blockDim.x >> 5) - 1;  // the last warp is the folder's
  unsigned char *base = ord_smem + (size_t)warp * L::warp_bytes(stages);
  longlong2 *table = (longlong2 *)base;
  T *tiles = (T *)(base + L::kTable);
  const int64_t P = teams * threads;
  const int64_t ngroups = (P + 31) / 32;
  const int64_t units = seg > 0 ? (int64_t)seg * ngroups : ngroups;
  const uint32_t bound = (uint32_t)(units + (int64_t)gridDim.x * nwarps - 1);
  uint32_t ndone = 0;
  int64_t next = (int64_t)blockIdx.x * nwarps + warp;  // static scheme
  for (;; ++ndone) {
    int64_t u;
    if (seg > 0) {
      uint32_t t = 0;
      if (lane == 0) t = atomic_inc_acq_rel_gpu(counter, bound);
      u = (int64_t)__shfl_sync(0xffffffffu, t, 0);
    } else {
      u = next;
      next += (int64_t)gridDim.x * nwarps;
    }
    if (u >= units) break;
    // dynamic order: waves of `wave` groups (one per streaming warp of the
    // grid), segment-major inside a wave, so groups still complete wave by
    // wave for the folder
    int64_t grp = u;
    int sidx = 0;
    if (seg > 0) {
      const int64_t wave = (int64_t)gridDim.x * nwarps;
      const int64_t per_wave = wave * seg;
      const int64_t wv = u / per_wave, r = u - wv * per_wave;
      const int64_t g0 = wv * wave;
      const int64_t gw = (ngroups - g0) < wave ? (ngroups - g0) : wave;  // groups in this wave
      sidx = (int)(r / gw);
      grp = g0 + r % gw;
    }
    const int64_t g = grp * 32 + lane;
    OrdRow<W, V> ld, fd;
    ld.init(la, g, teams, threads);
    if (seg > 0) {
      const uint32_t nwin = (uint32_t)ld.windows();
      const int64_t gmax = (int64_t)__reduce_max_sync(0xffffffffu, nwin);
      const int64_t K = (gmax + seg - 1) / seg, w0 = (int64_t)sidx * K;
      int64_t n = (int64_t)nwin - w0;
      n = n < 0 ? 0 : (n > K ? K : n);
      ld.seek(w0, n);
      if (sidx > 0) {
        if (lane == 0)
          while (ld_acquire_gpu(flags + grp) != epoch + (uint64_t)sidx) {
          }
        __syncwarp();
        if (g < P) fold.resume(g);
      }
    }
    fd = ld;
    for (int s = 0; s + 1 < stages; ++s)
      ord_issue<T, W, NS>(ld, src, la.lb, la.ub, table, tiles, s, lane);
    // ring positions kept incrementally (stages is a runtime value: no modulo)
    int st_fold = 0, st_issue = stages - 1;
    for (;;) {
      if (!__any_sync(0xffffffffu, fd.live())) break;
      ord_issue<T, W, NS>(ld, src, la.lb, la.ub, table, tiles, st_issue, lane);
      st_issue = (st_issue + 1 == stages) ? 0 : st_issue + 1;
      cp_async_wait(stages - 1);
      __syncwarp();
      const int st = st_fold;
      st_fold = (st_fold + 1 == stages) ? 0 : st_fold + 1;
      if (fd.live()) {
        const T *rows[NS];
#pragma unroll
        for (int s = 0; s < NS; ++s)
          rows[s] = tiles + (size_t)(st * NS + s) * (L::kTile / sizeof(T)) + lane * L::RS;
        fold(rows, fd.s(), fd.e());
        fd.advance();
      }
      __syncwarp();
    }
    cp_async_wait(0);
    __syncwarp();
    if constexpr (Fold::kAssoc) {
      // max/min: the group's last unit folds its 32 running partials as the
      // left-biased tree (bit-identical to the in-order chain, see
      // ord_folder) and publishes one group result for the folder
      if (seg == 0 || sidx == seg - 1) {
        typename Fold::P v = g < P ? fold.value() : fold.identity();
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) v = fold.comb(v, shfl_any(v, d, true));
        if (lane == 0) ((typename Fold::P *)(flags + ngroups))[grp] = v;
        fold.reset();
      } else if (g < P) {
        fold.publish(g);
      }
    } else if (g < P) {
      fold.publish(g);
    }
    // the lanes' partials, then the flag (release, gpu scope)
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release_gpu(flags + grp, epoch + (uint64_t)(seg > 0 ? sidx + 1 : 0));
  }
  // trace: one record per streaming warp (units it folded), slot = warp id
  if (lane == 0)
    trace_record(blockIdx.x * nwarps + warp, kTraceGroup, ndone, trace_t0());
}

// Load V elements (16 bytes) of a shared-memory row.
template <class T, int V> OMPRT_D void lds_vec(T (&v)[V], const T *p) {
  const uint4 q = *reinterpret_cast<const uint4 *>(p);
  memcpy(v, &q, 16);
}

// One row's in-order fold of a window: offsets s..e of `row`.
template <class T, int OP, int W> struct OrdReduceFold {
  static constexpr int V = 16 / (int)sizeof(T);
  static constexpr bool kAssoc = OP != OMPRT_OP_ADD;  // max/min: group trees
  using P = T;
  T part;
  T *tp;
  OMPRT_D T value() const { return part; }
  OMPRT_D static T identity() { return Red<OP, T>::identity(); }
  OMPRT_D static T comb(T a, T b) { return Red<OP, T>::apply(a, b); }
  OMPRT_D void reset() { part = identity(); }
  OMPRT_D void operator()(const T *const (&rows)[1], int s, int e) {
    const T *r = rows[0];
    if (s == 0 && e == W - 1) {
#pragma unroll 4
      for (int q = 0; q < W / V; ++q) {
        T v[V];
        lds_vec<T, V>(v, r + q * V);
#pragma unroll
        for (int k = 0; k < V; ++k) part = Red<OP, T>::apply(part, v[k]);
      }
    } else {
      for (int o = s; o <= e; ++o) part = Red<OP, T>::apply(part, r[o]);
    }
  }
  OMPRT_D void publish(int64_t g) {
    tp[g] = part;
    part = Red<OP, T>::identity();
  }
  OMPRT_D void resume(int64_t g) { part = ld_cg(tp + g); }
};

template <int W> struct OrdDotFold {
  static constexpr bool kAssoc = false;
  using P = double;
  OMPRT_D static double identity() { return 0.0; }
  OMPRT_D static double comb(double a, double b) { return a + b; }
  OMPRT_D double value() const { return part; }
  OMPRT_D void reset() { part = 0.0; }
  double part;
  double *tp;
  OMPRT_D void operator()(const double *const (&rows)[2], int s, int e) {
    const double *a = rows[0], *b = rows[1];
    if (s == 0 && e == W - 1) {
#pragma unroll 4
      for (int q = 0; q < W / 2; ++q) {
        double va[2], vb[2];
        lds_vec<double, 2>(va, a + 2 * q);
        lds_vec<double, 2>(vb, b + 2 * q);
        part = __fma_rn(va[0], vb[0], part);
        part = __fma_rn(va[1], vb[1], part);
      }
    } else {
      for (int o = s; o <= e; ++o) part = __fma_rn(a[o], b[o], part);
    }
  }
  OMPRT_D void publish(int64_t g) {
    tp[g] = part;
    part = 0.0;
  }
  OMPRT_D void resume(int64_t g) { part = ld_cg(tp + g); }
};

// The folder: one warp (the extra warp of CTA 0) folds the P per-thread
// partials into *out strictly in global thread order — the fallback's
// combine order (host.py:567-582) — following the streaming warps as their
// group flags turn to this launch's epoch, so the sequential chain overlaps
// the stream instead of trailing it.  Batches of kFoldB groups (256
// partials): lane l waits (ld.acquire) for the flag of group l/4 of batch
// b+2, loads its 8 partials into registers, and stores them into a 2-slot
// shared-memory ring one iteration later; meanwhile the warp folds batch b
// out of the ring with broadcast loads, one dependent add per partial (the
// chain is the floor: ~8 cycles per fp64 add).
constexpr int kFoldB = 8;                                 // groups per batch
constexpr int kFoldPer = kFoldB * 32;                     // partials per batch
constexpr size_t kFolderSmem = 2 * kFoldPer * 8;          // the ring (bytes)

template <class T> struct FoldLoad {
  static constexpr int N = kFoldPer / 32;  // partials per lane per batch
  T v[N];
};

template <class T>
OMPRT_D void ord_folder_load(const T *tp, int64_t P, const uint64_t *flags, uint64_t epoch,
                             int64_t b, FoldLoad<T> &L) {
  constexpr int N = FoldLoad<T>::N;
  const uint32_t lane = threadIdx.x & 31u;
  const int64_t first = b * kFoldPer + (int64_t)lane * N;  // this lane's partials
  if (first < P) {
    const int64_t grp = first / 32;
    while (ld_acquire_gpu(flags + grp) != epoch) {
    }
  }
#pragma unroll
  for (int k = 0; k < N; ++k) L.v[k] = (first + k < P) ? ld_cg(tp + first + k) : T();
}

// The folder warp: folds the P per-thread partials in global thread order
// into acc.  For max/min (Combine::kAssoc) the reference's step
// `acc < e ? e : acc` keeps the leftmost maximum of its operands (a partial
// is never NaN: it starts at the identity and only ever takes an e that
// compares greater; ±0 tie and the left one stays), which is associative —
// so a full batch folds as a left-biased tree (each lane its 8 partials in
// order, then lane i takes lane i+d for d = 1..16) with the sequential
// fold's exact bits; a NaN cell value stays absorbing because acc is
// combined first.  Sums fold strictly one by one.
template <class T, class Combine>
OMPRT_D T ord_folder(const T *tp, int64_t P, const uint64_t *flags, uint64_t epoch, T acc,
                     T *ring, Combine &&comb) {
  constexpr int N = FoldLoad<T>::N;
  const uint32_t lane = threadIdx.x & 31u;
  if constexpr (std::decay_t<Combine>::kAssoc) {
    // The streaming warps already folded every group's 32 partials as a
    // left-biased tree (ord_groups); the folder takes the ngroups group
    // results in order, kFoldB per lane per step: relaxed loads of the lane's
    // ready flags (retried until all show this launch's epoch), one acquire
    // fence, the lane's results folded in order, then the same tree across
    // the lanes.  One flag and one data round trip per 256 groups.
    const int64_t ng = (P + 31) / 32;
    const T *gres = (const T *)(flags + ng);
    for (int64_t b = 0; b < ng; b += 32 * kFoldB) {
      const int64_t j0 = b + (int64_t)lane * kFoldB;
      bool ready;
      do {
        ready = true;
#pragma unroll
        for (int k = 0; k < kFoldB; ++k)
          if (j0 + k < ng) ready &= ld_relaxed_gpu(flags + j0 + k) == epoch;
      } while (!ready);
      fence_acq_rel_gpu();
      T r[kFoldB];
#pragma unroll
      for (int k = 0; k < kFoldB; ++k) r[k] = j0 + k < ng ? ld_cg(gres + j0 + k) : comb.identity();
      T v = r[0];
#pragma unroll
      for (int k = 1; k < kFoldB; ++k) v = comb(v, r[k]);
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) v = comb(v, shfl_any<T>(v, d, true));
      acc = comb(acc, shfl_any<T>(v, 0, false));
    }
    if (lane == 0)
      trace_record(gridDim.x * ((blockDim.x >> 5) - 1), kTraceFolder,
                   (uint32_t)((ng + 32 * kFoldB - 1) / (32 * kFoldB)), trace_t0());
    return acc;
  }
  const int64_t nb = (P + kFoldPer - 1) / kFoldPer;
  FoldLoad<T> L;
  ord_folder_load<T>(tp, P, flags, epoch, 0, L);
#pragma unroll
  for (int k = 0; k < N; ++k) ring[lane * N + k] = L.v[k];
  if (nb > 1) ord_folder_load<T>(tp, P, flags, epoch, 1, L);
  // fp sums: a batch whose chain stays inside one binade folds 32 lanes wide
  // (exactfold.cuh, same bits); after a miss (a binade crossing, a tie, a
  // zero / non-finite value) the next attempts back off, so data that never
  // qualifies pays at most one attempt per 16 batches
  int wait = 0, miss = 0;
  for (int64_t b = 0; b < nb; ++b) {
    T *cur = ring + (b & 1) * kFoldPer;
    T *nxt = ring + ((b + 1) & 1) * kFoldPer;
    if (b + 1 < nb) {
#pragma unroll
      for (int k = 0; k < N; ++k) nxt[lane * N + k] = L.v[k];
    }
    if (b + 2 < nb) ord_folder_load<T>(tp, P, flags, epoch, b + 2, L);
    __syncwarp();
    const int64_t base = b * kFoldPer;
    if constexpr (std::is_floating_point<T>::value) {
      T mine[N];
#pragma unroll
      for (int k = 0; k < N; ++k) mine[k] = cur[lane * N + k];  // zero past P
      if (wait > 0) {
        --wait;
      } else if (exact_fold_batch<T, N>(acc, mine)) {
        miss = 0;
        __syncwarp();
        continue;
      } else {
        miss = miss < 4 ? miss + 1 : 4;
        wait = (1 << miss) - 1;
      }
    }
    if (base + kFoldPer <= P) {
#pragma unroll 32
      for (int j = 0; j < kFoldPer; ++j) acc = comb(acc, cur[j]);
    } else {
      for (int j = 0; base + j < P; ++j) acc = comb(acc, cur[j]);
    }
    __syncwarp();
  }
  if (lane == 0)
    trace_record(gridDim.x * ((blockDim.x >> 5) - 1), kTraceFolder, (uint32_t)nb, trace_t0());
  return acc;  // the same in every lane
}

template <int OP, class T> struct RedComb {
  static constexpr bool kAssoc = OP != OMPRT_OP_ADD;  // leftmost max / min (ord_folder)
  OMPRT_D T operator()(T a, T b) const { return Red<OP, T>::apply(a, b); }
  OMPRT_D static T identity() { return Red<OP, T>::identity(); }
};

// flags (one u64 per group) live after the P partials in the (2-slot)
// thread-partial area.  The workspace is shared with every other kernel, so
// a flag slot may hold anything when a launch starts: the per-launch key is
// a splitmix64 image of (process nonce, launch counter) — distinct for every
// launch of the process and a 2^-64 chance to equal stale data.
OMPRT_HD size_t ord_flags_offset(int64_t P) { return (size_t)P * 8; }

constexpr int kOrdMaxWarps = 16;  // streaming warps per CTA (+1 folder warp)

template <class T, int OP, int W>
__global__ void __launch_bounds__((kOrdMaxWarps + 1) * 32)
    k_reduce_ordered_rows(const T *__restrict__ x, LoopArgs la, int teams, int threads,
                          Workspace ws, T *out, int stages, uint64_t epoch, uint32_t ring_off,
                          int seg) {
  trace_begin();
  __syncthreads();  // the CTA's trace start time, read by every warp at its end
  const int64_t P = (int64_t)teams * threads;
  T *tp = (T *)ws.thread_partials;
  uint64_t *flags = (uint64_t *)(ws.thread_partials + ord_flags_offset(P));
  if ((threadIdx.x >> 5) == (blockDim.x >> 5) - 1) {
    extern __shared__ __align__(16) unsigned char ord_smem[];
    if (blockIdx.x == 0) {
      const T v = ord_folder<T>(tp, P, flags, epoch + (uint64_t)seg, *out,
                                (T *)(ord_smem + ring_off), RedComb<OP, T>());
      if ((threadIdx.x & 31u) == 0) *out = v;
    }
    return;
  }
  OrdReduceFold<T, OP, W> f{Red<OP, T>::identity(), tp};
  const T *src[1] = {x};
  ord_groups<T, W, 1>(la, teams, threads, src, stages, f, flags, epoch, seg, ws.ticket);
}

template <int W>
__global__ void __launch_bounds__((kOrdMaxWarps + 1) * 32)
    k_dot_ordered_rows(const double *__restrict__ x, const double *__restrict__ y, LoopArgs la,
                       int teams, int threads, Workspace ws, double *out, int stages,
                       uint64_t epoch, uint32_t ring_off, int seg) {
  trace_begin();
  __syncthreads();  // the CTA's trace start time, read by every warp at its end
  const int64_t P = (int64_t)teams * threads;
  double *tp = (double *)ws.thread_partials;
  uint64_t *flags = (uint64_t *)(ws.thread_partials + ord_flags_offset(P));
  if ((threadIdx.x >> 5) == (blockDim.x >> 5) - 1) {
    extern __shared__ __align__(16) unsigned char ord_smem[];
    if (blockIdx.x == 0) {
      const double v = ord_folder<double>(tp, P, flags, epoch + (uint64_t)seg, *out,
                                          (double *)(ord_smem + ring_off),
                                          RedComb<OMPRT_OP_ADD, double>());
      if ((threadIdx.x & 31u) == 0) *out = v;
    }
    return;
  }
  OrdDotFold<W> f{0.0, tp};
  const double *src[2] = {x, y};
  ord_groups<double, W, 2>(la, teams, threads, src, stages, f, flags, epoch, seg, ws.ticket);
}

// max and min folded together in one ORDERED pass (axpy's ORDERED mode):
// the per-thread partials are float2 {max, min}, the folder carries both
// chains (independent, so interleaved at the latency of one).
template <int W> struct OrdMinMaxFold {
  static constexpr int V = 4;
  static constexpr bool kAssoc = true;
  using P = float2;
  float mx, mn;
  float2 *tp;
  OMPRT_D float2 value() const { return make_float2(mx, mn); }
  OMPRT_D static float2 identity() {
    return make_float2(Limits<float>::lowest(), Limits<float>::highest());
  }
  OMPRT_D static float2 comb(float2 a, float2 b) {
    return make_float2(Red<OMPRT_OP_MAX, float>::apply(a.x, b.x),
                       Red<OMPRT_OP_MIN, float>::apply(a.y, b.y));
  }
  OMPRT_D void reset() {
    mx = Limits<float>::lowest();
    mn = Limits<float>::highest();
  }
  OMPRT_D void operator()(const float *const (&rows)[1], int s, int e) {
    const float *r = rows[0];
    if (s == 0 && e == W - 1) {
#pragma unroll 4
      for (int q = 0; q < W / V; ++q) {
        float v[V];
        lds_vec<float, V>(v, r + q * V);
#pragma unroll
        for (int k = 0; k < V; ++k) {
          mx = Red<OMPRT_OP_MAX, float>::apply(mx, v[k]);
          mn = Red<OMPRT_OP_MIN, float>::apply(mn, v[k]);
        }
      }
    } else {
      for (int o = s; o <= e; ++o) {
        mx = Red<OMPRT_OP_MAX, float>::apply(mx, r[o]);
        mn = Red<OMPRT_OP_MIN, float>::apply(mn, r[o]);
      }
    }
  }
  OMPRT_D void publish(int64_t g) {
    tp[g] = make_float2(mx, mn);
    mx = Limits<float>::lowest();
    mn = Limits<float>::highest();
  }
  OMPRT_D void resume(int64_t g) {
    const float2 v = ld_cg(tp + g);
    mx = v.x;
    mn = v.y;
  }
};

struct MinMaxComb {
  static constexpr bool kAssoc = true;
  OMPRT_D float2 operator()(float2 a, float2 b) const { return OrdMinMaxFold<4>::comb(a, b); }
  OMPRT_D static float2 identity() { return OrdMinMaxFold<4>::identity(); }
};

template <int W>
__global__ void __launch_bounds__((kOrdMaxWarps + 1) * 32)
    k_minmax_ordered_rows(const float *__restrict__ y, LoopArgs la, int teams, int threads,
                          Workspace ws, float *out_max, float *out_min, int stages,
                          uint64_t epoch, uint32_t ring_off, int seg) {
  trace_begin();
  __syncthreads();
  const int64_t P = (int64_t)teams * threads;
  float2 *tp = (float2 *)ws.thread_partials;
  uint64_t *flags = (uint64_t *)(ws.thread_partials + ord_flags_offset(P));
  if ((threadIdx.x >> 5) == (blockDim.x >> 5) - 1) {
    extern __shared__ __align__(16) unsigned char ord_smem[];
    if (blockIdx.x == 0) {
      const float2 v = ord_folder<float2>(tp, P, flags, epoch + (uint64_t)seg,
                                          make_float2(*out_max, *out_min),
                                          (float2 *)(ord_smem + ring_off), MinMaxComb());
      if ((threadIdx.x & 31u) == 0) {
        *out_max = v.x;
        *out_min = v.y;
      }
    }
    return;
  }
  OrdMinMaxFold<W> f{Limits<float>::lowest(), Limits<float>::highest(), tp};
  const float *src[1] = {y};
  ord_groups<float, W, 1>(la, teams, threads, src, stages, f, flags, epoch, seg, ws.ticket);
}

// Host side: can the row-group kernels take this launch?  x (and y) must be
// 16-byte aligned; chunked schedules need chunk >= kOrdMinChunk (smaller
// chunks keep the literal walk, which is coalesced across lanes for chunk 1).
constexpr int64_t kOrdMinChunk = 16;

__host__ inline bool ord_rows_ok(const LoopArgs &la, const void *x, const void *y = nullptr) {
  if (((uintptr_t)x & 15) != 0 || ((uintptr_t)y & 15) != 0) return false;
  const bool chunked = (la.sched == OMPRT_SCHED_STATIC_CHUNKED ||
                        la.sched == OMPRT_SCHED_DISTRIBUTE_CHUNKED);
  return !chunked || la.chunk >= kOrdMinChunk;
}

}  // namespace omprt
