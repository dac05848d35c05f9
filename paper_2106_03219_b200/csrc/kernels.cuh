// kernels.cuh — the `target teams distribute parallel for reduction` kernels.
//
//   k_reduce            SPMD: schedule -> coalesced team walk -> per-lane
//                       accumulators -> warp shuffle + smem tree -> team
//                       partial -> last-team-finishes ordered combine
//   k_reduce_ordered    ORDERED: literal per-thread chunk loops, per-thread
//                       partials combined in global thread order
//   k_axpy_minmax       fused y = a*x + y (fmaf) with max/min of y
//   k_dot               fp64 dot product
//   k_bounds_dump       every thread's schedule_init result (parity)
//   k_fill              counter-based synthetic data
//   k_combine           ordered combine of per-rank partials
#pragma once

#include "exactfold.cuh"
#include "loops.cuh"

namespace omprt {

constexpr int kMaxThreads = 1024;

// Workspace layout (bytes): [0,256) ticket + pad | team partials | thread partials
struct Workspace {
  uint32_t *ticket;
  unsigned char *team_partials;
  unsigned char *thread_partials;
};

// Team-partial slots: at least kMinPartialSlots so an SPMD launch may split
// each of a few teams over several CTAs (LoopArgs::split, team_set_cta).
constexpr int kMinPartialSlots = 256;
__host__ __device__ inline int partial_slots(int teams) {
  return teams < kMinPartialSlots ? kMinPartialSlots : teams;
}

__host__ inline size_t ws_bytes(int teams, int threads, int mode, int slots) {
  size_t b = 256 + (size_t)partial_slots(teams) * 8 * slots;
  b = (b + 255) & ~(size_t)255;
  if (mode == OMPRT_MODE_ORDERED) b += (size_t)teams * threads * 8 * slots;
  return b;
}

__host__ inline Workspace ws_carve(void *base, int teams, int slots) {
  Workspace w;
  unsigned char *p = (unsigned char *)base;
  w.ticket = (uint32_t *)p;
  w.team_partials = p + 256;
  size_t off = 256 + (size_t)partial_slots(teams) * 8 * slots;
  off = (off + 255) & ~(size_t)255;
  w.thread_partials = p + off;
  return w;
}

// Last-team-finishes (__kmpc_nvptx_teams_reduce_nowait_v2 analog): thread 0
// publishes the team value, takes a ticket with a device-scope acq_rel
// atomic inc bounded by teams-1 (so the counter wraps back to 0 for the next
// launch, step_inc devicert.py:105-107); the team holding the last ticket
// combines every team partial in team-id order — deterministic regardless of
// which team finished last.
template <int OP, class T>
OMPRT_D bool teams_ticket(T team_val, T *partials, uint32_t *ticket) {
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = team_val;
    fence_acq_rel_gpu();
    const uint32_t t = atomic_inc_acq_rel_gpu(ticket, gridDim.x - 1);
    s_last = (t == gridDim.x - 1);
    trace_record(blockIdx.x, kTraceTeam, t, trace_t0());
    if (s_last) trace_t0() = globaltimer();  // start of the combine
  }
  __syncthreads();
  const bool last = s_last != 0;
  if (last) fence_acq_rel_gpu();
  return last;
}

// the last team, after writing the result: the combine's trace record
OMPRT_D void trace_combine() {
  if (threadIdx.x == 0) trace_record(gridDim.x, kTraceCombine, gridDim.x - 1, trace_t0());
}

template <int OP, class T>
OMPRT_D T combine_team_partials(const T *partials, T *scratch) {
  T v = Red<OP, T>::identity();
  for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x)
    v = Red<OP, T>::apply(v, ld_cg(partials + i));
  return block_reduce<OP, T>(v, scratch, blockDim.x);
}

// ------------------------------------------------------------------ bodies

template <class T> OMPRT_D void unpack(const uint4 &r, T (&out)[16 / sizeof(T)]) {
  static_assert(sizeof(uint4) == 16, "vector width");
  union {
    uint4 u;
    T t[16 / sizeof(T)];
  } cv;
  cv.u = r;
#pragma unroll
  for (int j = 0; j < (int)(16 / sizeof(T)); ++j) out[j] = cv.t[j];
}

template <class T> OMPRT_D uint4 pack(const T (&in)[16 / sizeof(T)]) {
  union {
    uint4 u;
    T t[16 / sizeof(T)];
  } cv;
#pragma unroll
  for (int j = 0; j < (int)(16 / sizeof(T)); ++j) cv.t[j] = in[j];
  return cv.u;
}

// part = part OP x[i] — the PARTIAL_SUMS loop body (corpus.py:219-247).
// VB = bytes per lane per load (16: LDG.128, 32: LDG.256 on sm_100).
template <class T, int OP, int LP = kLoadDefault, int VB = 16> struct ReduceBody {
  static constexpr int V = VB / sizeof(T);
  static constexpr int V16 = 16 / sizeof(T);
  const T *__restrict__ x;
  T acc[V16];
  OMPRT_D explicit ReduceBody(const T *x_) : x(x_) {
#pragma unroll
    for (int j = 0; j < V16; ++j) acc[j] = Red<OP, T>::identity();
  }
  OMPRT_D bool head_ok(int64_t i) const { return (((uintptr_t)(x + i)) & (VB - 1)) == 0; }
  OMPRT_D void scalar(int64_t i) { acc[0] = Red<OP, T>::apply(acc[0], x[i]); }
  template <int U> OMPRT_D void vecs(const int64_t (&e)[U]) {
    if constexpr (VB == 32) {
      U8x32 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) r[u] = ld_v8<LP>(x + e[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        consume(r[u].lo);
        consume(r[u].hi);
      }
    } else {
      uint4 r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) r[u] = ld_v4<LP>(x + e[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) consume(r[u]);
    }
  }
  OMPRT_D void consume(const uint4 &r) {
    T t[V16];
    unpack<T>(r, t);
#pragma unroll
    for (int j = 0; j < V16; ++j) acc[j] = Red<OP, T>::apply(acc[j], t[j]);
  }
  OMPRT_D T total() const {
    T v = acc[0];
#pragma unroll
    for (int j = 1; j < V16; ++j) v = Red<OP, T>::apply(v, acc[j]);
    return v;
  }
};

// part = fma(x[i], y[i], part) — fp64 dot (config 5).
struct DotBody {
  static constexpr int V = 2;
  const double *__restrict__ x;
  const double *__restrict__ y;
  double acc[2];
  OMPRT_D DotBody(const double *x_, const double *y_) : x(x_), y(y_) { acc[0] = acc[1] = 0.0; }
  OMPRT_D bool head_ok(int64_t i) const {
    return ((((uintptr_t)(x + i)) | ((uintptr_t)(y + i))) & 15) == 0;
  }
  OMPRT_D void scalar(int64_t i) { acc[0] = __fma_rn(x[i], y[i], acc[0]); }
  template <int U> OMPRT_D void vecs(const int64_t (&e)[U]) {
    uint4 rx[U], ry[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      rx[u] = ld_stream_v4(x + e[u]);
      ry[u] = ld_stream_v4(y + e[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double a[2], b[2];
      unpack<double>(rx[u], a);
      unpack<double>(ry[u], b);
      acc[0] = __fma_rn(a[0], b[0], acc[0]);
      acc[1] = __fma_rn(a[1], b[1], acc[1]);
    }
  }
  OMPRT_D double total() const { return acc[0] + acc[1]; }
};

// y[i] = fmaf(a, x[i], y[i]); mx = max(mx, y[i]); mn = min(mn, y[i]) (config 3).
struct AxpyBody {
  static constexpr int V = 4;
  float a;
  const float *__restrict__ x;
  float *__restrict__ y;
  float mx[4], mn[4];
  OMPRT_D AxpyBody(float a_, const float *x_, float *y_) : a(a_), x(x_), y(y_) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      mx[j] = Limits<float>::lowest();
      mn[j] = Limits<float>::highest();
    }
  }
  OMPRT_D bool head_ok(int64_t i) const {
    return ((((uintptr_t)(x + i)) | ((uintptr_t)(y + i))) & 15) == 0;
  }
  OMPRT_D void scalar(int64_t i) {
    const float v = __fmaf_rn(a, x[i], y[i]);
    y[i] = v;
    mx[0] = Red<OMPRT_OP_MAX, float>::apply(mx[0], v);
    mn[0] = Red<OMPRT_OP_MIN, float>::apply(mn[0], v);
  }
  template <int U> OMPRT_D void vecs(const int64_t (&e)[U]) {
    uint4 rx[U], ry[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      rx[u] = ld_stream_v4(x + e[u]);
      ry[u] = ld_rw_v4(y + e[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float xv[4], yv[4];
      unpack<float>(rx[u], xv);
      unpack<float>(ry[u], yv);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        yv[j] = __fmaf_rn(a, xv[j], yv[j]);
        mx[j] = Red<OMPRT_OP_MAX, float>::apply(mx[j], yv[j]);
        mn[j] = Red<OMPRT_OP_MIN, float>::apply(mn[j], yv[j]);
      }
      st_stream_v4(y + e[u], pack<float>(yv));
    }
  }
  OMPRT_D float max_total() const {
    float v = mx[0];
#pragma unroll
    for (int j = 1; j < 4; ++j) v = Red<OMPRT_OP_MAX, float>::apply(v, mx[j]);
    return v;
  }
  OMPRT_D float min_total() const {
    float v = mn[0];
#pragma unroll
    for (int j = 1; j < 4; ++j) v = Red<OMPRT_OP_MIN, float>::apply(v, mn[j]);
    return v;
  }
};

// ------------------------------------------------------------------ kernels

struct LoopArgs {
  int64_t lb, ub, chunk;
  int sched;
  int split;    // SPMD: CTAs per OpenMP team (<= 1: one CTA per team)
  int balance;  // SPMD flat chunked: CTAs take balanced contiguous pieces
  int64_t tile;  // balance == 2 (tuning): CTAs take interleaved tiles of `tile` elements
  int threads;  // OpenMP threads per team (0: blockDim.x).  SPMD kernels may
                // run a team on a CTA of another size: the team's iteration
                // set depends on the OpenMP geometry only, which lane of the
                // CTA folds an iteration is unobservable
};

// Contiguous piece k of `cl` of [first, end): cut points on absolute
// 64-element boundaries (16-byte aligned pieces for every element size).
OMPRT_D void contiguous_piece(TeamSet &s, int64_t first, int64_t end, int64_t k, int64_t cl) {
  const int64_t piece = (end - first + cl - 1) / cl;
  auto cut = [&](int64_t j) {
    if (j <= 0) return first;
    if (j >= cl) return end;
    int64_t c = (first + j * piece + 63) & ~(int64_t)63;
    return c < end ? c : end;
  };
  const int64_t lo = cut(k), hi = cut(k + 1);
  s.seg_stride = 0;
  if (hi <= lo) {
    s.nseg = 0;
    s.seg_len = 0;
    return;
  }
  s.first = lo;
  s.seg_len = hi - lo;
  s.nseg = 1;
  s.ub = hi - 1;
}

// The iteration set of this CTA: its team's set (team_set, the schedule's
// contract) — or, when a launch splits each team over `split` CTAs (few
// teams: the rest of the SMs would idle), sub-CTA k's share of it: a
// contiguous set cut into split pieces on 64-element boundaries, a comb's
// teeth dealt round robin.  Which CTA of the team folds an iteration is as
// unobservable as which lane does (SPMD re-association; integers exact), and
// the team partials are still combined in (team, piece) order.
OMPRT_D TeamSet team_set_cta(const LoopArgs &la) {
  const int64_t cl = la.split > 1 ? la.split : 1;
  const int64_t teams = gridDim.x / cl, team = blockIdx.x / cl, sub = blockIdx.x % cl;
  if (la.balance == 2) {
    // tuning variant: CTA b takes tiles b, b + G, b + 2G, ... of [lb, ub]
    TeamSet s;
    s.ub = la.ub;
    s.first = la.lb + (int64_t)blockIdx.x * la.tile;
    s.seg_len = la.tile;
    s.seg_stride = (int64_t)gridDim.x * la.tile;
    s.nseg = (la.ub >= s.first) ? (la.ub - s.first) / s.seg_stride + 1 : 0;
    return s;
  }
  if (la.balance && la.sched == OMPRT_SCHED_STATIC_CHUNKED) {
    // The flat chunked teeth of all teams tile [lb, ub] exactly once, so the
    // union is contiguous: every CTA takes an equal contiguous piece of it
    // (a per-team comb of ceil(N / (threads*chunk)) teeth over `teams` CTAs
    // leaves a partial second wave, e.g. 171 teeth on 148 CTAs at C3's
    // 148 x 384 x 4096).  Same iterations, each exactly once; integers are
    // exact, max/min order-free, fp sums re-associated (SPMD).
    TeamSet s;
    s.ub = la.ub;
    if (la.ub < la.lb) {
      s.first = la.lb;
      s.seg_len = s.seg_stride = s.nseg = 0;
      return s;
    }
    contiguous_piece(s, la.lb, la.ub + 1, blockIdx.x, gridDim.x);
    return s;
  }
  TeamSet s = team_set(la.sched, la.lb, la.ub, la.chunk, team, teams,
                       la.threads > 0 ? la.threads : (int64_t)blockDim.x);
  if (cl == 1 || s.nseg <= 0) return s;
  if (s.seg_stride == 0 || s.nseg <= 1) {
    int64_t len = s.ub - s.first + 1;
    if (len > s.seg_len) len = s.seg_len;
    contiguous_piece(s, s.first, s.first + len, sub, cl);
    return s;
  }
  if (sub >= s.nseg) {
    s.nseg = 0;
    return s;
  }
  s.first += sub * s.seg_stride;
  s.nseg = (s.nseg - sub + cl - 1) / cl;
  s.seg_stride *= cl;
  return s;
}

template <class T, int OP, int U, int LP = kLoadDefault, int VB = 16>
__global__ void __launch_bounds__(kMaxThreads)
    k_reduce(const T *__restrict__ x, LoopArgs la, Workspace ws, T *out) {
  trace_begin();
  __shared__ T scratch[32];
  const TeamSet s = team_set_cta(la);
  ReduceBody<T, OP, LP, VB> body(x);
  run_team<U>(body, s, threadIdx.x, blockDim.x);
  const T team_val = block_reduce<OP, T>(body.total(), scratch, blockDim.x);
  T *partials = (T *)ws.team_partials;
  if (teams_ticket<OP, T>(team_val, partials, ws.ticket)) {
    // the cell's old value loaded alongside the partials (one round trip
    // less on the combine's critical path; nothing else writes it meanwhile)
    const T cell = threadIdx.x == 0 ? *out : Red<OP, T>::identity();
    const T v = combine_team_partials<OP, T>(partials, scratch);
    if (threadIdx.x == 0) *out = Red<OP, T>::apply(cell, v);
    trace_combine();
  }
}

// Sequential in-order fold used by ORDERED mode's final combine:
// acc = ((init OP p0) OP p1) ... — the fallback's atomic order, team-major and
// tid-minor (host.py:567-582, _atomic_step host.py:810-837).
template <int OP, class T> OMPRT_D T fold_in_order(T acc, const T *p, int64_t n) {
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    T v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = ld_cg(p + i + k);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc = Red<OP, T>::apply(acc, v[k]);
  }
  for (; i < n; ++i) acc = Red<OP, T>::apply(acc, ld_cg(p + i));
  return acc;
}

// The same fold with the whole (last) team staging the partials through
// shared memory in coalesced chunks; thread 0 still adds them strictly in
// order from shared memory (short-latency loads instead of one dependent
// global load per partial).  Every thread of the team must call it; the
// result is valid in thread 0.
template <int OP, class T>
OMPRT_D T fold_in_order_team(T acc, const T *p, int64_t n, T *buf, int cap) {
  for (int64_t base = 0; base < n; base += cap) {
    const int m = (int)((n - base) < cap ? (n - base) : cap);
    for (int k = threadIdx.x; k < m; k += blockDim.x) buf[k] = ld_cg(p + base + k);
    __syncthreads();
    if constexpr (OP != OMPRT_OP_ADD) {
      // max/min: the reference step keeps the leftmost of tied values and
      // per-thread partials are never NaN, so the in-order fold equals a
      // left-biased tree (see ord_folder, ordered.cuh): thread t folds the
      // t-th contiguous slice from the identity (±inf, neutral), each warp
      // combines lane i with lane i+d, thread 0 takes the warps in order.
      const int seg = (m + (int)blockDim.x - 1) / (int)blockDim.x;
      const int k0 = (int)threadIdx.x * seg;
      T v = Red<OP, T>::identity();
      for (int k = k0; k < k0 + seg && k < m; ++k) v = Red<OP, T>::apply(v, buf[k]);
      const uint32_t lane = threadIdx.x & 31u, wb = threadIdx.x & ~31u;
      const uint32_t lanes = blockDim.x - wb < 32u ? blockDim.x - wb : 32u;
      const uint32_t mask = lanes == 32u ? 0xffffffffu : ((1u << lanes) - 1u);
#pragma unroll
      for (uint32_t d = 1; d < 32; d <<= 1) {
        const T o = __shfl_down_sync(mask, v, d);
        if (lane + d < lanes) v = Red<OP, T>::apply(v, o);
      }
      __syncthreads();  // every thread is done reading buf
      if (lane == 0) buf[threadIdx.x >> 5] = v;
      __syncthreads();
      if (threadIdx.x == 0)
        for (uint32_t w = 0; w < (blockDim.x + 31u) / 32u; ++w) acc = Red<OP, T>::apply(acc, buf[w]);
      __syncthreads();
      continue;
    }
    if constexpr (std::is_floating_point<T>::value) {
      // fp sums: warp 0 folds the staged block 32 lanes wide where the chain
      // stays inside one binade (exactfold.cuh, the same bits)
      if (blockDim.x >= 32) {
        if (threadIdx.x < 32) acc = warp_sum_in_order<T>(acc, buf, m);
        __syncthreads();
        continue;
      }
    }
    if (threadIdx.x == 0) {
      int k = 0;
      for (; k + 8 <= m; k += 8) {
        T v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = buf[k + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = Red<OP, T>::apply(acc, v[u]);
      }
      for (; k < m; ++k) acc = Red<OP, T>::apply(acc, buf[k]);
    }
    __syncthreads();
  }
  return acc;
}

// One OpenMP thread's literal in-order fold of x[lo..hi] (the fallback's
// per-thread loop, host.py:567-582), fed by 32-byte loads (LDG.E.256) with
// 256-byte L2 promotion: every DRAM access brings 256 B of the thread's own
// row, which its next seven loads then find in L2 — the rows of a warp are
// far apart, so without the promotion DRAM would see 32-byte pieces.
// D: 32-byte loads in flight per step (2 for the literal ORDERED walk; the
// generic-mode ORDERED workers take 4 — their teams share the SM, so each
// lane needs more bytes in flight).
template <int OP, class T, int D = 2>
OMPRT_D T fold_row_in_order(const T *__restrict__ x, int64_t lo, int64_t hi, T part) {
  constexpr int V = 32 / (int)sizeof(T);
  int64_t i = lo;
  for (; i <= hi && (((uintptr_t)(x + i)) & 31u) != 0; ++i) part = Red<OP, T>::apply(part, x[i]);
  for (; i + D * V - 1 <= hi; i += D * V) {
    U8x32 r[D];
#pragma unroll
    for (int d = 0; d < D; ++d) r[d] = ld_v8<kLoadNcL2_256B>(x + i + d * V);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      T v[V];
      memcpy(v, &r[d], 32);
#pragma unroll
      for (int k = 0; k < V; ++k) part = Red<OP, T>::apply(part, v[k]);
    }
  }
  for (; i <= hi; ++i) part = Red<OP, T>::apply(part, x[i]);
  return part;
}

// The thread's iterations in order (block schedules: [lower, upper]; chunked:
// `chunk`-long runs from lower by stride up to limit), with D loads issued
// ahead of the in-order fold: only the fold is a dependent chain, the
// addresses are known, so each lane keeps D loads in flight instead of one
// round trip per element (small chunks otherwise walk at one element per
// L2/HBM latency: 0.63 TB/s for a chunk-1 ORDERED sum at 148 x 384).
template <int D, class V, class LoadF, class FoldF>
OMPRT_D void walk_in_order_ahead(const Bounds &bd, bool chunked, int64_t chunk, LoadF &&load,
                                 FoldF &&fold) {
  const int64_t limit = chunked ? bd.limit : bd.upper;
  int64_t lo = bd.lower;
  if (lo > limit) return;
  int64_t hi = chunked && lo + chunk - 1 < limit ? lo + chunk - 1 : limit;
  int64_t i = lo;
  bool live = true;
  while (live) {
    V v[D];
    int cnt = 0;
#pragma unroll
    for (int d = 0; d < D; ++d) {
      if (live) {
        v[d] = load(i);
        ++cnt;
        if (++i > hi) {
          lo += bd.stride;
          if (!chunked || lo > limit) {
            live = false;
          } else {
            i = lo;
            hi = lo + chunk - 1 < limit ? lo + chunk - 1 : limit;
          }
        }
      }
    }
#pragma unroll
    for (int d = 0; d < D; ++d)
      if (d < cnt) fold(v[d]);
  }
}

// This thread's schedule chunks as [lo, hi] runs, in order (block schedules:
// one run; chunked: run_thread_chunks' sequence, loops.cuh).
template <class F> OMPRT_D void for_each_thread_run(const LoopArgs &la, F &&f) {
  const Bounds bd = schedule_init(la.sched, la.lb, la.ub, la.chunk, blockIdx.x, gridDim.x,
                                  threadIdx.x, blockDim.x);
  if (la.sched != OMPRT_SCHED_STATIC_CHUNKED && la.sched != OMPRT_SCHED_DISTRIBUTE_CHUNKED) {
    if (bd.lower <= bd.upper) f(bd.lower, bd.upper);
    return;
  }
  for (int64_t lo = bd.lower; lo <= bd.limit; lo += bd.stride) {
    int64_t hi = lo + la.chunk - 1;
    if (hi > bd.limit) hi = bd.limit;
    f(lo, hi);
  }
}

// In-order y = a*x + y over [lo..hi] with max/min folded in iteration order:
// 16-byte loads (x non-coherent, y coherent: this kernel writes it) and
// 16-byte stores.
OMPRT_D void axpy_run_in_order(float a, const float *__restrict__ x, float *__restrict__ y,
                               int64_t lo, int64_t hi, float &mx, float &mn) {
  auto one = [&](int64_t i) {
    const float v = __fmaf_rn(a, x[i], y[i]);
    y[i] = v;
    mx = Red<OMPRT_OP_MAX, float>::apply(mx, v);
    mn = Red<OMPRT_OP_MIN, float>::apply(mn, v);
  };
  int64_t i = lo;
  if (((((uintptr_t)x) ^ ((uintptr_t)y)) & 15u) == 0) {
    for (; i <= hi && (((uintptr_t)(x + i)) & 15u) != 0; ++i) one(i);
    for (; i + 3 <= hi; i += 4) {
      float xv[4], yv[4];
      unpack<float>(ld_stream_v4(x + i), xv);
      unpack<float>(ld_rw_v4(y + i), yv);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        yv[k] = __fmaf_rn(a, xv[k], yv[k]);
        mx = Red<OMPRT_OP_MAX, float>::apply(mx, yv[k]);
        mn = Red<OMPRT_OP_MIN, float>::apply(mn, yv[k]);
      }
      st_stream_v4(y + i, pack<float>(yv));
    }
  }
  for (; i <= hi; ++i) one(i);
}

constexpr int kFoldBuf = 2048;  // elements of the static fold buffer

template <class T, int OP>
__global__ void __launch_bounds__(kMaxThreads)
    k_reduce_ordered(const T *__restrict__ x, LoopArgs la, Workspace ws, T *out) {
  trace_begin();
  T part = Red<OP, T>::identity();
  {
    const Bounds bd = schedule_init(la.sched, la.lb, la.ub, la.chunk, blockIdx.x, gridDim.x,
                                    threadIdx.x, blockDim.x);
    if (la.sched != OMPRT_SCHED_STATIC_CHUNKED && la.sched != OMPRT_SCHED_DISTRIBUTE_CHUNKED) {
      part = fold_row_in_order<OP, T>(x, bd.lower, bd.upper, part);
    } else if (la.chunk < 16) {
      // small chunks: element loads issued ahead of the fold
      walk_in_order_ahead<16, T>(
          bd, true, la.chunk, [&](int64_t i) { return __ldg(x + i); },
          [&](T v) { part = Red<OP, T>::apply(part, v); });
    } else {
      for (int64_t lo = bd.lower; lo <= bd.limit; lo += bd.stride) {
        int64_t hi = lo + la.chunk - 1;
        if (hi > bd.limit) hi = bd.limit;
        part = fold_row_in_order<OP, T>(x, lo, hi, part);
      }
    }
  }
  __shared__ T buf[kFoldBuf];
  T *tp = (T *)ws.thread_partials;
  tp[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = part;
  __syncthreads();
  if (teams_ticket<OP, T>(part, (T *)ws.team_partials, ws.ticket)) {
    const T v = fold_in_order_team<OP, T>(threadIdx.x == 0 ? *out : part, tp,
                                          (int64_t)gridDim.x * blockDim.x, buf, kFoldBuf);
    if (threadIdx.x == 0) *out = v;
    trace_combine();
  }
}

template <int U>
__global__ void __launch_bounds__(kMaxThreads)
    k_dot(const double *__restrict__ x, const double *__restrict__ y, LoopArgs la, Workspace ws,
          double *out) {
  trace_begin();
  __shared__ double scratch[32];
  const TeamSet s = team_set_cta(la);
  DotBody body(x, y);
  run_team<U>(body, s, threadIdx.x, blockDim.x);
  const double team_val = block_reduce<OMPRT_OP_ADD, double>(body.total(), scratch, blockDim.x);
  double *partials = (double *)ws.team_partials;
  if (teams_ticket<OMPRT_OP_ADD, double>(team_val, partials, ws.ticket)) {
    const double v = combine_team_partials<OMPRT_OP_ADD, double>(partials, scratch);
    if (threadIdx.x == 0) *out = *out + v;
    trace_combine();
  }
}

__global__ void __launch_bounds__(kMaxThreads)
    k_dot_ordered(const double *__restrict__ x, const double *__restrict__ y, LoopArgs la,
                  Workspace ws, double *out) {
  trace_begin();
  double part = 0.0;
  {
    const Bounds bd = schedule_init(la.sched, la.lb, la.ub, la.chunk, blockIdx.x, gridDim.x,
                                    threadIdx.x, blockDim.x);
    const bool chunked =
        la.sched == OMPRT_SCHED_STATIC_CHUNKED || la.sched == OMPRT_SCHED_DISTRIBUTE_CHUNKED;
    walk_in_order_ahead<8, double2>(
        bd, chunked, la.chunk, [&](int64_t i) { return make_double2(__ldg(x + i), __ldg(y + i)); },
        [&](double2 v) { part = __fma_rn(v.x, v.y, part); });
  }
  __shared__ double buf[kFoldBuf];
  double *tp = (double *)ws.thread_partials;
  tp[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = part;
  __syncthreads();
  if (teams_ticket<OMPRT_OP_ADD, double>(part, (double *)ws.team_partials, ws.ticket)) {
    const double v = fold_in_order_team<OMPRT_OP_ADD, double>(
        threadIdx.x == 0 ? *out : 0.0, tp, (int64_t)gridDim.x * blockDim.x, buf, kFoldBuf);
    if (threadIdx.x == 0) *out = v;
    trace_combine();
  }
}

// Two partial arrays (max, min) share one ticket: slots = 2 in ws_bytes.
template <int U>
__global__ void __launch_bounds__(kMaxThreads)
    k_axpy_minmax(float a, const float *__restrict__ x, float *__restrict__ y, LoopArgs la,
                  Workspace ws, float *out_max, float *out_min) {
  trace_begin();
  __shared__ float scratch[32];
  const TeamSet s = team_set_cta(la);
  AxpyBody body(a, x, y);
  run_team<U>(body, s, threadIdx.x, blockDim.x);
  const float tmax = block_reduce<OMPRT_OP_MAX, float>(body.max_total(), scratch, blockDim.x);
  const float tmin = block_reduce<OMPRT_OP_MIN, float>(body.min_total(), scratch, blockDim.x);
  float *pmax = (float *)ws.team_partials;
  float *pmin = pmax + gridDim.x;
  if (threadIdx.x == 0) pmin[blockIdx.x] = tmin;
  if (teams_ticket<OMPRT_OP_MAX, float>(tmax, pmax, ws.ticket)) {
    const float vmax = combine_team_partials<OMPRT_OP_MAX, float>(pmax, scratch);
    const float vmin = combine_team_partials<OMPRT_OP_MIN, float>(pmin, scratch);
    if (threadIdx.x == 0) {
      *out_max = Red<OMPRT_OP_MAX, float>::apply(*out_max, vmax);
      *out_min = Red<OMPRT_OP_MIN, float>::apply(*out_min, vmin);
    }
    trace_combine();
  }
}

__global__ void __launch_bounds__(kMaxThreads)
    k_axpy_minmax_ordered(float a, const float *__restrict__ x, float *__restrict__ y,
                          LoopArgs la, Workspace ws, float *out_max, float *out_min) {
  trace_begin();
  float mx = Limits<float>::lowest(), mn = Limits<float>::highest();
  for_each_thread_run(
      la, [&](int64_t lo, int64_t hi) { axpy_run_in_order(a, x, y, lo, hi, mx, mn); });
  const int64_t n = (int64_t)gridDim.x * blockDim.x;
  float *tmax = (float *)ws.thread_partials;
  float *tmin = tmax + n;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  tmax[g] = mx;
  tmin[g] = mn;
  __syncthreads();
  __shared__ float buf[kFoldBuf];
  if (teams_ticket<OMPRT_OP_MAX, float>(mx, (float *)ws.team_partials, ws.ticket)) {
    const float vmax = fold_in_order_team<OMPRT_OP_MAX, float>(
        threadIdx.x == 0 ? *out_max : mx, tmax, n, buf, kFoldBuf);
    const float vmin = fold_in_order_team<OMPRT_OP_MIN, float>(
        threadIdx.x == 0 ? *out_min : mn, tmin, n, buf, kFoldBuf);
    if (threadIdx.x == 0) {
      *out_max = vmax;
      *out_min = vmin;
    }
    trace_combine();
  }
}

// Every device thread runs the schedule's init routine (for_static_init,
// runtime.mc:193-203, and the chunked / distribute variants) and dumps it.
__global__ void k_bounds_dump(LoopArgs la, int64_t *__restrict__ out) {
  const Bounds b = schedule_init(la.sched, la.lb, la.ub, la.chunk, blockIdx.x, gridDim.x,
                                 threadIdx.x, blockDim.x);
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  out[4 * g + 0] = b.lower;
  out[4 * g + 1] = b.upper;
  out[4 * g + 2] = b.stride;
  out[4 * g + 3] = b.last;
}

template <class T>
__global__ void k_fill(T *__restrict__ x, int64_t n, uint64_t seed, int k, int64_t offset) {
  constexpr int V = 16 / sizeof(T);
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool aligned = (((uintptr_t)x) & 15) == 0;
  const int64_t nvec = aligned ? n / V : 0;
  for (int64_t v = g; v < nvec; v += nthr) {
    T t[V];
#pragma unroll
    for (int j = 0; j < V; ++j)
      t[j] = gen_value<T>(gen_bits(seed, k, (uint64_t)(offset + v * V + j)));
    st_stream_v4(x + v * V, pack<T>(t));
  }
  for (int64_t i = nvec * V + g; i < n; i += nthr)
    x[i] = gen_value<T>(gen_bits(seed, k, (uint64_t)(offset + i)));
}

template <class T, int OP> __global__ void k_combine(const T *p, int count, T *out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    T acc = *out;
    for (int i = 0; i < count; ++i) acc = Red<OP, T>::apply(acc, p[i]);
    *out = acc;
  }
}

}  // namespace omprt
