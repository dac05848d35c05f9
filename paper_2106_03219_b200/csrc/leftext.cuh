// leftext.cuh — ORDERED max/min at SPMD speed.
//
// The reference folds max/min with `acc < e ? e : acc` (max) and
// `acc > e ? e : acc` (min): per OpenMP thread over its chunks in order from
// the identity, then the per-thread partials into the cell in global thread
// order (host.py:567-582, step_max/step_min devicert.py:88-95).  That fold
// keeps the FIRST extremal element of the sequence (ties — +0 / -0, equal
// values — keep the earlier one) and never takes a NaN element.  So its bits
// are those of the extremal element with the smallest position in the
// reference sequence, which is a function of the set of (value, position)
// pairs, not of the order they are visited in:
//
//   (v, k) ⊕ (v', k') = whichever value is strictly more extreme, and on a
//                       tie (==) the one with the smaller position k
//
// is associative and commutative, so any lane / warp / team tree gives the
// literal fold's bits.  The position of iteration i in the reference
// sequence is (owner OpenMP thread, i): iteration order for the block
// schedules, (thread, i) for the chunked ones (OrderKey).  Keys are computed
// only when an element ties or beats the running extremum (rare after the
// first few elements), so the construct streams at the SPMD kernels' rate —
// this replaces the second, row-ordered max/min pass of C3's ORDERED mode and
// the row-group kernels for fp max/min.  The cell is combined last with the
// reference step (a NaN cell stays NaN, a tie keeps the cell).
#pragma once

#include <climits>

#include "bulk.cuh"

namespace omprt {

// Position of iteration i in the reference's sequence (global thread order,
// each thread's iterations in order), as one comparable int64:
// (thread << 40) | (i - lb).  Host-gated to spaces of < 2^40 iterations.
struct OrderKey {
  int64_t lb, chunk, team_chunk, threads, P;
  int sched;
  OMPRT_D int64_t operator()(int64_t i) const {
    if (sched != OMPRT_SCHED_STATIC_CHUNKED && sched != OMPRT_SCHED_DISTRIBUTE_CHUNKED)
      return i - lb;  // block schedules: thread order is iteration order
    return chunked(i);
  }
  // out of line: only ties between equal values need it during the stream
  // (and each lane's final extremum once), and its 64-bit divisions would
  // otherwise be inlined at every element of the unrolled loops
  __device__ __noinline__ int64_t chunked(int64_t i) const {
    const int64_t r = i - lb;
    if (sched == OMPRT_SCHED_STATIC_CHUNKED) return (((r / chunk) % P) << 40) | r;
    // distribute_chunked: the team's block (static_bounds over teams), then
    // chunks round robin over the team's threads
    const int64_t team = r / team_chunk;
    const int64_t tid = ((r - team * team_chunk) / chunk) % threads;
    return ((team * threads + tid) << 40) | r;
  }
};

OMPRT_D OrderKey make_order_key(const LoopArgs &la) {
  OrderKey k;
  const int64_t cl = la.split > 1 ? la.split : 1;
  const int64_t teams = gridDim.x / cl;
  const int64_t threads = la.threads > 0 ? la.threads : (int64_t)blockDim.x;
  const int64_t n = la.ub - la.lb + 1;
  k.lb = la.lb;
  k.chunk = la.chunk > 0 ? la.chunk : 1;
  k.team_chunk = n > 0 ? floordiv(n + teams - 1, teams) : 1;
  k.threads = threads;
  k.P = teams * threads;
  k.sched = la.sched;
  return k;
}

// (value, order key) of the extremum; k = INT64_MAX: none (the identity).
template <int OP, class T> struct LeftExt {
  T v = Red<OP, T>::identity();
  int64_t k = INT64_MAX;
  // strictly more extreme under the reference step's comparison
  static OMPRT_D bool beats(T e, T cur) {
    if constexpr (OP == OMPRT_OP_MAX) return cur < e;
    else return e < cur;
  }
  OMPRT_D void merge(T ov, int64_t ok) {
    if (beats(ov, v) || (ov == v && ok < k)) {
      v = ov;
      k = ok;
    }
  }
};

// One lane's running extremum while it streams: the value and the ITERATION
// it came from (keys are computed for ties only — a new extremum is a plain
// select — and once at the end, finish()).  A warp-level branch around a key
// computation at every new extremum would run nearly every step: 32 lanes'
// record-breaking elements together.
template <int OP, class T> struct LeftExtLane {
  T v = Red<OP, T>::identity();
  int64_t pos = -1;  // iteration of v, -1: the identity
  static OMPRT_D bool beats(T e, T cur) { return LeftExt<OP, T>::beats(e, cur); }
  OMPRT_D void take(T e, int64_t i, const OrderKey *key) {
    if (beats(e, v)) {
      v = e;
      pos = i;
    } else if (e == v) {  // a tie (never a NaN): the earlier in the reference sequence
      if (pos < 0 || (*key)(i) < (*key)(pos)) pos = i;
      v = pos == i ? e : v;
    }
  }
  // Could any of these values tie or beat the running extremum?  (One
  // NaN-ignoring max/min over the group; the extremum only moves further, so
  // a group that fails never matters.)
  template <int N> OMPRT_D bool screen(const T (&e)[N]) const {
    // a tree, not a chain: log2(N) dependent min/max steps
    T t[N];
#pragma unroll
    for (int j = 0; j < N; ++j) t[j] = e[j];
#pragma unroll
    for (int w = 1; w < N; w <<= 1) {
#pragma unroll
      for (int j = 0; j + w < N; j += 2 * w) {
        if constexpr (OP == OMPRT_OP_MAX) t[j] = fmax(t[j], t[j + w]);
        else t[j] = fmin(t[j], t[j + w]);
      }
    }
    return beats(t[0], v) || t[0] == v;
  }
  template <int N> OMPRT_D void take_vec(const T (&e)[N], int64_t i0, const OrderKey *key) {
    if (screen(e)) {
#pragma unroll
      for (int j = 0; j < N; ++j) take(e[j], i0 + j, key);
    }
  }
  OMPRT_D LeftExt<OP, T> finish(const OrderKey *key) const {
    LeftExt<OP, T> r;
    r.v = v;
    r.k = pos < 0 ? INT64_MAX : (*key)(pos);
    return r;
  }
};

template <int OP, class T> OMPRT_D void warp_merge(LeftExt<OP, T> &a) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    const T ov = __shfl_xor_sync(0xffffffffu, a.v, m);
    const int64_t ok = __shfl_xor_sync(0xffffffffu, a.k, m);
    a.merge(ov, ok);
  }
}

// Block-wide ⊕ (every thread calls; blockDim.x a multiple of 32 or not —
// missing lanes contribute the neutral (identity, INT64_MAX)).
template <int OP, class T> OMPRT_D LeftExt<OP, T> block_merge(LeftExt<OP, T> a) {
  __shared__ T sv[32];
  __shared__ int64_t sk[32];
  const uint32_t lane = lane_id(), warp = warp_id();
  const uint32_t nwarps = (blockDim.x + 31) >> 5;
  warp_merge(a);
  if (lane == 0) {
    sv[warp] = a.v;
    sk[warp] = a.k;
  }
  __syncthreads();
  if (warp == 0) {
    LeftExt<OP, T> b;
    if (lane < nwarps) {
      b.v = sv[lane];
      b.k = sk[lane];
    }
    warp_merge(b);
    a = b;
  }
  __syncthreads();
  return a;
}

// The team's (value, key) into the team slots, the ticket, and the last CTA
// merges every team's pair (any order) and applies the cell step.
// Returns true in the CTA that wrote the result.
template <int OP, class T>
OMPRT_D bool ext_teams_combine(LeftExt<OP, T> team, T *pv, int64_t *pk, uint32_t *ticket,
                               T *out) {
  if (threadIdx.x == 0) pk[blockIdx.x] = team.k;
  if (!teams_ticket<OP, T>(team.v, pv, ticket)) return false;
  LeftExt<OP, T> a;
  for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x) a.merge(ld_cg(pv + i), ld_cg(pk + i));
  a = block_merge(a);
  if (threadIdx.x == 0) *out = Red<OP, T>::apply(*out, a.v);
  return true;
}

// Body concept (loops.cuh) for reduce(max/min) with leftmost tie-breaking.
template <class T, int OP> struct ExtReduceBody {
  static constexpr int V = 16 / sizeof(T);
  const T *__restrict__ x;
  const OrderKey *key;  // in shared memory
  LeftExtLane<OP, T> acc;
  OMPRT_D ExtReduceBody(const T *x_, const OrderKey *k) : x(x_), key(k) {}
  OMPRT_D bool head_ok(int64_t i) const { return (((uintptr_t)(x + i)) & 15) == 0; }
  OMPRT_D void scalar(int64_t i) { acc.take(x[i], i, key); }
  OMPRT_D void consume(const uint4 &r, int64_t i0) {
    T t[V];
    unpack<T>(r, t);
    acc.take_vec(t, i0, key);
  }
  // the G vectors' elements against the running extremum
  template <int G> OMPRT_D bool screen(const uint4 (&r)[G]) const {
    T t[G * V];
#pragma unroll
    for (int u = 0; u < G; ++u) {
      T w[V];
      unpack<T>(r[u], w);
#pragma unroll
      for (int j = 0; j < V; ++j) t[u * V + j] = w[j];
    }
    return acc.screen(t);
  }
  template <int U> OMPRT_D void vecs(const int64_t (&e)[U]) {
    uint4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = ld_stream_v4(x + e[u]);
    if (screen(r)) {
#pragma unroll
      for (int u = 0; u < U; ++u) consume(r[u], e[u]);
    }
  }
};

// y = fmaf(a, x, y) with max and min over the new y, leftmost ties.
struct ExtAxpyBody {
  static constexpr int V = 4;
  float a;
  const float *__restrict__ x;
  float *__restrict__ y;
  const OrderKey *key;  // in shared memory
  LeftExtLane<OMPRT_OP_MAX, float> mx;
  LeftExtLane<OMPRT_OP_MIN, float> mn;
  OMPRT_D ExtAxpyBody(float a_, const float *x_, float *y_, const OrderKey *k)
      : a(a_), x(x_), y(y_), key(k) {}
  OMPRT_D bool head_ok(int64_t i) const {
    return ((((uintptr_t)(x + i)) | ((uintptr_t)(y + i))) & 15) == 0;
  }
  OMPRT_D void scalar(int64_t i) {
    const float v = __fmaf_rn(a, x[i], y[i]);
    y[i] = v;
    mx.take(v, i, key);
    mn.take(v, i, key);
  }
  // y' = fmaf(a, x, y) of G vectors (stored by the caller), then max and
  // min over them, screened as a group
  template <int G>
  OMPRT_D void group(const uint4 (&rx)[G], const uint4 (&ry)[G], float (&yv)[G * 4]) {
#pragma unroll
    for (int u = 0; u < G; ++u) {
      float xv[4], w[4];
      unpack<float>(rx[u], xv);
      unpack<float>(ry[u], w);
#pragma unroll
      for (int j = 0; j < 4; ++j) yv[u * 4 + j] = __fmaf_rn(a, xv[j], w[j]);
    }
  }
  template <int G, class Index>
  OMPRT_D void track(const float (&yv)[G * 4], Index &&index_of) {
    const bool hx = mx.screen(yv), hn = mn.screen(yv);
    if (hx || hn) {
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const float w[4] = {yv[u * 4], yv[u * 4 + 1], yv[u * 4 + 2], yv[u * 4 + 3]};
        const int64_t i0 = index_of(u);
        if (hx) mx.take_vec(w, i0, key);
        if (hn) mn.take_vec(w, i0, key);
      }
    }
  }
  template <int U> OMPRT_D void vecs(const int64_t (&e)[U]) {
    uint4 rx[U], ry[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      rx[u] = ld_stream_v4(x + e[u]);
      ry[u] = ld_rw_v4(y + e[u]);
    }
    float yv[U * 4];
    group<U>(rx, ry, yv);
#pragma unroll
    for (int u = 0; u < U; ++u)
      st_stream_v4(y + e[u], make_uint4(__float_as_uint(yv[u * 4]), __float_as_uint(yv[u * 4 + 1]),
                                        __float_as_uint(yv[u * 4 + 2]),
                                        __float_as_uint(yv[u * 4 + 3])));
    track<U>(yv, [&](int u) { return e[u]; });
  }
};

// ORDERED fp max/min reduction over the SPMD machinery (team_set_cta, the
// TMA ring, the LDG walker for what the ring cannot take).
template <class T, int OP, int STAGES, int STAGE_BYTES, int MAXT = kMaxThreads>
__global__ void __launch_bounds__(MAXT)
    k_reduce_ext(const T *__restrict__ x, LoopArgs la, Workspace ws, T *out) {
  trace_begin();
  extern __shared__ __align__(128) unsigned char stages[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];
  __shared__ OrderKey s_key;
  if (threadIdx.x == 0) s_key = make_order_key(la);
  __syncthreads();
  const TeamSet s = team_set_cta(la);
  ExtReduceBody<T, OP> body(x, &s_key);
  BulkPlan<STAGE_BYTES> plan;
  const void *const ptrs[1] = {x};
  if (team_bulk_plan<STAGE_BYTES>(s, (int)sizeof(T), ptrs, plan,
                                  [&](int64_t i) { body.scalar(i); })) {
    const unsigned char *const b[1] = {(const unsigned char *)x};
    bulk_stream_stages<1, STAGES, STAGE_BYTES>(
        b, plan, stages, full, empty,
        [&](const auto &where, const uint4 *sv, uint32_t nvec, uint32_t ct, uint32_t nc) {
          // four vectors per step, screened together: the loads of a group
          // issue back to back and the element-wise path runs only for a
          // group that could move the extremum
          uint32_t v = ct;
          for (; v + 3 * nc < nvec; v += 4 * nc) {
            uint4 r[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) r[u] = sv[v + u * nc];
            if (body.screen(r)) {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                body.consume(r[u], where.byte_of(v + u * nc) / (int64_t)sizeof(T));
            }
          }
          for (; v < nvec; v += nc) {
            const uint4 r[1] = {sv[v]};
            if (body.screen(r)) body.consume(r[0], where.byte_of(v) / (int64_t)sizeof(T));
          }
        });
  } else {
    run_team<4>(body, s, threadIdx.x, blockDim.x);
  }
  const LeftExt<OP, T> team = block_merge(body.acc.finish(&s_key));
  T *pv = (T *)ws.team_partials;
  int64_t *pk = (int64_t *)(ws.team_partials + (size_t)gridDim.x * 8);
  if (ext_teams_combine<OP, T>(team, pv, pk, ws.ticket, out)) trace_combine();
}

// ORDERED C3: y = a*x + y (elementwise: the SPMD y) with the reference
// order's max and min, in one pass.
template <int STAGES, int STAGE_BYTES, int MAXT>
__global__ void __launch_bounds__(MAXT)
    k_axpy_minmax_ext(float a, const float *__restrict__ x, float *__restrict__ y, LoopArgs la,
                      Workspace ws, float *out_max, float *out_min) {
  trace_begin();
  extern __shared__ __align__(128) unsigned char stages[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];
  __shared__ OrderKey s_key;
  if (threadIdx.x == 0) s_key = make_order_key(la);
  __syncthreads();
  const TeamSet s = team_set_cta(la);
  ExtAxpyBody body(a, x, y, &s_key);
  BulkPlan<STAGE_BYTES> plan;
  const void *const ptrs[2] = {x, y};
  if (team_bulk_plan<STAGE_BYTES>(s, 4, ptrs, plan, [&](int64_t i) { body.scalar(i); })) {
    const unsigned char *const b[2] = {(const unsigned char *)x, (const unsigned char *)y};
    unsigned char *yb = (unsigned char *)y;
    constexpr uint32_t SV = STAGE_BYTES / 16;  // vectors per stream per stage
    bulk_stream_stages<2, STAGES, STAGE_BYTES>(
        b, plan, stages, full, empty,
        [&](const auto &where, const uint4 *sv, uint32_t nvec, uint32_t ct, uint32_t nc) {
          uint32_t v = ct;
          for (; v < nvec; v += nc) {
            const uint4 rx[1] = {sv[v]};
            const uint4 ry[1] = {sv[SV + v]};
            float yv[4];
            body.group<1>(rx, ry, yv);
            const int64_t off = where.byte_of(v);
            st_stream_v4(yb + off, make_uint4(__float_as_uint(yv[0]), __float_as_uint(yv[1]),
                                              __float_as_uint(yv[2]), __float_as_uint(yv[3])));
            body.track<1>(yv, [&](int) { return off / 4; });
          }
        });
  } else {
    run_team<2>(body, s, threadIdx.x, blockDim.x);  // LDG walker: misaligned / tiny teeth
  }
  const LeftExt<OMPRT_OP_MAX, float> tmax = block_merge(body.mx.finish(&s_key));
  const LeftExt<OMPRT_OP_MIN, float> tmin = block_merge(body.mn.finish(&s_key));
  // slots: max values | min values | max keys | min keys
  const size_t G = gridDim.x;
  float *pmax = (float *)ws.team_partials;
  float *pmin = pmax + G;
  int64_t *kmax = (int64_t *)(ws.team_partials + G * 8);
  int64_t *kmin = kmax + G;
  if (threadIdx.x == 0) {
    pmin[blockIdx.x] = tmin.v;
    kmin[blockIdx.x] = tmin.k;
  }
  if (ext_teams_combine<OMPRT_OP_MAX, float>(tmax, pmax, kmax, ws.ticket, out_max)) {
    LeftExt<OMPRT_OP_MIN, float> m;
    for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x)
      m.merge(ld_cg(pmin + i), ld_cg(kmin + i));
    m = block_merge(m);
    if (threadIdx.x == 0) *out_min = Red<OMPRT_OP_MIN, float>::apply(*out_min, m.v);
    trace_combine();
  }
}

}  // namespace omprt
