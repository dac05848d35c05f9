// loops.cuh — how a team's lanes walk the iterations the schedule gives the
// team.  Bodies (reduce, axpy+max/min, dot) plug in through a small concept:
//
//   static constexpr int V;                 elements per 16-byte vector
//   bool head_ok(int64_t i) const;          can vectors start at element i (all streams)?
//   void scalar(int64_t i);                 process element i
//   template <int U> void vecs(const int64_t (&e)[U]);
//                                           process the U vectors starting at elements e[u]
//                                           (issue all U loads before any math)
//
// Physical mapping (SURVEY §7 hard part #1): the OpenMP schedule decides which
// team owns an iteration (team_set, bit-exact with schedule_init); inside the
// team, lane l takes vectors l, l+T, l+2T ... so every warp-wide load is 512
// contiguous bytes.  Which lane of the team touches an iteration is not
// observable for associative/commutative combines (integer add wraps, max,
// min) nor for elementwise bodies; fp sums are re-associated (ORDERED mode
// keeps the literal per-thread order when bit-identity is wanted).
#pragma once

#include "omprt.cuh"

namespace omprt {

// Contiguous run of `count` iterations starting at `lo`, covered by `nthr`
// threads (this thread is `tid`).  Unaligned head and ragged tail go scalar.
template <int U, class Body>
OMPRT_D void run_contiguous(Body &b, int64_t lo, int64_t count, uint32_t tid, uint32_t nthr) {
  constexpr int V = Body::V;
  if (count <= 0) return;
  int64_t head = 0;
  while (head < V && head < count && !b.head_ok(lo + head)) ++head;
  if (head == V || !b.head_ok(lo + head)) {
    // streams mutually misaligned (or too short): coalesced scalar walk
    for (int64_t i = tid; i < count; i += nthr) b.scalar(lo + i);
    return;
  }
  for (int64_t i = tid; i < head; i += nthr) b.scalar(lo + i);
  const int64_t base = lo + head;
  const int64_t nvec = (count - head) / V;
  const int64_t step = (int64_t)nthr;
  int64_t v = tid;
  for (; v + (U - 1) * step < nvec; v += U * step) {
    int64_t e[U];
#pragma unroll
    for (int u = 0; u < U; ++u) e[u] = base + (v + u * step) * V;
    b.template vecs<U>(e);
  }
  for (; v < nvec; v += step) {
    int64_t e[1] = {base + v * V};
    b.template vecs<1>(e);
  }
  for (int64_t i = head + nvec * V + tid; i < count; i += nthr) b.scalar(lo + i);
}

// The flat schedule(static, c) team set: teeth of seg_len iterations every
// seg_stride, last tooth clipped at ub.  The team's owned units (vectors when
// every tooth starts 16-byte aligned and seg_len is a multiple of V, else
// single elements) are numbered q = 0..Q-1 tooth-major and lane l walks
// q = l, l+T, ... keeping (tooth, offset) incrementally — no division in the
// loop.
template <int U, class Body>
OMPRT_D void run_comb(Body &b, const TeamSet &s, uint32_t tid, uint32_t nthr) {
  constexpr int V = Body::V;
  if (s.nseg <= 0) return;
  if (s.nseg == 1) {
    int64_t len = s.ub - s.first + 1;
    if (len > s.seg_len) len = s.seg_len;
    run_contiguous<U>(b, s.first, len, tid, nthr);
    return;
  }
  const int64_t last_first = s.first + (s.nseg - 1) * s.seg_stride;
  int64_t last_len = s.ub - last_first + 1;
  if (last_len > s.seg_len) last_len = s.seg_len;
  const bool vec_ok = (s.seg_len % V == 0) && (s.seg_stride % V == 0) && b.head_ok(s.first);
  const int64_t W = vec_ok ? V : 1;                 // elements per unit
  const int64_t useg = s.seg_len / W;               // units per full tooth
  const int64_t ulast = last_len / W;               // units in the last tooth
  const int64_t Q = (s.nseg - 1) * useg + ulast;    // total units
  // incremental decomposition of q = r*useg + o
  int64_t r = (int64_t)tid / useg, o = (int64_t)tid % useg;
  const int64_t dr = (int64_t)nthr / useg, dq = (int64_t)nthr % useg;
  int64_t e = s.first + r * s.seg_stride + o * W;
  const int64_t de = dr * s.seg_stride + dq * W;
  const int64_t wrap = s.seg_stride - useg * W;
  int64_t q = tid;
  auto advance = [&]() {
    q += nthr;
    o += dq;
    e += de;
    if (o >= useg) {
      o -= useg;
      e += wrap;
    }
  };
  if (vec_ok) {
    for (; q + (int64_t)(U - 1) * nthr < Q;) {
      int64_t es[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        es[u] = e;
        advance();
      }
      b.template vecs<U>(es);
    }
    for (; q < Q;) {
      int64_t es[1] = {e};
      b.template vecs<1>(es);
      advance();
    }
  } else {
    for (; q < Q;) {
      b.scalar(e);
      advance();
    }
  }
  // ragged remainder of the last tooth
  const int64_t rem_first = last_first + ulast * W;
  const int64_t rem = last_len - ulast * W;
  for (int64_t i = tid; i < rem; i += nthr) b.scalar(rem_first + i);
}

// Dispatch on the team's set shape.
template <int U, class Body>
OMPRT_D void run_team(Body &b, const TeamSet &s, uint32_t tid, uint32_t nthr) {
  if (s.seg_stride == 0 || s.nseg <= 1) {
    if (s.nseg <= 0) return;
    int64_t len = s.ub - s.first + 1;
    if (len > s.seg_len) len = s.seg_len;
    run_contiguous<U>(b, s.first, len, tid, nthr);
  } else {
    run_comb<U>(b, s, tid, nthr);
  }
}

// ORDERED mode: this thread walks exactly its own schedule chunks in
// iteration order (the host fallback's per-thread loop, host.py:567-582).
template <class F>
OMPRT_D void run_thread_chunks(int sched, int64_t lb, int64_t ub, int64_t chunk, F &&f) {
  const Bounds bd = schedule_init(sched, lb, ub, chunk, blockIdx.x, gridDim.x, threadIdx.x,
                                  blockDim.x);
  const bool chunked =
      (sched == OMPRT_SCHED_STATIC_CHUNKED || sched == OMPRT_SCHED_DISTRIBUTE_CHUNKED);
  if (!chunked) {
    for (int64_t i = bd.lower; i <= bd.upper; ++i) f(i);
    return;
  }
  for (int64_t lo = bd.lower; lo <= bd.limit; lo += bd.stride) {
    int64_t hi = lo + chunk - 1;
    if (hi > bd.limit) hi = bd.limit;
    for (int64_t i = lo; i <= hi; ++i) f(i);
  }
}

}  // namespace omprt
