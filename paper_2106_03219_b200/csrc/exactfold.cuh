// exactfold.cuh — the in-order fp sum chain s = RN(s + p_0), RN(.. + p_1), ...
// folded 32 lanes wide, bit-identical to the sequential chain.
//
// The reference combines the per-thread partials one after the other in
// global thread order (host.py:567-582): one dependent fp add per partial,
// ~8 cycles each on the folder warp, and the partials of the last wave of
// groups all arrive at the end (profiles/r2_trace_ordered.jsonl: 142 us of
// tail at 148 x 384).  The chain is sequential in general, but not inside one
// binade: while s stays in [2^e, 2^(e+1)) (magnitude, fixed sign), every s is
// a multiple of u = ulp(s) = 2^(e-M) (M = 52 for fp64, 23 for fp32), so
//
//     RN(s + p) = s + u * rint(p / u)       when p/u is not a half-integer
//
// (the grid of representable numbers around s + p is exactly the multiples of
// u; round-half-even of integer + y equals integer + rint(y) unless y is a
// tie).  With S = s/u an integer, the chain becomes S_j = S_0 + q_0 + ... +
// q_{j-1} in int64 — associative, so one warp scan folds a whole batch.  The
// fast path is taken only when it is provably the same computation:
//   * s finite, normal, exponent inside a margin (p * 2^(M-e) and 2^(e-M)
//     exact powers of two);
//   * every p finite with |p/u| <= 2^(M+2) and p/u not a half-integer;
//   * every intermediate |S_j| in [2^M + 1, 2^(M+1) - 1]: the exact s + p
//     then lies strictly inside the binade, so its rounding unit is u and
//     the rounded value does not reach the binade's ends.
// Otherwise the caller folds the batch one add at a time as before.  Zero,
// NaN and infinite partials, ties and binade crossings all take the serial
// chain, so signed zeros, NaN propagation and overflow are unchanged.
#pragma once

#include "omprt.cuh"

namespace omprt {

template <class T> struct ExactBits;
template <> struct ExactBits<double> {
  static constexpr int kMant = 52, kEmin = -900, kEmax = 900;
  OMPRT_D static int exponent(double s) {  // unbiased; out of range if zero/subnormal/inf/nan
    const int be = (int)((__double_as_longlong(s) >> 52) & 0x7ff);
    return (be == 0 || be == 0x7ff) ? -100000 : be - 1023;
  }
  OMPRT_D static double pow2(int k) { return __longlong_as_double((long long)(k + 1023) << 52); }
  OMPRT_D static long long to_ll_rn(double y) { return __double2ll_rn(y); }
};
template <> struct ExactBits<float> {
  static constexpr int kMant = 23, kEmin = -100, kEmax = 100;
  OMPRT_D static int exponent(float s) {
    const int be = (__float_as_int(s) >> 23) & 0xff;
    return (be == 0 || be == 0xff) ? -100000 : be - 127;
  }
  OMPRT_D static float pow2(int k) { return __int_as_float((k + 127) << 23); }
  OMPRT_D static long long to_ll_rn(float y) { return __float2ll_rn(y); }
};

// Fold this warp's batch (lane l holds partials l*N .. l*N+N-1 of the batch,
// in order) into acc (the same value in every lane).  Returns true with acc
// advanced past the whole batch, bit-identical to the sequential chain, or
// false with acc untouched (the caller folds the batch serially).  All 32
// lanes must call it.
template <class T, int N>
OMPRT_D bool exact_fold_batch(T &acc, const T (&v)[N]) {
  using B = ExactBits<T>;
  const int e = B::exponent(acc);
  if (e < B::kEmin || e > B::kEmax) return false;  // warp-uniform: acc is
  const T inv = B::pow2(B::kMant - e);
  const T lim = B::pow2(B::kMant + 2);
  bool ok = true;
  long long pre[N];  // this lane's inclusive prefix of the rounded quotients
  long long run = 0;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const T y = v[k] * inv;  // exact: a power-of-two scale (overflow -> inf fails below)
    ok &= fabs(y) <= lim;    // NaN fails too
    const long long q = B::to_ll_rn(y);
    ok &= fabs(y - (T)q) != (T)0.5;  // a tie: the rounding would depend on S's parity
    run += q;
    pre[k] = run;
  }
  // exclusive scan of the lanes' totals
  long long incl = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const long long t = __shfl_up_sync(0xffffffffu, incl, d);
    if ((int)(threadIdx.x & 31u) >= d) incl += t;
  }
  const long long s0 = B::to_ll_rn(acc * inv);  // exact: acc / u is an integer
  const long long base = s0 + (incl - run);
  constexpr long long lo = (1ll << B::kMant) + 1, hi = (1ll << (B::kMant + 1)) - 1;
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const long long sj = base + pre[k];
    const long long a = sj < 0 ? -sj : sj;
    ok &= a >= lo && a <= hi;
  }
  if (!__all_sync(0xffffffffu, ok)) return false;
  const long long sn = s0 + __shfl_sync(0xffffffffu, incl, 31);
  acc = (T)sn * B::pow2(e - B::kMant);  // exact: |sn| < 2^(M+1)
  return true;
}

// acc (lane 0's value on entry; the same in every lane on return) folded with
// p[0..m) in order, 256 partials a step through exact_fold_batch, lane 0's
// one-add-at-a-time chain for a step that does not qualify (after a miss the
// next attempts back off: at most one per 16 steps on data that never
// qualifies).  p is read in place (shared or global).  All 32 lanes of a
// full warp call.
template <class T> OMPRT_D T warp_sum_in_order(T acc, const T *p, int m) {
  constexpr int N = 8;
  const uint32_t lane = threadIdx.x & 31u;
  acc = __shfl_sync(0xffffffffu, acc, 0);
  int wait = 0, miss = 0;
  for (int k0 = 0; k0 < m; k0 += 32 * N) {
    const int mm = m - k0 < 32 * N ? m - k0 : 32 * N;
    if (wait == 0) {
      T mine[N];
#pragma unroll
      for (int u = 0; u < N; ++u) {
        const int i = (int)lane * N + u;
        mine[u] = i < mm ? p[k0 + i] : T(0);
      }
      if (exact_fold_batch<T, N>(acc, mine)) {
        miss = 0;
        continue;
      }
      miss = miss < 4 ? miss + 1 : 4;
      wait = (1 << miss) - 1;
    } else {
      --wait;
    }
    if (lane == 0)
      for (int k = 0; k < mm; ++k) acc = acc + p[k0 + k];
    acc = __shfl_sync(0xffffffffu, acc, 0);
  }
  return acc;
}

}  // namespace omprt
