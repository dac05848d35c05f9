/*
 * omprt_oracle.c — TEST INFRASTRUCTURE ONLY.  The CPU restatement of the
 * reference's semantics for the data-parallel path, used as the parity
 * checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg.  Never linked into or called by the product
 * (paper_2106_03219_b200/).
 *
 * Pinned: tests/test_oracle.py checks every function here against golden
 * vectors produced by running the reference itself (oracle/gen_golden.py ->
 * tests/golden/ JSON files): devicert.static_bounds, Arena, step_*, the host
 * fallback (TargetCall.fallback) and vgpu (tgt_target) on the same inputs.
 *
 * Each function cites the reference lines it restates
 * (paths relative to /root/reference/pkg/src/forge/).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { I32 = 0, U32 = 1, I64 = 2, U64 = 3, F32 = 4, F64 = 5 };
enum { OP_ADD = 0, OP_MAX = 1, OP_MIN = 2 };
enum { S_STATIC = 0, S_STATIC_CHUNKED = 1, S_DISTRIBUTE = 2, S_DISTRIBUTE_CHUNKED = 3 };
enum { A_ADD = 0, A_MAX = 1, A_MIN = 2, A_XCHG = 3, A_CAS = 4, A_INC = 5 };

/* ------------------------------------------------------------------ threads */

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

/* ------------------------------------------------------------ partitioning */

/* Python `//` (floor division), as devicert.static_bounds uses. */
static int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}

/* devicert.static_bounds (devicert.py:110-115); host.py:872-883 calls it with
 * to_signed 64-bit arguments.  Returns 7 (DivideByZero) for nthreads == 0,
 * the trap vgpu raises for the IR's sdiv. */
int oracle_static_bounds(int64_t lb, int64_t ub, int64_t tid, int64_t n, int64_t *my_lb,
                         int64_t *my_ub) {
  if (n == 0) return 7;
  int64_t chunk = floordiv(ub - lb + 1 + n - 1, n);
  int64_t lo = lb + tid * chunk;
  int64_t hi = lo + chunk - 1;
  if (hi > ub) hi = ub;
  *my_lb = lo;
  *my_ub = hi;
  return 0;
}

typedef struct {
  int64_t lower, upper, stride, last, limit;
} bounds_t;

static bounds_t block_init(int64_t lb, int64_t ub, int64_t tid, int64_t n) {
  bounds_t b;
  oracle_static_bounds(lb, ub, tid, n, &b.lower, &b.upper);
  b.stride = (ub >= lb) ? (ub - lb + 1) : 1;
  b.last = (ub >= lb && b.lower <= ub && b.upper >= ub) ? 1 : 0;
  b.limit = ub;
  return b;
}

/* OpenMP schedule(static, c): chunk k -> thread k mod n (extension; the
 * reference has no chunk parameter). */
static bounds_t chunked_init(int64_t lb, int64_t ub, int64_t tid, int64_t n, int64_t c) {
  bounds_t b;
  b.lower = lb + tid * c;
  b.upper = b.lower + c - 1;
  if (b.upper > ub) b.upper = ub;
  b.stride = n * c;
  b.last = 0;
  b.limit = ub;
  if (ub >= lb) b.last = (((ub - lb) / c) % n == tid) ? 1 : 0;
  return b;
}

static bounds_t schedule_init(int sched, int64_t lb, int64_t ub, int64_t c, int64_t team,
                              int64_t teams, int64_t tid, int64_t threads) {
  if (sched == S_STATIC) return block_init(lb, ub, team * threads + tid, teams * threads);
  if (sched == S_STATIC_CHUNKED)
    return chunked_init(lb, ub, team * threads + tid, teams * threads, c);
  bounds_t tb = block_init(lb, ub, team, teams);
  if (tb.lower > tb.upper) {
    bounds_t e = {tb.lower, tb.upper, 1, 0, tb.upper};
    return e;
  }
  bounds_t b = (sched == S_DISTRIBUTE) ? block_init(tb.lower, tb.upper, tid, threads)
                                       : chunked_init(tb.lower, tb.upper, tid, threads, c);
  b.last = (b.last && tb.last) ? 1 : 0;
  return b;
}

/* Every (team, thread)'s init result, 4 x int64 per flat id. */
void oracle_bounds_dump(int64_t lb, int64_t ub, int sched, int64_t chunk, int64_t teams,
                        int64_t threads, int64_t *out) {
  for (int64_t t = 0; t < teams; ++t)
    for (int64_t i = 0; i < threads; ++i) {
      bounds_t b = schedule_init(sched, lb, ub, chunk, t, teams, i, threads);
      int64_t g = t * threads + i;
      out[4 * g + 0] = b.lower;
      out[4 * g + 1] = b.upper;
      out[4 * g + 2] = b.stride;
      out[4 * g + 3] = b.last;
    }
}

/* Visit this thread's iterations in order (the fallback's per-thread loop). */
#define FOR_THREAD_ITERS(sched, lb, ub, c, team, teams, tid, threads, i, BODY)             \
  do {                                                                                     \
    bounds_t _b = schedule_init(sched, lb, ub, c, team, teams, tid, threads);              \
    if (sched == S_STATIC || sched == S_DISTRIBUTE) {                                      \
      for (int64_t i = _b.lower; i <= _b.upper; ++i) { BODY; }                             \
    } else {                                                                               \
      for (int64_t _lo = _b.lower; _lo <= _b.limit; _lo += _b.stride) {                    \
        int64_t _hi = _lo + c - 1;                                                         \
        if (_hi > _b.limit) _hi = _b.limit;                                                \
        for (int64_t i = _lo; i <= _hi; ++i) { BODY; }                                     \
      }                                                                                    \
    }                                                                                      \
  } while (0)

/* ---------------------------------------------------------- synthetic data */

static uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

static uint64_t gen_bits(uint64_t seed, int k, uint64_t i) {
  return splitmix64(seed ^ ((uint64_t)k << 56) ^ i);
}

static int64_t gen_i64(uint64_t h) { return ((int64_t)h) >> 24; }
static uint64_t gen_u64(uint64_t h) { return h >> 24; }
static int32_t gen_i32(uint64_t h) { return ((int32_t)(uint32_t)(h >> 32)) >> 8; }
static uint32_t gen_u32(uint64_t h) { return (uint32_t)(h >> 40); }
static double gen_f64(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }
static float gen_f32(uint64_t h) { return (float)(h >> 40) * 0x1.0p-24f; }

void oracle_fill(void *out, int64_t n, int dtype, uint64_t seed, int k, int64_t offset) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t h = gen_bits(seed, k, (uint64_t)(offset + i));
    switch (dtype) {
      case I32: ((int32_t *)out)[i] = gen_i32(h); break;
      case U32: ((uint32_t *)out)[i] = gen_u32(h); break;
      case I64: ((int64_t *)out)[i] = gen_i64(h); break;
      case U64: ((uint64_t *)out)[i] = gen_u64(h); break;
      case F32: ((float *)out)[i] = gen_f32(h); break;
      default: ((double *)out)[i] = gen_f64(h); break;
    }
  }
}

/* ------------------------------------------------------- combine semantics */

/* step_add / step_max / step_min (devicert.py:84-95) generalised to the
 * element type as _atomic_step does (host.py:810-837): add wraps mod 2^bits
 * (done in unsigned arithmetic), max/min compare signed for i32/i64. */
#define DEF_OPS(T, NAME, LOW, HIGH)                                                      \
  static T NAME##_apply(int op, T a, T e) {                                              \
    if (op == OP_ADD) return NAME##_add(a, e);                                           \
    if (op == OP_MAX) return a < e ? e : a;                                              \
    return a > e ? e : a;                                                                \
  }                                                                                      \
  static T NAME##_ident(int op) { return op == OP_ADD ? (T)0 : (op == OP_MAX ? LOW : HIGH); }

static int32_t i32_add(int32_t a, int32_t b) { return (int32_t)((uint32_t)a + (uint32_t)b); }
static uint32_t u32_add(uint32_t a, uint32_t b) { return a + b; }
static int64_t i64_add(int64_t a, int64_t b) { return (int64_t)((uint64_t)a + (uint64_t)b); }
static uint64_t u64_add(uint64_t a, uint64_t b) { return a + b; }
static float f32_add(float a, float b) { return a + b; }
static double f64_add(double a, double b) { return a + b; }

DEF_OPS(int32_t, i32, INT32_MIN, INT32_MAX)
DEF_OPS(uint32_t, u32, 0u, 0xffffffffu)
DEF_OPS(int64_t, i64, INT64_MIN, INT64_MAX)
DEF_OPS(uint64_t, u64, 0ull, ~0ull)
DEF_OPS(float, f32, -INFINITY, INFINITY)
DEF_OPS(double, f64, -INFINITY, INFINITY)

/* ---------------------------------------------------------------- reduces */

/* The reference-order reduction of a PARTIAL_SUMS-shaped region
 * (corpus.py:219-247) as the host fallback executes it (host.py:567-582):
 * teams in order, threads in order, each thread folds its own schedule
 * chunks in iteration order starting from the identity (part = 0), then
 * combines into the cell with one atomic (host.py:810-837):
 *     cell = ((cell OP p_0) OP p_1) OP ... p_{n-1}.
 * Per-thread parts are independent, so they are computed in parallel and
 * folded sequentially — bit-identical to the sequential fallback.
 * `x` may be NULL to regenerate element i from (seed, k) on the fly. */
#define DEF_REDUCE(T, NAME, GEN)                                                          \
  static void reduce_##NAME(const T *x, uint64_t seed, int k, int64_t lb, int64_t ub,     \
                            int op, int sched, int64_t c, int64_t teams, int64_t threads, \
                            T *cell) {                                                    \
    int64_t n = teams * threads;                                                          \
    T *parts = (T *)malloc(sizeof(T) * (size_t)n);                                        \
    _Pragma("omp parallel for schedule(dynamic, 64)")                                     \
    for (int64_t g = 0; g < n; ++g) {                                                     \
      T part = NAME##_ident(op);                                                          \
      int64_t team = g / threads, tid = g % threads;                                      \
      if (x) {                                                                            \
        FOR_THREAD_ITERS(sched, lb, ub, c, team, teams, tid, threads, i,                  \
                         part = NAME##_apply(op, part, x[i]));                            \
      } else {                                                                            \
        FOR_THREAD_ITERS(sched, lb, ub, c, team, teams, tid, threads, i,                  \
                         part = NAME##_apply(op, part, GEN(gen_bits(seed, k, (uint64_t)i)))); \
      }                                                                                   \
      parts[g] = part;                                                                    \
    }                                                                                     \
    T acc = *cell;                                                                        \
    for (int64_t g = 0; g < n; ++g) acc = NAME##_apply(op, acc, parts[g]);                \
    *cell = acc;                                                                          \
    free(parts);                                                                          \
  }

DEF_REDUCE(int32_t, i32, gen_i32)
DEF_REDUCE(uint32_t, u32, gen_u32)
DEF_REDUCE(int64_t, i64, gen_i64)
DEF_REDUCE(uint64_t, u64, gen_u64)
DEF_REDUCE(float, f32, gen_f32)
DEF_REDUCE(double, f64, gen_f64)

static int reduce_any(const void *x, uint64_t seed, int k, int64_t lb, int64_t ub, int dtype,
                      int op, int sched, int64_t c, int64_t teams, int64_t threads, void *cell) {
  if (teams < 1 || threads < 1) return -1;
  if ((sched == S_STATIC_CHUNKED || sched == S_DISTRIBUTE_CHUNKED) && c < 1) return -1;
  switch (dtype) {
    case I32: reduce_i32(x, seed, k, lb, ub, op, sched, c, teams, threads, cell); break;
    case U32: reduce_u32(x, seed, k, lb, ub, op, sched, c, teams, threads, cell); break;
    case I64: reduce_i64(x, seed, k, lb, ub, op, sched, c, teams, threads, cell); break;
    case U64: reduce_u64(x, seed, k, lb, ub, op, sched, c, teams, threads, cell); break;
    case F32: reduce_f32(x, seed, k, lb, ub, op, sched, c, teams, threads, cell); break;
    case F64: reduce_f64(x, seed, k, lb, ub, op, sched, c, teams, threads, cell); break;
    default: return -1;
  }
  return 0;
}

int oracle_reduce(const void *x, int64_t lb, int64_t ub, int dtype, int op, int sched,
                  int64_t chunk, int64_t teams, int64_t threads, void *cell) {
  return reduce_any(x, 0, 0, lb, ub, dtype, op, sched, chunk, teams, threads, cell);
}

int oracle_reduce_gen(uint64_t seed, int k, int64_t lb, int64_t ub, int dtype, int op, int sched,
                      int64_t chunk, int64_t teams, int64_t threads, void *cell) {
  return reduce_any(NULL, seed, k, lb, ub, dtype, op, sched, chunk, teams, threads, cell);
}

/* Order-free reduction of generated data (integer results only depend on
 * the multiset; used for full-size integer checks).  x[i] for i in [lb, ub]. */
int oracle_reduce_gen_flat(uint64_t seed, int k, int64_t lb, int64_t ub, int dtype, int op,
                           void *cell) {
  int nt = oracle_num_threads();
  int rc = reduce_any(NULL, seed, k, lb, ub, dtype, op, S_STATIC, 1, 1, nt * 16, cell);
  return rc;
}

/* Exactly rounded sum of generated fp data: every generated f64 is
 * m * 2^-53 with m < 2^53 (f32: m * 2^-24, m < 2^24), so the exact sum is
 * (sum m) * 2^-s computed in 128-bit integers, then rounded once. */
double oracle_exact_sum_gen(uint64_t seed, int k, int64_t lb, int64_t ub, int dtype) {
  unsigned __int128 total = 0;
#pragma omp parallel
  {
    unsigned __int128 loc = 0;
#pragma omp for schedule(static)
    for (int64_t i = lb; i <= ub; ++i) {
      uint64_t h = gen_bits(seed, k, (uint64_t)i);
      loc += (dtype == F32) ? (h >> 40) : (h >> 11);
    }
#pragma omp critical
    total += loc;
  }
  long double v = (long double)total; /* 64-bit mantissa: exact below 2^64 */
  return (double)(v * ((dtype == F32) ? 0x1.0p-24L : 0x1.0p-53L));
}

/* Exact-enough truth for an fp64 array: long double Kahan summation. */
double oracle_accurate_sum_f64(const double *x, int64_t n) {
  long double s = 0.0L, comp = 0.0L;
  for (int64_t i = 0; i < n; ++i) {
    long double y = (long double)x[i] - comp;
    long double t = s + y;
    comp = (t - s) - y;
    s = t;
  }
  return (double)s;
}

/* ------------------------------------------------------------- axpy / dot */

/* y[i] = fmaf(a, x[i], y[i]) with max/min of the new y, reference order
 * (same per-thread / global-id structure as oracle_reduce). */
int oracle_axpy_minmax(float a, const float *x, float *y, int64_t lb, int64_t ub, int sched,
                       int64_t c, int64_t teams, int64_t threads, float *mx, float *mn) {
  if (teams < 1 || threads < 1) return -1;
  int64_t n = teams * threads;
  float *pmax = (float *)malloc(sizeof(float) * (size_t)n);
  float *pmin = (float *)malloc(sizeof(float) * (size_t)n);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t g = 0; g < n; ++g) {
    float hi = -INFINITY, lo = INFINITY;
    FOR_THREAD_ITERS(sched, lb, ub, c, g / threads, teams, g % threads, threads, i, {
      float v = fmaf(a, x[i], y[i]);
      y[i] = v;
      hi = hi < v ? v : hi;
      lo = lo > v ? v : lo;
    });
    pmax[g] = hi;
    pmin[g] = lo;
  }
  float accx = *mx, accn = *mn;
  for (int64_t g = 0; g < n; ++g) {
    accx = accx < pmax[g] ? pmax[g] : accx;
    accn = accn > pmin[g] ? pmin[g] : accn;
  }
  *mx = accx;
  *mn = accn;
  free(pmax);
  free(pmin);
  return 0;
}

/* part = fma(x[i], y[i], part), reference order.  x/y NULL: generated
 * (x from stream k=0, y from stream k=1). */
int oracle_dot(const double *x, const double *y, uint64_t seed, int64_t lb, int64_t ub,
               int sched, int64_t c, int64_t teams, int64_t threads, double *cell) {
  if (teams < 1 || threads < 1) return -1;
  int64_t n = teams * threads;
  double *parts = (double *)malloc(sizeof(double) * (size_t)n);
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t g = 0; g < n; ++g) {
    double part = 0.0;
    if (x) {
      FOR_THREAD_ITERS(sched, lb, ub, c, g / threads, teams, g % threads, threads, i,
                       part = fma(x[i], y[i], part));
    } else {
      FOR_THREAD_ITERS(sched, lb, ub, c, g / threads, teams, g % threads, threads, i,
                       part = fma(gen_f64(gen_bits(seed, 0, (uint64_t)i)),
                                  gen_f64(gen_bits(seed, 1, (uint64_t)i)), part));
    }
    parts[g] = part;
  }
  double acc = *cell;
  for (int64_t g = 0; g < n; ++g) acc += parts[g];
  *cell = acc;
  free(parts);
  return 0;
}

/* Accurate dot of generated data (long double Kahan over the exact products
 * a*b*2^-106 — each product is exact in a 106-bit integer, rounded once into
 * long double), for the rel-tol checks at full size. */
double oracle_accurate_dot_gen(uint64_t seed, int64_t lb, int64_t ub) {
  long double total = 0.0L;
#pragma omp parallel
  {
    long double s = 0.0L, comp = 0.0L;
#pragma omp for schedule(static)
    for (int64_t i = lb; i <= ub; ++i) {
      uint64_t a = gen_bits(seed, 0, (uint64_t)i) >> 11, b = gen_bits(seed, 1, (uint64_t)i) >> 11;
      long double p = (long double)((unsigned __int128)a * b) * 0x1.0p-106L;
      long double yy = p - comp;
      long double t = s + yy;
      comp = (t - s) - yy;
      s = t;
    }
#pragma omp critical
    total += s;
  }
  return (double)total;
}

/* Exactly accumulated dot of generated data: every product a*b (a, b < 2^53
 * integers, value a*b*2^-106) is exact in 128 bits; its high and low 64-bit
 * halves are summed separately in 128-bit integers (exact for any N below
 * 2^64), then combined and rounded once into long double and once into
 * double.  Same truth as oracle_accurate_dot_gen,
 * an order of magnitude faster (the full-size config-5 check, N = 2^33). */
double oracle_exact_dot_gen(uint64_t seed, int64_t lb, int64_t ub) {
  unsigned __int128 hi_tot = 0, lo_tot = 0;
#pragma omp parallel
  {
    unsigned __int128 hi = 0, lo = 0;
#pragma omp for schedule(static)
    for (int64_t i = lb; i <= ub; ++i) {
      const uint64_t a = gen_bits(seed, 0, (uint64_t)i) >> 11, b = gen_bits(seed, 1, (uint64_t)i) >> 11;
      const unsigned __int128 p = (unsigned __int128)a * b;
      hi += (uint64_t)(p >> 64);
      lo += (uint64_t)p;
    }
#pragma omp critical
    {
      hi_tot += hi;
      lo_tot += lo;
    }
  }
  /* total = hi_tot * 2^64 + lo_tot; fold lo's carries into hi first */
  hi_tot += lo_tot >> 64;
  lo_tot &= (unsigned __int128)UINT64_MAX;
  long double v = (long double)hi_tot * 0x1.0p64L + (long double)(uint64_t)lo_tot;
  return (double)(v * 0x1.0p-106L);
}

/* -------------------------------------------------------- generic pattern */

/* The generic-mode globalisation kernel in reference order:
 * team t takes its distribute block of [lb, ub] (static_bounds over teams);
 * worker w of P folds its static_bounds share of that block in order into
 * parts[w] (in the arena); the main thread folds parts[0..P) in order into
 * the team value starting from the identity; teams combine into the cell in
 * team order (the fallback runs teams sequentially, host.py:567-582). */
int oracle_generic_reduce(const void *x, uint64_t seed, int k, int64_t lb, int64_t ub, int dtype,
                          int op, int64_t teams, int64_t P, void *cell) {
  if (teams < 1 || P < 1) return -1;
  if (dtype == I64) {
    int64_t *tv = (int64_t *)malloc(sizeof(int64_t) * (size_t)teams);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < teams; ++t) {
      int64_t tlb, tub;
      oracle_static_bounds(lb, ub, t, teams, &tlb, &tub);
      int64_t v = i64_ident(op);
      for (int64_t w = 0; w < P; ++w) {
        int64_t mlb = tlb, mub = tlb - 1;
        if (tub >= tlb) oracle_static_bounds(tlb, tub, w, P, &mlb, &mub);
        int64_t part = i64_ident(op);
        for (int64_t i = mlb; i <= mub; ++i)
          part = i64_apply(op, part, x ? ((const int64_t *)x)[i] : gen_i64(gen_bits(seed, k, i)));
        v = i64_apply(op, v, part);
      }
      tv[t] = v;
    }
    int64_t acc = *(int64_t *)cell;
    for (int64_t t = 0; t < teams; ++t) acc = i64_apply(op, acc, tv[t]);
    *(int64_t *)cell = acc;
    free(tv);
    return 0;
  }
  if (dtype == U64) {
    uint64_t *tv = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)teams);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < teams; ++t) {
      int64_t tlb, tub;
      oracle_static_bounds(lb, ub, t, teams, &tlb, &tub);
      uint64_t v = u64_ident(op);
      for (int64_t w = 0; w < P; ++w) {
        int64_t mlb = tlb, mub = tlb - 1;
        if (tub >= tlb) oracle_static_bounds(tlb, tub, w, P, &mlb, &mub);
        uint64_t part = u64_ident(op);
        for (int64_t i = mlb; i <= mub; ++i)
          part = u64_apply(op, part, x ? ((const uint64_t *)x)[i] : gen_u64(gen_bits(seed, k, i)));
        v = u64_apply(op, v, part);
      }
      tv[t] = v;
    }
    uint64_t acc = *(uint64_t *)cell;
    for (int64_t t = 0; t < teams; ++t) acc = u64_apply(op, acc, tv[t]);
    *(uint64_t *)cell = acc;
    free(tv);
    return 0;
  }
  if (dtype == F64) {
    double *tv = (double *)malloc(sizeof(double) * (size_t)teams);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < teams; ++t) {
      int64_t tlb, tub;
      oracle_static_bounds(lb, ub, t, teams, &tlb, &tub);
      double v = f64_ident(op);
      for (int64_t w = 0; w < P; ++w) {
        int64_t mlb = tlb, mub = tlb - 1;
        if (tub >= tlb) oracle_static_bounds(tlb, tub, w, P, &mlb, &mub);
        double part = f64_ident(op);
        for (int64_t i = mlb; i <= mub; ++i)
          part = f64_apply(op, part, x ? ((const double *)x)[i] : gen_f64(gen_bits(seed, k, i)));
        v = f64_apply(op, v, part);
      }
      tv[t] = v;
    }
    double acc = *(double *)cell;
    for (int64_t t = 0; t < teams; ++t) acc = f64_apply(op, acc, tv[t]);
    *(double *)cell = acc;
    free(tv);
    return 0;
  }
  return -1;
}

/* ------------------------------------------------------------------ arena */

/* devicert.Arena (devicert.py:124-148) + the runtime's thread-0 check
 * (runtime.mc:76, 87 -> trap 3) + the heap-fallback extension (one LIFO
 * stack continuing past `capacity` into a heap of heap_cap bytes) + the
 * arena's data: 0xAA loader_uninitialized poison (vgpu.py:64-77), WRITE /
 * READ ops, and vgpu's check_uninit shadow (vgpu.py:365-369, trap 4) over the
 * shared-memory part.  script: nops x {op (0 alloc, 1 free, 2 write, 3 read),
 * bytes, offset, value}.  results: offset / 0 / 0 / u64 read, -code at the
 * trapping op, -0x7fff after it.  Returns the trap code (0 if none). */
int oracle_arena_replay(const int64_t *script, int nops, int caller_tid, int64_t capacity,
                        int heap_fallback, int64_t heap_cap, int check_uninit,
                        int64_t *results) {
  uint64_t cursor = 0, heap_cursor = 0;
  int code = 0;
  int64_t total = capacity + (heap_fallback ? heap_cap : 0);
  unsigned char *mem = (unsigned char *)malloc((size_t)(total > 0 ? total : 1));
  unsigned char *shadow = (unsigned char *)calloc((size_t)(capacity > 0 ? capacity : 1), 1);
  memset(mem, 0xAA, (size_t)(total > 0 ? total : 1));
  for (int op = 0; op < nops; ++op) {
    if (code) {
      results[op] = -0x7fff;
      continue;
    }
    const int64_t *o = script + 4 * op;
    int64_t kind = o[0];
    uint64_t bytes = (uint64_t)o[1], off = (uint64_t)o[2], value = (uint64_t)o[3];
    uint64_t need = (bytes + 7) / 8 * 8;
    if (kind == 2) { /* WRITE: little-endian value repeated by address */
      for (uint64_t j = 0; j < bytes; ++j) {
        uint64_t b = off + j;
        mem[b] = (unsigned char)((value >> (8 * (b & 7))) & 0xff);
        if ((int64_t)b < capacity) shadow[b] = 1;
      }
      results[op] = 0;
      continue;
    }
    if (kind == 3) { /* READ of (up to) 8 bytes */
      uint64_t v = 0;
      int init = 1;
      for (uint64_t j = 0; j < 8 && j < bytes; ++j) {
        v |= (uint64_t)mem[off + j] << (8 * j);
        if ((int64_t)(off + j) < capacity && !shadow[off + j]) init = 0;
      }
      if (check_uninit && !init) {
        code = 4;
        results[op] = -4;
      } else {
        results[op] = (int64_t)v;
      }
      continue;
    }
    if (caller_tid != 0) {
      code = 3;
    } else if (kind == 0) {
      if (heap_cursor == 0 && bytes <= (uint64_t)capacity && cursor + need <= (uint64_t)capacity) {
        results[op] = (int64_t)cursor;
        cursor += need;
        continue;
      }
      if (!heap_fallback || need > (uint64_t)heap_cap - heap_cursor) {
        code = 1;
      } else {
        results[op] = (int64_t)((uint64_t)capacity + heap_cursor);
        heap_cursor += need;
        continue;
      }
    } else {
      if (heap_fallback && off >= (uint64_t)capacity) {
        if (off + need - (uint64_t)capacity != heap_cursor) {
          code = 2;
        } else {
          heap_cursor = off - (uint64_t)capacity;
          results[op] = 0;
          continue;
        }
      } else if (heap_cursor != 0 || off + need != cursor) {
        code = 2;
      } else {
        cursor = off;
        results[op] = 0;
        continue;
      }
    }
    results[op] = -code;
  }
  free(mem);
  free(shadow);
  return code;
}

/* ---------------------------------------------------------------- atomics */

/* One RMW on a cell of `dtype` (bits 32/64, signed i32/i64): the
 * _atomic_step semantics (host.py:810-837) over step_* (devicert.py:84-107).
 * Values are little-endian words zero-extended to 64 bits. */
int oracle_atomic_step(int kind, int dtype, uint64_t x, uint64_t e, uint64_t d, uint64_t *new_out,
                       uint64_t *old_out) {
  int bits = (dtype == I32 || dtype == U32) ? 32 : 64;
  int sgn = (dtype == I32 || dtype == I64);
  uint64_t m = bits == 64 ? ~0ull : 0xffffffffull;
  x &= m;
  e &= m;
  d &= m;
  int64_t sx = bits == 64 ? (int64_t)x : (int64_t)(int32_t)(uint32_t)x;
  int64_t se = bits == 64 ? (int64_t)e : (int64_t)(int32_t)(uint32_t)e;
  uint64_t nv;
  switch (kind) {
    case A_ADD: nv = (x + e) & m; break;
    case A_MAX: nv = sgn ? (sx < se ? e : x) : (x < e ? e : x); break;
    case A_MIN: nv = sgn ? (sx > se ? e : x) : (x > e ? e : x); break;
    case A_XCHG: nv = e; break;
    case A_CAS: nv = (x == e) ? d : x; break;
    case A_INC:
      if (bits != 32) return -1;
      nv = (x >= e) ? 0 : ((x + 1) & m);
      break;
    default: return -1;
  }
  *new_out = nv;
  *old_out = x;
  return 0;
}
