// bulk.cuh — the SPMD reduction fed by the Tensor Memory Accelerator's bulk
// copy engine (cp.async.bulk, SASS UBLKCP) instead of per-thread LDGs.
//
// One elected producer thread (warp 0, lane 0) streams the team's contiguous
// block through a ring of STAGES shared-memory stages of STAGE_BYTES each;
// every stage completes on an mbarrier (complete_tx::bytes); the consumer
// warps fold the stage out of shared memory and release it on an `empty`
// mbarrier (one arrive per warp).  Bytes in flight per team =
// STAGES * STAGE_BYTES, independent of registers.  Only for schedules whose
// team set is contiguous (static, distribute, distribute_chunked).
#pragma once

#include "kernels.cuh"

namespace omprt {

OMPRT_D uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

OMPRT_D void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count)
               : "memory");
}

OMPRT_D void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}

OMPRT_D void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}

OMPRT_D void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

OMPRT_D uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

OMPRT_D void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Default ring: 3 x 48 KiB, one team per SM.  The ring shape trades two
// regimes against each other (same process, alternating blocks,
// profiles/r2_ring_regimes.jsonl):
//  * the round-end bench's regime (20 launches after a short warm-up, SM
//    clocks near max): 3 x 48 KiB 7.40-7.41 TB/s, 2 x 80 7.39-7.40, 4 x 32
//    7.39, 2 x 72 7.37, 2 x 96 7.31-7.34, 4 x 40 7.34, 5 x 32 7.28, 3 x 64
//    7.07, 4 x 48 6.98, 6 x 32 6.73, 8 x 16 4.94, 12 x 8 2.36;
//  * the sustained power-capped regime (after 2,000 launches, SM clock
//    1.5-1.6 GHz): 2 x 96 7.28-7.36, 4 x 40 7.25, 3 x 48 7.17-7.25, 2 x 80
//    7.10-7.22, 4 x 32 6.94-7.21.
// Copies below ~32 KiB cost ~0.5 us each per SM whatever the wait mode
// (test_wait spin and try_wait with a suspend hint measured identical), and
// more stages of the same size lose; 3 x 48 KiB is the best shape in the
// regime the bench measures and within 1 % of the best sustained one.
constexpr int kBulkStages = 3;
constexpr int kBulkStageBytes = 49152;
// Two-stream rings: axpy 4 stages x 2 streams x 16 KiB = 128 KiB (bigger
// stages lose 3-4 %: its consumers also store y); dot 2 x 2 x 48 KiB.
constexpr int kBulk2Stages = 4;
constexpr int kBulk2StageBytes = 16384;
constexpr int kDotStages = 2;
constexpr int kDotStageBytes = 49152;

template <int STAGES, int STAGE_BYTES> struct BulkSmem {
  static constexpr size_t bytes = (size_t)STAGES * STAGE_BYTES;
};

// The bytes a team streams, as teeth: `nteeth` runs of `tooth` bytes,
// `stride` bytes apart, the last one `last` bytes long; all 16-byte aligned
// multiples of 16 (relative to each stream's base pointer).  A contiguous team
// block is one tooth.  Stages never straddle a tooth boundary: a tooth larger
// than a stage is cut into stage-sized pieces (case A), smaller teeth are
// packed `per` to a stage (case B), so every stage is a handful of bulk copies.
template <int STAGE_BYTES> struct BulkPlan {
  int64_t first = 0, tooth = 0, stride = 0, nteeth = 0, last = 0;
  int64_t spt = 0;  // case A: stages per full tooth
  int64_t per = 0;  // case B: teeth per stage

  OMPRT_D void finish() {
    if (nteeth > 0 && last == 0) {
      --nteeth;
      last = tooth;
    }
    if (tooth > STAGE_BYTES) {
      spt = (tooth + STAGE_BYTES - 1) / STAGE_BYTES;
    } else if (tooth > 0) {
      per = STAGE_BYTES / tooth;
    }
  }
  OMPRT_D int64_t nstages() const {
    if (nteeth <= 0) return 0;
    if (spt) return (nteeth - 1) * spt + (last + STAGE_BYTES - 1) / STAGE_BYTES;
    return (nteeth + per - 1) / per;
  }
  OMPRT_D int64_t tooth_len(int64_t r) const { return r == nteeth - 1 ? last : tooth; }
  // case A: stage k -> (tooth r, byte offset inside the tooth, bytes)
  // case B: stage k -> teeth [k*per, min(k*per+per, nteeth))
  OMPRT_D int64_t stage_bytes(int64_t k) const {
    if (spt) {
      const int64_t r = k / spt, c = k % spt;
      const int64_t rem = tooth_len(r) - c * STAGE_BYTES;
      return rem < STAGE_BYTES ? rem : STAGE_BYTES;
    }
    const int64_t r0 = k * per;
    const int64_t r1 = (r0 + per < nteeth) ? r0 + per : nteeth;
    return (r1 - r0 - 1) * tooth + tooth_len(r1 - 1);
  }
  // Where the vectors of stage k live (computed once per stage, so the
  // per-vector position is 32-bit arithmetic): byte offset (relative to the
  // stream base) of vector v = base + (v / vpt) * stride + (v % vpt) * 16.
  struct Loc {
    int64_t base;
    int64_t stride;
    uint32_t vpt;  // 0: the stage is one contiguous piece
    OMPRT_D int64_t byte_of(uint32_t v) const {
      if (vpt == 0) return base + (int64_t)v * 16;
      return base + (int64_t)(v / vpt) * stride + (int64_t)(v % vpt) * 16;
    }
  };
  OMPRT_D Loc loc(int64_t k) const {
    Loc l;
    if (spt) {
      const int64_t r = k / spt, c = k % spt;
      l.base = first + r * stride + c * STAGE_BYTES;
      l.stride = 0;
      l.vpt = 0;
    } else {
      l.base = first + k * per * stride;
      l.stride = stride;
      l.vpt = (uint32_t)(tooth >> 4);
    }
    return l;
  }
  // Issue the bulk copies of stage k; lane `lane` of the producer warp takes
  // pieces lane, lane+32, ... (a packed stage holds up to STAGE_BYTES/512).
  template <class Issue> OMPRT_D void issue(int64_t k, uint32_t lane, Issue &&copy) const {
    if (spt) {
      if (lane == 0) {
        const int64_t r = k / spt, c = k % spt;
        copy(first + r * stride + c * STAGE_BYTES, 0, stage_bytes(k));
      }
      return;
    }
    const int64_t r0 = k * per;
    const int64_t r1 = (r0 + per < nteeth) ? r0 + per : nteeth;
    for (int64_t r = r0 + lane; r < r1; r += 32)
      copy(first + r * stride, (r - r0) * tooth, tooth_len(r));
  }
};

// Stream NS byte streams (same plan, different base pointers) through the
// stage ring (stage st of stream j lives at stages + (st*NS + j)*STAGE_BYTES).
// `stage_fn(loc, sv, nvec, ct, nc)` is called by every consumer thread (all
// warps but warp 0; consumer index ct of nc) once per stage, with the stage's
// vectors at sv (stream j's vector v at sv[j * STAGE_BYTES/16 + v]); `loc`
// (BulkPlan::Loc) locates vector v in the streams.
// The consumers release a stage with an mbarrier arrive only (the
// producer's wait on that mbarrier orders the stage's reads before the next
// bulk copy into it — the CUTLASS TMA-pipeline consumer_release pattern);
// PROXY_FENCE adds a fence.proxy.async per stage (tuning variant 17).
template <int NS, int STAGES, int STAGE_BYTES, bool PROXY_FENCE = false, class F>
OMPRT_D void bulk_stream_stages(const unsigned char *const (&base)[NS],
                                const BulkPlan<STAGE_BYTES> &plan, unsigned char *stages,
                                uint64_t *full, uint64_t *empty, F &&stage_fn) {
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t nwarps = blockDim.x >> 5;
  const int64_t nst = plan.nstages();
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwarps - 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    // producer warp: lane 0 arms the stage's transaction count, then the
    // lanes issue its bulk copies in parallel
    const uint64_t pol = policy_evict_first();
    for (int64_t k = 0; k < nst; ++k) {
      const int st = (int)(k % STAGES);
      if (k >= STAGES) mbar_wait(&empty[st], (uint32_t)((k / STAGES - 1) & 1));
      if (lane == 0) mbar_expect_tx(&full[st], (uint32_t)(plan.stage_bytes(k) * NS));
      __syncwarp();
      plan.issue(k, lane, [&](int64_t src, int64_t dst, int64_t bytes) {
#pragma unroll
        for (int j = 0; j < NS; ++j)
          bulk_g2s(stages + ((size_t)st * NS + j) * STAGE_BYTES + dst, base[j] + src,
                   (uint32_t)bytes, &full[st], pol);
      });
    }
  } else {
    const uint32_t ct = threadIdx.x - 32, nc = blockDim.x - 32;
    for (int64_t k = 0; k < nst; ++k) {
      const int st = (int)(k % STAGES);
      mbar_wait(&full[st], (uint32_t)((k / STAGES) & 1));
      const uint32_t nvec = (uint32_t)(plan.stage_bytes(k) >> 4);
      stage_fn(plan.loc(k), (const uint4 *)(stages + (size_t)st * NS * STAGE_BYTES), nvec, ct,
               nc);
      if constexpr (PROXY_FENCE)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
}

// The per-vector form: `consume(loc, v, r[0..NS))` is called by the consumer
// threads exactly once for every 16-byte vector v of every stage.
template <int NS, int STAGES, int STAGE_BYTES, class F, bool PROXY_FENCE = false>
OMPRT_D void bulk_stream_n(const unsigned char *const (&base)[NS],
                           const BulkPlan<STAGE_BYTES> &plan, unsigned char *stages,
                           uint64_t *full, uint64_t *empty, F &&consume) {
  bulk_stream_stages<NS, STAGES, STAGE_BYTES, PROXY_FENCE>(
      base, plan, stages, full, empty,
      [&](const typename BulkPlan<STAGE_BYTES>::Loc &where, const uint4 *sv, uint32_t nvec,
          uint32_t ct, uint32_t nc) {
        for (uint32_t v = ct; v < nvec; v += nc) {
          uint4 r[NS];
#pragma unroll
          for (int j = 0; j < NS; ++j) r[j] = sv[(size_t)j * (STAGE_BYTES / 16) + v];
          consume(where, v, r);
        }
      });
}

// Split the team's iteration set into a bulk plan (16-byte aligned teeth for
// every stream in `ptrs`) and the element-wise remainder walked by `scalar`:
// an unaligned head (contiguous sets), the ragged end of the last tooth.
// Returns false when the streams cannot be vectorised (mutually misaligned
// or a comb whose teeth are not 16-byte multiples): the caller then walks
// the set with per-lane loads instead.
template <int STAGE_BYTES, int NP, class Scalar>
OMPRT_D bool team_bulk_plan(const TeamSet &s, int elem, const void *const (&ptrs)[NP],
                            BulkPlan<STAGE_BYTES> &plan, Scalar &&scalar) {
  auto aligned = [&](int64_t i) {
    uintptr_t a = 0;
#pragma unroll
    for (int j = 0; j < NP; ++j) a |= (uintptr_t)ptrs[j] + (uintptr_t)(i * elem);
    return (a & 15) == 0;
  };
  if (s.nseg <= 0) return true;
  const uint32_t tid = threadIdx.x, nthr = blockDim.x;
  if (s.nseg == 1 || s.seg_stride == 0) {
    int64_t count = s.ub - s.first + 1;
    if (count > s.seg_len) count = s.seg_len;
    const int V = 16 / elem;
    int64_t head = 0;
    while (head < V && head < count && !aligned(s.first + head)) ++head;
    if (head < count && !aligned(s.first + head)) return false;
    for (int64_t i = tid; i < head && i < count; i += nthr) scalar(s.first + i);
    if (head >= count) return true;
    const int64_t vb = ((count - head) * elem) & ~(int64_t)15;
    plan.first = (s.first + head) * elem;
    plan.tooth = plan.last = vb;
    plan.nteeth = vb > 0 ? 1 : 0;
    plan.stride = 0;
    plan.finish();
    for (int64_t i = head + vb / elem + tid; i < count; i += nthr) scalar(s.first + i);
    return true;
  }
  // teeth below 512 bytes would cost one bulk copy per few vectors: the
  // per-lane walker (run_comb) is the better engine there
  if (!aligned(s.first) || (s.seg_len * elem) % 16 || (s.seg_stride * elem) % 16 ||
      s.seg_len * elem < 512)
    return false;
  const int64_t last_first = s.first + (s.nseg - 1) * s.seg_stride;
  int64_t last_len = s.ub - last_first + 1;
  if (last_len > s.seg_len) last_len = s.seg_len;
  plan.first = s.first * elem;
  plan.tooth = s.seg_len * elem;
  plan.stride = s.seg_stride * elem;
  plan.nteeth = s.nseg;
  plan.last = (last_len * elem) & ~(int64_t)15;
  plan.finish();
  for (int64_t i = (((last_len * elem) & ~(int64_t)15) / elem) + tid; i < last_len; i += nthr)
    scalar(last_first + i);
  return true;
}

// fp64 dot over the TMA ring: x and y chunks land in paired stages.
template <int STAGES, int STAGE_BYTES, int U>
__global__ void __launch_bounds__(kMaxThreads)
    k_dot_bulk(const double *__restrict__ x, const double *__restrict__ y, LoopArgs la,
               Workspace ws, double *out) {
  trace_begin();
  extern __shared__ __align__(128) unsigned char stages[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];
  __shared__ double scratch[32];
  const TeamSet s = team_set_cta(la);
  DotBody body(x, y);
  BulkPlan<STAGE_BYTES> plan;
  const void *const ptrs[2] = {x, y};
  if (team_bulk_plan<STAGE_BYTES>(s, 8, ptrs, plan, [&](int64_t i) { body.scalar(i); })) {
    const unsigned char *const b[2] = {(const unsigned char *)x, (const unsigned char *)y};
    bulk_stream_n<2, STAGES, STAGE_BYTES>(b, plan, stages, full, empty,
                                          [&](const auto &, uint32_t, const uint4 (&r)[2]) {
                                            double a[2], c[2];
                                            unpack<double>(r[0], a);
                                            unpack<double>(r[1], c);
                                            body.acc[0] = __fma_rn(a[0], c[0], body.acc[0]);
                                            body.acc[1] = __fma_rn(a[1], c[1], body.acc[1]);
                                          });
  } else {
    run_team<U>(body, s, threadIdx.x, blockDim.x);
  }
  const double team_val = block_reduce<OMPRT_OP_ADD, double>(body.total(), scratch, blockDim.x);
  double *partials = (double *)ws.team_partials;
  if (teams_ticket<OMPRT_OP_ADD, double>(team_val, partials, ws.ticket)) {
    const double v = combine_team_partials<OMPRT_OP_ADD, double>(partials, scratch);
    if (threadIdx.x == 0) *out = *out + v;
    trace_combine();
  }
}

// Chunked-schedule axpy + max/min over the TMA ring: x and y arrive by bulk
// copy, the new y leaves by coalesced 16-byte stores.
// MAXT: launch bound (256 for the default 148x256 grid: no 64-register cap,
// no spills; kMaxThreads for bigger teams).
template <int STAGES, int STAGE_BYTES, int U, int MAXT = kMaxThreads>
__global__ void __launch_bounds__(MAXT)
    k_axpy_minmax_bulk(float a, const float *__restrict__ x, float *__restrict__ y, LoopArgs la,
                       Workspace ws, float *out_max, float *out_min) {
  trace_begin();
  extern __shared__ __align__(128) unsigned char stages[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];
  __shared__ float scratch[32];
  const TeamSet s = team_set_cta(la);
  AxpyBody body(a, x, y);
  BulkPlan<STAGE_BYTES> plan;
  const void *const ptrs[2] = {x, y};
  if (team_bulk_plan<STAGE_BYTES>(s, 4, ptrs, plan, [&](int64_t i) { body.scalar(i); })) {
    const unsigned char *const b[2] = {(const unsigned char *)x, (const unsigned char *)y};
    unsigned char *yb = (unsigned char *)y;
    bulk_stream_n<2, STAGES, STAGE_BYTES>(
        b, plan, stages, full, empty, [&](const auto &where, uint32_t v, const uint4 (&r)[2]) {
          float xv[4], yv[4];
          unpack<float>(r[0], xv);
          unpack<float>(r[1], yv);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            yv[j] = __fmaf_rn(a, xv[j], yv[j]);
            body.mx[j] = Red<OMPRT_OP_MAX, float>::apply(body.mx[j], yv[j]);
            body.mn[j] = Red<OMPRT_OP_MIN, float>::apply(body.mn[j], yv[j]);
          }
          st_stream_v4(yb + where.byte_of(v), pack<float>(yv));
        });
  } else {
    run_team<U>(body, s, threadIdx.x, blockDim.x);
  }
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

template <class T, int OP, int STAGES, int STAGE_BYTES, bool PROXY_FENCE = false>
__global__ void __launch_bounds__(kMaxThreads)
    k_reduce_bulk(const T *__restrict__ x, LoopArgs la, Workspace ws, T *out) {
  trace_begin();
  extern __shared__ __align__(128) unsigned char stages[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];
  __shared__ T scratch[32];
  const TeamSet s = team_set_cta(la);
  ReduceBody<T, OP> body(x);
  BulkPlan<STAGE_BYTES> plan;
  const void *const ptrs[1] = {x};
  if (team_bulk_plan<STAGE_BYTES>(s, (int)sizeof(T), ptrs, plan,
                                  [&](int64_t i) { body.scalar(i); })) {
    const unsigned char *const b[1] = {(const unsigned char *)x};
    auto consume = [&](const auto &, uint32_t, const uint4 (&r)[1]) { body.consume(r[0]); };
    bulk_stream_n<1, STAGES, STAGE_BYTES, decltype(consume) &, PROXY_FENCE>(b, plan, stages, full,
                                                                           empty, consume);
  } else {
    run_team<4>(body, s, threadIdx.x, blockDim.x);
  }
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

}  // namespace omprt
