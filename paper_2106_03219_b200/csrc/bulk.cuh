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

// Default ring: 4 x 32 KiB = 128 KiB in flight per team, one team per SM.
// Measured steady state (power-capped, back to back) on B200: a 256-thread
// team streams as fast as a 1024-thread one in isolation but draws less
// power, so it keeps ~7.46 TB/s where 1024 threads settle at ~7.13 TB/s
// (profiles/r1_steady_bulk.jsonl).
constexpr int kBulkStages = 4;
constexpr int kBulkStageBytes = 32768;

template <int STAGES, int STAGE_BYTES> struct BulkSmem {
  static constexpr size_t bytes = (size_t)STAGES * STAGE_BYTES;
};

// Stream [base, base + nbytes) (16-byte aligned, nbytes % 16 == 0) through
// the stage ring; `consume(const uint4&)` is called by the consumer threads
// (all warps but warp 0) for every 16-byte vector exactly once.
template <int STAGES, int STAGE_BYTES, class F>
OMPRT_D void bulk_stream(const unsigned char *base, int64_t nbytes, unsigned char *stages,
                         uint64_t *full, uint64_t *empty, F &&consume) {
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t nwarps = blockDim.x >> 5;
  const int64_t nchunks = (nbytes + STAGE_BYTES - 1) / STAGE_BYTES;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwarps - 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      for (int64_t k = 0; k < nchunks; ++k) {
        const int st = (int)(k % STAGES);
        if (k >= STAGES) mbar_wait(&empty[st], (uint32_t)((k / STAGES - 1) & 1));
        const int64_t rem = nbytes - k * STAGE_BYTES;
        const uint32_t b = (uint32_t)(rem < STAGE_BYTES ? rem : STAGE_BYTES);
        mbar_expect_tx(&full[st], b);
        bulk_g2s(stages + (size_t)st * STAGE_BYTES, base + k * STAGE_BYTES, b, &full[st], pol);
      }
    }
  } else {
    const uint32_t ct = threadIdx.x - 32, nc = blockDim.x - 32;
    for (int64_t k = 0; k < nchunks; ++k) {
      const int st = (int)(k % STAGES);
      mbar_wait(&full[st], (uint32_t)((k / STAGES) & 1));
      const int64_t rem = nbytes - k * STAGE_BYTES;
      const uint32_t nvec = (uint32_t)((rem < STAGE_BYTES ? rem : STAGE_BYTES) >> 4);
      const uint4 *sv = (const uint4 *)(stages + (size_t)st * STAGE_BYTES);
      for (uint32_t v = ct; v < nvec; v += nc) consume(sv[v]);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
}

template <class T, int OP, int STAGES, int STAGE_BYTES>
__global__ void __launch_bounds__(kMaxThreads)
    k_reduce_bulk(const T *__restrict__ x, LoopArgs la, Workspace ws, T *out) {
  extern __shared__ __align__(128) unsigned char stages[];
  __shared__ __align__(8) uint64_t full[STAGES];
  __shared__ __align__(8) uint64_t empty[STAGES];
  __shared__ T scratch[32];
  const TeamSet s = team_set(la.sched, la.lb, la.ub, la.chunk, blockIdx.x, gridDim.x, blockDim.x);
  int64_t count = 0;
  if (s.nseg > 0) {
    count = s.ub - s.first + 1;
    if (count > s.seg_len) count = s.seg_len;
  }
  ReduceBody<T, OP> body(x);
  constexpr int V = ReduceBody<T, OP>::V;
  int64_t head = 0;
  while (head < V && head < count && !body.head_ok(s.first + head)) ++head;
  for (int64_t i = threadIdx.x; i < head; i += blockDim.x) body.scalar(s.first + i);
  const int64_t nbytes = ((count - head) * (int64_t)sizeof(T)) & ~(int64_t)15;
  if (nbytes > 0)
    bulk_stream<STAGES, STAGE_BYTES>((const unsigned char *)(x + s.first + head), nbytes, stages,
                                     full, empty, [&](const uint4 &r) { body.consume(r); });
  const int64_t done = head + nbytes / (int64_t)sizeof(T);
  for (int64_t i = done + threadIdx.x; i < count; i += blockDim.x) body.scalar(s.first + i);
  const T team_val = block_reduce<OP, T>(body.total(), scratch, blockDim.x);
  T *partials = (T *)ws.team_partials;
  if (teams_ticket<OP, T>(team_val, partials, ws.ticket)) {
    const T v = combine_team_partials<OP, T>(partials, scratch);
    if (threadIdx.x == 0) *out = Red<OP, T>::apply(*out, v);
  }
}

}  // namespace omprt
