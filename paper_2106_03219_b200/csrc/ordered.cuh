// ordered.cuh — ORDERED mode at HBM speed for the block schedules.
//
// In ORDERED mode every OpenMP thread folds exactly its own for_static_init
// block in iteration order (the host fallback's order, host.py:567-582), so fp
// results are bit-identical to the CPU reference.  Done literally (one lane
// walking its own block) the lanes of a warp touch 32 blocks c elements
// apart: uncoalesced.  Here a team's blocks are viewed as a matrix — row i is
// thread i's block, the columns are iterations — and streamed column window
// by column window: one elected warp issues one cp.async.bulk per row window
// (P bytes of row i, 16-byte-aligned superset) into a shared-memory stage;
// then every thread folds its own row of the stage, in order, with 16-byte
// shared loads (row pitch P+16 = an odd number of 16-byte units: conflict
// free per quarter warp).  DRAM sees P-byte contiguous pieces; the fold order
// of every thread is exactly the literal one.
#pragma once

#include "bulk.cuh"

namespace omprt {

constexpr int kOrderedStages = 3;

template <int P> struct OrderedGeom {
  static constexpr int kPitch = P + 16;  // odd multiple of 16 for P in {256, 512}
  static_assert((kPitch / 16) % 2 == 1, "row pitch must be an odd number of 16-byte units");
  static __host__ __device__ size_t smem_bytes(int threads) {
    return (size_t)kOrderedStages * threads * kPitch;
  }
};

// Block rows of this team: row i = [r0 + i*c, min(r0 + i*c + c - 1, hi)].
struct BlockRows {
  int64_t r0, c, hi;
  OMPRT_D int64_t start(int64_t i) const { return r0 + i * c; }
  OMPRT_D int64_t len(int64_t i) const {
    const int64_t s = start(i);
    if (c <= 0 || s > hi) return 0;
    const int64_t e = s + c - 1 < hi ? s + c - 1 : hi;
    return e - s + 1;
  }
};

OMPRT_D BlockRows block_rows(int sched, int64_t lb, int64_t ub) {
  BlockRows b;
  if (sched == OMPRT_SCHED_STATIC) {
    const int64_t n = (int64_t)gridDim.x * blockDim.x;
    b.c = floordiv(ub - lb + 1 + n - 1, n);
    b.r0 = lb + (int64_t)blockIdx.x * blockDim.x * b.c;
    b.hi = ub;
  } else {  // DISTRIBUTE: block over teams, then block over the team's threads
    const Bounds tb = team_block(lb, ub, blockIdx.x, gridDim.x);
    const int64_t len = tb.upper - tb.lower + 1;
    b.r0 = tb.lower;
    b.hi = tb.upper;
    b.c = len > 0 ? floordiv(len + blockDim.x - 1, blockDim.x) : 0;
  }
  return b;
}

template <class T, int OP, int P>
__global__ void __launch_bounds__(256)
    k_reduce_ordered_bulk(const T *__restrict__ x, LoopArgs la, Workspace ws, T *out) {
  constexpr int kPitch = OrderedGeom<P>::kPitch;
  constexpr int W = P / (int)sizeof(T);  // iterations per row window
  constexpr int V = 16 / (int)sizeof(T);
  extern __shared__ __align__(128) unsigned char stages[];
  __shared__ __align__(8) uint64_t full[kOrderedStages];
  __shared__ __align__(8) uint64_t empty[kOrderedStages];
  const uint32_t tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const uint32_t nwarps = blockDim.x >> 5;
  const BlockRows rows = block_rows(la.sched, la.lb, la.ub);
  const int64_t nwin = rows.c > 0 ? (rows.c + W - 1) / W : 0;
  const unsigned char *xb = (const unsigned char *)x;
  if (tid == 0) {
    for (int s = 0; s < kOrderedStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  // window j of row i: global bytes [gs, ge) -> copy [gs & ~15, (ge + 15) & ~15).
  // The producer warp sums its lanes' copy sizes first and arms the stage's
  // mbarrier once (one arrive.expect_tx), then the lanes issue the copies.
  auto window = [&](uint32_t i, int64_t j, int64_t &a0, int64_t &a1) -> bool {
    const int64_t len = rows.len(i) - j * W;
    if (len <= 0) return false;
    const int64_t n = len < W ? len : W;
    const int64_t gs = (rows.start(i) + j * W) * (int64_t)sizeof(T);
    a0 = gs & ~(int64_t)15;
    a1 = (gs + n * (int64_t)sizeof(T) + 15) & ~(int64_t)15;
    return true;
  };
  auto issue = [&](int64_t j) {
    const int st = (int)(j % kOrderedStages);
    unsigned char *stage = stages + (size_t)st * blockDim.x * kPitch;
    const uint64_t pol = policy_evict_first();
    uint32_t bytes = 0;
    for (uint32_t i = lane; i < blockDim.x; i += 32) {
      int64_t a0, a1;
      if (window(i, j, a0, a1)) bytes += (uint32_t)(a1 - a0);
    }
    bytes = __reduce_add_sync(0xffffffffu, bytes);
    if (lane == 0) mbar_expect_tx(&full[st], bytes);
    __syncwarp();
    for (uint32_t i = lane; i < blockDim.x; i += 32) {
      int64_t a0, a1;
      if (window(i, j, a0, a1))
        bulk_g2s(stage + (size_t)i * kPitch, xb + a0, (uint32_t)(a1 - a0), &full[st], pol);
    }
  };

  if (warp == 0)
    for (int64_t j = 0; j < nwin && j < kOrderedStages; ++j) issue(j);

  T part = Red<OP, T>::identity();
  const int64_t my_len = rows.len(tid);
  const int64_t my_off = ((rows.start(tid) * (int64_t)sizeof(T)) & 15) / (int64_t)sizeof(T);
  for (int64_t j = 0; j < nwin; ++j) {
    const int st = (int)(j % kOrderedStages);
    mbar_wait(&full[st], (uint32_t)((j / kOrderedStages) & 1));
    int64_t n = my_len - j * W;
    if (n > W) n = W;
    if (n > 0) {
      // this thread's window starts `off` elements into its 16-byte-aligned
      // copy; fold elements off .. off+n-1 in order (off is the same in
      // every window because W*sizeof(T) is a multiple of 16)
      const unsigned char *row = stages + ((size_t)st * blockDim.x + tid) * kPitch;
      const int64_t off = my_off;
      const int64_t nq = (off + n + V - 1) / V;
      for (int64_t q = 0; q < nq; ++q) {
        T t[V];
        unpack<T>(*(const uint4 *)(row + q * 16), t);
#pragma unroll
        for (int e = 0; e < V; ++e) {
          const int64_t k = q * V + e - off;
          if (k >= 0 && k < n) part = Red<OP, T>::apply(part, t[e]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (warp == 0 && j + kOrderedStages < nwin) {
      mbar_wait(&empty[st], (uint32_t)((j / kOrderedStages) & 1));
      issue(j + kOrderedStages);
    }
  }

  T *tp = (T *)ws.thread_partials;
  tp[(int64_t)blockIdx.x * blockDim.x + tid] = part;
  __syncthreads();
  if (teams_ticket<OP, T>(part, (T *)ws.team_partials, ws.ticket)) {
    // the stage ring is drained: reuse it as the fold buffer
    const int cap = (int)(OrderedGeom<P>::smem_bytes(blockDim.x) / sizeof(T));
    const T v = fold_in_order_team<OP, T>(tid == 0 ? *out : part, tp,
                                          (int64_t)gridDim.x * blockDim.x, (T *)stages, cap);
    if (tid == 0) *out = v;
  }
}

}  // namespace omprt
