// exchange.cuh — the multi-GPU combine fused into the reduction kernel
// (SURVEY §8(e)): instead of a separate collective after the construct, the
// team that draws the last ticket on each GPU stores its GPU partial straight
// into every rank's mailbox over NVLink peer memory (CUDA IPC mappings) and
// then folds the G partials of its own mailbox in rank order into the cell —
// one kernel per step, no collective launch, the same bits on every rank.
//
// Mailbox (one per rank, cudaMalloc'd, exported by cudaIpcGetMemHandle):
// two banks (step parity) of `world` slots {u64 value bits, u64 key}.  The
// writer stores the value, then the key with st.release.sys; the reader
// spins with ld.acquire.sys until the slot holds this step's key.  Keys are
// a per-step image of a nonce all ranks agreed on, so stale slots never
// match; two banks suffice because a rank cannot start step k+2's exchange
// before every rank has finished step k+1's, which needs this rank's step-k
// kernel to have completed.  A peer that never arrives raises the Deadlock
// trap after `timeout_ns` instead of hanging the GPU.
#pragma once

#include "kernels.cuh"

namespace omprt {

struct Exchange {
  uint64_t *const *peers;  // device array [world]: every rank's mailbox (own included)
  int rank, world;
  uint64_t key;            // this step's key (same on every rank)
  uint32_t bank;           // step parity
  uint64_t timeout_ns;
};

OMPRT_D void st_release_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
OMPRT_D void st_relaxed_sys(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
OMPRT_D uint64_t ld_acquire_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
OMPRT_D uint64_t ld_relaxed_sys(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <class T> OMPRT_D uint64_t to_bits(T v) {
  uint64_t b = 0;
  memcpy(&b, &v, sizeof(T));
  return b;
}
template <class T> OMPRT_D T from_bits(uint64_t b) {
  T v;
  memcpy(&v, &b, sizeof(T));
  return v;
}

// Thread 0 of the last team: publish `v` (this GPU's partial), then fold the
// world's partials in rank order into *out.  Returns false on timeout.
template <int OP, class T>
OMPRT_D bool exchange_fold(const Exchange &xc, T v, T *out) {
  const uint64_t bits = to_bits<T>(v);
  const size_t slot = ((size_t)xc.bank * xc.world + xc.rank) * 2;
  for (int r = 0; r < xc.world; ++r) {
    uint64_t *mb = xc.peers[r];
    st_relaxed_sys(mb + slot, bits);
    st_release_sys(mb + slot + 1, xc.key);
  }
  const uint64_t *own = xc.peers[xc.rank];
  T acc = *out;
  const uint64_t t0 = globaltimer();
  for (int r = 0; r < xc.world; ++r) {
    const uint64_t *s = own + ((size_t)xc.bank * xc.world + r) * 2;
    while (ld_acquire_sys(s + 1) != xc.key) {
      if (globaltimer() - t0 > xc.timeout_ns) {
        raise_trap(OMPRT_TRAP_DEADLOCK, r);
        return false;
      }
    }
    acc = Red<OP, T>::apply(acc, from_bits<T>(ld_relaxed_sys(s)));
  }
  *out = acc;
  return true;
}

// The SPMD bulk reduction (bulk.cuh k_reduce_bulk) with the exchange as its
// epilogue.
template <class T, int OP, int STAGES, int STAGE_BYTES>
__global__ void __launch_bounds__(kMaxThreads)
    k_reduce_bulk_exchange(const T *__restrict__ x, LoopArgs la, Workspace ws, T *out,
                           Exchange xc) {
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
    bulk_stream_n<1, STAGES, STAGE_BYTES, decltype(consume) &>(b, plan, stages, full, empty,
                                                               consume);
  } else {
    run_team<4>(body, s, threadIdx.x, blockDim.x);
  }
  const T team_val = block_reduce<OP, T>(body.total(), scratch, blockDim.x);
  T *partials = (T *)ws.team_partials;
  if (teams_ticket<OP, T>(team_val, partials, ws.ticket)) {
    const T v = combine_team_partials<OP, T>(partials, scratch);
    if (threadIdx.x == 0) exchange_fold<OP, T>(xc, v, out);
    trace_combine();
  }
}

}  // namespace omprt
