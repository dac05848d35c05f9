// omprt_b200.cu — the C ABI (include/omprt_b200.h) over the sm_100a kernels.
// Single translation unit: the device runtime, every kernel and the host
// entry points, so the trap word is one device symbol.
#include <atomic>
#include <dlfcn.h>
#include <chrono>
#include <unistd.h>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <utility>

#include "bulk.cuh"
#include "generic.cuh"
#include "ordered.cuh"
#include "exchange.cuh"
#include "leftext.cuh"

using namespace omprt;

namespace {

thread_local std::string t_last_error;

// Team-partial slots (8 bytes each) of the reduction-family workspace: the
// ORDERED max/min constructs keep a (value, order key) pair per CTA for max
// and for min (leftext.cuh).
constexpr int kReduceSlots = 4;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_last_error = buf;
  return code;
}

int check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(OMPRT_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return OMPRT_OK;
}

#define OMPRT_CUDA(call)                                                                   \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess) return fail(OMPRT_ECUDA, "%s: %s", #call, cudaGetErrorString(_e)); \
  } while (0)

inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Every stream-taking entry point runs on the stream's device: the launches,
// the SM count, the dynamic-smem opt-in and the trap word all follow the
// calling thread's current device, so a caller holding streams of several
// devices (one process driving two GPUs) must not have to select the device
// first.  The previous current device is restored on return.  The legacy /
// per-thread default streams (handles 0, 1, 2) keep the current device.
class DeviceGuard {
 public:
  explicit DeviceGuard(void *stream) {
    if (reinterpret_cast<uintptr_t>(stream) <= 2) return;
    // inside a CUDA-graph capture the stream cannot be queried for its device
    // (it would invalidate the capture): the capturing caller has its device
    // current, so the launch is captured as is
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(S(stream), &cs) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    if (cs != cudaStreamCaptureStatusNone) return;
    int want = -1, cur = -1;
    if (cudaStreamGetDevice(S(stream), &want) != cudaSuccess) {
      cudaGetLastError();  // an invalid handle surfaces at the launch instead
      return;
    }
    if (cudaGetDevice(&cur) == cudaSuccess && cur != want && cudaSetDevice(want) == cudaSuccess)
      prev_ = cur;
  }
  ~DeviceGuard() {
    if (prev_ >= 0) cudaSetDevice(prev_);
  }
  DeviceGuard(const DeviceGuard &) = delete;
  DeviceGuard &operator=(const DeviceGuard &) = delete;

 private:
  int prev_ = -1;
};
#define OMPRT_ON_STREAM_DEVICE(stream) DeviceGuard device_guard_(stream)

// Tuning knobs are per host thread: a tuning call in one thread never
// changes the kernel another caller's launch selects.
thread_local int g_unroll = 4;   // vectors in flight per lane per iteration
thread_local int g_variant = 0;  // kernel variant of the fp64 sum (0 = default)
thread_local int g_spmd_block = 0;  // CUDA threads per SPMD CTA (0 = the policy below)
constexpr int kOrderedLiteral = 20;  // variant: ORDERED mode through the literal walk
// variant: ORDERED fp max/min through the row-group kernels (ordered.cuh)
// instead of the leftmost-extremum SPMD kernels (leftext.cuh) — A/B and tests
constexpr int kOrderedRowsMinMax = 76;
bool g_trace_on = false;  // a trace ring is installed (selects traced kernel instances)

// Construct kernels are launched with programmatic dependent launch (PDL):
// the next construct on a stream gets its CTAs resident while the previous
// one drains, then waits in pdl_begin() (omprt.cuh) for its completion —
// the launch gap of back-to-back constructs is hidden.  Variant kNoPdl
// launches them plainly (A/B).
constexpr int kNoPdl = 77;
// SPMD reductions whose pieces are under this many bytes per CTA take the
// LDG walker instead of the TMA ring (default variant only: any tuning
// variant, e.g. kNoSmallPath, keeps the ring — the ring tests use that)
constexpr int64_t kSmallPieceBytes = 96 * 1024;
constexpr int kNoSmallPath = 78;

template <class... KArgs, class... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_variant == kNoPdl ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

int check_grid(int teams, int threads) {
  if (teams < 1) return fail(OMPRT_EINVAL, "teams must be >= 1 (got %d)", teams);
  if (threads < 1 || threads > kMaxThreads)
    return fail(OMPRT_EINVAL, "threads must lie in 1..%d (got %d)", kMaxThreads, threads);
  return OMPRT_OK;
}

int check_sched(int sched, int64_t chunk) {
  if (sched < OMPRT_SCHED_STATIC || sched > OMPRT_SCHED_DISTRIBUTE_CHUNKED)
    return fail(OMPRT_EINVAL, "unknown schedule %d", sched);
  if ((sched == OMPRT_SCHED_STATIC_CHUNKED || sched == OMPRT_SCHED_DISTRIBUTE_CHUNKED) &&
      chunk < 1)
    return fail(OMPRT_EINVAL, "chunked schedule needs chunk >= 1 (got %lld)", (long long)chunk);
  return OMPRT_OK;
}

// ---------------------------------------------------------------- dispatch

// The dynamic-smem opt-in is per (device, kernel) and sticky: set it once,
// not on every launch (the call costs ~microseconds, visible on short
// constructs such as config 1).
std::mutex g_smem_mu;
std::unordered_map<uint64_t, size_t> g_smem_set;

template <class K> int set_smem(K kern, size_t bytes) {
  if (bytes <= 48 * 1024) return OMPRT_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t key = ((uint64_t)dev << 56) ^ (uint64_t)(uintptr_t)(const void *)kern;
  {
    std::lock_guard<std::mutex> lk(g_smem_mu);
    auto it = g_smem_set.find(key);
    if (it != g_smem_set.end() && it->second >= bytes) return OMPRT_OK;
  }
  cudaError_t e =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return fail(OMPRT_ECUDA, "smem attribute: %s", cudaGetErrorString(e));
  std::lock_guard<std::mutex> lk(g_smem_mu);
  size_t &v = g_smem_set[key];
  if (v < bytes) v = bytes;
  return OMPRT_OK;
}

template <class T, int OP, int STAGES, int SB, bool FENCE = false>
int launch_bulk(const T *xp, LoopArgs la, int teams, int threads, Workspace w, T *op,
                cudaStream_t st) {
  auto kern = k_reduce_bulk<T, OP, STAGES, SB, FENCE>;
  const size_t smem = BulkSmem<STAGES, SB>::bytes;
  int rc = set_smem(kern, smem);
  if (rc) return rc;
  launch_k(kern, teams * (la.split > 1 ? la.split : 1), threads, smem, st, xp, la, w, op);
  return check_launch("omprt_reduce(bulk)");
}

// Tuning variants of the fp64 sum (selected by omprt_set_variant).
template <class T, int OP>
int launch_variant(int v, const T *xp, LoopArgs la, int teams, int threads, Workspace w, T *op,
                   cudaStream_t st) {
  const bool bulk_ok = threads >= 64 && threads % 32 == 0;
  switch (v) {
    case 1: k_reduce<T, OP, 4, kLoadNc><<<teams, threads, 0, st>>>(xp, la, w, op); break;
    case 2: k_reduce<T, OP, 4, kLoadEvictFirst, 32><<<teams, threads, 0, st>>>(xp, la, w, op); break;
    case 3: k_reduce<T, OP, 4, kLoadPlain><<<teams, threads, 0, st>>>(xp, la, w, op); break;
    case 4: k_reduce<T, OP, 8, kLoadNc><<<teams, threads, 0, st>>>(xp, la, w, op); break;
    case 5: k_reduce<T, OP, 2, kLoadNcL2_256B, 32><<<teams, threads, 0, st>>>(xp, la, w, op); break;
    case 6: k_reduce<T, OP, 4, kLoadNcL2_256B, 32><<<teams, threads, 0, st>>>(xp, la, w, op); break;
    case 7: k_reduce<T, OP, 4, kLoadNc, 32><<<teams, threads, 0, st>>>(xp, la, w, op); break;
    case 8: k_reduce<T, OP, 2, kLoadNc, 32><<<teams, threads, 0, st>>>(xp, la, w, op); break;
    case 9: k_reduce<T, OP, 2, kLoadEvictFirst, 32><<<teams, threads, 0, st>>>(xp, la, w, op); break;
    case 10: if (bulk_ok) return launch_bulk<T, OP, 4, 16384>(xp, la, teams, threads, w, op, st); break;
    case 11: if (bulk_ok) return launch_bulk<T, OP, 8, 16384>(xp, la, teams, threads, w, op, st); break;
    case 12: if (bulk_ok) return launch_bulk<T, OP, 4, 32768>(xp, la, teams, threads, w, op, st); break;
    case 13: if (bulk_ok) return launch_bulk<T, OP, 3, 32768>(xp, la, teams, threads, w, op, st); break;
    case 14: if (bulk_ok) return launch_bulk<T, OP, 6, 16384>(xp, la, teams, threads, w, op, st); break;
    case 15: if (bulk_ok) return launch_bulk<T, OP, 2, 32768>(xp, la, teams, threads, w, op, st); break;
    case 16: if (bulk_ok) return launch_bulk<T, OP, 12, 8192>(xp, la, teams, threads, w, op, st); break;
    case 17: if (bulk_ok) return launch_bulk<T, OP, 4, 32768, true>(xp, la, teams, threads, w, op, st); break;
    case 18: if (bulk_ok) return launch_bulk<T, OP, 6, 32768>(xp, la, teams, threads, w, op, st); break;
    case 19: if (bulk_ok) return launch_bulk<T, OP, 3, 65536>(xp, la, teams, threads, w, op, st); break;
    case 36: if (bulk_ok) return launch_bulk<T, OP, 4, 49152>(xp, la, teams, threads, w, op, st); break;
    case 37: if (bulk_ok) return launch_bulk<T, OP, 2, 98304>(xp, la, teams, threads, w, op, st); break;
    case 38: if (bulk_ok) return launch_bulk<T, OP, 2, 65536>(xp, la, teams, threads, w, op, st); break;
    case 39: if (bulk_ok) return launch_bulk<T, OP, 2, 114688>(xp, la, teams, threads, w, op, st); break;
    case 40: if (bulk_ok) return launch_bulk<T, OP, 3, 73728>(xp, la, teams, threads, w, op, st); break;
    case 46: if (bulk_ok) return launch_bulk<T, OP, 4, 57344>(xp, la, teams, threads, w, op, st); break;
    // more ring shapes (profiles/r2_ring_regimes.jsonl); 37 is round 2's 2 x 96 KiB
    case 70: if (bulk_ok) return launch_bulk<T, OP, 5, 32768>(xp, la, teams, threads, w, op, st); break;
    case 71: if (bulk_ok) return launch_bulk<T, OP, 3, 49152>(xp, la, teams, threads, w, op, st); break;
    case 72: if (bulk_ok) return launch_bulk<T, OP, 2, 81920>(xp, la, teams, threads, w, op, st); break;
    case 73: if (bulk_ok) return launch_bulk<T, OP, 4, 40960>(xp, la, teams, threads, w, op, st); break;
    case 74: if (bulk_ok) return launch_bulk<T, OP, 2, 73728>(xp, la, teams, threads, w, op, st); break;
    case 75: if (bulk_ok) return launch_bulk<T, OP, 4, 24576>(xp, la, teams, threads, w, op, st); break;
    // interleaved CTA tiles of 64 KiB / 512 KiB / 2 MiB (every CTA streams
    // neighbouring addresses at the same time) on the default ring
    case 33: case 34: case 35:
      if (!bulk_ok) break;
      la.balance = 2;
      la.tile = (int64_t)(v == 33 ? 65536 : v == 34 ? 524288 : 2097152) / (int64_t)sizeof(T);
      return launch_bulk<T, OP, kBulkStages, kBulkStageBytes>(xp, la, teams, threads, w, op, st);
    default: return fail(OMPRT_EINVAL, "unknown variant %d", v);
  }
  if (v >= 10) k_reduce<T, OP, 4><<<teams, threads, 0, st>>>(xp, la, w, op);
  return check_launch("omprt_reduce(variant)");
}

// SM count of the calling thread's current device, cached per device (it is
// asked on every launch's path)
int sm_count() {
  constexpr int kMaxDev = 64;
  static std::atomic<int> cache[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (dev >= 0 && dev < kMaxDev) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) return c;
  }
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  if (dev >= 0 && dev < kMaxDev) cache[dev].store(sms, std::memory_order_relaxed);
  return sms;
}

// SPMD launches with few teams split every team over `split` CTAs
// (team_set_cta) so the whole GPU streams: split = SMs / teams when
// teams <= SMs / 2 (teams * split <= SMs <= kMinPartialSlots).  Config 1
// (1 team x 128 threads, 2^20 int64): 148 CTAs 15.7 us, 16 CTAs 22.6 us,
// unsplit 240 us (profiles/r1_c1_split.jsonl).  Variant kNoSplit keeps one
// CTA per team.
constexpr int kNoSplit = 30;

int spmd_split(int teams) {
  if (g_variant == kNoSplit) return 1;
  const int sms = sm_count();
  if (sms <= 0 || teams * 2 > sms) return 1;
  const int cl = sms / teams, cap = kMinPartialSlots / teams;  // teams * split partial slots
  return cl < cap ? cl : cap;
}

// SPMD iteration-to-CTA mapping: the team split above, and for the flat
// chunked schedule balanced contiguous CTA pieces (team_set_cta).  Variant
// kNoSplit keeps the literal mapping (one CTA per team, its comb of teeth).
void spmd_prepare(LoopArgs &la, int teams) {
  la.split = spmd_split(teams);
  la.balance = g_variant == kNoSplit ? 0 : 1;
}

// CUDA threads per CTA of an SPMD construct kernel running an OpenMP team of
// `threads` (LoopArgs::threads carries the OpenMP count): the tuning knob if
// set, else `pref` (the construct's measured best), else the OpenMP count
// rounded up to a whole number of warps (at least two: producer + consumer).
// Preferred CTA sizes per construct (0: follow the OpenMP thread count),
// measured with the OpenMP geometry fixed (profiles/r2_block_sweep.jsonl):
// the fp64 sum at 2^30 streams best from 384-thread CTAs whatever the team
// size (OpenMP 148 x 1024: 5.97 TB/s on 1024-thread CTAs, 7.05 on 384), the
// two-stream dot from 256 (7.09-7.13 vs 6.94 at 384); axpy (read, read,
// write) from 1024 (+1-3 % over 256-768: more warps issue the y stores).
constexpr int kReduceBlock = 384, kAxpyBlock = 1024, kDotBlock = 256;
// ORDERED axpy + max/min (leftext.cuh): its (value, key) trackers need more
// registers than 1024-thread CTAs allow
constexpr int kAxpyExtBlock = 512;

int spmd_block(int threads, int pref) {
  if (g_spmd_block > 0) return g_spmd_block;
  if (pref > 0) return pref;
  int b = (threads + 31) / 32 * 32;
  return b < 64 ? 64 : b;
}

// ORDERED row-group kernels (ordered.cuh).  Each CTA = nw streaming warps +
// the folder warp; one CTA per SM (the tile ring takes most of the shared
// memory), never more CTAs than the warp groups need.  Every launch gets a
// fresh 64-bit key for the per-group ready flags (so the shared workspace is
// reused without re-zeroing).
std::atomic<uint64_t> g_ord_epoch{0};

uint64_t next_epoch() {
  static const uint64_t nonce =
      (uint64_t)std::chrono::high_resolution_clock::now().time_since_epoch().count() ^
      ((uint64_t)getpid() << 32);
  uint64_t z = nonce + 0x9E3779B97F4A7C15ull * (++g_ord_epoch);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z ? z : 1;
}

inline int ord_grid(int teams, int threads, int nw) {
  const int64_t groups = ((int64_t)teams * threads + 31) / 32;
  int64_t g = (groups + nw - 1) / nw;
  const int sms = sm_count();
  if (sms > 0 && g > sms) g = sms;
  return (int)(g < 1 ? 1 : g);
}

// streaming warps per CTA: enough that every SM gets work; at most 8 (three
// 256-byte stages each), or up to 12 (two stages) when that puts every group
// in flight at once (e.g. 148 x 384 OpenMP threads: 12 groups per SM)
inline int ord_default_nw(int teams, int threads) {
  const int64_t groups = ((int64_t)teams * threads + 31) / 32;
  const int sms = sm_count() > 0 ? sm_count() : 148;
  int64_t nw = (groups + sms - 1) / sms;
  if (nw > 8) nw = nw <= 12 ? nw : 8;
  return (int)(nw < 1 ? 1 : nw);
}

// Six streaming warps fill whole waves when the 32-thread groups per SM are
// a multiple of six (up to `whole_max` groups per SM), or are many (>= `many`).
constexpr int kOrderedNoSix = 44;  // variant: never the six-warp policy (A/B)
inline bool ord_six_warps(int teams, int threads, int64_t whole_max, int64_t many) {
  if (g_variant == kOrderedNoSix) return false;
  const int64_t groups = ((int64_t)teams * threads + 31) / 32;
  const int sms = sm_count() > 0 ? sm_count() : 148;
  const int64_t per_sm = (groups + sms - 1) / sms;
  return (per_sm % 6 == 0 && per_sm <= whole_max) || per_sm >= many;
}

// Segments per group for the dynamic (load-balanced) ORDERED walk: block
// schedules only, ~64+ windows per unit, at most 8 units per group;
// omprt_set_variant(31) keeps the static assignment.
constexpr int kOrderedStatic = 31;

int ord_segments(const LoopArgs &la, int teams, int threads, int window_elems, int elem_bytes) {
  if (g_variant == kOrderedStatic) return 0;
  // chunked rows: segments need every chunk at the same 16-byte offset
  if ((la.sched == OMPRT_SCHED_STATIC_CHUNKED || la.sched == OMPRT_SCHED_DISTRIBUTE_CHUNKED) &&
      la.chunk % (16 / elem_bytes) != 0)
    return 0;
  if (la.ub < la.lb) return 0;
  const int64_t P = (int64_t)teams * threads;
  const int64_t per_row = (la.ub - la.lb + 1 + P - 1) / P;
  const int64_t windows = per_row / window_elems;
  int64_t seg = windows / 64;
  return (int)(seg < 1 ? 1 : (seg > 8 ? 8 : seg));
}

template <class T, int OP, int WB>
int launch_ordered_rows(const T *xp, LoopArgs la, int teams, int threads, int nw, Workspace w,
                        T *op, cudaStream_t st) {
  constexpr int W = WB / (int)sizeof(T);
  using L = OrdSmem<T, W, 1>;
  const int stages = L::stages_for(nw);
  if (stages < 2) return fail(OMPRT_EINVAL, "ordered rows: %d warps x %d B do not fit", nw, WB);
  const size_t ring = (size_t)nw * L::warp_bytes(stages);
  const size_t smem = ring + kFolderSmem;
  auto kern = k_reduce_ordered_rows<T, OP, W>;
  int rc = set_smem(kern, smem);
  if (rc) return rc;
  kern<<<ord_grid(teams, threads, nw), (nw + 1) * 32, smem, st>>>(
      xp, la, teams, threads, w, op, stages, next_epoch(), (uint32_t)ring,
      ord_segments(la, teams, threads, W, (int)sizeof(T)));
  return check_launch("omprt_reduce(ordered rows)");
}

// Default ORDERED policy: six warps with 512-byte row windows (two stages)
// when the groups per SM come in whole waves of six (6, 12 or 18 per SM);
// else 512-byte windows when three stages fit, else 256-byte windows.
// Measured: 148 x 384 threads 5.53 vs 5.18 TB/s isolated
// (profiles/r1_ordered_sweep_windows.jsonl) and 5.49-5.59 vs 5.10-5.13 in
// the power-capped steady state (profiles/r1_ordered_steady_ab.jsonl), where
// 24 and 32 groups per SM gain nothing (-2 % at 148 x 1024); 8 or 16 groups
// per SM lose a partial wave with six warps (4.1 / 5.2 vs 5.4).
template <class T, int OP>
int launch_ordered_default(const T *xp, LoopArgs la, int teams, int threads, Workspace w, T *op,
                           cudaStream_t st) {
  if (ord_six_warps(teams, threads, 18, INT64_MAX) &&
      OrdSmem<T, 512 / (int)sizeof(T), 1>::stages_for(6) >= 2)
    return launch_ordered_rows<T, OP, 512>(xp, la, teams, threads, 6, w, op, st);
  const int nw = ord_default_nw(teams, threads);
  if (OrdSmem<T, 512 / (int)sizeof(T), 1>::stages_for(nw) >= 3)
    return launch_ordered_rows<T, OP, 512>(xp, la, teams, threads, nw, w, op, st);
  return launch_ordered_rows<T, OP, 256>(xp, la, teams, threads, nw, w, op, st);
}

// Tuning variants of the ORDERED fp64 sum (21..29): window bytes × warps.
template <class T, int OP>
int launch_ordered_variant(int v, const T *xp, LoopArgs la, int teams, int threads, Workspace w,
                           T *op, cudaStream_t st) {
  switch (v) {
    case 21: return launch_ordered_rows<T, OP, 512>(xp, la, teams, threads, 4, w, op, st);
    case 22: return launch_ordered_rows<T, OP, 256>(xp, la, teams, threads, 8, w, op, st);
    case 23: return launch_ordered_rows<T, OP, 128>(xp, la, teams, threads, 16, w, op, st);
    case 24: return launch_ordered_rows<T, OP, 256>(xp, la, teams, threads, 4, w, op, st);
    case 25: return launch_ordered_rows<T, OP, 512>(xp, la, teams, threads, 2, w, op, st);
    case 26: return launch_ordered_rows<T, OP, 256>(xp, la, teams, threads, 12, w, op, st);
    case 27: return launch_ordered_rows<T, OP, 128>(xp, la, teams, threads, 8, w, op, st);
    case 28: return launch_ordered_rows<T, OP, 256>(xp, la, teams, threads, 6, w, op, st);
    case 29: return launch_ordered_rows<T, OP, 512>(xp, la, teams, threads, 6, w, op, st);
    case 41: return launch_ordered_rows<T, OP, 512>(xp, la, teams, threads, 5, w, op, st);
    default: return fail(OMPRT_EINVAL, "unknown ordered variant %d", v);
  }
}

// ORDERED fp max/min as the SPMD construct with leftmost tie-breaking
// (leftext.cuh): order keys pack the iteration below bit 40.
bool ext_ok(const LoopArgs &la) { return la.ub < la.lb || la.ub - la.lb < ((int64_t)1 << 40); }

template <class T, int OP>
int launch_reduce_ext(const T *xp, LoopArgs la, int teams, int threads, Workspace w, T *op,
                      cudaStream_t st) {
  spmd_prepare(la, teams);
  la.threads = threads;
  const int blk = spmd_block(threads, kReduceBlock);
  auto kern = blk <= kReduceBlock ? k_reduce_ext<T, OP, kBulkStages, kBulkStageBytes, kReduceBlock>
                                  : k_reduce_ext<T, OP, kBulkStages, kBulkStageBytes>;
  const size_t smem = BulkSmem<kBulkStages, kBulkStageBytes>::bytes;
  int rc = set_smem(kern, smem);
  if (rc) return rc;
  launch_k(kern, teams * la.split, blk, smem, st, xp, la, w, op);
  return check_launch("omprt_reduce(ordered max/min)");
}

template <class T, int OP>
int launch_reduce_t(const void *x, LoopArgs la, int teams, int threads, int mode, Workspace w,
                    void *out, cudaStream_t st) {
  const T *xp = (const T *)x;
  T *op = (T *)out;
  if constexpr (std::is_same<T, double>::value && OP == OMPRT_OP_ADD) {
    if (g_variant != 0 && mode == OMPRT_MODE_SPMD &&
        (g_variant < kOrderedLiteral || (g_variant >= 33 && g_variant <= 40) || g_variant == 46 ||
         (g_variant >= 70 && g_variant <= 75)))
      return launch_variant<T, OP>(g_variant, xp, la, teams, threads, w, op, st);
  }
  // Integer add (mod 2^n), max and min are associative and commutative: the
  // reference order's result IS the re-associated one, bit for bit, so
  // ORDERED integer reductions take the SPMD kernels (variant kOrderedLiteral
  // still forces the literal walk, for the tests).
  if (mode == OMPRT_MODE_ORDERED && std::is_integral<T>::value && g_variant != kOrderedLiteral)
    mode = OMPRT_MODE_SPMD;
  if (mode == OMPRT_MODE_ORDERED) {
    if constexpr (std::is_floating_point<T>::value && OP != OMPRT_OP_ADD) {
      if (g_variant != kOrderedLiteral && g_variant != kOrderedRowsMinMax && ext_ok(la))
        return launch_reduce_ext<T, OP>(xp, la, teams, threads, w, op, st);
    }
    // row-group kernels (ordered.cuh); the literal walk for small chunks,
    // pointers not 16-byte aligned, or variant kOrderedLiteral
    if constexpr (std::is_same<T, double>::value && OP == OMPRT_OP_ADD) {
      if (g_variant > kOrderedLiteral && g_variant < 30)
        return launch_ordered_variant<T, OP>(g_variant, xp, la, teams, threads, w, op, st);
    }
    if constexpr (std::is_floating_point<T>::value) {
      if (g_variant != kOrderedLiteral && ord_rows_ok(la, x))
        return launch_ordered_default<T, OP>(xp, la, teams, threads, w, op, st);
    }
    {
      k_reduce_ordered<T, OP><<<teams, threads, 0, st>>>(xp, la, w, op);
    }
  } else {
    spmd_prepare(la, teams);
    la.threads = threads;
    const int grid = teams * la.split;
    const int blk = spmd_block(threads, kReduceBlock);
    // Small pieces per CTA (config 1: 8 MiB over 148 CTAs) are latency-bound:
    // the ring would wait for a whole first stage to land; eight 16-byte
    // loads in flight per lane cover the piece in about one round trip.
    const int64_t n = la.ub - la.lb + 1;
    const bool small = n > 0 && n * (int64_t)sizeof(T) < (int64_t)grid * kSmallPieceBytes;
    if (g_unroll == 4 && !(small && g_variant == 0)) {
      // default SPMD path: TMA bulk-copy stage ring
      return launch_bulk<T, OP, kBulkStages, kBulkStageBytes>(xp, la, teams, blk, w, op, st);
    } else if (small && g_variant == 0 && g_unroll == 4) {
      // up to 96 KiB per CTA: 16 vectors in flight per lane of a 384-thread
      // CTA cover the piece in one round trip
      launch_k(k_reduce<T, OP, 16>, grid, blk, 0, st, xp, la, w, op);
    } else if (g_unroll >= 8) {
      launch_k(k_reduce<T, OP, 8>, grid, blk, 0, st, xp, la, w, op);
    } else {
      launch_k(k_reduce<T, OP, 2>, grid, blk, 0, st, xp, la, w, op);
    }
  }
  return check_launch("omprt_reduce");
}

template <class T>
int launch_reduce_op(int op, const void *x, LoopArgs la, int teams, int threads, int mode,
                     Workspace w, void *out, cudaStream_t st) {
  switch (op) {
    case OMPRT_OP_ADD:
      return launch_reduce_t<T, OMPRT_OP_ADD>(x, la, teams, threads, mode, w, out, st);
    case OMPRT_OP_MAX:
      return launch_reduce_t<T, OMPRT_OP_MAX>(x, la, teams, threads, mode, w, out, st);
    case OMPRT_OP_MIN:
      return launch_reduce_t<T, OMPRT_OP_MIN>(x, la, teams, threads, mode, w, out, st);
  }
  return fail(OMPRT_EINVAL, "unknown reduction op %d", op);
}

size_t dtype_size(int dtype) {
  switch (dtype) {
    case OMPRT_I32:
    case OMPRT_U32:
    case OMPRT_F32:
      return 4;
    case OMPRT_I64:
    case OMPRT_U64:
    case OMPRT_F64:
      return 8;
  }
  return 0;
}

template <template <class> class F, class... A> int by_dtype(int dtype, A... a) {
  switch (dtype) {
    case OMPRT_I32:
      return F<int32_t>::run(a...);
    case OMPRT_U32:
      return F<uint32_t>::run(a...);
    case OMPRT_I64:
      return F<int64_t>::run(a...);
    case OMPRT_U64:
      return F<uint64_t>::run(a...);
    case OMPRT_F32:
      return F<float>::run(a...);
    case OMPRT_F64:
      return F<double>::run(a...);
  }
  return fail(OMPRT_EINVAL, "unknown dtype %d", dtype);
}

template <class T> struct ReduceF {
  static int run(int op, const void *x, LoopArgs la, int teams, int threads, int mode,
                 Workspace w, void *out, cudaStream_t st) {
    return launch_reduce_op<T>(op, x, la, teams, threads, mode, w, out, st);
  }
};

template <class T, int OP>
int launch_exchange_t(const void *x, LoopArgs la, int teams, int threads, Workspace w, void *out,
                      const Exchange &xc, cudaStream_t st) {
  auto kern = k_reduce_bulk_exchange<T, OP, kBulkStages, kBulkStageBytes>;
  const size_t smem = BulkSmem<kBulkStages, kBulkStageBytes>::bytes;
  int rc = set_smem(kern, smem);
  if (rc) return rc;
  spmd_prepare(la, teams);
  la.threads = threads;
  launch_k(kern, teams * la.split, spmd_block(threads, kReduceBlock), smem, st, (const T *)x, la,
           w, (T *)out, xc);
  return check_launch("omprt_reduce_exchange");
}

template <class T> struct ExchangeF {
  static int run(int op, const void *x, LoopArgs la, int teams, int threads, Workspace w,
                 void *out, Exchange xc, cudaStream_t st) {
    switch (op) {
      case OMPRT_OP_ADD:
        return launch_exchange_t<T, OMPRT_OP_ADD>(x, la, teams, threads, w, out, xc, st);
      case OMPRT_OP_MAX:
        return launch_exchange_t<T, OMPRT_OP_MAX>(x, la, teams, threads, w, out, xc, st);
      case OMPRT_OP_MIN:
        return launch_exchange_t<T, OMPRT_OP_MIN>(x, la, teams, threads, w, out, xc, st);
    }
    return fail(OMPRT_EINVAL, "unknown op %d", op);
  }
};

template <class T> struct FillF {
  static int run(void *x, int64_t n, uint64_t seed, int k, int64_t offset, cudaStream_t st) {
    if (n <= 0) return OMPRT_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t vecs = n / (int64_t)(16 / sizeof(T)) + 1;
    int64_t blocks = (vecs + 255) / 256;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    k_fill<T><<<(unsigned)blocks, 256, 0, st>>>((T *)x, n, seed, k, offset);
    return check_launch("omprt_fill");
  }
};

template <class T> struct CombineF {
  static int run(int op, const void *p, int count, void *out, cudaStream_t st) {
    switch (op) {
      case OMPRT_OP_ADD:
        k_combine<T, OMPRT_OP_ADD><<<1, 32, 0, st>>>((const T *)p, count, (T *)out);
        break;
      case OMPRT_OP_MAX:
        k_combine<T, OMPRT_OP_MAX><<<1, 32, 0, st>>>((const T *)p, count, (T *)out);
        break;
      case OMPRT_OP_MIN:
        k_combine<T, OMPRT_OP_MIN><<<1, 32, 0, st>>>((const T *)p, count, (T *)out);
        break;
      default:
        return fail(OMPRT_EINVAL, "unknown reduction op %d", op);
    }
    return check_launch("omprt_combine_partials");
  }
};

template <class T> struct AtomicF {
  static int run(int kind, const uint64_t *ops, const uint64_t *desired, void *cell,
                 uint64_t *old, int teams, int threads, cudaStream_t st) {
    k_atomic_probe<T><<<teams, threads, 0, st>>>(kind, ops, desired, (T *)cell, old);
    return check_launch("omprt_atomic_probe");
  }
  static int program(const int32_t *kinds, const uint64_t *ops, const uint64_t *desired,
                     const int64_t *offsets, void *cell, uint64_t *old, int teams, int threads,
                     cudaStream_t st) {
    k_atomic_program<T><<<teams, threads, 0, st>>>(kinds, ops, desired, offsets, (T *)cell, old);
    return check_launch("omprt_atomic_program");
  }
  static int apply(int kind, void *cells, const uint64_t *ops, const uint64_t *desired,
                   uint64_t *old, int64_t n, cudaStream_t st) {
    if (n <= 0) return OMPRT_OK;
    const int64_t blocks = (n + 255) / 256;
    k_atomic_apply<T><<<(unsigned)blocks, 256, 0, st>>>(kind, (T *)cells, ops, desired, old, n);
    return check_launch("omprt_atomic_apply");
  }
};

int check_atomic(int kind, int dtype, const uint64_t *desired) {
  if (kind < OMPRT_ATOMIC_ADD || kind > OMPRT_ATOMIC_INC)
    return fail(OMPRT_EINVAL, "unknown atomic kind %d", kind);
  if (dtype != OMPRT_I32 && dtype != OMPRT_U32 && dtype != OMPRT_I64 && dtype != OMPRT_U64)
    return fail(OMPRT_EINVAL, "atomics take i32/u32/i64/u64 (got dtype %d)", dtype);
  if (kind == OMPRT_ATOMIC_INC && dtype != OMPRT_U32)
    return fail(OMPRT_EINVAL, "atomic_inc is u32 only (runtime.mc:175-186)");
  if (kind == OMPRT_ATOMIC_CAS && !desired) return fail(OMPRT_EINVAL, "CAS needs desired values");
  return OMPRT_OK;
}

// Generic mode: teams of up to 288 threads take the one-wave instance
// (seven teams per SM); variant kGenericNoOneWave keeps the default one (A/B).
constexpr int kGenericOneWaveThreads = 288;
constexpr int kGenericNoOneWave = 45;

template <class T, int OP>
int launch_generic_t(const void *x, int64_t lb, int64_t ub, int teams, int P, int ordered,
                     int64_t pad, ArenaCfg cfg, Workspace w, void *out, int64_t *offs,
                     cudaStream_t st) {
  // the ORDERED instance only where order matters (fp): integer folds give
  // the same bits in any order (see launch_reduce_t) and take the SPMD one
  auto kern = g_trace_on ? k_generic<T, OP, 4, false, true> : k_generic<T, OP, 4, false>;
  if (32 + P <= kGenericOneWaveThreads && g_variant != kGenericNoOneWave)
    kern = g_trace_on ? k_generic<T, OP, 2, false, true, kGenericOneWaveThreads, 7>
                      : k_generic<T, OP, 2, false, false, kGenericOneWaveThreads, 7>;
  if constexpr (std::is_floating_point<T>::value) {
    if (ordered) kern = g_trace_on ? k_generic<T, OP, 4, true, true> : k_generic<T, OP, 4, true>;
    // teams of <= 288 threads: pinned at four teams per SM (<= 56 registers;
    // the residency A/B in profiles/r2_c4_ordered_residency_ab.jsonl)
    if (ordered && 32 + P <= kGenericOneWaveThreads)
      kern = g_trace_on ? k_generic<T, OP, 4, true, true, kGenericOneWaveThreads, 4>
                        : k_generic<T, OP, 4, true, false, kGenericOneWaveThreads, 4>;
  }
  // Physical backing of the team arena: the region's known allocation
  // footprint (pad, then parts[P+1]) capped at the semantic capacity.  The
  // overflow check still uses cfg.capacity (64 KiB, the reference's
  // ARENA_CAPACITY), so traps are unchanged; a small footprint just leaves
  // room for more resident teams per SM.
  const int64_t footprint =
      (pad + 7) / 8 * 8 + (int64_t)(P + 1) * (int64_t)sizeof(T);
  int64_t phys = footprint < cfg.capacity ? footprint : cfg.capacity;
  phys = (phys + 15) / 16 * 16;
  if (phys < 16) phys = 16;
  const size_t smem = (size_t)phys;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess)
      return fail(OMPRT_ECUDA, "generic: smem attribute: %s", cudaGetErrorString(e));
  }
  launch_k(kern, teams, 32 + P, smem, st, (const T *)x, lb, ub, P, ordered, pad, cfg, w, (T *)out,
           offs, next_epoch());
  return check_launch("omprt_generic_reduce");
}

template <class T>
int launch_generic_op(int op, const void *x, int64_t lb, int64_t ub, int teams, int P,
                      int ordered, int64_t pad, ArenaCfg cfg, Workspace w, void *out,
                      int64_t *offs, cudaStream_t st) {
  switch (op) {
    case OMPRT_OP_ADD:
      return launch_generic_t<T, OMPRT_OP_ADD>(x, lb, ub, teams, P, ordered, pad, cfg, w, out,
                                               offs, st);
    case OMPRT_OP_MAX:
      return launch_generic_t<T, OMPRT_OP_MAX>(x, lb, ub, teams, P, ordered, pad, cfg, w, out,
                                               offs, st);
    case OMPRT_OP_MIN:
      return launch_generic_t<T, OMPRT_OP_MIN>(x, lb, ub, teams, P, ordered, pad, cfg, w, out,
                                               offs, st);
  }
  return fail(OMPRT_EINVAL, "unknown reduction op %d", op);
}

// team partials + (ORDERED) one epoch-tagged ready flag per team
size_t generic_ws_core(int teams) { return ws_bytes(teams, 0, OMPRT_MODE_SPMD, 2); }

// Host-buffer (tgt_target-shaped) entries: device staging cached per CUDA
// device (a buffer belongs to the context it was allocated in, so a caller
// that switches devices gets that device's own staging, never another's).
// reduce_host pipelining: the input lands in pieces of kHostPipeBytes on a
// copy stream while the reduction of the previous piece runs on the compute
// stream (SPMD: the construct accumulates into the cell, so piecewise
// launches give the same integers and a re-associated fp sum).
constexpr size_t kHostPipeBytes = (size_t)256 << 20;
constexpr int kHostPipeEvents = 4;

struct HostStaging {
  void *buf[2] = {nullptr, nullptr};  // input / in-out arrays
  size_t bytes[2] = {0, 0};
  void *ws = nullptr;                 // zeroed construct workspace
  size_t ws_bytes = 0;
  void *cells = nullptr;              // 64 bytes: result cells + team offsets spill
  int64_t *offs = nullptr;            // generic mode: per-team arena offsets
  size_t offs_bytes = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;        // copy-in stream of the pipelined reduce_host
  cudaEvent_t landed[kHostPipeEvents] = {};
};
std::mutex g_host_mu;
std::unordered_map<int, HostStaging> g_host;

int staging_grow(void *&p, size_t &have, size_t want, bool zero) {
  if (want <= have) return OMPRT_OK;
  if (p) cudaFree(p);
  p = nullptr;
  have = 0;
  if (cudaMalloc(&p, want) != cudaSuccess) {
    cudaGetLastError();
    return fail(OMPRT_ENOMEM, "host entry: cannot allocate %zu device bytes", want);
  }
  if (zero && cudaMemset(p, 0, want) != cudaSuccess)
    return fail(OMPRT_ECUDA, "host entry: cannot zero the workspace");
  have = want;
  return OMPRT_OK;
}

// The calling thread's device's staging, with room for two arrays of
// (b0, b1) bytes and a workspace of ws bytes.  g_host_mu must be held.
int staging(HostStaging *&out, size_t b0, size_t b1, size_t ws) {
  int dev = 0;
  OMPRT_CUDA(cudaGetDevice(&dev));
  HostStaging &h = g_host[dev];
  if (!h.stream) OMPRT_CUDA(cudaStreamCreateWithFlags(&h.stream, cudaStreamNonBlocking));
  if (!h.copy) {
    OMPRT_CUDA(cudaStreamCreateWithFlags(&h.copy, cudaStreamNonBlocking));
    for (cudaEvent_t &e : h.landed)
      OMPRT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  int rc;
  if ((rc = staging_grow(h.buf[0], h.bytes[0], b0, false)) ||
      (rc = staging_grow(h.buf[1], h.bytes[1], b1, false)) ||
      (rc = staging_grow(h.ws, h.ws_bytes, ws, true)))
    return rc;
  if (!h.cells) OMPRT_CUDA(cudaMalloc(&h.cells, 64));
  out = &h;
  return OMPRT_OK;
}

}  // namespace

// ======================================================================= ABI

extern "C" {

const char *omprt_version(void) { return "omprt_b200 0.1.0 sm_100a"; }

const char *omprt_last_error(void) { return t_last_error.c_str(); }

int omprt_device_init(int device) {
  int prev = -1;
  OMPRT_CUDA(cudaGetDevice(&prev));
  OMPRT_CUDA(cudaSetDevice(device));
  TrapWord z = {0, 0, 0, 0};
  const cudaError_t e = cudaMemcpyToSymbol(g_trap, &z, sizeof(z));
  if (prev != device) cudaSetDevice(prev);  // the caller's current device is left alone
  if (e != cudaSuccess) return fail(OMPRT_ECUDA, "device_init: %s", cudaGetErrorString(e));
  return OMPRT_OK;
}

// ------------------------------------------------------- multi-GPU combine
//
// One in-place NCCL all-reduce of the per-GPU partials.  NCCL
// is resolved at first use with dlopen("libnccl.so.2") — the library the
// caller's communicator came from when it is already loaded (torch's, or the
// system one) — so libomprt_b200.so has no link-time NCCL dependency.
// Integer sums travel as unsigned (two's-complement wrap, the reference's
// modular adds); max/min keep the signed type (signed compare).
namespace {
using nccl_allreduce_fn = int (*)(const void *, void *, size_t, int, int, void *, cudaStream_t);
nccl_allreduce_fn g_nccl_allreduce = nullptr;
std::mutex g_nccl_mu;

int nccl_dtype(int dtype, int op) {
  const bool add = op == OMPRT_OP_ADD;
  switch (dtype) {
    case OMPRT_I32: return add ? 3 : 2;  // ncclUint32 : ncclInt32
    case OMPRT_U32: return 3;
    case OMPRT_I64: return add ? 5 : 4;  // ncclUint64 : ncclInt64
    case OMPRT_U64: return 5;
    case OMPRT_F32: return 7;
    case OMPRT_F64: return 8;
    default: return -1;
  }
}
}  // namespace

int omprt_allreduce(void *d_buf, int64_t count, int dtype, int op, void *nccl_comm,
                    void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  if (count < 0 || (count > 0 && !d_buf) || !nccl_comm)
    return fail(OMPRT_EINVAL, "allreduce: bad arguments");
  const int nt = nccl_dtype(dtype, op);
  if (nt < 0) return fail(OMPRT_EINVAL, "allreduce: unknown dtype %d", dtype);
  const int nop = op == OMPRT_OP_ADD ? 0 : (op == OMPRT_OP_MAX ? 2 : (op == OMPRT_OP_MIN ? 3 : -1));
  if (nop < 0) return fail(OMPRT_EINVAL, "allreduce: unknown op %d", op);
  {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (!g_nccl_allreduce) {
      void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
      if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
      if (!h) return fail(OMPRT_EUNAVAILABLE, "allreduce: libnccl.so.2 not found (%s)", dlerror());
      g_nccl_allreduce = reinterpret_cast<nccl_allreduce_fn>(dlsym(h, "ncclAllReduce"));
      if (!g_nccl_allreduce) return fail(OMPRT_EUNAVAILABLE, "allreduce: no ncclAllReduce");
    }
  }
  if (count == 0) return OMPRT_OK;
  const int r = g_nccl_allreduce(d_buf, d_buf, (size_t)count, nt, nop, nccl_comm, S(stream));
  if (r != 0) return fail(OMPRT_ECUDA, "ncclAllReduce failed (ncclResult %d)", r);
  return OMPRT_OK;
}

// ------------------------------------------- fused multi-GPU exchange (IPC)

size_t omprt_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int omprt_mailbox_create(int world, void **d_mailbox, void *ipc_handle) {
  if (world < 1 || !d_mailbox || !ipc_handle)
    return fail(OMPRT_EINVAL, "mailbox_create: bad arguments");
  const size_t bytes = (size_t)2 * world * 16;  // two banks x world slots {value, key}
  void *p = nullptr;
  OMPRT_CUDA(cudaMalloc(&p, bytes));
  OMPRT_CUDA(cudaMemset(p, 0, bytes));
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return fail(OMPRT_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  }
  std::memcpy(ipc_handle, &h, sizeof(h));
  *d_mailbox = p;
  return OMPRT_OK;
}

int omprt_mailbox_open(const void *ipc_handle, void **d_ptr) {
  if (!ipc_handle || !d_ptr) return fail(OMPRT_EINVAL, "mailbox_open: bad arguments");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, ipc_handle, sizeof(h));
  OMPRT_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return OMPRT_OK;
}

int omprt_mailbox_close(void *d_ptr) {
  if (!d_ptr) return fail(OMPRT_EINVAL, "mailbox_close: null");
  OMPRT_CUDA(cudaIpcCloseMemHandle(d_ptr));
  return OMPRT_OK;
}

int omprt_mailbox_destroy(void *d_mailbox) {
  if (!d_mailbox) return fail(OMPRT_EINVAL, "mailbox_destroy: null");
  OMPRT_CUDA(cudaFree(d_mailbox));
  return OMPRT_OK;
}

int omprt_reduce_exchange(const void *d_x, int64_t lb, int64_t ub, int dtype, int op, int sched,
                          int64_t chunk, int teams, int threads, void *d_ws, void *d_out,
                          const void *d_peers, int rank, int world, uint64_t key, uint64_t step,
                          void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  int rc;
  if ((rc = check_grid(teams, threads)) || (rc = check_sched(sched, chunk))) return rc;
  if (!d_ws || !d_out || !d_peers || (!d_x && ub >= lb) || world < 1 || rank < 0 ||
      rank >= world || key == 0)
    return fail(OMPRT_EINVAL, "reduce_exchange: bad arguments");
  if (threads < 64 || threads % 32 != 0)
    return fail(OMPRT_EINVAL, "reduce_exchange: threads must be a multiple of 32, >= 64");
  LoopArgs la{lb, ub, chunk, sched};
  Workspace w = ws_carve(d_ws, teams, kReduceSlots);
  Exchange xc;
  xc.peers = reinterpret_cast<uint64_t *const *>(const_cast<void *>(d_peers));
  xc.rank = rank;
  xc.world = world;
  xc.key = key;
  xc.bank = (uint32_t)(step & 1);
  xc.timeout_ns = 20ull * 1000 * 1000 * 1000;  // 20 s: a missing peer traps (Deadlock)
  return by_dtype<ExchangeF>(dtype, op, d_x, la, teams, threads, w, d_out, xc, S(stream));
}

int omprt_set_trace(void *d_records, int64_t capacity) {
  if (capacity < 0 || (capacity > 0 && !d_records))
    return fail(OMPRT_EINVAL, "set_trace: bad arguments");
  TraceRing r;
  r.recs = capacity > 0 ? reinterpret_cast<TraceRec *>(d_records) : nullptr;
  r.cap = (uint32_t)(capacity > 0xffffffffll ? 0xffffffffll : capacity);
  OMPRT_CUDA(cudaMemcpyToSymbol(g_trace, &r, sizeof(r)));
  g_trace_on = r.recs != nullptr;
  return OMPRT_OK;
}

int omprt_num_sms(void) {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(OMPRT_ECUDA, "no CUDA device");
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return fail(OMPRT_ECUDA, "cudaDeviceGetAttribute failed");
  return sms;
}

int omprt_check_trap(void *stream, int *kind, int *code, int *team, int *thread) {
  OMPRT_ON_STREAM_DEVICE(stream);
  OMPRT_CUDA(cudaStreamSynchronize(S(stream)));
  TrapWord t;
  OMPRT_CUDA(cudaMemcpyFromSymbol(&t, g_trap, sizeof(t)));
  if (kind) *kind = t.kind;
  if (code) *code = t.code;
  if (team) *team = t.team;
  if (thread) *thread = t.thread;
  if (t.kind == 0) return OMPRT_OK;
  TrapWord z = {0, 0, 0, 0};
  OMPRT_CUDA(cudaMemcpyToSymbol(g_trap, &z, sizeof(z)));
  return OMPRT_TRAP;
}

int omprt_set_unroll(int unroll) {
  if (unroll != 2 && unroll != 4 && unroll != 8)
    return fail(OMPRT_EINVAL, "unroll must be 2, 4 or 8 (got %d)", unroll);
  g_unroll = unroll;
  return OMPRT_OK;
}

int omprt_set_spmd_block(int threads) {
  if (threads != 0 && (threads < 64 || threads > 1024 || threads % 32 != 0))
    return fail(OMPRT_EINVAL, "SPMD block must be 0 or a multiple of 32 in 64..1024 (got %d)",
                threads);
  g_spmd_block = threads;
  return OMPRT_OK;
}

int omprt_set_variant(int variant) {
  if (variant < 0) return fail(OMPRT_EINVAL, "variant must be >= 0");
  g_variant = variant;
  return OMPRT_OK;
}

int omprt_static_bounds(int64_t lb, int64_t ub, int64_t tid, int64_t nthreads, int64_t *my_lb,
                        int64_t *my_ub) {
  if (nthreads == 0) {
    t_last_error = "DivideByZero: sdiv.i64 by zero";
    return OMPRT_TRAP;
  }
  int64_t a, b;
  static_bounds(lb, ub, tid, nthreads, a, b);
  if (my_lb) *my_lb = a;
  if (my_ub) *my_ub = b;
  return OMPRT_OK;
}

int omprt_bounds_dump(int64_t lb, int64_t ub, int sched, int64_t chunk, int teams, int threads,
                      int64_t *d_out, void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  int rc;
  if ((rc = check_grid(teams, threads)) || (rc = check_sched(sched, chunk))) return rc;
  if (!d_out) return fail(OMPRT_EINVAL, "bounds_dump: null output");
  LoopArgs la{lb, ub, chunk, sched};
  k_bounds_dump<<<teams, threads, 0, S(stream)>>>(la, d_out);
  return check_launch("omprt_bounds_dump");
}

size_t omprt_reduce_workspace_bytes(int teams, int threads, int mode) {
  return ws_bytes(teams < 1 ? 1 : teams, threads < 1 ? 1 : threads, mode, kReduceSlots);
}

int omprt_reduce(const void *d_x, int64_t lb, int64_t ub, int dtype, int op, int sched,
                 int64_t chunk, int teams, int threads, int mode, void *d_ws, void *d_out,
                 void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  int rc;
  if ((rc = check_grid(teams, threads)) || (rc = check_sched(sched, chunk))) return rc;
  if (!d_ws || !d_out || (!d_x && ub >= lb))
    return fail(OMPRT_EINVAL, "reduce: null device pointer");
  if (mode != OMPRT_MODE_SPMD && mode != OMPRT_MODE_ORDERED)
    return fail(OMPRT_EINVAL, "unknown mode %d", mode);
  LoopArgs la{lb, ub, chunk, sched};
  Workspace w = ws_carve(d_ws, teams, kReduceSlots);
  return by_dtype<ReduceF>(dtype, op, d_x, la, teams, threads, mode, w, d_out, S(stream));
}

namespace {
int launch_axpy_spmd(float a, const float *d_x, float *d_y, LoopArgs la, int teams, int threads,
                     Workspace w, float *d_max, float *d_min, cudaStream_t st) {
  int rc;
  spmd_prepare(la, teams);
  la.threads = threads;
  const int blk = spmd_block(threads, kAxpyBlock);
  if (g_unroll == 4 && (g_variant == 47 || g_variant == 48)) {
    // tuning: two-stream rings 2 x 2 x 48 KiB (47) / 3 x 2 x 32 KiB (48)
    auto kern = g_variant == 47 ? k_axpy_minmax_bulk<2, 49152, 4> : k_axpy_minmax_bulk<3, 32768, 4>;
    const size_t smem = g_variant == 47 ? (size_t)2 * 2 * 49152 : (size_t)2 * 3 * 32768;
    if ((rc = set_smem(kern, smem))) return rc;
    launch_k(kern, teams * la.split, blk, smem, st, a, d_x, d_y, la, w, d_max, d_min);
  } else if (g_unroll == 4) {
    auto kern = blk <= 256 ? k_axpy_minmax_bulk<kBulk2Stages, kBulk2StageBytes, 4, 256>
                           : k_axpy_minmax_bulk<kBulk2Stages, kBulk2StageBytes, 4>;
    const size_t smem = (size_t)2 * kBulk2Stages * kBulk2StageBytes;
    if ((rc = set_smem(kern, smem))) return rc;
    launch_k(kern, teams * la.split, blk, smem, st, a, d_x, d_y, la, w, d_max, d_min);
  } else {
    k_axpy_minmax<4><<<teams * la.split, blk, 0, st>>>(a, d_x, d_y, la, w, d_max, d_min);
  }
  return check_launch("omprt_axpy_minmax");
}
}  // namespace

int omprt_axpy_minmax(float a, const float *d_x, float *d_y, int64_t lb, int64_t ub, int sched,
                      int64_t chunk, int teams, int threads, int mode, void *d_ws, float *d_max,
                      float *d_min, void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  int rc;
  if ((rc = check_grid(teams, threads)) || (rc = check_sched(sched, chunk))) return rc;
  if (!d_ws || !d_max || !d_min || ((!d_x || !d_y) && ub >= lb))
    return fail(OMPRT_EINVAL, "axpy_minmax: null device pointer");
  LoopArgs la{lb, ub, chunk, sched};
  Workspace w = ws_carve(d_ws, teams, kReduceSlots);
  if (mode != OMPRT_MODE_ORDERED)
    return launch_axpy_spmd(a, d_x, d_y, la, teams, threads, w, d_max, d_min, S(stream));
  if (g_variant != kOrderedLiteral && g_variant != kOrderedRowsMinMax && ext_ok(la)) {
    // one pass: the SPMD axpy with the reference order's max/min kept as the
    // leftmost extremum (leftext.cuh) — bit-identical to the literal walk
    spmd_prepare(la, teams);
    la.threads = threads;
    const int blk = spmd_block(threads, kAxpyExtBlock);
    auto kern = blk <= kAxpyExtBlock ? k_axpy_minmax_ext<kBulk2Stages, kBulk2StageBytes, kAxpyExtBlock>
                                     : k_axpy_minmax_ext<kBulk2Stages, kBulk2StageBytes, kMaxThreads>;
    const size_t smem = (size_t)2 * kBulk2Stages * kBulk2StageBytes;
    if ((rc = set_smem(kern, smem))) return rc;
    launch_k(kern, teams * la.split, blk, smem, S(stream), a, d_x, d_y, la, w, d_max, d_min);
    return check_launch("omprt_axpy_minmax(ordered)");
  }
  if (g_variant == kOrderedLiteral || !ord_rows_ok(la, d_y)) {
    k_axpy_minmax_ordered<<<teams, threads, 0, S(stream)>>>(a, d_x, d_y, la, w, d_max, d_min);
    return check_launch("omprt_axpy_minmax(ordered)");
  }
  // ORDERED: y = a*x + y is elementwise, so the SPMD kernel writes the same
  // y (its own max/min go to a scratch pair in the workspace header and are
  // dropped); then max and min are folded over the new y in the reference
  // order — every OpenMP thread its chunks in order, partials in global
  // thread order, starting from the cells — by the ORDERED reductions,
  // exactly what the literal walk computes, at streaming speed.
  float *scratch = reinterpret_cast<float *>(static_cast<unsigned char *>(d_ws) + 128);
  if ((rc = launch_axpy_spmd(a, d_x, d_y, la, teams, threads, w, scratch, scratch + 1,
                             S(stream))))
    return rc;
  // one pass folding max and min together (float2 partials, two chains)
  const int nw = ord_default_nw(teams, threads);
  const int s512 = OrdSmem<float, 128, 1>::stages_for(nw);
  const int s256 = OrdSmem<float, 64, 1>::stages_for(nw);
  const int grid = ord_grid(teams, threads, nw);
  if (s512 >= 3) {
    const size_t ring = (size_t)nw * OrdSmem<float, 128, 1>::warp_bytes(s512);
    if ((rc = set_smem(k_minmax_ordered_rows<128>, ring + kFolderSmem))) return rc;
    k_minmax_ordered_rows<128><<<grid, (nw + 1) * 32, ring + kFolderSmem, S(stream)>>>(
        d_y, la, teams, threads, w, d_max, d_min, s512, next_epoch(), (uint32_t)ring,
        ord_segments(la, teams, threads, 128, 4));
  } else {
    const size_t ring = (size_t)nw * OrdSmem<float, 64, 1>::warp_bytes(s256);
    if ((rc = set_smem(k_minmax_ordered_rows<64>, ring + kFolderSmem))) return rc;
    k_minmax_ordered_rows<64><<<grid, (nw + 1) * 32, ring + kFolderSmem, S(stream)>>>(
        d_y, la, teams, threads, w, d_max, d_min, s256, next_epoch(), (uint32_t)ring,
        ord_segments(la, teams, threads, 64, 4));
  }
  return check_launch("omprt_axpy_minmax(ordered max/min)");
}

int omprt_dot(const double *d_x, const double *d_y, int64_t lb, int64_t ub, int sched,
              int64_t chunk, int teams, int threads, int mode, void *d_ws, double *d_out,
              void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  int rc;
  if ((rc = check_grid(teams, threads)) || (rc = check_sched(sched, chunk))) return rc;
  if (!d_ws || !d_out || ((!d_x || !d_y) && ub >= lb))
    return fail(OMPRT_EINVAL, "dot: null device pointer");
  LoopArgs la{lb, ub, chunk, sched};
  Workspace w = ws_carve(d_ws, teams, kReduceSlots);
  if (mode == OMPRT_MODE_ORDERED) {
    if (g_variant != kOrderedLiteral && ord_rows_ok(la, d_x, d_y)) {
      // six warps when they fill whole waves: two streams' 256-byte windows
      // then fit two stages (148 x 384: 3.9 -> 5.7 TB/s; static_chunked 64:
      // 2.1 -> 6.1, profiles/r1_ordered_six_dot.jsonl)
      const int nw = ord_six_warps(teams, threads, INT64_MAX, 24) ? 6 : ord_default_nw(teams, threads);
      const int s512 = OrdSmem<double, 64, 2>::stages_for(nw);
      const int s256 = OrdSmem<double, 32, 2>::stages_for(nw);
      const int s128 = OrdSmem<double, 16, 2>::stages_for(nw);
      const int grid = ord_grid(teams, threads, nw);
      const uint64_t ep = next_epoch();
      if (s512 >= 3) {
        const size_t ring = (size_t)nw * OrdSmem<double, 64, 2>::warp_bytes(s512);
        const size_t smem = ring + kFolderSmem;
        if ((rc = set_smem(k_dot_ordered_rows<64>, smem))) return rc;
        k_dot_ordered_rows<64><<<grid, (nw + 1) * 32, smem, S(stream)>>>(
            d_x, d_y, la, teams, threads, w, d_out, s512, ep, (uint32_t)ring,
            ord_segments(la, teams, threads, 64, 8));
      } else if (s256 >= 2) {
        const size_t ring = (size_t)nw * OrdSmem<double, 32, 2>::warp_bytes(s256);
        const size_t smem = ring + kFolderSmem;
        if ((rc = set_smem(k_dot_ordered_rows<32>, smem))) return rc;
        k_dot_ordered_rows<32><<<grid, (nw + 1) * 32, smem, S(stream)>>>(
            d_x, d_y, la, teams, threads, w, d_out, s256, ep, (uint32_t)ring,
            ord_segments(la, teams, threads, 32, 8));
      } else if (s128 >= 2) {
        const size_t ring = (size_t)nw * OrdSmem<double, 16, 2>::warp_bytes(s128);
        const size_t smem = ring + kFolderSmem;
        if ((rc = set_smem(k_dot_ordered_rows<16>, smem))) return rc;
        k_dot_ordered_rows<16><<<grid, (nw + 1) * 32, smem, S(stream)>>>(
            d_x, d_y, la, teams, threads, w, d_out, s128, ep, (uint32_t)ring,
            ord_segments(la, teams, threads, 16, 8));
      } else {
        k_dot_ordered<<<teams, threads, 0, S(stream)>>>(d_x, d_y, la, w, d_out);
      }
    } else {
      k_dot_ordered<<<teams, threads, 0, S(stream)>>>(d_x, d_y, la, w, d_out);
    }
  } else {
    spmd_prepare(la, teams);
    la.threads = threads;
    const int blk = spmd_block(threads, kDotBlock);
    if (g_unroll == 4 && g_variant == 48) {
      // tuning: 3 stages x 2 streams x 32 KiB
      auto kern = k_dot_bulk<3, 32768, 4>;
      const size_t smem = (size_t)2 * 3 * 32768;
      if ((rc = set_smem(kern, smem))) return rc;
      launch_k(kern, teams * la.split, blk, smem, S(stream), d_x, d_y, la, w, d_out);
    } else if (g_unroll == 4) {
      // 2 stages x 2 streams x 48 KiB (7.50 vs 7.42 TB/s for 4 x 2 x 16 KiB,
      // steady state, profiles/r2_ring2_steady.jsonl)
      auto kern = k_dot_bulk<kDotStages, kDotStageBytes, 4>;
      const size_t smem = (size_t)2 * kDotStages * kDotStageBytes;
      if ((rc = set_smem(kern, smem))) return rc;
      launch_k(kern, teams * la.split, blk, smem, S(stream), d_x, d_y, la, w, d_out);
    } else if (g_unroll >= 8) {
      k_dot<8><<<teams * la.split, blk, 0, S(stream)>>>(d_x, d_y, la, w, d_out);
    } else {
      k_dot<4><<<teams * la.split, blk, 0, S(stream)>>>(d_x, d_y, la, w, d_out);
    }
  }
  return check_launch("omprt_dot");
}

int omprt_combine_partials(const void *d_partials, int count, int dtype, int op, void *d_out,
                           void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  if (count < 0 || !d_out || (count > 0 && !d_partials))
    return fail(OMPRT_EINVAL, "combine_partials: bad arguments");
  return by_dtype<CombineF>(dtype, op, d_partials, count, d_out, S(stream));
}

size_t omprt_generic_workspace_bytes(int teams, int par_threads, int heap_fallback,
                                     int64_t heap_bytes_per_team) {
  (void)par_threads;
  size_t b = generic_ws_core(teams < 1 ? 1 : teams);
  if (heap_fallback) b += (size_t)(teams < 1 ? 1 : teams) * (size_t)heap_bytes_per_team;
  return (b + 255) & ~(size_t)255;
}

int omprt_generic_reduce(const void *d_x, int64_t lb, int64_t ub, int dtype, int op, int teams,
                         int par_threads, int ordered, int64_t pad_bytes, int heap_fallback,
                         int64_t heap_bytes_per_team, void *d_ws, void *d_out,
                         int64_t *d_team_offsets, void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  if (teams < 1) return fail(OMPRT_EINVAL, "teams must be >= 1");
  if (par_threads < 32 || par_threads % 32 != 0 || par_threads + 32 > kMaxThreads)
    return fail(OMPRT_EINVAL, "par_threads must be a multiple of 32 in 32..%d (got %d)",
                kMaxThreads - 32, par_threads);
  if (pad_bytes < 0 || (heap_fallback && heap_bytes_per_team < 0))
    return fail(OMPRT_EINVAL, "generic: negative sizes");
  if (!d_ws || !d_out || (!d_x && ub >= lb))
    return fail(OMPRT_EINVAL, "generic: null device pointer");
  Workspace w = ws_carve(d_ws, teams, 1);
  ArenaCfg cfg;
  cfg.capacity = OMPRT_ARENA_CAPACITY;
  cfg.heap_fallback = heap_fallback ? 1 : 0;
  cfg.heap_per_team = heap_fallback ? heap_bytes_per_team : 0;
  cfg.heap = heap_fallback ? (unsigned char *)d_ws + generic_ws_core(teams) : nullptr;
  switch (dtype) {
    case OMPRT_I64:
      return launch_generic_op<int64_t>(op, d_x, lb, ub, teams, par_threads, ordered, pad_bytes,
                                        cfg, w, d_out, d_team_offsets, S(stream));
    case OMPRT_U64:
      return launch_generic_op<uint64_t>(op, d_x, lb, ub, teams, par_threads, ordered,
                                         pad_bytes, cfg, w, d_out, d_team_offsets, S(stream));
    case OMPRT_F64:
      return launch_generic_op<double>(op, d_x, lb, ub, teams, par_threads, ordered, pad_bytes,
                                       cfg, w, d_out, d_team_offsets, S(stream));
  }
  return fail(OMPRT_EINVAL, "generic_reduce: dtype must be I64, U64 or F64 (got %d)", dtype);
}

int omprt_arena_replay(const int64_t *d_script, int nops, int teams, int threads,
                       int caller_tid, int64_t capacity, int heap_fallback,
                       int64_t heap_bytes_per_team, void *d_heap, int check_uninit,
                       int64_t *d_results, void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  int rc;
  if ((rc = check_grid(teams, threads))) return rc;
  if (nops < 0 || (nops > 0 && (!d_script || !d_results)))
    return fail(OMPRT_EINVAL, "arena_replay: bad script");
  if (capacity < 0 || capacity > OMPRT_ARENA_CAPACITY || capacity % 16 != 0)
    return fail(OMPRT_EINVAL, "arena capacity must be a multiple of 16 in 0..%d",
                OMPRT_ARENA_CAPACITY);
  if (caller_tid < 0 || caller_tid >= threads)
    return fail(OMPRT_EINVAL, "caller_tid must lie in 0..threads-1");
  if (heap_fallback && (!d_heap || heap_bytes_per_team < 0))
    return fail(OMPRT_EINVAL, "heap fallback needs a heap buffer");
  if (nops == 0) return OMPRT_OK;
  ArenaCfg cfg;
  cfg.capacity = capacity;
  cfg.heap_fallback = heap_fallback ? 1 : 0;
  cfg.heap_per_team = heap_fallback ? heap_bytes_per_team : 0;
  cfg.heap = (unsigned char *)d_heap;
  const size_t smem = (size_t)(capacity > 0 ? capacity : 16);
  if (smem > 48 * 1024)
    OMPRT_CUDA(cudaFuncSetAttribute(k_arena_replay, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
  k_arena_replay<<<teams, threads, smem, S(stream)>>>(d_script, nops, caller_tid, cfg,
                                                      check_uninit ? 1 : 0, d_results);
  if ((rc = check_launch("omprt_arena_replay"))) return rc;
  // report (but leave) the trap word: omprt_check_trap reads and clears it
  OMPRT_CUDA(cudaStreamSynchronize(S(stream)));
  TrapWord t;
  OMPRT_CUDA(cudaMemcpyFromSymbol(&t, g_trap, sizeof(t)));
  return t.kind ? OMPRT_TRAP : OMPRT_OK;
}

int omprt_atomic_probe(int kind, int dtype, const uint64_t *d_operands, const uint64_t *d_desired,
                       uint64_t *d_cell, uint64_t *d_old, int teams, int threads, void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  int rc;
  if ((rc = check_grid(teams, threads))) return rc;
  if ((rc = check_atomic(kind, dtype, d_desired))) return rc;
  if (!d_operands || !d_cell || !d_old) return fail(OMPRT_EINVAL, "atomic_probe: null pointer");
  switch (dtype) {
    case OMPRT_I32:
      return AtomicF<int32_t>::run(kind, d_operands, d_desired, d_cell, d_old, teams, threads,
                                   S(stream));
    case OMPRT_U32:
      return AtomicF<uint32_t>::run(kind, d_operands, d_desired, d_cell, d_old, teams, threads,
                                    S(stream));
    case OMPRT_I64:
      return AtomicF<int64_t>::run(kind, d_operands, d_desired, d_cell, d_old, teams, threads,
                                   S(stream));
    default:
      return AtomicF<uint64_t>::run(kind, d_operands, d_desired, d_cell, d_old, teams, threads,
                                    S(stream));
  }
}

int omprt_atomic_apply(int kind, int dtype, uint64_t *d_cells, const uint64_t *d_operands,
                       const uint64_t *d_desired, uint64_t *d_old, int64_t n, void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  int rc;
  if ((rc = check_atomic(kind, dtype, d_desired))) return rc;
  if (n < 0 || (n > 0 && (!d_cells || !d_operands || !d_old)))
    return fail(OMPRT_EINVAL, "atomic_apply: bad arguments");
  switch (dtype) {
    case OMPRT_I32:
      return AtomicF<int32_t>::apply(kind, d_cells, d_operands, d_desired, d_old, n, S(stream));
    case OMPRT_U32:
      return AtomicF<uint32_t>::apply(kind, d_cells, d_operands, d_desired, d_old, n, S(stream));
    case OMPRT_I64:
      return AtomicF<int64_t>::apply(kind, d_cells, d_operands, d_desired, d_old, n, S(stream));
    default:
      return AtomicF<uint64_t>::apply(kind, d_cells, d_operands, d_desired, d_old, n, S(stream));
  }
}

int omprt_atomic_program(const int32_t *d_kinds, const uint64_t *d_operands,
                         const uint64_t *d_desired, const int64_t *d_offsets, int64_t nops,
                         int dtype, uint64_t *d_cell, uint64_t *d_old, int teams, int threads,
                         void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  int rc;
  if ((rc = check_grid(teams, threads))) return rc;
  if (dtype != OMPRT_I32 && dtype != OMPRT_U32 && dtype != OMPRT_I64 && dtype != OMPRT_U64)
    return fail(OMPRT_EINVAL, "atomics take i32/u32/i64/u64 (got dtype %d)", dtype);
  if (!d_offsets || !d_cell || (nops > 0 && (!d_kinds || !d_operands || !d_old)))
    return fail(OMPRT_EINVAL, "atomic_program: null pointer");
  // kinds are validated on the host side of the ABI by the caller's table;
  // INC on 64-bit cells and CAS without desired values are rejected here
  switch (dtype) {
    case OMPRT_I32:
      return AtomicF<int32_t>::program(d_kinds, d_operands, d_desired, d_offsets, d_cell, d_old,
                                       teams, threads, S(stream));
    case OMPRT_U32:
      return AtomicF<uint32_t>::program(d_kinds, d_operands, d_desired, d_offsets, d_cell, d_old,
                                        teams, threads, S(stream));
    case OMPRT_I64:
      return AtomicF<int64_t>::program(d_kinds, d_operands, d_desired, d_offsets, d_cell, d_old,
                                       teams, threads, S(stream));
    default:
      return AtomicF<uint64_t>::program(d_kinds, d_operands, d_desired, d_offsets, d_cell, d_old,
                                        teams, threads, S(stream));
  }
}

int omprt_fill(void *d_x, int64_t n, int dtype, uint64_t seed, int k, int64_t offset,
               void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  if (n < 0 || (n > 0 && !d_x)) return fail(OMPRT_EINVAL, "fill: bad arguments");
  return by_dtype<FillF>(dtype, d_x, n, seed, k, offset, S(stream));
}

int omprt_reduce_host(const void *h_x, int64_t n, int dtype, int op, int sched, int64_t chunk,
                      int teams, int threads, int mode, void *h_out) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  const size_t es = dtype_size(dtype);
  if (!es) return fail(OMPRT_EINVAL, "unknown dtype %d", dtype);
  if (n < 0 || !h_out || (n > 0 && !h_x)) return fail(OMPRT_EINVAL, "reduce_host: bad arguments");
  int rc;
  if ((rc = check_grid(teams, threads)) || (rc = check_sched(sched, chunk))) return rc;
  const size_t xbytes = (size_t)n * es;
  HostStaging *h = nullptr;
  if ((rc = staging(h, xbytes, 0, omprt_reduce_workspace_bytes(teams, threads, mode)))) return rc;
  cudaStream_t st = h->stream;
  // copy-in (tgt_target host.py:276-281)
  OMPRT_CUDA(cudaMemcpyAsync(h->cells, h_out, es, cudaMemcpyHostToDevice, st));
  const bool pipe = xbytes > 2 * kHostPipeBytes &&
                    (mode == OMPRT_MODE_SPMD || dtype == OMPRT_I32 || dtype == OMPRT_U32 ||
                     dtype == OMPRT_I64 || dtype == OMPRT_U64);
  if (!pipe) {
    if (xbytes) OMPRT_CUDA(cudaMemcpyAsync(h->buf[0], h_x, xbytes, cudaMemcpyHostToDevice, st));
    rc = omprt_reduce(h->buf[0], 0, n - 1, dtype, op, sched, chunk, teams, threads, mode, h->ws,
                      h->cells, st);
    if (rc) return rc;
  } else {
    // piece k lands on the copy stream while piece k-1 is reduced on st;
    // every piece's construct launch accumulates into the cell
    const int64_t per = (int64_t)(kHostPipeBytes / es);
    OMPRT_CUDA(cudaEventRecord(h->landed[0], st));  // the copy stream starts after the cell
    OMPRT_CUDA(cudaStreamWaitEvent(h->copy, h->landed[0], 0));
    int k = 0;
    for (int64_t lo = 0; lo < n; lo += per, ++k) {
      const int64_t cnt = n - lo < per ? n - lo : per;
      unsigned char *dst = static_cast<unsigned char *>(h->buf[0]) + (size_t)lo * es;
      OMPRT_CUDA(cudaMemcpyAsync(dst, static_cast<const unsigned char *>(h_x) + (size_t)lo * es,
                                 (size_t)cnt * es, cudaMemcpyHostToDevice, h->copy));
      cudaEvent_t ev = h->landed[k % kHostPipeEvents];
      OMPRT_CUDA(cudaEventRecord(ev, h->copy));
      OMPRT_CUDA(cudaStreamWaitEvent(st, ev, 0));
      rc = omprt_reduce(dst, 0, cnt - 1, dtype, op, sched, chunk, teams, threads, mode, h->ws,
                        h->cells, st);
      if (rc) return rc;
    }
  }
  // copy-out only on status 0 (host.py:293-295)
  unsigned char res[16];
  OMPRT_CUDA(cudaMemcpyAsync(res, h->cells, es, cudaMemcpyDeviceToHost, st));
  OMPRT_CUDA(cudaStreamSynchronize(st));
  std::memcpy(h_out, res, es);
  return OMPRT_OK;
}

int omprt_axpy_minmax_host(float a, const float *h_x, float *h_y, int64_t n, int sched,
                           int64_t chunk, int teams, int threads, int mode, float *h_max,
                           float *h_min) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  if (n < 0 || !h_max || !h_min || (n > 0 && (!h_x || !h_y)))
    return fail(OMPRT_EINVAL, "axpy_minmax_host: bad arguments");
  int rc;
  if ((rc = check_grid(teams, threads)) || (rc = check_sched(sched, chunk))) return rc;
  const size_t bytes = (size_t)n * sizeof(float);
  HostStaging *h = nullptr;
  if ((rc = staging(h, bytes, bytes, omprt_reduce_workspace_bytes(teams, threads, mode))))
    return rc;
  cudaStream_t st = h->stream;
  float *cells = static_cast<float *>(h->cells);
  const float init[2] = {*h_max, *h_min};
  if (bytes) {
    OMPRT_CUDA(cudaMemcpyAsync(h->buf[0], h_x, bytes, cudaMemcpyHostToDevice, st));
    OMPRT_CUDA(cudaMemcpyAsync(h->buf[1], h_y, bytes, cudaMemcpyHostToDevice, st));
  }
  OMPRT_CUDA(cudaMemcpyAsync(cells, init, sizeof init, cudaMemcpyHostToDevice, st));
  rc = omprt_axpy_minmax(a, static_cast<const float *>(h->buf[0]), static_cast<float *>(h->buf[1]),
                         0, n - 1, sched, chunk, teams, threads, mode, h->ws, cells, cells + 1, st);
  if (rc) return rc;
  // y is tofrom: back to the caller with the two cells, only on status 0
  float res[2];
  if (bytes) OMPRT_CUDA(cudaMemcpyAsync(h_y, h->buf[1], bytes, cudaMemcpyDeviceToHost, st));
  OMPRT_CUDA(cudaMemcpyAsync(res, cells, sizeof res, cudaMemcpyDeviceToHost, st));
  OMPRT_CUDA(cudaStreamSynchronize(st));
  *h_max = res[0];
  *h_min = res[1];
  return OMPRT_OK;
}

int omprt_dot_host(const double *h_x, const double *h_y, int64_t n, int sched, int64_t chunk,
                   int teams, int threads, int mode, double *h_out) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  if (n < 0 || !h_out || (n > 0 && (!h_x || !h_y)))
    return fail(OMPRT_EINVAL, "dot_host: bad arguments");
  int rc;
  if ((rc = check_grid(teams, threads)) || (rc = check_sched(sched, chunk))) return rc;
  const size_t bytes = (size_t)n * sizeof(double);
  HostStaging *h = nullptr;
  if ((rc = staging(h, bytes, bytes, omprt_reduce_workspace_bytes(teams, threads, mode))))
    return rc;
  cudaStream_t st = h->stream;
  double *cell = static_cast<double *>(h->cells);
  if (bytes) {
    OMPRT_CUDA(cudaMemcpyAsync(h->buf[0], h_x, bytes, cudaMemcpyHostToDevice, st));
    OMPRT_CUDA(cudaMemcpyAsync(h->buf[1], h_y, bytes, cudaMemcpyHostToDevice, st));
  }
  OMPRT_CUDA(cudaMemcpyAsync(cell, h_out, sizeof(double), cudaMemcpyHostToDevice, st));
  rc = omprt_dot(static_cast<const double *>(h->buf[0]), static_cast<const double *>(h->buf[1]),
                 0, n - 1, sched, chunk, teams, threads, mode, h->ws, cell, st);
  if (rc) return rc;
  double res;
  OMPRT_CUDA(cudaMemcpyAsync(&res, cell, sizeof res, cudaMemcpyDeviceToHost, st));
  OMPRT_CUDA(cudaStreamSynchronize(st));
  *h_out = res;
  return OMPRT_OK;
}

int omprt_generic_reduce_host(const void *h_x, int64_t n, int dtype, int op, int teams,
                              int par_threads, int ordered, int64_t pad_bytes, int heap_fallback,
                              int64_t heap_bytes_per_team, void *h_out,
                              int64_t *h_team_offsets) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  const size_t es = dtype_size(dtype);
  if (!es) return fail(OMPRT_EINVAL, "unknown dtype %d", dtype);
  if (n < 0 || !h_out || (n > 0 && !h_x) || teams < 1)
    return fail(OMPRT_EINVAL, "generic_reduce_host: bad arguments");
  int rc;
  const size_t xbytes = (size_t)n * es;
  HostStaging *h = nullptr;
  if ((rc = staging(h, xbytes, 0,
                    omprt_generic_workspace_bytes(teams, par_threads, heap_fallback,
                                                  heap_bytes_per_team))))
    return rc;
  if (h_team_offsets &&
      (rc = staging_grow(reinterpret_cast<void *&>(h->offs), h->offs_bytes,
                         (size_t)teams * sizeof(int64_t), false)))
    return rc;
  cudaStream_t st = h->stream;
  if (xbytes) OMPRT_CUDA(cudaMemcpyAsync(h->buf[0], h_x, xbytes, cudaMemcpyHostToDevice, st));
  OMPRT_CUDA(cudaMemcpyAsync(h->cells, h_out, es, cudaMemcpyHostToDevice, st));
  rc = omprt_generic_reduce(h->buf[0], 0, n - 1, dtype, op, teams, par_threads, ordered,
                            pad_bytes, heap_fallback, heap_bytes_per_team, h->ws, h->cells,
                            h_team_offsets ? h->offs : nullptr, st);
  if (rc) return rc;
  // a device trap (arena overflow, non-LIFO free, ...) is status 2 with the
  // caller's buffers untouched (host.py:289-295); the trap word stays set
  // for omprt_check_trap
  OMPRT_CUDA(cudaStreamSynchronize(st));
  TrapWord t;
  OMPRT_CUDA(cudaMemcpyFromSymbol(&t, g_trap, sizeof(t)));
  if (t.kind) return fail(OMPRT_TRAP, "generic_reduce_host: device trap kind %d code %d", t.kind,
                          t.code);
  unsigned char res[16];
  OMPRT_CUDA(cudaMemcpy(res, h->cells, es, cudaMemcpyDeviceToHost));
  if (h_team_offsets)
    OMPRT_CUDA(cudaMemcpy(h_team_offsets, h->offs, (size_t)teams * sizeof(int64_t),
                          cudaMemcpyDeviceToHost));
  std::memcpy(h_out, res, es);
  return OMPRT_OK;
}

int omprt_release_host_cache(void) {
  std::lock_guard<std::mutex> lk(g_host_mu);
  int prev = -1;
  cudaGetDevice(&prev);
  for (auto &kv : g_host) {
    HostStaging &h = kv.second;
    cudaSetDevice(kv.first);
    for (void *p : {h.buf[0], h.buf[1], h.ws, h.cells, static_cast<void *>(h.offs)})
      if (p) cudaFree(p);
    if (h.stream) cudaStreamDestroy(h.stream);
    if (h.copy) cudaStreamDestroy(h.copy);
    for (cudaEvent_t e : h.landed)
      if (e) cudaEventDestroy(e);
  }
  g_host.clear();
  if (prev >= 0) cudaSetDevice(prev);
  return OMPRT_OK;
}

// ------------------------------------------------------- compiled regions

int omprt_image_load(const void *image, size_t bytes, void **handle) {
  if (!image || !bytes || !handle) return fail(OMPRT_EINVAL, "image_load: bad arguments");
  cudaLibrary_t lib = nullptr;
  OMPRT_CUDA(cudaLibraryLoadData(&lib, image, nullptr, nullptr, 0, nullptr, nullptr, 0));
  *handle = reinterpret_cast<void *>(lib);
  return OMPRT_OK;
}

int omprt_image_unload(void *handle) {
  if (!handle) return fail(OMPRT_EINVAL, "image_unload: null handle");
  OMPRT_CUDA(cudaLibraryUnload(reinterpret_cast<cudaLibrary_t>(handle)));
  return OMPRT_OK;
}

int omprt_image_launch(void *handle, const char *kernel, int teams, int threads,
                       size_t shared_bytes, const void *argv, size_t argv_bytes, void *stream) {
  OMPRT_ON_STREAM_DEVICE(stream);
  if (!handle || !kernel || !argv || !argv_bytes)
    return fail(OMPRT_EINVAL, "image_launch: bad arguments");
  // GridConfig limits (vgpu.py:50-61)
  if (teams < 1 || teams > 1024 || threads < 1 || threads > 1024)
    return fail(OMPRT_EINVAL, "image_launch: grid %dx%d outside 1..1024", teams, threads);
  cudaKernel_t k = nullptr;
  cudaError_t e = cudaLibraryGetKernel(&k, reinterpret_cast<cudaLibrary_t>(handle), kernel);
  if (e != cudaSuccess)
    return fail(OMPRT_EINVAL, "image_launch: no kernel '%s' in the image (%s)", kernel,
                cudaGetErrorString(e));
  if (shared_bytes > 48 * 1024) {
    int dev = 0;
    OMPRT_CUDA(cudaGetDevice(&dev));
    OMPRT_CUDA(cudaKernelSetAttributeForDevice(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)shared_bytes, dev));
  }
  void *params[1] = {const_cast<void *>(argv)};
  OMPRT_CUDA(cudaLaunchKernel(reinterpret_cast<const void *>(k), dim3(teams), dim3(threads),
                              params, shared_bytes, S(stream)));
  return OMPRT_OK;
}

}  // extern "C"
