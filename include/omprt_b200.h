/*
 * omprt_b200.h — C ABI of the B200-native OpenMP device-runtime data-parallel core.
 *
 * This is the drop-in boundary between the reference's Python entry points
 * (forge: pkg/src/forge/devicert.py, pkg/src/forge/host.py) and hand-written
 * sm_100a kernels in libomprt_b200.so.  Plain C types only: pointers, sizes,
 * enums.  Device pointers are raw CUDA device addresses (e.g. a torch
 * tensor's data_ptr()); `stream` is a cudaStream_t passed as void* (NULL =
 * legacy default stream).  Every launch is stream-ordered and asynchronous
 * unless the function says it synchronises.
 *
 * Status convention (mirrors tgt_target, /root/reference/pkg/src/forge/host.py:255-296):
 *   0  OMPRT_OK        ran on the device
 *   1  OMPRT_FALLBACK  could not launch (the reference then runs its host fallback;
 *                      this library never does — callers treat it as an error)
 *   2  OMPRT_TRAP      device trap; omprt_last_trap() says which (vgpu.py:28-43)
 *  <0  argument / CUDA errors; omprt_last_error() has the message
 */
#ifndef OMPRT_B200_H
#define OMPRT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- element types: forge ScalarType (ast.py:18-34) plus the fp types the
 *      north star adds (the reference itself has no float type, parser.py:23-24) */
enum omprt_dtype {
  OMPRT_I32 = 0,
  OMPRT_U32 = 1,
  OMPRT_I64 = 2,
  OMPRT_U64 = 3,
  OMPRT_F32 = 4,
  OMPRT_F64 = 5
};

/* ---- reduction operators: the combine of __atomic_add/max/min
 *      (intrinsics.py:40-42; vgpu.py:586-625; host.py:810-837).
 *      Integer add wraps mod 2^bits; max/min compare signed for i32/i64. */
enum omprt_op { OMPRT_OP_ADD = 0, OMPRT_OP_MAX = 1, OMPRT_OP_MIN = 2 };

/* ---- worksharing schedules.
 *  STATIC                 for_static_init block partition over the flattened id
 *                         g = team*threads + tid, n = teams*threads
 *                         (runtime.mc:193-203; devicert.static_bounds devicert.py:110-115)
 *  STATIC_CHUNKED         schedule(static, chunk) over g: chunk k -> thread k mod n
 *                         (__kmpc_for_static_init kmp_sch_static_chunked; extension)
 *  DISTRIBUTE             __kmpc_distribute_static_init block over teams, then the
 *                         block rule again over the team's threads (nested)
 *  DISTRIBUTE_CHUNKED     distribute block over teams, schedule(static, chunk) inside */
enum omprt_sched {
  OMPRT_SCHED_STATIC = 0,
  OMPRT_SCHED_STATIC_CHUNKED = 1,
  OMPRT_SCHED_DISTRIBUTE = 2,
  OMPRT_SCHED_DISTRIBUTE_CHUNKED = 3
};

/* ---- execution modes for the reductions.
 *  SPMD     every thread runs the loop; the lanes of a team cover the team's
 *           iterations with coalesced 16-byte vector loads, and for the flat
 *           chunked schedule the CTAs take balanced contiguous pieces of
 *           [lb, ub] (a legal re-association: every iteration runs exactly
 *           once; integer results stay bit-exact).  Floating-point sums are
 *           within the stated tolerance (1e-6 fp64, 1e-4 fp32); fp max/min
 *           return the exact extreme value, but when +0.0 and -0.0 tie for it
 *           the sign of the returned zero is unspecified (step_max keeps the
 *           first of tied values, and which zero comes first depends on the
 *           order).  Use ORDERED for the reference order's zero sign.
 *  ORDERED  every device thread runs exactly its own schedule chunks in
 *           iteration order and the per-thread partials are combined in
 *           global thread order — the host fallback's order (host.py:567-582),
 *           so fp results are bit-identical to the CPU reference order.
 *           Integer reductions give the same bits in either order (add wraps
 *           mod 2^n, max/min are exact), so ORDERED integer launches run the
 *           SPMD kernels. */
enum omprt_mode { OMPRT_MODE_SPMD = 0, OMPRT_MODE_ORDERED = 1 };

/* ---- status and trap kinds (TrapKind / TRAP_CODES, vgpu.py:28-43) */
enum omprt_status {
  OMPRT_OK = 0,
  OMPRT_FALLBACK = 1,
  OMPRT_TRAP = 2,
  OMPRT_EINVAL = -1,
  OMPRT_ECUDA = -2,
  OMPRT_ENOMEM = -3,
  OMPRT_EUNAVAILABLE = -4  /* a runtime dependency (NCCL) is not installed */
};

enum omprt_trap_kind {
  OMPRT_TRAP_NONE = 0,
  OMPRT_TRAP_SHARED_OVERFLOW = 1,   /* __trap(1), runtime.mc:76-79 */
  OMPRT_TRAP_NON_LIFO_FREE = 2,     /* __trap(2), runtime.mc:89 */
  OMPRT_TRAP_NON_UNIFORM_ALLOC = 3, /* __trap(3), runtime.mc:76, 87 */
  OMPRT_TRAP_UNINITIALIZED_READ = 4,
  OMPRT_TRAP_OUT_OF_BOUNDS = 5,
  OMPRT_TRAP_DEADLOCK = 6,
  OMPRT_TRAP_DIVIDE_BY_ZERO = 7,    /* for_static_init with nthreads == 0 (sdiv) */
  OMPRT_TRAP_ABORT = 8
};

/* ---- atomic kinds for the device atomic probe (IntrinsicKind, intrinsics.py:14-28) */
enum omprt_atomic_kind {
  OMPRT_ATOMIC_ADD = 0,
  OMPRT_ATOMIC_MAX = 1,
  OMPRT_ATOMIC_MIN = 2,
  OMPRT_ATOMIC_XCHG = 3,
  OMPRT_ATOMIC_CAS = 4,
  OMPRT_ATOMIC_INC = 5
};

/* ---- arena script opcodes for omprt_arena_replay */
enum omprt_arena_op {
  OMPRT_ARENA_ALLOC = 0,
  OMPRT_ARENA_FREE = 1,
  OMPRT_ARENA_WRITE = 2,
  OMPRT_ARENA_READ = 3
};

#define OMPRT_ARENA_CAPACITY 65536 /* devicert.ARENA_CAPACITY, devicert.py:54 */
#define OMPRT_ARENA_ALIGN 8        /* devicert.ARENA_ALIGN,    devicert.py:55 */

/* ========================================================================= */
/* Library state                                                              */
/* ========================================================================= */

/* Version string of the built library. */
const char *omprt_version(void);

/* Message of the last failing call on this host thread ("" if none). */
const char *omprt_last_error(void);

/* Clear the trap word of CUDA device `device`.  The calling thread's current
 * device is left unchanged: every stream-taking entry point below runs on
 * its stream's device (cudaStreamGetDevice), restoring the caller's current
 * device on return; with a NULL (legacy default) stream it runs on the
 * current device. */
int omprt_device_init(int device);

/* Tuning knobs are per host thread (a tuning call never changes the kernel
 * another thread's launch selects). */

/* Tuning knob (not part of the reference interface): 16-byte vectors each
 * lane keeps in flight per loop iteration in the LDG-fed SPMD loops (2, 4 or
 * 8).  4 (the default) lets contiguous-schedule reductions use the TMA
 * bulk-copy path; 2 or 8 force the LDG path. */
int omprt_set_unroll(int unroll);

/* Tuning knob (not part of the reference interface): CUDA threads per CTA of
 * the SPMD construct kernels (reduce, axpy_minmax, dot, reduce_exchange) for
 * this calling thread — 0 (default) = each construct's measured policy; else a
 * multiple of 32 in 64..1024.  The OpenMP geometry (teams x threads) still
 * defines every team's iteration set; in SPMD mode which lane of the CTA
 * folds an iteration is unobservable, so the CTA size is a pure performance
 * choice. */
int omprt_set_spmd_block(int threads);

/* Tuning knob (not part of the reference interface): kernel variant used by
 * the fp64 sum in SPMD mode — 0 default; 1-5 LDG load-policy / unroll
 * variants; 10-16 TMA bulk-copy (cp.async.bulk + mbarrier) stage rings;
 * 20 = ORDERED mode through the literal per-thread walk instead of the
 * row-group kernels (cp.async shared-memory row windows + folder warp);
 * 21-29, 41 = row-group kernels with a forced window size x warps per SM;
 * 44 = ORDERED without the six-warp window policy;
 * 30 = SPMD without splitting few teams over several CTAs; 31 = ORDERED
 * row-group kernels with the static group assignment (no dynamic segments). */
int omprt_set_variant(int variant);

/* One in-place all-reduce of `count` elements of d_buf over an NCCL
 * communicator (`nccl_comm` = an ncclComm_t): the combine of the per-GPU
 * partials of a sharded construct (the GPU level of the
 * static_bounds partition).  Integer sums are reduced as unsigned (wrap
 * mod 2^n like the reference's adds), max/min as signed.  NCCL is loaded at
 * first use (dlopen libnccl.so.2: the instance the communicator came from
 * when it is already loaded); OMPRT_EUNAVAILABLE without it.  Stream-ordered.
 * Python callers use torch.distributed (paper_2106_03219_b200.parallel). */
int omprt_allreduce(void *d_buf, int64_t count, int dtype, int op, void *nccl_comm,
                    void *stream);

/* Fused multi-GPU combine (the all-reduce inside the reduction kernel):
 * each rank creates a mailbox (two banks x world slots of 16 bytes, zeroed)
 * and exports it as a CUDA IPC handle (omprt_ipc_handle_bytes() bytes); the
 * ranks exchange handles out of band and open each other's mailboxes; a
 * device array of the world's mailbox pointers (rank order, own included)
 * is passed to omprt_reduce_exchange.  Its last team stores this GPU's
 * partial into every rank's slot over NVLink peer memory and folds the
 * world's partials in rank order into d_out — one kernel, identical bits on
 * every rank.  `key` (nonzero, the same on all ranks) must differ at every
 * call; `step` selects the bank (calls on one mailbox alternate).  A peer
 * that does not arrive within 20 s raises OMPRT_TRAP_DEADLOCK. */
size_t omprt_ipc_handle_bytes(void);
int omprt_mailbox_create(int world, void **d_mailbox, void *ipc_handle);
int omprt_mailbox_open(const void *ipc_handle, void **d_ptr);
int omprt_mailbox_close(void *d_ptr);
int omprt_mailbox_destroy(void *d_mailbox);
int omprt_reduce_exchange(const void *d_x, int64_t lb, int64_t ub, int dtype, int op, int sched,
                          int64_t chunk, int teams, int threads, void *d_ws, void *d_out,
                          const void *d_peers, int rank, int world, uint64_t key, uint64_t step,
                          void *stream);

/* Per-team trace ring — the B200 analog of the vgpu's collect_trace
 * (vgpu.py:351-353, tgt_target(collect_trace=True) host.py:255-296).  While a
 * device buffer of `capacity` 32-byte records is installed, every construct
 * kernel's CTA writes one record {u64 t_begin_ns, u64 t_end_ns, u32 cta,
 * u32 smid, u32 ticket, u32 kind} at index blockIdx.x: kind 1 = team (ticket
 * = the value its atom.inc returned), 2 = the last team's ordered combine
 * (index gridDim.x), 3 = an ORDERED streaming warp (index = warp id, ticket
 * = groups folded), 4 = the ORDERED folder.  Times are %globaltimer ns.
 * Pass NULL/0 to uninstall (then kernels write nothing).  Synchronous. */
int omprt_set_trace(void *d_records, int64_t capacity);

/* Number of streaming multiprocessors of the current device (148 on B200). */
int omprt_num_sms(void);

/* Last device trap: replaces ExecResult.trap / out["trap"] (host.py:289-292).
 * Synchronises `stream`, copies the device trap word, clears it.  Returns
 * OMPRT_OK if no trap was raised, else OMPRT_TRAP with *kind (omprt_trap_kind),
 * *code (the __trap code), *team and *thread of the first trapping thread. */
int omprt_check_trap(void *stream, int *kind, int *code, int *team, int *thread);

/* ========================================================================= */
/* Worksharing (for_static_init / __kmpc_for_static_init /                    */
/*              __kmpc_distribute_static_init)                                */
/* ========================================================================= */

/* Host execution of the device's __host__ __device__ block-partition routine.
 * Replaces devicert.static_bounds (devicert.py:110-115): chunk = ceil((ub-lb+1)/n)
 * with floor division, my_lb = lb + tid*chunk, my_ub = min(my_lb+chunk-1, ub).
 * nthreads == 0 -> OMPRT_TRAP (DivideByZero), as vgpu's sdiv (vgpu.py:528-565). */
int omprt_static_bounds(int64_t lb, int64_t ub, int64_t tid, int64_t nthreads,
                        int64_t *my_lb, int64_t *my_ub);

/* Every device thread of a (teams x threads) launch runs the schedule's init
 * routine and writes its result, 4 x int64 per thread, flat id g = team*threads+tid:
 *   d_out[4g+0] = lower   first iteration of the thread's first chunk
 *   d_out[4g+1] = upper   last iteration of that chunk (lower > ub: no iterations)
 *   d_out[4g+2] = stride  distance between the thread's consecutive chunks
 *   d_out[4g+3] = last    1 if the thread owns iteration ub (lastprivate), else 0
 * For STATIC (chunk ignored) lower/upper are exactly for_static_init's
 * bounds[0..1] (runtime.mc:193-203).  chunk must be >= 1 for the chunked kinds. */
int omprt_bounds_dump(int64_t lb, int64_t ub, int sched, int64_t chunk, int teams,
                      int threads, int64_t *d_out, void *stream);

/* ========================================================================= */
/* teams distribute parallel for reduction                                    */
/* ========================================================================= */

/* Bytes of device workspace the reductions need (team partials — for
 * ORDERED max/min a (value, order key) pair per team for max and for min —,
 * per-thread partials for ORDERED, the last-team-finishes ticket, ORDERED's
 * per-group ready flags).  The workspace must be zeroed once before first use; the
 * ticket self-resets (atomic inc wraps, devicert.step_inc
 * devicert.py:105-107) and the ready flags carry a fresh 64-bit key per
 * launch, so it can be reused across launches (of any kernel) on one
 * stream. */
size_t omprt_reduce_workspace_bytes(int teams, int threads, int mode);

/* out = out OP reduce_{i in [lb,ub]} x[i], x indexed by the iteration number
 * (x points at element 0).  The PARTIAL_SUMS idiom (corpus.py:219-247) as the
 * combined construct: schedule -> per-thread/lane accumulate -> warp
 * __shfl_xor_sync tree -> smem tree (__kmpc_nvptx_parallel_reduce_nowait_v2)
 * -> team partial buffer + atomic-inc last-team-finishes combine in team order
 * (__kmpc_nvptx_teams_reduce_nowait_v2).  d_out holds the initial value on
 * entry (the original list item).  Deterministic for every dtype. */
int omprt_reduce(const void *d_x, int64_t lb, int64_t ub, int dtype, int op, int sched,
                 int64_t chunk, int teams, int threads, int mode, void *d_ws,
                 void *d_out, void *stream);

/* Fused chunked-schedule axpy + fp32 max/min (config 3):
 *   y[i] = fmaf(a, x[i], y[i]);  max = max(max, y[i]);  min = min(min, y[i])
 * d_max / d_min hold the initial values on entry. */
int omprt_axpy_minmax(float a, const float *d_x, float *d_y, int64_t lb, int64_t ub,
                      int sched, int64_t chunk, int teams, int threads, int mode,
                      void *d_ws, float *d_max, float *d_min, void *stream);

/* fp64 dot product: out = out + sum fma(x[i], y[i], part) (config 5, per shard). */
int omprt_dot(const double *d_x, const double *d_y, int64_t lb, int64_t ub, int sched,
              int64_t chunk, int teams, int threads, int mode, void *d_ws,
              double *d_out, void *stream);

/* Combine `count` partials (one per rank / shard, in rank order) into d_out:
 * d_out = d_out OP p[0] OP p[1] ...  — the deterministic tail of the
 * multi-GPU reduction after an all-gather of per-GPU partials. */
int omprt_combine_partials(const void *d_partials, int count, int dtype, int op,
                           void *d_out, void *stream);

/* ========================================================================= */
/* Generic mode: __kmpc_alloc_shared globalisation + nested parallel reduce    */
/* ========================================================================= */

/* Bytes of device workspace for omprt_generic_reduce. */
size_t omprt_generic_workspace_bytes(int teams, int par_threads, int heap_fallback,
                                     int64_t heap_bytes_per_team);

/* Generic-mode target region (config 4).  Each team has one main warp (its
 * lane 0 is the OpenMP initial thread, omp thread 0) and par_threads/32
 * worker warps waiting in a state machine on named barriers.  Per team the
 * main thread: takes its distribute block of [lb,ub] (static_bounds over
 * teams); if pad_bytes > 0 first allocates pad_bytes from the arena; then
 * globalises `parts` with __kmpc_alloc_shared((par_threads+1)*8); forks the
 * parallel region (workers reduce their for_static_init share of the team
 * block — ordered: each worker folds its own block in order into parts[tid];
 * SPMD: coalesced walk + warp/named-barrier tree into parts[par_threads]);
 * joins; folds the parts in order; frees LIFO; publishes the team value to
 * the teams-reduction buffer (last-team-finishes).  dtype I64, U64 or F64.
 * A pad that pushes parts past the 64 KiB arena traps 1 (SharedOverflow, the
 * reference semantics) unless heap_fallback spills it to the global heap.
 * d_team_offsets (optional, [teams]) receives the offset of `parts` returned
 * to each team, for parity against devicert.Arena and the vgpu run. */
int omprt_generic_reduce(const void *d_x, int64_t lb, int64_t ub, int dtype, int op,
                         int teams, int par_threads, int ordered, int64_t pad_bytes,
                         int heap_fallback, int64_t heap_bytes_per_team, void *d_ws,
                         void *d_out, int64_t *d_team_offsets, void *stream);

/* ========================================================================= */
/* Shared-memory smart stack and atomics (parity probes)                      */
/* ========================================================================= */

/* Replays an arena script on the device arena of every team.
 * d_script: nops x 4 int64 {opcode (omprt_arena_op), bytes, offset, value}:
 *   ALLOC bytes -> offset; FREE bytes, offset -> 0; WRITE bytes, offset, value
 *   (the team stores the little-endian u64 `value`, repeated) -> 0;
 *   READ 8, offset -> the u64 there.
 * Each team executes the script (ALLOC/FREE/READ from thread `caller_tid`;
 * 3 = NonUniformAlloc when it is not 0) against its shared-memory arena
 * (capacity bytes, <= 64 KiB, plus heap spill if heap_fallback), initialised
 * to the 0xAA loader_uninitialized poison.  d_results: teams x nops int64 —
 * the op's result, -code at the trapping op (later ops -0x7fff).  After each
 * alloc every thread writes and re-reads a tag through the returned offset
 * and restores the bytes (data-path check; mismatch -> trap Abort).
 * check_uninit != 0: a READ of any byte no WRITE covered traps
 * UninitializedRead (kind 4; vgpu's check_uninit, vgpu.py:365-369).
 * Synchronises; returns OMPRT_TRAP if any team trapped (the trap word is
 * left set for omprt_check_trap), else OMPRT_OK. */
int omprt_arena_replay(const int64_t *d_script, int nops, int teams, int threads,
                       int caller_tid, int64_t capacity, int heap_fallback,
                       int64_t heap_bytes_per_team, void *d_heap, int check_uninit,
                       int64_t *d_results, void *stream);

/* Every thread of a (teams x threads) grid applies one atomic RMW of `kind`
 * (omprt_atomic_kind) to the single cell *d_cell (dtype I32/U32/I64/U64),
 * operand d_operands[g] (and d_desired[g] for CAS), storing the returned old
 * value in d_old[g].  Values travel as uint64 little-endian words.
 * seq_cst scoped atomics (atom.*.gpu), atomicInc for INC (u32 only). */
int omprt_atomic_probe(int kind, int dtype, const uint64_t *d_operands,
                       const uint64_t *d_desired, uint64_t *d_cell, uint64_t *d_old,
                       int teams, int threads, void *stream);

/* Per-thread atomic programs on one cell (corpus.probe_source, corpus.py:374-408):
 * thread g of the (teams x threads) grid executes ops [d_offsets[g], d_offsets[g+1])
 * in program order — kind d_kinds[k] (omprt_atomic_kind; every kind valid for
 * dtype, INC only on U32), operand d_operands[k], desired d_desired[k] (CAS) —
 * on *d_cell and writes the old value of op k to d_old[k].  d_offsets has
 * teams*threads+1 entries; nops = d_offsets[teams*threads]. */
int omprt_atomic_program(const int32_t *d_kinds, const uint64_t *d_operands,
                         const uint64_t *d_desired, const int64_t *d_offsets, int64_t nops,
                         int dtype, uint64_t *d_cell, uint64_t *d_old, int teams, int threads,
                         void *stream);

/* Batched step semantics: thread g applies one RMW of `kind` to its own cell
 * d_cells[g] (element type dtype, packed; i32/u32 cells are 4 bytes apart)
 * with operand d_operands[g] (d_desired[g] for CAS); the old value goes to
 * d_old[g].  Replaces devicert.step_add/max/min/exchange/cas/inc
 * (devicert.py:84-107) as executed by a device. */
int omprt_atomic_apply(int kind, int dtype, uint64_t *d_cells, const uint64_t *d_operands,
                       const uint64_t *d_desired, uint64_t *d_old, int64_t n, void *stream);

/* ========================================================================= */
/* Synthetic inputs and host-buffer (tgt_target-shaped) entry                 */
/* ========================================================================= */

/* Counter-based synthetic data: element i of array k is derived from
 * h = splitmix64(seed ^ (k << 56) ^ (offset + i)):
 *   I64 (int64)h >> 24   U64 h >> 24   I32 (int32)(h >> 32) >> 8   U32 h >> 40
 *   F64 (h >> 11) * 2^-53                F32 (h >> 40) * 2^-24               */
int omprt_fill(void *d_x, int64_t n, int dtype, uint64_t seed, int k, int64_t offset,
               void *stream);

/* Host-buffer offload of one reduction region, the shape of tgt_target
 * (host.py:255-296): copy-in of h_x (n elements; pinned or pageable host
 * memory) to a device buffer, omprt_reduce over [0, n-1], copy-out of the
 * scalar result into *h_out (which holds the initial value on entry), only on
 * status 0.  Synchronous.  The device buffers are cached across calls, per
 * CUDA device (the calling thread's current device runs the region).  Above
 * 512 MiB an SPMD (or integer) reduction is pipelined: the input lands in
 * 256 MiB pieces on a copy stream while the previous piece is reduced, each
 * piece's launch accumulating into the cell (integers bit-exact, fp within
 * the SPMD tolerance); ORDERED fp copies everything first. */
int omprt_reduce_host(const void *h_x, int64_t n, int dtype, int op, int sched,
                      int64_t chunk, int teams, int threads, int mode, void *h_out);

/* Host-buffer offload of the config-3 region (axpy + max/min): copy-in of
 * h_x and h_y (n floats each), omprt_axpy_minmax over [0, n-1], copy-out of
 * y (tofrom) and the two cells *h_max / *h_min (which hold the initial
 * values on entry) — only on status 0 (host.py:293-295).  Synchronous. */
int omprt_axpy_minmax_host(float a, const float *h_x, float *h_y, int64_t n, int sched,
                           int64_t chunk, int teams, int threads, int mode, float *h_max,
                           float *h_min);

/* Host-buffer offload of the fp64 dot product: copy-in of h_x, h_y,
 * omprt_dot over [0, n-1], copy-out of *h_out only on status 0. */
int omprt_dot_host(const double *h_x, const double *h_y, int64_t n, int sched, int64_t chunk,
                   int teams, int threads, int mode, double *h_out);

/* Host-buffer offload of the generic-mode region (omprt_generic_reduce over
 * [0, n-1]): copy-in, launch, synchronise, and on a device trap return
 * OMPRT_TRAP with *h_out and h_team_offsets untouched (the trap word stays
 * set for omprt_check_trap: tgt_target's status 2, host.py:289-292);
 * otherwise copy-out of the cell and, when h_team_offsets is not NULL, the
 * `teams` arena offsets. */
int omprt_generic_reduce_host(const void *h_x, int64_t n, int dtype, int op, int teams,
                              int par_threads, int ordered, int64_t pad_bytes, int heap_fallback,
                              int64_t heap_bytes_per_team, void *h_out,
                              int64_t *h_team_offsets);

/* Release the device staging cached by the host-buffer entries (on every
 * device that has any: the staging is kept per CUDA device). */
int omprt_release_host_cache(void);

/* ========================================================================= */
/* Compiled target regions (B200 device images)                               */
/* ========================================================================= */

/* Load an sm_100a cubin produced by the region compiler
 * (paper_2106_03219_b200/regionc.py: forge IR image -> CUDA C++ over
 * csrc/region_rt.cuh -> NVRTC) into the current context.  Replaces parsing a
 * device image for the runnable arch (host._image_for, host.py:233-252, and
 * VirtualGPU construction, vgpu.py:154-167).  *handle is opaque. */
int omprt_image_load(const void *image, size_t bytes, void **handle);

/* Unload an image loaded by omprt_image_load. */
int omprt_image_unload(void *handle);

/* Launch kernel `kernel` (an __omp_offload_<id> entry) of a loaded image on a
 * (teams x threads) grid with `shared_bytes` of dynamic shared memory (the
 * image's team-shared globals).  `argv` is the kernel's single by-value
 * parameter block of argv_bytes (u64 words: trap record, global-space blob,
 * its init shadow, the team-shared init shadow, the dead-barrier wait mask,
 * then per IR parameter: buffer -> device pointer, byte length, vgpu offset;
 * scalar -> masked value).  Replaces VirtualGPU.launch (vgpu.py:254-347).
 * Stream-ordered, asynchronous: the trap record is read by the caller. */
int omprt_image_launch(void *handle, const char *kernel, int teams, int threads,
                       size_t shared_bytes, const void *argv, size_t argv_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* OMPRT_B200_H */
