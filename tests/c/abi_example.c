/*
 * A plain C caller of the B200 runtime — no Python, no torch: the drop-in
 * boundary as a C/C++ host program would use it.
 *
 *   gcc -std=c11 -I include tests/c/abi_example.c \
 *       -L paper_2106_03219_b200 -lomprt_b200 -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2106_03219_b200 -o abi_example && ./abi_example
 *
 * Checks: the for_static_init worked example (test_devicert.py:89-90), the
 * PARTIAL_SUMS corpus result 5050 (corpus.py:219-247) through omprt_reduce,
 * the host-buffer entry, a device trap (arena overflow, code 1) reported as
 * status 2 with the trap word, and a fp64 sum against the exact value.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "omprt_b200.h"

/* the few CUDA runtime entry points we need, declared to avoid the header */
int cudaMalloc(void **p, size_t n);
int cudaFree(void *p);
int cudaMemcpy(void *dst, const void *src, size_t n, int kind);
int cudaMemset(void *p, int v, size_t n);
int cudaDeviceSynchronize(void);

#define H2D 1
#define D2H 2
#define CHECK(c)                                                              \
  do {                                                                        \
    int _s = (c);                                                             \
    if (_s != 0) {                                                            \
      fprintf(stderr, "%s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #c, _s,   \
              omprt_last_error());                                            \
      return 1;                                                               \
    }                                                                         \
  } while (0)

int main(void) {
  int64_t lo, hi;
  CHECK(omprt_device_init(0));
  CHECK(omprt_static_bounds(0, 99, 1, 4, &lo, &hi));
  if (lo != 25 || hi != 49) return fprintf(stderr, "static_bounds %lld %lld\n",
                                           (long long)lo, (long long)hi), 1;

  /* PARTIAL_SUMS: u32 sum of i over for_static_init(1, 100) on 2 teams x 4 threads */
  uint32_t h[101];
  for (int i = 0; i <= 100; ++i) h[i] = (uint32_t)i;
  void *dx, *dws, *dout;
  /* one workspace big enough for every launch below (148 teams at most) */
  size_t wsb = omprt_reduce_workspace_bytes(omprt_num_sms(), 256, OMPRT_MODE_SPMD);
  CHECK(cudaMalloc(&dx, sizeof h));
  CHECK(cudaMalloc(&dws, wsb));
  CHECK(cudaMalloc(&dout, 8));
  CHECK(cudaMemset(dws, 0, wsb));
  CHECK(cudaMemset(dout, 0, 8));
  CHECK(cudaMemcpy(dx, h, sizeof h, H2D));
  CHECK(omprt_reduce(dx, 1, 100, OMPRT_U32, OMPRT_OP_ADD, OMPRT_SCHED_STATIC, 1, 2, 4,
                     OMPRT_MODE_SPMD, dws, dout, NULL));
  uint32_t cell = 0;
  CHECK(cudaMemcpy(&cell, dout, 4, D2H));
  if (cell != 5050) return fprintf(stderr, "partial_sums %u\n", cell), 1;

  /* host-buffer entry: int64 sum of 0..n-1 */
  const int64_t n = 1 << 20;
  int64_t *hx = (int64_t *)malloc(n * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) hx[i] = i;
  int64_t s = 0;
  CHECK(omprt_reduce_host(hx, n, OMPRT_I64, OMPRT_OP_ADD, OMPRT_SCHED_DISTRIBUTE, 1, 148, 256,
                          OMPRT_MODE_SPMD, &s));
  if (s != n * (n - 1) / 2) return fprintf(stderr, "reduce_host %lld\n", (long long)s), 1;

  /* fp64 sum of synthetic data (the test compares it with the exact value) */
  void *df;
  const int64_t m = 1 << 24;
  CHECK(cudaMalloc(&df, m * 8));
  CHECK(omprt_fill(df, m, OMPRT_F64, 0x210603219ull, 0, 0, NULL));
  double fs = 0.0;
  CHECK(cudaMemset(dout, 0, 8));
  CHECK(omprt_reduce(df, 0, m - 1, OMPRT_F64, OMPRT_OP_ADD, OMPRT_SCHED_DISTRIBUTE, 1,
                     omprt_num_sms(), 256, OMPRT_MODE_SPMD, dws, dout, NULL));
  CHECK(cudaMemcpy(&fs, dout, 8, D2H));

  /* generic region whose pad overflows the 64 KiB arena: status-2 trap, code 1 */
  void *dws2;
  size_t wsb2 = omprt_generic_workspace_bytes(4, 64, 0, 0);
  CHECK(cudaMalloc(&dws2, wsb2));
  CHECK(cudaMemset(dws2, 0, wsb2));
  CHECK(omprt_generic_reduce(df, 0, 100, OMPRT_I64, OMPRT_OP_ADD, 4, 64, 0,
                             65536 - 64, 0, 0, dws2, dout, NULL, NULL));
  int kind = 0, code = 0, team = 0, thread = 0;
  int st = omprt_check_trap(NULL, &kind, &code, &team, &thread);
  if (st != OMPRT_TRAP || kind != OMPRT_TRAP_SHARED_OVERFLOW || code != 1)
    return fprintf(stderr, "trap %d kind %d code %d\n", st, kind, code), 1;

  printf("abi_example ok: static_bounds (25,49), partial_sums 5050, reduce_host %lld, "
         "trap kind %d code %d team %d, fp64 sum %.17g\n",
         (long long)s, kind, code, team, fs);
  cudaFree(dx);
  cudaFree(dws);
  cudaFree(dws2);
  cudaFree(dout);
  cudaFree(df);
  free(hx);
  return 0;
}
