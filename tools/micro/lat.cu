// Microbenchmark: dependent-chain latency of DADD, FADD, DFMA, SHFL+DADD on
// this GPU (one warp, clock64).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
__global__ void k(double *o, float *of, long long *t, double a, float af) {
  double x = a; float y = af;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) x = x + a;
  long long t1 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) y = y + af;
  long long t2 = clock64();
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) x = __fma_rn(x, a, a);
  long long t3 = clock64();
  double v = a * threadIdx.x;
#pragma unroll 64
  for (int i = 0; i < 4096; ++i) x = x + __shfl_sync(0xffffffffu, v, i & 31);
  long long t4 = clock64();
  o[threadIdx.x] = x; of[threadIdx.x] = y;
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; }
}
int main() {
  double *o; float *of; long long *t;
  cudaMalloc(&o, 256); cudaMalloc(&of, 256); cudaMallocManaged(&t, 64);
  for (int r = 0; r < 3; ++r) { k<<<1, 32>>>(o, of, t, 1.0000001, 1.0001f); cudaDeviceSynchronize(); }
  printf("{\"dadd_cyc\": %.2f, \"fadd_cyc\": %.2f, \"dfma_cyc\": %.2f, \"shfl_dadd_cyc\": %.2f}\n",
         t[0] / 4096.0, t[1] / 4096.0, t[2] / 4096.0, t[3] / 4096.0);
  return 0;
}
