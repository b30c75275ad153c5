// Microbenchmark: do FP64 DMMA (mma.sync m16n8k4 f64) and DFMA share one pipe
// on B200? Warps 0..D-1 of each CTA run DMMA chains, warps D..7 run DFMA
// chains, for the same wall time budget; prints each stream's TFLOP/s and the
// sum. If the sum exceeds the single-pipe rate, the two run on separate units
// and part of the update contraction could move onto DFMA.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void mixed(double *out, double seed, int ndmma_warps, int dmma_iters, int dfma_iters) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp < ndmma_warps) {
    double a0 = seed + threadIdx.x, a1 = a0 * 0.5, b0 = seed - threadIdx.x;
    double c[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
    for (int it = 0; it < dmma_iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                     : "d"(a0), "d"(a1), "d"(b0));
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  } else {
    double a = seed + threadIdx.x, b = seed * 0.999;
    double c[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = i;
    for (int it = 0; it < dfma_iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; ++i) c[i] = fma(a, c[i], b);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) s += c[i];
  }
  if (s == 1.2345) out[0] = s;
}
int main() {
  double *d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int threads = 256, grid = sms;
  // per-warp flops: DMMA 8 x 1024 per iter, DFMA 16 x 2 x 32 per iter
  struct Cfg { int nd, di, fi; } cfgs[] = {
      {8, ITERS, 0}, {0, 0, ITERS * 4}, {4, ITERS, 0}, {4, 0, ITERS * 4},
      {4, ITERS, ITERS * 4}, {4, ITERS, ITERS * 8}, {2, ITERS, ITERS * 4}, {6, ITERS, ITERS * 4}};
  for (auto c : cfgs) {
    mixed<<<grid, threads>>>(d, 1.0, c.nd, c.di, c.fi);
    cudaEventRecord(e0);
    mixed<<<grid, threads>>>(d, 1.0, c.nd, c.di, c.fi);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fd = 8.0 * 1024 * c.di * c.nd * (double)grid;
    const double ff = 16.0 * 64 * c.fi * (8 - c.nd) * (double)grid;
    printf("dmma_warps=%d dmma_iters=%d dfma_iters=%d : %.3f ms  DMMA %.2f  DFMA %.2f  sum %.2f TFLOP/s\n", c.nd, c.di,
           c.fi, ms, fd / ms / 1e9, ff / ms / 1e9, (fd + ff) / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
