// Microbenchmark: FP64 DMMA (mma.sync f64) vs DFMA peak throughput on one B200.
// Used to pick the update-kernel contraction path and as the measured FP64
// roofline denominator.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
__global__ void dmma_kernel(double* out, double seed) {
  double a0 = seed + threadIdx.x, a1 = a0 * 0.5, b0 = seed - threadIdx.x;
  double c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b0));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1.2345) out[0] = s;
}
__global__ void dfma_kernel(double* out, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.999;
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int grid = sms * bps;
      dmma_kernel<<<grid, threads>>>(d, 1.0);
      cudaEventRecord(e0);
      dmma_kernel<<<grid, threads>>>(d, 1.0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * 8 * 4 * 8.0 * ITERS * (threads / 32) * (double)grid;
      printf("DMMA m16n8k4 threads=%d blocks/SM=%d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
      dfma_kernel<<<grid, threads>>>(d, 1.0);
      cudaEventRecord(e0);
      dfma_kernel<<<grid, threads>>>(d, 1.0);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 16 * ITERS * threads * (double)grid;
      printf("DFMA         threads=%d blocks/SM=%d : %.2f TFLOP/s\n", threads, bps, flops / ms / 1e9);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
