// DMMA rate vs SM clock: clock64 and globaltimer around a register-fed DMMA loop on every SM
// (development aid: is the FP64 tensor pipe bound by issue cycles or by clock throttling?).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b0));
}
__device__ unsigned long long gt() { unsigned long long v; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v)); return v; }
__global__ void k(double *out, unsigned long long *o, int iters, double x) {
  double acc[8][4];
  for (int c = 0; c < 8; ++c) for (int e = 0; e < 4; ++e) acc[c][e] = 0;
  double a0 = x * threadIdx.x, a1 = x + threadIdx.x, b = x * 0.5;
  __syncthreads();
  unsigned long long c0 = clock64(), g0 = gt();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) dmma(acc[c], a0, a1, b);
    a0 += 1e-30; b -= 1e-30;
  }
  unsigned long long c1 = clock64(), g1 = gt();
  double s = 0; for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { o[0] = c1 - c0; o[1] = g1 - g0; }
}
int main() {
  double *out; unsigned long long *o, h[2];
  cudaMalloc(&out, 8 * 148 * 1024); cudaMalloc(&o, 16);
  for (int grid : {1, 2, 8, 37, 74, 111, 148})
  for (int thr : {128, 256}) {
    int iters = 100000;
    k<<<grid, thr>>>(out, o, 1000, 1.0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<grid, thr>>>(out, o, iters, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
    double dm = 8.0 * iters * (thr / 32) * grid;
    printf("grid %3d threads %d: %.2f TFLOP/s  cycles %llu  ns %llu  => SM clock %.0f MHz, %.2f cycles/DMMA/SMSP\n", thr,
           grid, dm * 1024 / (ms * 1e-3) / 1e12, h[0], h[1], 1e3 * h[0] / (double)h[1],
           (double)h[0] / (8.0 * iters * (thr / 32) / 4));
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
