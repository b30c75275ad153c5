// DMMA (mma.sync m16n8k4 f64) latency / throughput vs independent chains per warp (development aid).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b0));
}
template <int C>
__global__ void k(double *out, long long *cyc, int iters) {
  double acc[C][4];
  for (int c = 0; c < C; ++c) for (int e = 0; e < 4; ++e) acc[c][e] = 0;
  double a0 = threadIdx.x * 1e-3, a1 = 0.5, b = 0.25;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) dmma(acc[c], a0, a1, b);
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < C; ++c) s += acc[c][0];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int C> void run(int warps, double *out, long long *cyc) {
  long long h;
  int it = 2000;
  k<C><<<1, 32 * warps>>>(out, cyc, it);
  k<C><<<1, 32 * warps>>>(out, cyc, it);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  double per = (double)h / (it * C);
  printf("chains/warp=%d warps=%2d : %6.1f cycles per DMMA per warp, SM rate %.3f DMMA/cycle (%.1f flop/cyc)\n", C, warps,
         per, warps / per, warps / per * 1024);
}
int main() {
  double *out; long long *cyc;
  cudaMalloc(&out, 8 * 1024 * 8); cudaMalloc(&cyc, 8);
  for (int w : {1, 4, 8}) { run<1>(w, out, cyc); run<2>(w, out, cyc); run<4>(w, out, cyc); run<8>(w, out, cyc); }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
