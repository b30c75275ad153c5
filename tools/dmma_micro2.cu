// DMMA under runtime-uniform conditionals / fed by smem loads (development aid).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[4], double a0, double a1, double b0) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b0));
}
__global__ void k(double *out, long long *cyc, int iters, int mt) {
  __shared__ double sh[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sh[i] = i * 1e-4;
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double acc[8][4];
  for (int c = 0; c < 8; ++c) for (int e = 0; e < 4; ++e) acc[c][e] = 0;
  // A: 8 unconditional DMMAs with register operands
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) dmma(acc[c], 0.5, 0.25, 0.125);
  }
  long long t1 = clock64();
  // B: 8 DMMAs each under if (c < mt)
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) if (c < mt) dmma(acc[c], 0.5, 0.25, 0.125);
  }
  long long t2 = clock64();
  // C: 8 DMMAs fed by smem loads (as in phase 3)
  for (int i = 0; i < iters; ++i) {
    const int k = (i & 7) * 4;
    const double b = sh[(k + t) + g * 36];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const double a0 = sh[(c * 16 + g) + (k + t) * 128], a1 = sh[(c * 16 + g + 8) + (k + t) * 128];
      dmma(acc[c], a0, a1, b);
    }
  }
  long long t3 = clock64();
  // D: C under if
  for (int i = 0; i < iters; ++i) {
    const int k = (i & 7) * 4;
    const double b = sh[(k + t) + g * 36];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < mt) {
        const double a0 = sh[(c * 16 + g) + (k + t) * 128], a1 = sh[(c * 16 + g + 8) + (k + t) * 128];
        dmma(acc[c], a0, a1, b);
      }
    }
  }
  long long t4 = clock64();
  double s = 0; for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][3];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double *out; long long *cyc, h[4];
  cudaMalloc(&out, 8 * 1024); cudaMalloc(&cyc, 32);
  for (int w : {1, 8}) {
    k<<<1, 32 * w>>>(out, cyc, 1000, 8);
    k<<<1, 32 * w>>>(out, cyc, 1000, 8);
    cudaMemcpy(h, cyc, 32, cudaMemcpyDeviceToHost);
    printf("warps=%d per 8-DMMA iteration: reg %.1f | if %.1f | smem-fed %.1f | smem-fed+if %.1f ticks\n", w, h[0] / 1000.0,
           h[1] / 1000.0, h[2] / 1000.0, h[3] / 1000.0);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
