// Microbenchmark of the latency of the per-column primitives of the panel
// factorization on one SM (development aid): fp64 division/sqrt chains, the
// warp butterfly sum, __syncthreads, and an STG + LDS round.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void k_micro(double *out, long long *cyc, double seed, int iters) {
  __shared__ double sh[256];
  double x = seed + threadIdx.x * 1e-3, y = 1.0;
  long long t0, t1;
  // 1. division chain
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = 1.0 / (x + 1.5);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = (t1 - t0) / iters;
  // 2. sqrt chain
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x + 2.0);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = (t1 - t0) / iters;
  // 3. warp butterfly chain
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = warp_sum(x) * 1e-2;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = (t1 - t0) / iters;
  // 4. __syncthreads + smem round trip chain
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    sh[threadIdx.x] = x;
    __syncthreads();
    x = sh[(threadIdx.x + 1) & 255] * 0.5 + 1.0;
    __syncthreads();
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = (t1 - t0) / iters;
  // 5. full larfg-like chain
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double s = fma(x, x, y);
    double nrm = sqrt(s);
    double beta = x >= 0 ? -nrm : nrm;
    double tau = (beta - x) / beta;
    double sc = 1.0 / (x - beta);
    x = tau + sc * 1e-3;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = (t1 - t0) / iters;
  // 6. DFMA dependent chain
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, 0.999, 1e-3);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = (t1 - t0) / iters;
  // 7. STG + syncthreads
  __syncthreads();
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    out[threadIdx.x + 256 * (i & 63)] = x;
    __syncthreads();
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = (t1 - t0) / iters;
  out[threadIdx.x + 256 * 64] = x + y;
}

int main() {
  double *out;
  long long *cyc, h[8] = {0};
  cudaMalloc(&out, sizeof(double) * 256 * 65);
  cudaMalloc(&cyc, sizeof(long long) * 8);
  k_micro<<<1, 256>>>(out, cyc, 0.3, 1000);
  k_micro<<<1, 256>>>(out, cyc, 0.3, 1000);
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  const char *nm[] = {"div chain", "sqrt chain", "warp_sum chain", "bar+smem chain (2 bars)", "larfg chain",
                      "dfma chain", "stg+bar"};
  for (int i = 0; i < 7; ++i) printf("%-26s %lld cycles/iter\n", nm[i], h[i]);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
