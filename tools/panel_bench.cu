// Standalone timing of one 32-column panel block of nb = 200 (GEQRT, TTQRT) on
// one CTA and on 148 CTAs at once (development aid; -DTQR_PROF=1 for the phases).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DTQR_PROF=1 -o tools/panel_bench tools/panel_bench.cu
#include <cstdio>
#include <vector>
#include <random>
#include "../paper_1104_4475_b200/csrc/tqr_device.cuh"
using namespace tqr;

__global__ void __launch_bounds__(kThreads, 1) k_panel(double *X, double *T, int nb, int ib, unsigned long long *out, int mode) {
  extern __shared__ __align__(16) double smem[];
  const SmemLayout L = smem_layout(nb, ib, 32);
  for (size_t x = threadIdx.x; x < L.total; x += kThreads) smem[x] = 0.0;
  if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) s_prof[i] = 0; s_prof_on = 1; }
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) s_prof_last = t0;
  double *Xb = X + (size_t)blockIdx.x * 2 * nb * nb, *Tb = T + (size_t)blockIdx.x * 2 * ib * nb;
  if (mode == 0)
    panel_block<0>(Xb, nullptr, Tb, nb, ib, 0, 32, smem + L.offV[0], smem + L.offT[0], smem + L.offWp);
  else
    panel_block<1>(Xb, Xb + nb * nb, Tb, nb, ib, nb - 32, 32, smem + L.offV[0], smem + L.offT[0], smem + L.offWp);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; for (int i = 0; i < 8; ++i) out[1 + i] = s_prof[i]; }
}

int main() {
  const int nb = 200, ib = 32;
  const int ncta = 148;
  std::vector<double> h((size_t)2 * nb * nb * ncta);
  std::mt19937_64 g(1); std::normal_distribution<double> d;
  for (auto &x : h) x = d(g);
  double *X, *T; unsigned long long *o, ho[9];
  cudaMalloc(&X, h.size() * 8); cudaMalloc(&T, (size_t)2 * ib * nb * 8 * ncta); cudaMalloc(&o, 9 * 8);
  size_t sm = smem_bytes(nb, ib, 32);
  cudaFuncSetAttribute(k_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const char *nm[] = {"load", "fix", "mma1", "tri", "mma3", "columns", "gram+T", "store"};
  for (int mode = 0; mode < 2; ++mode)
    for (int nc : {1, ncta}) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(X, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        k_panel<<<nc, kThreads, sm>>>(X, T, nb, ib, o, mode);
        cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
      }
      printf("%s ctas=%3d: %llu cycles per 32-column block (%.0f per column)\n", mode ? "TTQRT" : "GEQRT", nc, ho[0],
             ho[0] / 32.0);
      for (int i = 0; i < 8; ++i)
        if (ho[1 + i]) printf("   %-8s %8llu\n", nm[i], ho[1 + i]);
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
