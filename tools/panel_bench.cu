// Standalone timing of one 32-column GEQRT panel block (development aid).
//   nvcc ... -DTQR_PANEL_PROF tools/panel_bench.cu
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
  if (mode == 0)
    panel_block<0>(X, nullptr, T, nb, ib, 0, 32, smem + L.offV[0], L.ldv, smem + L.offT[0], smem + L.offW);
  else
    panel_block<1>(X, X + nb * nb, T, nb, ib, nb - 32, 32, smem + L.offV[0], L.ldv, smem + L.offT[0], smem + L.offW);
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; for (int i = 0; i < 8; ++i) out[1 + i] = s_prof[i]; }
}

int main() {
  const int nb = 200, ib = 32;
  std::vector<double> h(2 * nb * nb);
  std::mt19937_64 g(1); std::normal_distribution<double> d;
  for (auto &x : h) x = d(g);
  double *X, *T; unsigned long long *o, ho[9];
  cudaMalloc(&X, h.size() * 8); cudaMalloc(&T, 2 * ib * nb * 8); cudaMalloc(&o, 9 * 8);
  size_t sm = smem_bytes(nb, ib, 32);
  cudaFuncSetAttribute(k_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  const char *nm[] = {"owner norm", "larfg", "publish", "barrier", "update", "panel", "trec", "loop-top"};
  for (int mode = 0; mode < 2; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemcpy(X, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
      k_panel<<<1, kThreads, sm>>>(X, T, nb, ib, o, mode);
      cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
    }
    printf("mode %d: total %llu cycles for 32 columns (%.0f/col)\n", mode, ho[0], ho[0] / 32.0);
    for (int i = 0; i < 8; ++i) printf("   %-10s %8llu  (%.0f/col)\n", nm[i], ho[1 + i], ho[1 + i] / 32.0);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
