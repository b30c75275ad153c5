// Standalone timing of apply_block (one compact-WY block on a smem strip), development aid.
#include <cstdio>
#include "../paper_1104_4475_b200/csrc/tqr_device.cuh"
using namespace tqr;

__global__ void __launch_bounds__(kThreads, 1) k_apply(int nb, int nrows, int reps, int tt, unsigned long long *out) {
  extern __shared__ __align__(16) double smem[];
  const SmemLayout L = smem_layout(nb, 32, 32);
  for (size_t x = threadIdx.x; x < L.total; x += kThreads) smem[x] = 1e-3 * (double)((x * 2654435761u) % 1000);
  if (threadIdx.x == 0) { s_prof_on = 1; for (int i = 0; i < 8; ++i) s_prof[i] = 0; s_prof_last = clock64(); }
  __syncthreads();
  double *Cb = smem + L.offC, *Vb = smem + L.offV[0], *Wb = smem + L.offW, *Ts = smem + L.offT[0];
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
    apply_block(tt ? Cb : nullptr, Cb + kWinRows, L.ldc, nrows, Vb, L.ldv, Ts, 32, 32, true, Wb, Wb + L.ldw * L.wcols);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / reps; for (int i = 0; i < 8; ++i) out[1 + i] = s_prof[i] / reps; }
}

int main() {
  unsigned long long *o, h, hp[9];
  cudaMalloc(&o, 9 * 8);
  const int nb = 200;
  size_t sm = smem_bytes(nb, 32, 32);
  cudaFuncSetAttribute(k_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int nrows : {32, 104, 200})
    for (int tt = 0; tt < 2; ++tt) {
      k_apply<<<1, kThreads, sm>>>(nb, nrows, 50, tt, o);
      k_apply<<<1, kThreads, sm>>>(nb, nrows, 50, tt, o);
      cudaMemcpy(hp, o, 9 * 8, cudaMemcpyDeviceToHost);
      h = hp[0];
      double fl = 4.0 * 32 * 32 * nrows + 2.0 * 32 * 32 * 32;
      printf("nrows=%3d Ctop=%d: %llu ticks per apply_block (%.1f flop/tick)  phase1 %llu  phase2 %llu  phase3 %llu\n",
             nrows, tt, h, fl / h, hp[1 + PH_MMA1], hp[1 + PH_TRI], hp[1 + PH_MMA3]);
    }
  // full-chip: 148 CTAs
  for (int nrows : {104, 200}) {
    k_apply<<<148, kThreads, sm>>>(nb, nrows, 200, 0, o);
    cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("148 CTAs nrows=%3d: %llu ticks per apply_block\n", nrows, h);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
