// Standalone timing of strip_update (one UNMQR / TTMQR strip task of nb = 200,
// 7 inner blocks) on 1 CTA and on 148 CTAs (development aid).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/strip_bench tools/strip_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>
#include "../paper_1104_4475_b200/csrc/tqr_device.cuh"
using namespace tqr;

struct BenchArgs {
  CUtensorMap map, map4;
  double *A, *T;
  int nb, ib, reps, kind, tma;
  unsigned long long *out;
};

__global__ void __launch_bounds__(kThreads, 1) k_strip(const __grid_constant__ BenchArgs b) {
  extern __shared__ __align__(128) double smem[];   // (TMA tensor copies need 128-byte-aligned destinations)
  const SmemLayout L = smem_layout(b.nb, b.ib, 32);
  for (size_t x = threadIdx.x; x < L.total; x += kThreads) smem[x] = 0.0;
  if (threadIdx.x == 0) {
#if TQR_EXP & 16
    asm volatile("prefetch.tensormap [%0];" ::"l"(&b.map) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&b.map4) : "memory");
#endif
    mbar_init_all();
    s_prof_on = 1;
    for (int i = 0; i < 8; ++i) s_prof[i] = 0;
    s_prof_last = clock64();
  }
  __syncthreads();
  unsigned ph = 0;
  const int nb = b.nb, ib = b.ib, nblk = (nb + ib - 1) / ib;
  // CTA c: tiles 2c (reflectors / C1) and 2c + 1 (C2)
  double *X = b.A + (size_t)(2 * blockIdx.x) * nb * nb, *C = X + (size_t)nb * nb;
  const double *Ts = b.T + (size_t)blockIdx.x * ib * nb;
  const CUtensorMap *m = b.tma ? &b.map : nullptr, *m4 = b.tma ? &b.map4 : nullptr;
  long long t0 = clock64();
  for (int r = 0; r < b.reps; ++r) {
    const StripJob J{X, Ts, X, C, nb, ib, 0, 32, 0, nblk, true, false, m, m4, 2 * (int)blockIdx.x * nb,
                     2 * (int)blockIdx.x * nb};
    if (b.kind == 0) strip_update<SU_UN>(J, smem, L, ph);
    else if (b.kind == 1) strip_update<SU_TT>(J, smem, L, ph);
    else strip_update<SU_TS>(J, smem, L, ph);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    b.out[0] = (t1 - t0) / b.reps;
    for (int i = 0; i < 8; ++i) b.out[1 + i] = s_prof[i] / b.reps;
  }
}

int main() {
  const int nb = 200, ib = 32, nblk = 7, ncta = 148;
  double *A, *T;
  unsigned long long *o, h[9];
  cudaMalloc(&A, sizeof(double) * 2 * ncta * nb * nb);
  cudaMalloc(&T, sizeof(double) * ncta * ib * nb);
  cudaMalloc(&o, 9 * 8);
  std::vector<double> ha((size_t)2 * ncta * nb * nb), ht((size_t)ncta * ib * nb);
  unsigned s = 1;
  for (auto &x : ha) { s = s * 1664525u + 1013904223u; x = ((s >> 8) & 0xffff) / 65536.0 - 0.5; }
  for (auto &x : ht) { s = s * 1664525u + 1013904223u; x = 1e-3 * (((s >> 8) & 0xffff) / 65536.0); }
  cudaMemcpy(A, ha.data(), ha.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(T, ht.data(), ht.size() * 8, cudaMemcpyHostToDevice);
  void *f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  BenchArgs b{};
  const cuuint64_t dims[3] = {8, (cuuint64_t)2 * ncta * nb, (cuuint64_t)(nb / 8)};
  const cuuint64_t strides[2] = {(cuuint64_t)nb * 8, 64};
  const cuuint32_t box[3] = {8, 32, (cuuint32_t)kBoxTiles}, box4[3] = {8, 32, 4}, estr[3] = {1, 1, 1};
  CUresult cr = enc(&b.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&b.map4, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, dims, strides, box4, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  b.A = A; b.T = T; b.nb = nb; b.ib = ib; b.out = o;
  const size_t sm = smem_bytes(nb, ib, 32);
  cudaFuncSetAttribute(k_strip, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  // ideal cycles: 8 per m16n8k4 per SM (FP64 tensor pipe), phases 1 + 3 + 2
  const char *names[3] = {"UNMQR", "TTMQR", "TSMQR"};
  for (int kind = 0; kind < 3; ++kind) {
    long long dm = 0;
    for (int blk = 0; blk < nblk; ++blk) {
      const int j0 = 32 * blk, bw = j0 + 32 <= nb ? 32 : nb - j0;
      const int rows = kind == 0 ? nb - j0 : (kind == 1 ? j0 + bw : nb);
      const int tiles = (rows + 7) / 8;
      dm += 2 * 8 * tiles * 2 + 64;   // phase 1 (2 halves x 8 per tile) + phase 3 (same) + phase 2
    }
    for (int tma = 0; tma < 2; ++tma)
      for (int nc : {1, ncta}) {
        b.kind = kind; b.tma = tma; b.reps = 20;
        k_strip<<<nc, kThreads, sm>>>(b);
        k_strip<<<nc, kThreads, sm>>>(b);
        cudaMemcpy(h, o, 9 * 8, cudaMemcpyDeviceToHost);
        printf("%s tma=%d ctas=%3d: %6llu cyc/task (ideal %lld, %.0f%%)  load0 %llu wait %llu fix %llu mma1 %llu tri %llu mma3 %llu\n",
               names[kind], tma, nc, h[0], dm * 8, 100.0 * dm * 8 / h[0], h[1 + PH_LOAD], h[1 + PH_PANEL], h[1 + PH_FIX],
               h[1 + PH_MMA1], h[1 + PH_TRI], h[1 + PH_MMA3]);
      }
  }
  printf("encode=%d err=%s\n", (int)cr, cudaGetErrorString(cudaGetLastError()));
}
