// Copy-engine latency / throughput for moving one 200 x 32 fp64 reflector block
// (a column strip of a column-major 200 x 200 tile) into shared memory, by box
// shape (development aid):
//   3d4   : 3-D row-tile boxes {8 rows, 32 cols, 4 row tiles}  (7 copies, 64-byte global runs)
//   3d25  : one 3-D row-tile box {8, 32, 25}                   (1 copy, 64-byte runs)
//   2d    : one 2-D box {200 rows, 32 cols}                    (1 copy, 1600-byte runs, column-major smem)
//   cpa   : cp.async 16-byte copies by 256 threads (row-tile layout)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_bench tools/tma_bench.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <vector>

struct Args {
  CUtensorMap m3d4, m3d25, m2d;
  double *A;
  int mode, reps;
  unsigned long long *out;
};
__device__ __forceinline__ unsigned su(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__shared__ __align__(8) unsigned long long mbar;

__global__ void __launch_bounds__(256, 1) k(const __grid_constant__ Args a) {
  extern __shared__ __align__(128) double sm[];
  const int nb = 200;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  unsigned ph = 0;
  const long long col0 = (long long)blockIdx.x * 2 * nb;   // CTA's own tile pair
  unsigned long long t_sum = 0;
  for (int r = 0; r < a.reps; ++r) {
    const int cs = 32 * (r % 6);
    __syncthreads();
    const unsigned long long t0 = clock64();
    if (a.mode == 3) {   // cp.async, row-tile layout
      const double *X = a.A + col0 * nb;
      for (int i = threadIdx.x; i < 25 * 32 * 4; i += 256) {
        const int tl = i >> 7, c = (i >> 2) & 31, pr = 2 * (i & 3);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(sm + tl * 256 + c * 8 + pr)),
                     "l"(X + 8 * tl + pr + (size_t)(cs + c) * nb));
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
    } else {
      if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&mbar)), "r"(a.mode == 5 ? 102400 : 200 * 32 * 8 + (a.mode == 0 ? 3 * 2048 : 0)));
        if (a.mode == 0) {
          for (int e = 25, x = 0; x < 7; ++x, e -= 4) {
            const int st = e - 4 > 0 ? e - 4 : 0;
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(su(sm + st * 256)), "l"(&a.m3d4), "r"(0), "r"((int)col0 + cs), "r"(st), "r"(su(&mbar)) : "memory");
          }
        } else if (a.mode == 4) {   // one 1-D bulk copy of the contiguous 51200-byte block
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su(sm)), "l"(a.A + col0 * nb + (size_t)cs * nb), "r"(51200), "r"(su(&mbar)) : "memory");
        } else if (a.mode == 5) {   // two 1-D bulk copies (V and Y of a block)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su(sm)), "l"(a.A + col0 * nb + (size_t)cs * nb), "r"(51200), "r"(su(&mbar)) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su(sm + 6400)), "l"(a.A + col0 * nb + (size_t)cs * nb + 40000), "r"(51200), "r"(su(&mbar)) : "memory");
        } else if (a.mode == 1) {
          asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                       ::"r"(su(sm)), "l"(&a.m3d25), "r"(0), "r"((int)col0 + cs), "r"(0), "r"(su(&mbar)) : "memory");
        } else {
          asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                       ::"r"(su(sm)), "l"(&a.m2d), "r"(0), "r"((int)col0 + cs), "r"(su(&mbar)) : "memory");
        }
      }
      asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}\n" ::"r"(su(&mbar)), "r"(ph) : "memory");
      ph ^= 1;
    }
    t_sum += clock64() - t0;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) a.out[0] = t_sum / a.reps;
}

int main() {
  const int nb = 200, ncta = 148;
  double *A;
  unsigned long long *o, h;
  const size_t n = (size_t)2 * ncta * nb * nb;
  cudaMalloc(&A, n * 8);
  cudaMemset(A, 0, n * 8);
  cudaMalloc(&o, 8);
  void *f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  Args a{};
  const cuuint32_t e3[3] = {1, 1, 1};
  {
    const cuuint64_t d[3] = {8, (cuuint64_t)2 * ncta * nb, (cuuint64_t)(nb / 8)}, st[2] = {(cuuint64_t)nb * 8, 64};
    const cuuint32_t b4[3] = {8, 32, 4}, b25[3] = {8, 32, 25};
    enc(&a.m3d4, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, d, st, b4, e3, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&a.m3d25, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, A, d, st, b25, e3, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const cuuint64_t d2[2] = {(cuuint64_t)nb, (cuuint64_t)2 * ncta * nb}, st2[1] = {(cuuint64_t)nb * 8};
    const cuuint32_t b2[2] = {200, 32};
    enc(&a.m2d, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, d2, st2, b2, e3, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  a.A = A; a.out = o; a.reps = 200;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
  const char *nm[6] = {"3d4 (7 boxes)", "3d25 (1 box) ", "2d (1 box)   ", "cp.async     ", "1d bulk 51KB ", "2x1d bulk    "};
  for (int mode = 0; mode < 6; ++mode)
    for (int nc : {1, ncta}) {
      a.mode = mode;
      k<<<nc, 256, 110 * 1024>>>(a);
      k<<<nc, 256, 110 * 1024>>>(a);
      cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
      printf("%s ctas=%3d: %6llu cycles per 200x32 block (%.1f B/cycle/SM)\n", nm[mode], nc, h, 51200.0 / h);
    }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
