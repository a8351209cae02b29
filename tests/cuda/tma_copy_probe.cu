// Test-only micro-benchmark: the forward kernel's I/O pattern with no compute.
// y[n][0:C][p] = y[n][C:2C][p] = x[n][0:C][p] for 32-pixel blocks, each CTA a
// contiguous run of blocks; TMA loads of {32 px, C rows} and TMA stores of the
// same box to both halves; `depth` load buffers in flight per CTA.
#include <cstdio>
#include "sm100.cuh"
#include "tmap.hpp"
using namespace scc::sm100;

__global__ void __launch_bounds__(128, 1) copy_kernel(const __grid_constant__ CUtensorMap tx,
                                                      const __grid_constant__ CUtensorMap ty, int units,
                                                      int nbps, int C, int depth) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar[16];
  const int box = C * 128;
  const int u0 = (int)((long long)blockIdx.x * units / gridDim.x);
  const int u1 = (int)((long long)(blockIdx.x + 1) * units / gridDim.x);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // prime: issue `depth` loads
    int issued = u0;
    for (int d = 0; d < depth && issued < u1; ++d, ++issued) {
      const int n = issued / nbps, b = issued % nbps;
      mbar_expect_tx(&bar[d], box);
      tma_load_3d(smem + d * box, &tx, &bar[d], b * 32, 0, n);
    }
    uint32_t ph[16] = {0};
    for (int u = u0; u < u1; ++u) {
      const int d = (u - u0) % depth;
      mbar_wait(&bar[d], ph[d]);
      ph[d] ^= 1;
      const int n = u / nbps, b = u % nbps;
      tma_store_3d(&ty, smem + d * box, b * 32, 0, 2 * n);
      tma_store_3d(&ty, smem + d * box, b * 32, 0, 2 * n + 1);
      bulk_commit();
      if (issued < u1) {
        // the buffer we reuse next is d; its stores must have read it
        bulk_wait_read<0>();
        const int n2 = issued / nbps, b2 = issued % nbps;
        mbar_expect_tx(&bar[d], box);
        tma_load_3d(smem + d * box, &tx, &bar[d], b2 * 32, 0, n2);
        ++issued;
      }
    }
    bulk_wait<0>();
  }
  __syncthreads();
}

extern "C" float tma_copy(const float* x, float* y, int n, int C, int P, int depth, int grid) {
  CUtensorMap tx, ty;
  {
    const uint64_t dims[3] = {(uint64_t)P, (uint64_t)C, (uint64_t)n};
    const uint64_t strides[2] = {(uint64_t)P * 4, (uint64_t)P * 4 * C};
    const uint32_t box[3] = {32, (uint32_t)C, 1};
    if (!scc::encode_f32(&tx, x, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE)) return -1;
  }
  {
    const uint64_t dims[3] = {(uint64_t)P, (uint64_t)C, (uint64_t)(2 * n)};
    const uint64_t strides[2] = {(uint64_t)P * 4, (uint64_t)P * 4 * C};
    const uint32_t box[3] = {32, (uint32_t)C, 1};
    if (!scc::encode_f32(&ty, y, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE)) return -1;
  }
  const int nbps = P / 32;
  const int units = n * nbps;
  const int smem = depth * C * 128;
  cudaFuncSetAttribute(copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int r = 0; r < 3; ++r) copy_kernel<<<grid, 128, smem>>>(tx, ty, units, nbps, C, depth);
  cudaEventRecord(e0);
  for (int r = 0; r < 20; ++r) copy_kernel<<<grid, 128, smem>>>(tx, ty, units, nbps, C, depth);
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1) != cudaSuccess) return -2;
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1e3f / 20;  // us per launch
}
