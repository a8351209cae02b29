// Diagnostic: aggregate TMA load throughput with all SMs busy, vs the width of
// the contiguous row segment (box inner dim) and box height.
#include <cstdio>
#include "sm100.cuh"
#include "tmap.hpp"
using namespace scc::sm100;

__global__ void __launch_bounds__(128, 1) chip_kernel(const __grid_constant__ CUtensorMap tm, int box_bytes, int bw,
                                                      int bh, int iters, int rows_total, int cols_total) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar[8];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // each warp: 2 buffers, ping-pong; iters boxes per warp
  const int ncolblk = cols_total / bw;
  uint32_t ph[2] = {0, 0};
  for (int i = 0; i < iters; ++i) {
    const int b = i & 1;
    uint8_t* dst = smem + (w * 2 + b) * box_bytes;
    if (i >= 2) {
      mbar_wait(&bar[w * 2 + b], ph[b]);
      ph[b] ^= 1;
    }
    if (lane == 0) {
      const long long g = (long long)(blockIdx.x * 4 + w) * iters + i;
      const int cb = (int)(g % ncolblk);
      const int rb = (int)((g / ncolblk) % (rows_total / bh));
      mbar_expect_tx(&bar[w * 2 + b], box_bytes);
      tma_load_2d(dst, &tm, &bar[w * 2 + b], cb * bw, rb * bh);
    }
    __syncwarp();
  }
  for (int b = 0; b < 2; ++b) {
    mbar_wait(&bar[w * 2 + b], ph[b]);
  }
}

extern "C" float tma_chip(const float* g, int cols, int rows, int bw, int bh, int iters) {
  CUtensorMap tm;
  const uint64_t dims[2] = {(uint64_t)cols, (uint64_t)rows};
  const uint64_t strides[1] = {(uint64_t)cols * 4};
  const uint32_t box[2] = {(uint32_t)bw, (uint32_t)bh};
  if (!scc::encode_f32(&tm, g, 2, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE)) return -1;
  const int box_bytes = bw * bh * 4;
  const int smem = 8 * box_bytes + 1024;
  cudaFuncSetAttribute(chip_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  chip_kernel<<<148, 128, smem>>>(tm, box_bytes, bw, bh, iters, rows, cols);
  cudaEventRecord(e0);
  chip_kernel<<<148, 128, smem>>>(tm, box_bytes, bw, bh, iters, rows, cols);
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1) != cudaSuccess) return -2;
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 148.0 * 4 * iters * box_bytes;
  return (float)(bytes / (ms * 1e-3) / 1e9);
}
