// Test/diagnostic: TMA issue and completion time vs box shape (one CTA).
#include <cstdio>
#include "sm100.cuh"
#include "tmap.hpp"
using namespace scc::sm100;

__global__ void tma_kernel(const __grid_constant__ CUtensorMap tm, int rows, int nbox, int rows_total,
                           unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int nwarps = blockDim.x / 32;
  const int w = threadIdx.x / 32;
  const int box_bytes = rows * 128;
  const int per = (128 * 1024) / box_bytes;  // boxes fitting in 128 KB
  if (threadIdx.x == 0) mbar_expect_tx(&bar, nbox * box_bytes);
  __syncthreads();
  unsigned long long t0 = globaltimer();
  if ((threadIdx.x & 31) == 0) {
    for (int i = w; i < nbox; i += nwarps) {
      const int r0 = (i * rows) % rows_total;
      tma_load_2d(smem + (i % per) * box_bytes, &tm, &bar, 0, r0);
    }
  }
  unsigned long long t1 = globaltimer();
  mbar_wait(&bar, 0);
  unsigned long long t2 = globaltimer();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
}

extern "C" int tma_probe(const float* g, int rows_total, int rows, int nbox, int swz,
                         unsigned long long* out_dev, int warps) {
  CUtensorMap tm;
  const uint64_t dims[2] = {1024, (uint64_t)rows_total};
  const uint64_t strides[1] = {1024 * 4};
  const uint32_t box[2] = {32, (uint32_t)rows};
  if (!scc::encode_f32(&tm, g, 2, dims, strides, box, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE)) return -1;
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024);
  tma_kernel<<<1, 32 * warps, 140 * 1024>>>(tm, rows, nbox, rows_total, out_dev);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -2;
}
