// Test-only micro-benchmark: cost of the band-kernel epilogue pieces on one
// SM (clock64 cycles, CTA 0), to size the pipeline:
//   mode 0: 4 warps x G groups of tcgen05.ld.32x32b.x32 + wait
//   mode 1: mode 0 + 32 STS per group (staging writes, conflict-free)
//   mode 2: 32 STS per group only
//   mode 3: mode 1 while warp 4 issues back-to-back SS MMAs (M=128, N=128, K=8)
// out[0] = cycles of the slowest epilogue warp, out[1] = MMAs issued.
#include <cstdio>

#include "sm100.cuh"

using namespace scc::sm100;

__global__ void __launch_bounds__(192, 1) epi_kernel(unsigned long long* out, int mode, int groups) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tbase;
  __shared__ uint64_t mbar;
  __shared__ int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    stop = 0;
    mbar_init(&mbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (warp < 4) {
    float* buf = reinterpret_cast<float*>(smem + 32768) + warp * 1024;
    float acc = 0.f;
    __syncwarp();
    const unsigned long long t0 = clock64();
    for (int g = 0; g < groups; ++g) {
      uint32_t v[32];
      if (mode != 2) {
        tmem_ld32_nowait(tm + ((warp * 32) << 16) + (g & 7) * 32, v);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = g + j;
      }
      if (mode == 0) {
#pragma unroll
        for (int j = 0; j < 32; ++j) acc += __uint_as_float(v[j]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) buf[j * 32 + lane] = __uint_as_float(v[j]);
      }
    }
    __syncwarp();
    const unsigned long long t1 = clock64();
    if (lane == 0) atomicMax(out, t1 - t0);
    if (acc == 12345.f) out[2] = 1;
    if (warp == 0 && lane == 0) atomicExch(&stop, 1);
  } else if (mode == 3) {
    // back-to-back MMAs reading 4 KB A + 4 KB B from smem per instruction
    unsigned long long n = 0;
    const uint64_t da = desc_sw128(smem_u32(smem), 16, 1024);
    const uint64_t db = desc_sw128(smem_u32(smem + 16384), 16, 1024);
    const uint32_t idesc = idesc_tf32(128, 128, 0, 0);
    while (atomicAdd(&stop, 0) == 0) {
      if (elect_one()) {
        for (int i = 0; i < 16; ++i) mma_tf32(tm + 256, da, db, idesc, 1);
        mma_commit(&mbar);
      }
      __syncwarp();
      mbar_wait(&mbar, static_cast<uint32_t>(n & 1));
      ++n;
    }
    if (lane == 0) out[1] = n * 16;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tm);
}

extern "C" int epi_probe(unsigned long long* out, int mode, int groups) {
  const int smem = 64 * 1024;
  cudaFuncSetAttribute(epi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  epi_kernel<<<1, 192, smem>>>(out, mode, groups);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "epi_probe: %s\n", cudaGetErrorString(e));
    return -2;
  }
  return 0;
}
