// Test-only probe: issue rate of tcgen05.mma kind::tf32 (M=64/128, K=8) per
// operand layout.  One CTA per SM; the elected thread of warp 0 issues R MMAs
// back to back into one accumulator and waits for the commit; %clock64 from
// the first issue to the commit arrival, per MMA, is written per CTA.
//   ts:     A from TMEM (cols 256..) / A from SMEM (K-major SW128)
//   b_mn:   B MN-major (SWIZZLE_128B_BASE32B) / K-major (SWIZZLE_128B)
//   n:      MMA N (multiple of 16 up to 256)
// Operand contents are whatever SMEM / TMEM hold (only the timing matters).
#include <cstdio>

#include "sm100.cuh"

using namespace scc::sm100;

__global__ void __launch_bounds__(128) rate_kernel(int m, int n, int ts, int b_mn, int reps, int noise, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const uint32_t warp = warp_id();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(&tbase);
  for (int i = threadIdx.x; i < 65536 / 4; i += 128) reinterpret_cast<float*>(smem)[i] = 0.f;
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (warp != 0 && noise) {
    // shared-memory traffic from the other warps while warp 0 issues MMAs
    float4* p = reinterpret_cast<float4*>(smem + 16384 + (threadIdx.x - 32) * 128);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < reps * noise; ++r) {
      const float4 v = p[r & 7];
      acc.x += v.x;
      p[(r + 3) & 7] = acc;
    }
  } else if (warp == 0) {
    if (elect_one()) {
      const uint32_t idesc = idesc_tf32(static_cast<uint32_t>(m), static_cast<uint32_t>(n), 0, static_cast<uint32_t>(b_mn));
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      const long long t0 = clock64();
      for (int r = 0; r < reps; ++r) {
        const int k = r & 15;
        const uint64_t bd = b_mn ? desc_mn32(b + (k & 3) * 1024, 4096, 512) : desc_sw128(b + (k & 3) * 32, 16, 1024);
        if (ts) {
          mma_tf32_ts(tmem + 256, tmem + 8 * k, bd, idesc, r > 0);
        } else {
          mma_tf32(tmem, desc_sw128(a + (k & 3) * 32, 16, 1024), bd, idesc, r > 0);
        }
      }
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      const long long t1 = clock64();
      out[blockIdx.x] = static_cast<unsigned long long>(t1 - t0);
    }
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

extern "C" int mma_rate(int m, int n, int ts, int b_mn, int reps, int grid, int noise, unsigned long long* out_dev) {
  cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
  rate_kernel<<<grid, 128, 65536 + 1024>>>(m, n, ts, b_mn, reps, noise, out_dev);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("mma_rate: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : -1;
}
