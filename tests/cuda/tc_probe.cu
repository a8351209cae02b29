// Test-only probe of the tcgen05 building blocks the SCC tensor-core kernels
// use (csrc/sm100.cuh): one CTA computes D[p][oc] = sum_k X[k][p] * W[oc][k]
// for M=128 pixels, N=128 channels, K=32, with A (X) MN-major loaded by TMA
// (SWIZZLE_128B, box {32, 8}) and B (W) K-major written with a manual 128B
// swizzle.  mode 0: one pass with raw fp32 operands (reveals how the tensor
// core reduces fp32 bits to tf32); mode 1: 3xTF32 split.
#include <cstdio>

#include "sm100.cuh"
#include "tmap.hpp"

using namespace scc::sm100;

constexpr int M = 128, N = 128, K = 32;

__global__ void __launch_bounds__(128) probe_kernel(const __grid_constant__ CUtensorMap tx,
                                                    const float* __restrict__ w, float* out,
                                                    int mode) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* a_hi = reinterpret_cast<float*>(smem);            // 4 col blocks x 32 rows x 128B = 16 KB
  float* a_lo = reinterpret_cast<float*>(smem + 16384);    // 16 KB
  float* b_hi = reinterpret_cast<float*>(smem + 32768);    // 128 rows x 128B = 16 KB
  float* b_lo = reinterpret_cast<float*>(smem + 49152);    // 16 KB
  __shared__ uint64_t bar_tma, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  const uint32_t warp = warp_id();
  if (tid == 0) {
    mbar_init(&bar_tma, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<128>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_expect_tx(&bar_tma, M * K * 4);
    for (int cb = 0; cb < 4; ++cb)
      for (int r8 = 0; r8 < K / 8; ++r8)
        tma_load_2d(reinterpret_cast<uint8_t*>(a_hi) + cb * (K * 128) + r8 * 1024, &tx, &bar_tma,
                    cb * 32, r8 * 8);
  }
  // B: K-major SW128, row oc (128B = 32 k), 8-row groups of 1 KB.
  for (int i = tid; i < N * K; i += 128) {
    const int oc = i / K, k = i % K;
    const float v = w[oc * K + k];
    const int g = oc / 8, r = oc % 8;
    const int off = g * 1024 + r * 128 + (((k / 4) ^ r) * 16) + (k % 4) * 4;
    const float hi = mode == 0 ? v : tf32_hi(v);
    *reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(b_hi) + off) = hi;
    *reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(b_lo) + off) = v - hi;
  }
  mbar_wait(&bar_tma, 0);
  // A lo (same swizzled layout, elementwise)
  for (int i = tid; i < M * K; i += 128) {
    const float v = a_hi[i];
    a_lo[i] = v - tf32_hi(v);
    if (mode == 1) a_hi[i] = tf32_hi(v);
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (elect_one()) {
      const uint32_t idesc = idesc_tf32(M, N, 1, 0);
      for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t ad_hi = desc_sw128(smem_u32(a_hi) + ks * 1024, K * 128, 1024);
        const uint64_t ad_lo = desc_sw128(smem_u32(a_lo) + ks * 1024, K * 128, 1024);
        const uint64_t bd_hi = desc_sw128(smem_u32(b_hi) + ks * 32, 16, 1024);
        const uint64_t bd_lo = desc_sw128(smem_u32(b_lo) + ks * 32, 16, 1024);
        mma_tf32(tmem_base, ad_hi, bd_hi, idesc, ks > 0);
        if (mode == 1) {
          mma_tf32(tmem_base, ad_lo, bd_hi, idesc, 1);
          mma_tf32(tmem_base, ad_hi, bd_lo, idesc, 1);
        }
      }
      mma_commit(&bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  // epilogue: warp w reads lanes 32w..32w+31
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tmem_base + ((warp * 32) << 16) + c, v);
    const int p = warp * 32 + (tid & 31);
    for (int j = 0; j < 16; ++j) out[p * N + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tmem_base);
}

extern "C" int tc_probe(const float* x, const float* w, float* out, int mode) {
  CUtensorMap tm;
  const uint64_t dims[2] = {M, K};
  const uint64_t strides[1] = {M * 4};
  const uint32_t box[2] = {32, 8};
  if (!scc::encode_f32_sw128(&tm, x, 2, dims, strides, box)) return -1;
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_kernel<<<1, 128, smem>>>(tm, w, out, mode);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "tc_probe: %s\n", cudaGetErrorString(e));
    return -2;
  }
  return 0;
}
