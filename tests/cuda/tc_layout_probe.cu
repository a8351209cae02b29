// Test-only: operand-layout probe for kind::tf32 tcgen05.mma.  D[p][oc] =
// sum_k X[k][p] W[oc][k], M=N=128, K=32, A staged manually in either K-major
// or MN-major SWIZZLE_128B form with caller-chosen LBO/SBO and major flag.
#include <cstdio>

#include "sm100.cuh"

using namespace scc::sm100;

constexpr int M = 128, N = 128, K = 32;

__global__ void __launch_bounds__(128) layout_kernel(const float* __restrict__ xg,
                                                     const float* __restrict__ w, float* out,
                                                     int a_kmajor, int a_flag, int lbo, int sbo) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* A = smem;
  uint8_t* B = smem + 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  const uint32_t warp = warp_id();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<128>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  for (int i = tid; i < M * K; i += 128) {
    const int k = i / M, p = i % M;
    int off;
    if (a_kmajor) {
      off = (p / 8) * 1024 + (p % 8) * 128 + (((k / 4) ^ (p % 8)) * 16) + (k % 4) * 4;
    } else {
      const int cb = p / 32, pp = p % 32;
      off = cb * (K * 128) + k * 128 + (((pp / 4) ^ (k % 8)) * 16) + (pp % 4) * 4;
    }
    *reinterpret_cast<float*>(A + off) = xg[k * M + p];
  }
  for (int i = tid; i < N * K; i += 128) {
    const int oc = i / K, k = i % K;
    const int off = (oc / 8) * 1024 + (oc % 8) * 128 + (((k / 4) ^ (oc % 8)) * 16) + (k % 4) * 4;
    *reinterpret_cast<float*>(B + off) = w[oc * K + k];
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (elect_one()) {
      const uint32_t idesc = idesc_tf32(M, N, a_flag, 0);
      for (int ks = 0; ks < K / 8; ++ks) {
        const uint32_t astart = smem_u32(A) + (a_kmajor ? ks * 32 : ks * 1024);
        const uint64_t ad = desc_sw128(astart, lbo, sbo);
        const uint64_t bd = desc_sw128(smem_u32(B) + ks * 32, 16, 1024);
        mma_tf32(tbase, ad, bd, idesc, ks > 0);
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tbase + ((warp * 32) << 16) + c, v);
    const int p = warp * 32 + (tid & 31);
    for (int j = 0; j < 16; ++j) out[p * N + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tbase);
}

extern "C" int tc_layout(const float* x, const float* w, float* out, int a_kmajor, int a_flag,
                         int lbo, int sbo) {
  const int smem = 32768 + 1024;
  cudaFuncSetAttribute(layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  layout_kernel<<<1, 128, smem>>>(x, w, out, a_kmajor, a_flag, lbo, sbo);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "tc_layout: %s\n", cudaGetErrorString(e));
    return -2;
  }
  return 0;
}
