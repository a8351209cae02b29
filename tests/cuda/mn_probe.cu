// Test-only probe: MN-major kind::tf32 operands in the SWIZZLE_128B_BASE32B
// layout (descriptor layout type 1), loaded straight from an NCHW-style
// [k rows][pixels] fp32 array by TMA with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.
//
//   mode 0: D[p][oc] = sum_k X[k][p] W[oc][k]   A = X^T MN-major (TMA), B = W K-major
//   mode 1: D[oc][p] = sum_k W[oc][k] X[k][p]   A = W K-major, B = X MN-major (TMA)
//
// X is [K=64][P=128] (pixels contiguous); the TMA box is {32 px, 64 rows, 4
// pixel blocks} -> smem [pblk][k][32 px] (128 B rows, 32 B chunks swizzled).
#include <cstdio>

#include "sm100.cuh"
#include "tmap.hpp"

using namespace scc::sm100;

constexpr int M = 128, N = 128, K = 64;

__device__ __forceinline__ uint64_t desc_any(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t type) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(type) << 61;
  return d;
}

__global__ void __launch_bounds__(128) mn_kernel(const __grid_constant__ CUtensorMap tx,
                                                 const float* __restrict__ w, float* out, int mode,
                                                 int lbo, int sbo) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* X = smem;           // 32 KB
  uint8_t* W = smem + 32768;   // 32 KB: [oc/8][8 rows][128 B] per 32-k chunk, 2 chunks
  __shared__ uint64_t bar_ld, bar_mma;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  const uint32_t warp = warp_id();
  if (tid == 0) {
    mbar_init(&bar_ld, 1);
    mbar_init(&bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<128>(&tbase);
  // W K-major SWIZZLE_128B: chunk c (k 32c..32c+31) at W + c*16384, row oc at
  // (oc/8)*1024 + (oc%8)*128, 16 B unit u at ((u ^ oc%8) * 16).
  for (int i = tid; i < N * K; i += 128) {
    const int oc = i / K, k = i % K;
    const int c = k / 32, kk = k % 32;
    const int off = c * 16384 + (oc / 8) * 1024 + (oc % 8) * 128 + (((kk / 4) ^ (oc % 8)) * 16) + (kk % 4) * 4;
    *reinterpret_cast<float*>(W + off) = w[oc * K + k];
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_expect_tx(&bar_ld, 32768);
    tma_load_3d(X, &tx, &bar_ld, 0, 0, 0);
  }
  mbar_wait(&bar_ld, 0);
  if (warp == 0) {
    tc_fence_after();
    if (elect_one()) {
      const uint32_t idesc = mode == 0 ? idesc_tf32(M, N, 1, 0) : idesc_tf32(M, N, 0, 1);
      for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t xd = desc_any(smem_u32(X) + ks * 1024, lbo, sbo, 1);
        const uint64_t wd = desc_sw128(smem_u32(W) + (ks / 4) * 16384 + (ks % 4) * 32, 16, 1024);
        if (mode == 0)
          mma_tf32(tbase, xd, wd, idesc, ks > 0);
        else
          mma_tf32(tbase, wd, xd, idesc, ks > 0);
      }
      mma_commit(&bar_mma);
    }
    __syncwarp();
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tbase + ((warp * 32) << 16) + c, v);
    const int r = warp * 32 + (tid & 31);
    for (int j = 0; j < 16; ++j) out[r * N + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<128>(tbase);
}

extern "C" int mn_probe(const float* x, const float* w, float* out, int mode, int lbo, int sbo) {
  CUtensorMap tm;
  // dims {32 px in block, 64 rows, 4 blocks}; strides rows = 512 B, blocks = 128 B
  const uint64_t dims[3] = {32, K, 4};
  const uint64_t strides[2] = {128 * 4, 32 * 4};
  const uint32_t box[3] = {32, K, 4};
  if (!scc::encode_f32(&tm, x, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
    fprintf(stderr, "mn_probe: tensor map encode failed\n");
    return -1;
  }
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(mn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mn_kernel<<<1, 128, smem>>>(tm, w, out, mode, lbo, sbo);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "mn_probe: %s\n", cudaGetErrorString(e));
    return -2;
  }
  return 0;
}
