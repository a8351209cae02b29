// Test-only probe: tcgen05.mma kind::f16 with bf16 operands, A in TMEM
// (TS mode), B from shared memory in the two layouts the bf16x3 backward
// uses, plus the issue rate.
//
//   bf16_probe(mode 0): D[m][n] = sum_k A[m][k] B[k][n], B MN-major SWIZZLE_128B
//       (element (k, n), n < 64, at (k/8)*sbo + (k%8)*128 + ((n/8 ^ k%8)*16) + (n%8)*2)
//   bf16_probe(mode 1): the same product, B stored K-major SWIZZLE_128B
//       (row n, element k at (k/64)*(N/8*1024) + (n/8)*1024 + (n%8)*128 + (((k%64)/8 ^ n%8)*16) + (k%8)*2)
//   A in TMEM: lane m, column c holds bf16 pair (k = 2c, 2c+1); `swap` puts
//   k = 2c in the high half instead of the low half.
//   M = 128, N = 64, K = 128 (8 MMAs of K = 16).
//
//   bf16_rate: cycles per kind::f16 TS MMA (M = 128, K = 16) for N and B layout.
#include <cuda_bf16.h>

#include <cstdio>

#include "sm100.cuh"

using namespace scc::sm100;

constexpr int M = 128, N = 64, K = 128;

__device__ __forceinline__ uint64_t desc_t(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t type) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(type) << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_bf16_p(uint32_t m, uint32_t n, uint32_t a_mn, uint32_t b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (a_mn << 15) | (b_mn << 16) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16_ts_p(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void __launch_bounds__(128) bf16_kernel(const float* a, const float* b, float* out, int mode, int swap,
                                                   int lbo, int sbo) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  const uint32_t warp = warp_id();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(&tbase);
  for (int i = tid; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  __syncthreads();
  for (int i = tid; i < K * N; i += 128) {
    const int k = i / N, n = i % N;
    int off;
    if (mode == 0) {
      off = (k / 8) * sbo + (k % 8) * 128 + (((n / 8) ^ (k % 8)) * 16) + (n % 8) * 2;
    } else {
      off = (k / 64) * (N / 8 * 1024) + (n / 8) * 1024 + (n % 8) * 128 + ((((k % 64) / 8) ^ (n % 8)) * 16) + (k % 8) * 2;
    }
    *reinterpret_cast<__nv_bfloat16*>(smem + off) = __float2bfloat16_rn(b[k * N + n]);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  {
    // A: lane = row m = tid, 64 columns of bf16 pairs
    const int m = tid;
    for (int c0 = 0; c0 < K / 2; c0 += 32) {
      uint32_t r[32];
      for (int c = 0; c < 32; ++c) {
        const int k = 2 * (c0 + c);
        const uint32_t lo = __bfloat16_as_ushort(__float2bfloat16_rn(a[m * K + k]));
        const uint32_t hi = __bfloat16_as_ushort(__float2bfloat16_rn(a[m * K + k + 1]));
        r[c] = swap ? (lo << 16) | hi : (hi << 16) | lo;
      }
      tmem_st32(tmem + 128 + c0 + ((warp * 32) << 16), r);
    }
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16_p(M, N, 0, mode == 0 ? 1 : 0);
      const uint32_t bb = smem_u32(smem);
      for (int ks = 0; ks < K / 16; ++ks) {
        uint64_t bd;
        if (mode == 0)
          bd = desc_t(bb + ks * 2 * sbo, lbo, sbo, 2);
        else
          bd = desc_t(bb + (ks / 4) * (N / 8 * 1024) + (ks % 4) * 32, 16, 1024, 2);
        mma_bf16_ts_p(tmem, tmem + 128 + 8 * ks, bd, idesc, ks > 0);
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((warp * 32) << 16) + c, v);
    const int r = warp * 32 + (tid & 31);
    for (int j = 0; j < 16; ++j) out[r * N + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

extern "C" int bf16_probe(const float* a, const float* b, float* out, int mode, int swap, int lbo, int sbo) {
  const int smem = 65536;
  cudaFuncSetAttribute(bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  bf16_kernel<<<1, 128, smem>>>(a, b, out, mode, swap, lbo, sbo);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "bf16_probe: %s\n", cudaGetErrorString(e));
    return -2;
  }
  return 0;
}

__global__ void __launch_bounds__(128) bf16_rate_kernel(int m, int n, int b_mn, int reps, unsigned long long* out) {
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
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16_p(static_cast<uint32_t>(m), static_cast<uint32_t>(n), 0, static_cast<uint32_t>(b_mn));
      const uint32_t b = smem_u32(smem);
      const long long t0 = clock64();
      for (int r = 0; r < reps; ++r) {
        const int k = r & 15;
        const uint64_t bd = b_mn ? desc_t(b + (k & 3) * 2048, 8192, 1024, 2) : desc_t(b + (k & 3) * 32, 16, 1024, 2);
        mma_bf16_ts_p(tmem + 256, tmem + 8 * k, bd, idesc, r > 0);
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

extern "C" int bf16_rate(int m, int n, int b_mn, int reps, int grid, unsigned long long* out_dev) {
  cudaFuncSetAttribute(bf16_rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  bf16_rate_kernel<<<grid, 128, 65536>>>(m, n, b_mn, reps, out_dev);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("bf16_rate: %s\n", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : -1;
}

// M = 64 layout probe: A rows (bf16 pairs) at TMEM lanes [lb, lb + 64), D at
// lanes [lb, lb + 64) of columns [0, 64); every lane of D's columns is first
// filled with a sentinel so the caller sees which lanes the MMA wrote.
// out[128][64]: all 128 lanes of the D columns.
__global__ void __launch_bounds__(128) m64_kernel(const float* a, const float* b, float* out, int lb) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  const uint32_t warp = warp_id();
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<256>(&tbase);
  for (int i = tid; i < 65536 / 4; i += 128) reinterpret_cast<uint32_t*>(smem)[i] = 0u;
  __syncthreads();
  // B: K-major SWIZZLE_128B, N = 64 rows, K = 128
  for (int i = tid; i < K * N; i += 128) {
    const int k = i / N, n = i % N;
    const int off = (k / 64) * (N / 8 * 1024) + (n / 8) * 1024 + (n % 8) * 128 + ((((k % 64) / 8) ^ (n % 8)) * 16) + (k % 8) * 2;
    *reinterpret_cast<__nv_bfloat16*>(smem + off) = __float2bfloat16_rn(b[k * N + n]);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  {
    // A rows: lb < 0: row r at lane (r % 16) + 32 * (r / 16) (the M = 64
    // datapath layout); else lane m holds row (m - lb) for m in [lb, lb + 64).
    // D sentinel 7777.
    const int m = tid;
    const bool m64l = lb < 0;
    const bool live = m64l ? (m & 31) < 16 : (m >= lb && m < lb + 64);
    const int row = m64l ? (m & 15) + 16 * (m >> 5) : m - lb;
    if (m64l) lb = 0;
    for (int c0 = 0; c0 < K / 2; c0 += 32) {
      uint32_t r[32];
      for (int c = 0; c < 32; ++c) {
        const int k = 2 * (c0 + c);
        const uint32_t lo = live ? __bfloat16_as_ushort(__float2bfloat16_rn(a[row * K + k])) : 0u;
        const uint32_t hi = live ? __bfloat16_as_ushort(__float2bfloat16_rn(a[row * K + k + 1])) : 0u;
        r[c] = (hi << 16) | lo;
      }
      tmem_st32(tmem + 128 + c0 + ((warp * 32) << 16), r);
    }
    uint32_t s[32];
    for (int c = 0; c < 32; ++c) s[c] = __float_as_uint(7777.f);
    tmem_st32(tmem + ((warp * 32) << 16), s);
    tmem_st32(tmem + 32 + ((warp * 32) << 16), s);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {
    if (elect_one()) {
      const uint32_t idesc = idesc_bf16_p(64, N, 0, 0);
      const uint32_t bb = smem_u32(smem);
      for (int ks = 0; ks < K / 16; ++ks) {
        const uint64_t bd = desc_t(bb + (ks / 4) * (N / 8 * 1024) + (ks % 4) * 32, 16, 1024, 2);
        mma_bf16_ts_p(tmem + (static_cast<uint32_t>(lb) << 16), tmem + 128 + 8 * ks + (static_cast<uint32_t>(lb) << 16), bd,
                      idesc, ks > 0);
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c = 0; c < N; c += 16) {
    float v[16];
    tmem_ld16(tmem + ((warp * 32) << 16) + c, v);
    const int r = warp * 32 + (tid & 31);
    for (int j = 0; j < 16; ++j) out[r * N + c + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

extern "C" int m64_probe(const float* a, const float* b, float* out, int lb) {
  cudaFuncSetAttribute(m64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  m64_kernel<<<1, 128, 65536>>>(a, b, out, lb);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    fprintf(stderr, "m64_probe: %s\n", cudaGetErrorString(e));
    return -2;
  }
  return 0;
}
