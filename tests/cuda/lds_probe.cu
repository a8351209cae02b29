// Test-only micro-benchmark: dependent-LDS latency (pointer chase) and STS
// throughput on one SM, with `busy` extra warps issuing LDS traffic and a
// configurable dynamic shared-memory footprint.
#include <cstdio>
#include <cstdint>

__global__ void __launch_bounds__(384, 1) lds_kernel(unsigned long long* out, int busy, int n, int sts_mode) {
  extern __shared__ __align__(1024) int sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = (i * 97 + 13) & 8191;
  __syncthreads();
  if (warp == 0) {
    if (sts_mode == 0) {
      int p = lane;
      const unsigned long long t0 = clock64();
      for (int i = 0; i < n; ++i) p = sm[p];
      const unsigned long long t1 = clock64();
      if (lane == 0) { out[0] = t1 - t0; out[1] = p; }
    } else {
      // STS: 32 distinct words of one 128 B line per instruction, rows r
      const unsigned long long t0 = clock64();
      for (int i = 0; i < n; ++i) {
        const int r = i & 127;
        const int off = (r >> 3) * 256 + (r & 7) * 32 + (((lane >> 2) ^ (r & 7)) << 2) + (lane & 3);
        sm[8192 + off] = i;
      }
      __syncwarp();
      const unsigned long long t1 = clock64();
      if (lane == 0) out[0] = t1 - t0;
    }
  } else if (warp <= busy) {
    int acc = 0;
    for (int i = 0; i < n; ++i) acc += sm[(lane + i * 32) & 8191];
    if (acc == 123456789) out[2] = acc;
  }
}

extern "C" int lds_probe(unsigned long long* out, int busy, int n, int sts_mode, int smem) {
  cudaFuncSetAttribute(lds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  lds_kernel<<<1, 384, smem>>>(out, busy, n, sts_mode);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -2;
}
