// Depthwise 3x3 stage of a dsc_block (model.cpp:213-220: groups = c, kernel
// 3, padding 1, stride 1 or 2), sm_100a CUDA-core kernels.  HBM-bound
// (9 MACs per output element): thread per element, taps through L1, so every
// input element is read from HBM about once.
//
//   dw_fwd_kernel   y[n,c,oy,ox] = b[c] + sum_{i,j} w[c][i][j] * x[n,c,oy*s-1+i,ox*s-1+j]
//                   (conv_forward_impl, reference.cpp:74-123; taps i, j ascending)
//   dw_bwd_data_kernel  dx[n,c,iy,ix] = sum_{i,j : (iy+1-i)%s==0, (ix+1-j)%s==0}
//                   w[c][i][j] * dy[n,c,(iy+1-i)/s,(ix+1-j)/s]
//   dw_bwd_kernel (stride 1): dx and the weight partials in one pass
//   dw_bwd_weight_kernel + dw_bwd_weight_finalize
//                   dw[c][i][j] = sum_{n,oy,ox} dy * x[...tap...], db[c] = sum dy:
//                   per (c, sample slice) partials in a fixed order, then a fixed
//                   order sum over slices (deterministic, no atomics).
#include <algorithm>

#include "scc_kernels.hpp"

namespace scc {
namespace {

constexpr int kDwThreads = 256;
constexpr int kDwMaxSlices = 32;  // sample slices of the weight gradient

// Thread per output element, straight from global memory: neighbouring
// threads read neighbouring pixels, so the 9 taps of a warp hit the same few
// L1 lines and every input element comes from HBM about once.  The stride is
// a template parameter so the tap arithmetic has no runtime division.
// Stride 1: a thread computes an R x 4 output block from an (R+2) x 6 register
// window of the input (R=2: 24 loads for 8 outputs; per element needed 72).
// The host guarantees n*c*h*w < 2^31, so index math is 32-bit (a 64-bit
// division per element cost more than the element's traffic).
// FLIP: the 3x3 taps reversed -- at stride 1 backward-data is exactly this
// kernel applied to dy (dx[iy,ix] = sum w[i][j] dy[iy+1-i, ix+1-j]).
// R = 2 pays on large planes (32x32: 27 -> 20 us); on small planes the halved
// thread count costs more than the saved loads, so R = 1 there.
template <int S, bool FLIP = false, int R = 2>
__global__ void __launch_bounds__(kDwThreads) dw_fwd_kernel(DwArgs a) {
  static_assert(S == 1, "the register-window kernel is stride 1");
  constexpr int V = 4;
  const int hi = a.h, wi = a.w, ho = a.ho, wo = a.wo;
  const int wq = (wo + V - 1) / V, hq = (ho + R - 1) / R;
  const uint32_t per = static_cast<uint32_t>(hq * wq), nc = static_cast<uint32_t>(a.c);
  const uint32_t total = static_cast<uint32_t>(a.n * a.c) * per;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const uint32_t pl = e / per;
    const int q = static_cast<int>(e - pl * per);
    const int c = static_cast<int>(pl % nc);
    const int oy0 = (q / wq) * R, ox0 = (q - (q / wq) * wq) * V;
    const float* src = a.x + static_cast<size_t>(pl) * hi * wi;
    float wk[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) wk[t] = __ldg(a.wt + c * 9 + (FLIP ? 8 - t : t));
    const float b = a.b != nullptr ? __ldg(a.b + c) : 0.f;
    float out[R][V];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int v = 0; v < V; ++v) out[r][v] = b;
#pragma unroll
    for (int yy = 0; yy < R + 2; ++yy) {
      const int iy = oy0 - 1 + yy;
      float win[V + 2];
#pragma unroll
      for (int k = 0; k < V + 2; ++k) {
        const int ix = ox0 - 1 + k;
        win[k] = (iy >= 0 && iy < hi && ix >= 0 && ix < wi) ? __ldg(src + iy * wi + ix) : 0.f;
      }
      // input row yy feeds output row r through tap row i = yy - r
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = yy - r;
        if (i < 0 || i > 2) continue;
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int j = 0; j < 3; ++j) out[r][v] = fmaf(wk[3 * i + j], win[v + j], out[r][v]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (oy0 + r >= ho) break;
      float* dst = a.y + (static_cast<size_t>(pl) * ho + oy0 + r) * wo + ox0;
#pragma unroll
      for (int v = 0; v < V; ++v)
        if (ox0 + v < wo) dst[v] = out[r][v];
    }
  }
}

// Stride 2: thread per output element (the 4-wide register window measured
// slower there: the strided window doubles its loads and the rows are short).
__global__ void __launch_bounds__(kDwThreads) dw_fwd_s2_kernel(DwArgs a) {
  const int hi = a.h, wi = a.w, ho = a.ho, wo = a.wo;
  const uint32_t plane = static_cast<uint32_t>(ho * wo), nc = static_cast<uint32_t>(a.c);
  const uint32_t total = static_cast<uint32_t>(a.n * a.c) * plane;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const uint32_t pl = e / plane;
    const int o = static_cast<int>(e - pl * plane);
    const int c = static_cast<int>(pl % nc);
    const int oy = o / wo, ox = o - oy * wo;
    const float* src = a.x + static_cast<size_t>(pl) * hi * wi;
    const float* wk = a.wt + c * 9;
    float sum = a.b != nullptr ? __ldg(a.b + c) : 0.f;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int iy = oy * 2 - 1 + i;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int ix = ox * 2 - 1 + j;
        const float v = (iy >= 0 && iy < hi && ix >= 0 && ix < wi) ? __ldg(src + iy * wi + ix) : 0.f;
        sum = fmaf(__ldg(wk + 3 * i + j), v, sum);
      }
    }
    a.y[e] = sum;
  }
}

// Thread per input element: dx[iy, ix] gathers the outputs whose taps cover
// it (oy*S - 1 + i == iy), taps i, j ascending.
template <int S>
__global__ void __launch_bounds__(kDwThreads) dw_bwd_data_kernel(DwArgs a) {
  const int hi = a.h, wi = a.w, ho = a.ho, wo = a.wo;
  const uint32_t plane = static_cast<uint32_t>(hi * wi), nc = static_cast<uint32_t>(a.c);
  const uint32_t total = static_cast<uint32_t>(a.n * a.c) * plane;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const uint32_t pl = e / plane;
    const int q = static_cast<int>(e - pl * plane);
    const int c = static_cast<int>(pl % nc);
    const int iy = q / wi, ix = q - iy * wi;
    const float* src = a.dy + static_cast<size_t>(pl) * ho * wo;
    const float* wk = a.wt + c * 9;
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int ty = iy + 1 - i;
      if (ty < 0 || ty % S != 0 || ty / S >= ho) continue;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int tx = ix + 1 - j;
        if (tx < 0 || tx % S != 0 || tx / S >= wo) continue;
        sum = fmaf(__ldg(wk + 3 * i + j), __ldg(src + (ty / S) * wo + tx / S), sum);
      }
    }
    a.dx[e] = sum;
  }
}

// Stride-2 backward-data: a thread owns a 2x2 input block (2a.., 2b..), which
// gathers from the 2x2 output window (a.., b..): input row 2a takes tap row 1
// of output row a, row 2a+1 takes tap row 0 of output row a+1 and tap row 2
// of output row a (same for columns).  4 loads for 4 outputs, no divergence
// (the per-element form branched on the parity of each lane's column).
__global__ void __launch_bounds__(kDwThreads) dw_bwd_data_s2_kernel(DwArgs a) {
  const int hi = a.h, wi = a.w, ho = a.ho, wo = a.wo;
  const int bh = (hi + 1) / 2, bw = (wi + 1) / 2;
  const uint32_t per = static_cast<uint32_t>(bh * bw), nc = static_cast<uint32_t>(a.c);
  const uint32_t total = static_cast<uint32_t>(a.n * a.c) * per;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
    const uint32_t pl = e / per;
    const int q = static_cast<int>(e - pl * per);
    const int c = static_cast<int>(pl % nc);
    const int ya = q / bw, xb = q - ya * bw;
    const float* gp = a.dy + static_cast<size_t>(pl) * ho * wo;
    float w[9];
#pragma unroll
    for (int t = 0; t < 9; ++t) w[t] = __ldg(a.wt + c * 9 + t);
    const bool y1 = ya + 1 < ho, x1 = xb + 1 < wo;
    const float g00 = __ldg(gp + ya * wo + xb);
    const float g01 = x1 ? __ldg(gp + ya * wo + xb + 1) : 0.f;
    const float g10 = y1 ? __ldg(gp + (ya + 1) * wo + xb) : 0.f;
    const float g11 = (y1 && x1) ? __ldg(gp + (ya + 1) * wo + xb + 1) : 0.f;
    // taps in ascending (i, j) order per output
    const float d00 = w[4] * g00;
    const float d01 = fmaf(w[5], g00, w[3] * g01);
    const float d10 = fmaf(w[7], g00, w[1] * g10);
    const float d11 = fmaf(w[8], g00, fmaf(w[6], g01, fmaf(w[2], g10, w[0] * g11)));
    float* dst = a.dx + static_cast<size_t>(pl) * hi * wi;
    const int iy = 2 * ya, ix = 2 * xb;
    dst[iy * wi + ix] = d00;
    if (ix + 1 < wi) dst[iy * wi + ix + 1] = d01;
    if (iy + 1 < hi) {
      dst[(iy + 1) * wi + ix] = d10;
      if (ix + 1 < wi) dst[(iy + 1) * wi + ix + 1] = d11;
    }
  }
}

// Block (c, slice): samples n = slice, slice + S, ... ascending, pixels
// strided by the block; then a fixed shuffle tree and fixed warp order.
template <int S>
__global__ void __launch_bounds__(kDwThreads) dw_bwd_weight_kernel(DwArgs a) {
  const int hi = a.h, wi = a.w, ho = a.ho, wo = a.wo;
  const int c = blockIdx.x, slice = blockIdx.y;
  float acc[10];
#pragma unroll
  for (int t = 0; t < 10; ++t) acc[t] = 0.f;
  const int cnt = static_cast<int>((a.n - slice + gridDim.y - 1) / gridDim.y);
  if (S == 1) {
    // stride 1: a thread takes 4 consecutive outputs of a row and a 3 x 6
    // register window of x (22 loads for 40 MACs instead of 40 loads)
    constexpr int V = 4;
    const int wq = (wo + V - 1) / V;
    const int per = ho * wq;
    for (int k = threadIdx.x; k < cnt * per; k += blockDim.x) {
      const int kn = k / per, r = k - kn * per;
      const int oy = r / wq, ox0 = (r - oy * wq) * V;
      const int64_t n = slice + static_cast<int64_t>(kn) * gridDim.y;
      const float* xp = a.x + (n * a.c + c) * hi * wi;
      const float* gp = a.dy + (n * a.c + c) * ho * wo + oy * wo;
      float g[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        g[v] = ox0 + v < wo ? __ldg(gp + ox0 + v) : 0.f;
        acc[9] += g[v];
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int iy = oy - 1 + i;
        float win[V + 2];
#pragma unroll
        for (int q = 0; q < V + 2; ++q) {
          const int ix = ox0 - 1 + q;
          win[q] = (iy >= 0 && iy < hi && ix >= 0 && ix < wi) ? __ldg(xp + iy * wi + ix) : 0.f;
        }
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
          for (int v = 0; v < V; ++v) acc[3 * i + j] = fmaf(g[v], win[v + j], acc[3 * i + j]);
      }
    }
  }
  // flattened (sample of the slice, pixel) index, so small planes keep every
  // thread busy; the per-thread order is fixed by the shape
  const int P = ho * wo;
  for (int k = threadIdx.x; S != 1 && k < cnt * P; k += blockDim.x) {
    const int kn = k / P, o = k - kn * P;
    const int64_t n = slice + static_cast<int64_t>(kn) * gridDim.y;
    const float* xp = a.x + (n * a.c + c) * hi * wi;
    const float* gp = a.dy + (n * a.c + c) * ho * wo;
    {
      const int oy = o / wo, ox = o - oy * wo;
      const float g = __ldg(gp + o);
      acc[9] += g;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int iy = oy * S - 1 + i;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int ix = ox * S - 1 + j;
          if (iy >= 0 && iy < hi && ix >= 0 && ix < wi) acc[3 * i + j] = fmaf(g, __ldg(xp + iy * wi + ix), acc[3 * i + j]);
        }
      }
    }
  }
  __shared__ float red[kDwThreads / 32][10];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < 10; ++t) {
    float v = acc[t];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    if (lane == 0) red[warp][t] = v;
  }
  __syncthreads();
  if (threadIdx.x < 10) {
    float v = 0.f;
    for (int w = 0; w < kDwThreads / 32; ++w) v += red[w][threadIdx.x];
    a.part[(static_cast<int64_t>(c) * gridDim.y + slice) * 10 + threadIdx.x] = v;
  }
}

// Block (c, slice) partial sums of the 10 weight-gradient taps: a fixed
// shuffle tree per warp, then warps in order.
__device__ __forceinline__ void dw_block_partials(const float (&acc)[10], const DwArgs& a, int c, int slice) {
  __shared__ float red[kDwThreads / 32][10];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int t = 0; t < 10; ++t) {
    float v = acc[t];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
    if (lane == 0) red[warp][t] = v;
  }
  __syncthreads();
  if (threadIdx.x < 10) {
    float v = 0.f;
    for (int w = 0; w < kDwThreads / 32; ++w) v += red[w][threadIdx.x];
    a.part[(static_cast<int64_t>(c) * gridDim.y + slice) * 10 + threadIdx.x] = v;
  }
}

// One pass at R = 1 with its own code: on planes under 32 rows it measured
// faster than the generic kernel's R = 1 instance (e.g. 4x4 planes 15.5 vs
// 17.6 us at 512 channels, batch 128); dx, dW and db are bitwise the two
// separate kernels'.
__global__ void __launch_bounds__(kDwThreads) dw_bwd1_kernel(DwArgs a) {
  const int hi = a.h, wi = a.w;
  const int c = blockIdx.x, slice = blockIdx.y;
  float wf[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) wf[t] = __ldg(a.wt + c * 9 + 8 - t);
  float acc[10];
#pragma unroll
  for (int t = 0; t < 10; ++t) acc[t] = 0.f;
  const int cnt = static_cast<int>((a.n - slice + gridDim.y - 1) / gridDim.y);
  constexpr int V = 4;
  const int wq = (wi + V - 1) / V;
  const int per = hi * wq;
  for (int k = threadIdx.x; k < cnt * per; k += blockDim.x) {
    const int kn = k / per, r = k - kn * per;
    const int oy = r / wq, ox0 = (r - oy * wq) * V;
    const int64_t n = slice + static_cast<int64_t>(kn) * gridDim.y;
    const int64_t pl = (n * a.c + c) * hi * wi;
    const float* xp = a.x + pl;
    const float* gp = a.dy + pl;
    float gw[3][V + 2];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int iy = oy - 1 + i;
#pragma unroll
      for (int q = 0; q < V + 2; ++q) {
        const int ix = ox0 - 1 + q;
        gw[i][q] = (iy >= 0 && iy < hi && ix >= 0 && ix < wi) ? __ldg(gp + iy * wi + ix) : 0.f;
      }
    }
    float d[V];
#pragma unroll
    for (int v = 0; v < V; ++v) d[v] = 0.f;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int v = 0; v < V; ++v)
#pragma unroll
        for (int j = 0; j < 3; ++j) d[v] = fmaf(wf[3 * i + j], gw[i][v + j], d[v]);
    float* dxp = a.dx + pl + oy * wi + ox0;
#pragma unroll
    for (int v = 0; v < V; ++v)
      if (ox0 + v < wi) dxp[v] = d[v];
#pragma unroll
    for (int v = 0; v < V; ++v) acc[9] += gw[1][v + 1];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int iy = oy - 1 + i;
      float win[V + 2];
#pragma unroll
      for (int q = 0; q < V + 2; ++q) {
        const int ix = ox0 - 1 + q;
        win[q] = (iy >= 0 && iy < hi && ix >= 0 && ix < wi) ? __ldg(xp + iy * wi + ix) : 0.f;
      }
#pragma unroll
      for (int j = 0; j < 3; ++j)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[3 * i + j] = fmaf(gw[1][v + 1], win[v + j], acc[3 * i + j]);
    }
  }
  dw_block_partials(acc, a, c, slice);
}

// The whole depthwise backward at stride 1 in one pass over dy and x
// (block (c, slice), the weight kernel's work split).  A thread takes an
// R x 4 output block: its (R + 2) x 6 dy window gives the R x 4 dx outputs
// (the flipped-tap sum of dw_fwd_kernel<1, true>, taps in the same order, so
// dx is bitwise that kernel's) and, from its centre rows, the gradient
// samples the weight taps need; the x window streams through row by row.
// Taps come through L1, whose wavefronts bound these kernels: R = 4 reads
// 4.5 values per pixel where the two separate kernels read 3 + 5.5 (planes of
// >= 32 rows: 64 ch at 32x32, batch 128, 40 vs 49 us; smaller planes use
// dw_bwd1_kernel).
template <int R>
__global__ void __launch_bounds__(kDwThreads, R > 1 ? 2 : 1) dw_bwd_kernel(DwArgs a) {
  const int hi = a.h, wi = a.w;
  const int c = blockIdx.x, slice = blockIdx.y;
  float wf[9];
#pragma unroll
  for (int t = 0; t < 9; ++t) wf[t] = __ldg(a.wt + c * 9 + 8 - t);
  float acc[10];
#pragma unroll
  for (int t = 0; t < 10; ++t) acc[t] = 0.f;
  const int cnt = static_cast<int>((a.n - slice + gridDim.y - 1) / gridDim.y);
  constexpr int V = 4;
  const int wq = (wi + V - 1) / V, hq = (hi + R - 1) / R;
  const int per = hq * wq;
  for (int k = threadIdx.x; k < cnt * per; k += blockDim.x) {
    const int kn = k / per, rr = k - kn * per;
    const int oyq = rr / wq;
    const int oy0 = oyq * R, ox0 = (rr - oyq * wq) * V;
    const int64_t n = slice + static_cast<int64_t>(kn) * gridDim.y;
    const int64_t pl = (n * a.c + c) * hi * wi;
    const float* xp = a.x + pl;
    const float* gp = a.dy + pl;
    float gw[R + 2][V + 2];
#pragma unroll
    for (int i = 0; i < R + 2; ++i) {
      const int iy = oy0 - 1 + i;
#pragma unroll
      for (int q = 0; q < V + 2; ++q) {
        const int ix = ox0 - 1 + q;
        gw[i][q] = (iy >= 0 && iy < hi && ix >= 0 && ix < wi) ? __ldg(gp + iy * wi + ix) : 0.f;
      }
    }
    // dx (the flipped-tap forward over dy)
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float d[V];
#pragma unroll
      for (int v = 0; v < V; ++v) d[v] = 0.f;
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
          for (int j = 0; j < 3; ++j) d[v] = fmaf(wf[3 * i + j], gw[r + i][v + j], d[v]);
      if (oy0 + r < hi) {
        float* dxp = a.dx + pl + (oy0 + r) * wi + ox0;
#pragma unroll
        for (int v = 0; v < V; ++v)
          if (ox0 + v < wi) dxp[v] = d[v];
      }
    }
    // dW, db: g[r][v] = dy[oy0 + r][ox0 + v] = gw[r + 1][v + 1] (zero past
    // the plane)
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int v = 0; v < V; ++v) acc[9] += gw[r + 1][v + 1];
#pragma unroll
    for (int yy = 0; yy < R + 2; ++yy) {
      const int iy = oy0 - 1 + yy;
      float win[V + 2];
#pragma unroll
      for (int q = 0; q < V + 2; ++q) {
        const int ix = ox0 - 1 + q;
        win[q] = (iy >= 0 && iy < hi && ix >= 0 && ix < wi) ? __ldg(xp + iy * wi + ix) : 0.f;
      }
      // x row yy meets output row r through tap row i = yy - r
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int i = yy - r;
        if (i < 0 || i > 2) continue;
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
          for (int v = 0; v < V; ++v) acc[3 * i + j] = fmaf(gw[r + 1][v + 1], win[v + j], acc[3 * i + j]);
      }
    }
  }
  dw_block_partials(acc, a, c, slice);
}

__global__ void dw_bwd_weight_finalize(DwArgs a, int slices) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.c * 10) return;
  const int c = i / 10, t = i - c * 10;
  float v = 0.f;
  for (int s = 0; s < slices; ++s) v += a.part[(static_cast<int64_t>(c) * slices + s) * 10 + t];
  if (t < 9) a.dw[c * 9 + t] = v;
  else if (a.db != nullptr) a.db[c] = v;
}

int dw_grid(int64_t elements) {
  return static_cast<int>(std::min<int64_t>((elements + kDwThreads - 1) / kDwThreads, 148 * 16));
}

}  // namespace

size_t dw_workspace_bytes(int64_t c) { return static_cast<size_t>(c) * kDwMaxSlices * 10 * sizeof(float); }

cudaError_t launch_dw(DwArgs a, int op, cudaStream_t s) {
  const int64_t planes = a.n * a.c;
  if (planes <= 0) return cudaSuccess;
  const bool s2 = a.stride == 2;
  if (op == 0) {
    if (s2) dw_fwd_s2_kernel<<<dw_grid(planes * a.ho * a.wo), kDwThreads, 0, s>>>(a);
    else if (a.ho * a.wo >= 1024)
      dw_fwd_kernel<1, false, 2><<<dw_grid(planes * ((a.ho + 1) / 2) * ((a.wo + 3) / 4)), kDwThreads, 0, s>>>(a);
    else
      dw_fwd_kernel<1, false, 1><<<dw_grid(planes * a.ho * ((a.wo + 3) / 4)), kDwThreads, 0, s>>>(a);
    note_launches(1);
  } else if (op == 1) {
    if (s2) {
      dw_bwd_data_s2_kernel<<<dw_grid(planes * ((a.h + 1) / 2) * ((a.w + 1) / 2)), kDwThreads, 0, s>>>(a);
    } else {
      DwArgs f = a;  // stride 1: the flipped-tap forward over dy
      f.x = a.dy;
      f.y = a.dx;
      f.b = nullptr;
      if (a.ho * a.wo >= 1024)
        dw_fwd_kernel<1, true, 2><<<dw_grid(planes * ((a.ho + 1) / 2) * ((a.wo + 3) / 4)), kDwThreads, 0, s>>>(f);
      else
        dw_fwd_kernel<1, true, 1><<<dw_grid(planes * a.ho * ((a.wo + 3) / 4)), kDwThreads, 0, s>>>(f);
    }
    note_launches(1);
  } else if (op == 3 && s2) {
    // stride 2: backward-data then backward-weight
    cudaError_t e = launch_dw(a, 1, s);
    if (e != cudaSuccess) return e;
    return launch_dw(a, 2, s);
  } else {
    // enough (channel, slice) blocks to fill the chip; the slice count depends
    // only on the shape, so the summation order is fixed per shape
    const int64_t want = (148 * 8 + a.c - 1) / a.c;
    const int slices = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>({want, a.n, kDwMaxSlices})));
    dim3 grid(static_cast<unsigned>(a.c), static_cast<unsigned>(slices));
    if (op == 3 && a.h >= 32) dw_bwd_kernel<4><<<grid, kDwThreads, 0, s>>>(a);
    else if (op == 3) dw_bwd1_kernel<<<grid, kDwThreads, 0, s>>>(a);
    else if (s2) dw_bwd_weight_kernel<2><<<grid, kDwThreads, 0, s>>>(a);
    else dw_bwd_weight_kernel<1><<<grid, kDwThreads, 0, s>>>(a);
    const int fb = static_cast<int>((a.c * 10 + 255) / 256);
    dw_bwd_weight_finalize<<<fb, 256, 0, s>>>(a, slices);
    note_launches(2);
  }
  return cudaGetLastError();
}

}  // namespace scc
