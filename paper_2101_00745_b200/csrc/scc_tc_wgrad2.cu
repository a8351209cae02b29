// Tensor-core backward-weight, generation 2 (tcgen05, 3xTF32), sm_100a
// (replaces scc_backward_params, kernel.cpp:140-181):
//
//   dWband[oc, ic] = sum_{n,p} dy[n, oc, p] * x[n, ic, p]     (ic in the arc of oc's row tile)
//   db[oc]         = sum_{n,p} dy[n, oc, p]                    (a ones row appended to x)
//
// GEMM per row tile of 128 cycle-sorted filters: M = 128 filters (TMEM lanes),
// N = the tile's input-channel arc plus one ones row (db) rounded to 16,
// K = pixels, one 32-pixel block per pipeline stage.  Both operands are
// pixel-contiguous (K-major) and land by TMA in the SWIZZLE_128B layout:
//   * dy [128 rows][32 px]: row-converter warps (thread = filter row) split it
//     into tf32 hi/lo and store it to TMEM ([filter lane][pixel column]), so
//     the MMAs run in TS mode and only x is read from shared memory;
//   * x [arc rows][32 px] plus a converted lo copy (SS operand B); the ones row
//     and zero padding rows are written once and never overwritten by TMA.
// 3xTF32 per k-step: dy_hi*x + dy_lo*x + dy_hi*x_lo (x raw = x_hi: the tensor
// core truncates).
//
// The pixel blocks are cut into a fixed number of contiguous slices (not tied
// to the grid size); each slice accumulates in TMEM (two accumulators, so one
// slice's epilogue overlaps the next slice's MMAs) and the epilogue writes the
// slice's window-relative partial dW / db to the workspace.  A second, PDL-
// chained kernel sums the partials in a fixed order.  No atomics on the data:
// the bits of dW do not depend on how many CTAs run.

// Warp roles (384 threads, one CTA per SM):
//   warp 0      TMA producer
//   warp 1      TMEM allocator + MMA issuer
//   warps 2-3   x lo converters (+ the constant ones / zero rows)
//   warps 4-7   dy row converters (warp q: filter rows 32q..32q+31)
//   warps 8-11  epilogue (TMEM -> smem row dump -> window-relative partial)
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "scc_kernels.hpp"
#include "scc_plan.hpp"
#include "sm100.cuh"
#include "tmap.hpp"

namespace scc {
namespace {

using namespace sm100;

__device__ unsigned long long g_w2trace[64];
__device__ unsigned long long g_w2cta[3 * 256];  // per CTA: start, accfull, barrier arrival
#if defined(SCC_TRACE)
#define W2T(slot)                                              \
  do {                                                         \
    if (blockIdx.x == 0) g_w2trace[(slot)] = globaltimer();    \
  } while (0)
#define W2CTA(k)                                                            \
  do {                                                                      \
    if (blockIdx.x < 256) g_w2cta[3 * blockIdx.x + (k)] = globaltimer();    \
  } while (0)
#else
#define W2T(slot) \
  do {            \
  } while (0)
#define W2CTA(k) \
  do {           \
  } while (0)
#endif

constexpr int kThreads = 384;
constexpr int kDyBytes = 128 * 128;   // [128 rows][32 px]
constexpr int kMaxStages = 6;
constexpr int kTStages = 4;           // TMEM A stages (hi + lo, 64 columns each)
constexpr int kACol0 = 256;           // TMEM: two 128-column accumulators, then A stages
constexpr int kSlices = 74;           // pixel slices (partials) of a launch: one per CTA of
                                      // the concurrent backward (half of a B200's 148 SMs);
                                      // the reduce kernel sums at most 8 x 10 slices
constexpr int kMaxRt = 16;
constexpr int kMaxCls = 64;
constexpr int kSmemLimit = 227 * 1024;
constexpr int kMaxGw = 32;            // window slots per filter handled in registers

struct W2Args {
  float* part;               // [grid][c_out*gw + c_out] partial dW | db
  float* dweight;            // [c_out*gw]
  float* dbias;              // [c_out] or nullptr
  const int32_t* perm;       // sorted position -> oc
  const int32_t* starts;     // oc -> window start
  int32_t rt_start8[kMaxRt]; // per row tile: first arc ring position (input channel)
  int32_t class_d[kMaxCls];
  int32_t n_rt, c_in, c_out, gw, cls;
  int32_t nx;                // arc rows loaded per tile (max over tiles, 8-aligned)
  int32_t xr;                // x stage rows (nx + ones row, rounded to 16) = MMA N
  int32_t rba, rbb;          // TMA box rows (dy, x)
  int32_t dybox;             // 1: one dy box {32 px, cls, D} per block, row i = d*cls + j (oc = d + D*j)
  int32_t xbox;              // 1: one x box {32 px, nx rows} per block (arc does not wrap)
  int32_t n_class;
  int32_t stages;
  int32_t nbps;              // 32-pixel blocks per sample
  int32_t units;             // n * nbps
  int32_t elems;             // per-slice partial floats: n_rt * (128*gw + 128)
  int32_t slices;            // pixel slices (partials), fixed per launch geometry
};

// Filter of tile row `pos` (row tile * 128 + row): cycle-sorted order, or the
// class-major order of the single dy box.
__device__ __forceinline__ int row_oc(const W2Args& a, int pos) {
  if (a.dybox) {
    const int d = pos / a.cls;
    return d + a.n_class * (pos - d * a.cls);
  }
  return __ldg(a.perm + pos);
}

// Pixel slices: a fixed number of contiguous block ranges (independent of the
// grid size), each accumulated in its own TMEM pass and written as its own
// partial, so the reduction order -- and the bits of dW -- do not depend on
// how many CTAs run.
__device__ __forceinline__ int slice_u(const W2Args& a, int k) {
  return static_cast<int>((static_cast<int64_t>(k) * a.units) / a.slices);
}
__device__ __forceinline__ void advance(int& stage, uint32_t& phase, int stages) {
  if (++stage == stages) {
    stage = 0;
    phase ^= 1u;
  }
}

struct WLayout {
  int stage, ring, xoff, xlo, stg, bars, total;
  __host__ __device__ WLayout(int xr, int stages) {
    const int xb = xr * 128;
    stage = kDyBytes + 2 * xb;   // dy | x | x_lo
    xoff = kDyBytes;
    xlo = kDyBytes + xb;
    ring = 0;
    stg = stages * stage;        // epilogue row dump: [128][xr + 4] floats
    bars = stg + ((128 * (xr + 4) * 4 + 1023) & ~1023);
    total = bars + (3 * kMaxStages + 2 * kTStages + 6) * 8 + 16;
  }
};

__global__ void __launch_bounds__(kThreads, 1)
    tc_wgrad2_kernel(const __grid_constant__ CUtensorMap tdy, const __grid_constant__ CUtensorMap tx,
                     const __grid_constant__ W2Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const WLayout L(a.xr, a.stages);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* full = bars;                       // TMA landed (dy + x)
  uint64_t* sfree = full + kMaxStages;         // 4 row converters + MMA commit
  uint64_t* xlo = sfree + kMaxStages;          // 2 lo-converter warps
  uint64_t* conv = xlo + kMaxStages;           // 4 row converters
  uint64_t* tfree = conv + kTStages;           // MMA commit
  uint64_t* accfull = tfree + kTStages;        // [2] MMA final commit of a (slice, row tile)
  uint64_t* accempty = accfull + 2;            // [2] 4 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + 2);
  float* stg = reinterpret_cast<float*>(smem + L.stg);

  const uint32_t warp = warp_id();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    W2T(0);
    W2CTA(0);
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sfree[s], 5);
      mbar_init(&xlo[s], 2);
    }
    for (int s = 0; s < kTStages; ++s) {
      mbar_init(&conv[s], 4);
      mbar_init(&tfree[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accfull[i], 1);
      mbar_init(&accempty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tdy);
    prefetch_tmap(&tx);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  cudaGridDependencySynchronize();
  // the dependent reduce kernel may launch now (it waits for this grid)
  cudaTriggerProgrammaticLaunchCompletion();
  if (threadIdx.x == 0) W2T(1);

  if (warp == 0) {
    // ---------------- producer ----------------
    if (elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      const uint32_t bytes = (a.dybox ? a.c_out * 128 : kDyBytes) + a.nx * 128;
      for (int sl = blockIdx.x; sl < a.slices; sl += gridDim.x) {
        const int u0 = slice_u(a, sl), u1 = slice_u(a, sl + 1);
        for (int rt = 0; rt < a.n_rt; ++rt) {
          const int start8 = a.rt_start8[rt];
          for (int u = u0; u < u1; ++u) {
            if (u == u0) W2T(40);
            const int n = u / a.nbps, px0 = (u - n * a.nbps) * 32;
            mbar_wait(&sfree[s], ph ^ 1u);
            if (u == u0) W2T(41);
            mbar_expect_tx(&full[s], bytes);
            if (u == u0) W2T(42);
            uint8_t* st = smem + s * L.stage;
            if (a.dybox) {
              tma_load_4d(st, &tdy, &full[s], px0, 0, 0, n);
            } else
            for (int r = 0; r < 128; r += a.rba) {
              // sorted filter position rt*128 + r -> (class, j); positions past
              // c_out read the next rows (zero-filled past the tensor) and feed
              // accumulator rows the epilogue ignores
              int pos = rt * 128 + r;
              pos = pos < a.c_out ? pos : a.c_out - a.rba;
              const int cl = pos / a.cls, j = pos - cl * a.cls;
              tma_load_4d(st + r * 128, &tdy, &full[s], px0, j, a.class_d[cl], n);
              if (u == u0 && r == 0) W2T(43);
            }
            if (u == u0) W2T(44);
            if (a.xbox) {
              tma_load_3d(st + L.xoff, &tx, &full[s], px0, start8, n);
            } else
            for (int r = 0; r < a.nx; r += a.rbb) {
              int ic = start8 + r;
              ic -= ic >= a.c_in ? a.c_in : 0;
              tma_load_3d(st + L.xoff + r * 128, &tx, &full[s], px0, ic, n);
            }
            if (u - u0 < 8) W2T(2 + u - u0);
            advance(s, ph, a.stages);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = idesc_tf32(128, static_cast<uint32_t>(a.xr), 0, 0);
    int s = 0, st = 0, acc = 0;
    uint32_t ph = 0, tph = 0, aph = 0;
    for (int sl = blockIdx.x; sl < a.slices; sl += gridDim.x) {
      const int u0 = slice_u(a, sl), u1 = slice_u(a, sl + 1);
      for (int rt = 0; rt < a.n_rt; ++rt) {
        mbar_wait(&accempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t dacc = tmem + acc * 128;
        bool first = true;
        for (int u = u0; u < u1; ++u) {
          mbar_wait(&xlo[s], ph);
          mbar_wait(&conv[st], tph);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t bx = smem_u32(smem + s * L.stage + L.xoff);
            const uint32_t bl = smem_u32(smem + s * L.stage + L.xlo);
            const uint32_t ah = tmem + kACol0 + st * 64, al = ah + 32;
            for (int k = 0; k < 4; ++k) {
              const uint64_t dbx = desc_sw128(bx + k * 32, 16, 1024);
              const uint64_t dbl = desc_sw128(bl + k * 32, 16, 1024);
              mma_tf32_ts(dacc, ah + 8 * k, dbx, idesc, (first && k == 0) ? 0u : 1u);
              mma_tf32_ts(dacc, al + 8 * k, dbx, idesc, 1);
              mma_tf32_ts(dacc, ah + 8 * k, dbl, idesc, 1);
            }
            mma_commit(&tfree[st]);
            mma_commit(&sfree[s]);
            if (u - u0 < 8) W2T(10 + u - u0);
          }
          __syncwarp();
          first = false;
          advance(s, ph, a.stages);
          advance(st, tph, kTStages);
        }
        // (an empty slice accumulates nothing; the epilogue writes zeros)
        if (elect_one()) mma_commit(&accfull[acc]);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          aph ^= 1u;
        }
      }
    }
  } else if (warp < 4) {
    // ---------------- x lo converters ----------------
    const int ct = threadIdx.x - 64;  // 0..63
    // constant rows [nx, xr): row nx = 1 (x) / 0 (x_lo), the rest 0
    for (int s = 0; s < a.stages; ++s) {
      float* xs = reinterpret_cast<float*>(smem + s * L.stage + L.xoff);
      float* xl = reinterpret_cast<float*>(smem + s * L.stage + L.xlo);
      for (int i = ct; i < (a.xr - a.nx) * 32; i += 64) {
        const int r = a.nx + (i >> 5), c = i & 31;
        // SWIZZLE_128B: 16 B chunk c/4 of row r sits at chunk (c/4) ^ (r%8)
        const int off = r * 32 + ((((c >> 2) ^ (r & 7)) << 2) | (c & 3));
        xs[off] = r == a.nx ? 1.f : 0.f;
        xl[off] = 0.f;
      }
    }
    fence_proxy_async_smem();
    int s = 0;
    uint32_t ph = 0;
    const int words = a.nx * 8;  // float4 per x stage
    for (int sl = blockIdx.x; sl < a.slices; sl += gridDim.x) {
      const int u0 = slice_u(a, sl), u1 = slice_u(a, sl + 1);
      for (int rt = 0; rt < a.n_rt; ++rt) {
        for (int u = u0; u < u1; ++u) {
          mbar_wait(&full[s], ph);
          const float4* src = reinterpret_cast<const float4*>(smem + s * L.stage + L.xoff);
          const uint32_t dst = smem_u32(smem + s * L.stage + L.xlo);
          for (int i0 = ct; i0 < words; i0 += 64 * 4) {
            float4 v[4];
  #pragma unroll
            for (int b = 0; b < 4; ++b) v[b] = src[min(i0 + 64 * b, words - 1)];
  #pragma unroll
            for (int b = 0; b < 4; ++b) {
              if (i0 + 64 * b < words) {
                float4 o;
                o.x = v[b].x - tf32_hi(v[b].x);
                o.y = v[b].y - tf32_hi(v[b].y);
                o.z = v[b].z - tf32_hi(v[b].z);
                o.w = v[b].w - tf32_hi(v[b].w);
                sts_v4(dst + (i0 + 64 * b) * 16, o);
              }
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&xlo[s]);
          advance(s, ph, a.stages);
        }
      }
    }
  } else if (warp < 8) {
    // ---------------- dy row converters: smem [row][32 px] -> TMEM [row lane][px] hi / lo ----------------
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    int s = 0, st = 0;
    uint32_t ph = 0, tph = 0;
    for (int sl = blockIdx.x; sl < a.slices; sl += gridDim.x) {
      const int u0 = slice_u(a, sl), u1 = slice_u(a, sl + 1);
      for (int rt = 0; rt < a.n_rt; ++rt) {
        for (int u = u0; u < u1; ++u) {
          mbar_wait(&full[s], ph);
          if (row == 0 && u - u0 < 8) W2T(18 + u - u0);
          const float4* rp = reinterpret_cast<const float4*>(smem + s * L.stage + row * 128);
          uint32_t hi[32], lo[32];
  #pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 v = rp[j ^ (row & 7)];  // SWIZZLE_128B: logical chunk j
            const float e[4] = {v.x, v.y, v.z, v.w};
  #pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float h = tf32_hi(e[t]);
              hi[4 * j + t] = __float_as_uint(h);
              lo[4 * j + t] = __float_as_uint(e[t] - h);
            }
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&sfree[s]);
          mbar_wait(&tfree[st], tph ^ 1u);
          tc_fence_after();
          const uint32_t col = tmem + kACol0 + st * 64 + lane_base;
          tmem_st32(col, hi);
          tmem_st32(col + 32, lo);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv[st]);
          if (row == 0 && u - u0 < 8) W2T(26 + u - u0);
          advance(s, ph, a.stages);
          advance(st, tph, kTStages);
        }
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> window-relative partial ----------------
    const int q = warp & 3;
    const int i = q * 32 + lane;  // tile row
    const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const int rstride = a.xr + 4;  // dump row stride (floats): 16 B rows, conflict-free STS.128
    float* prow = stg + i * rstride;
    const uint32_t prow_a = smem_u32(prow);
    uint32_t aph = 0;
    int acc = 0;
    for (int sl = blockIdx.x; sl < a.slices; sl += gridDim.x) {
      const int u0 = slice_u(a, sl), u1 = slice_u(a, sl + 1);
      for (int rt = 0; rt < a.n_rt; ++rt) {
        mbar_wait(&accfull[acc], aph);
        tc_fence_after();
        if (i == 0) {
          W2T(34);
          W2CTA(1);
        }
        // own TMEM row (lane = tile row) -> own smem dump row
        for (int c0 = 0; c0 < a.xr; c0 += 32) {
          uint32_t v[32];
          tmem_ld32_nowait(taddr + acc * 128 + c0, v);
          tmem_ld_wait();
  #pragma unroll
          for (int t = 0; t < 32; t += 4)
            if (c0 + t < a.xr)
              sts_v4(prow_a + (c0 + t) * 4, make_float4(__uint_as_float(v[t]), __uint_as_float(v[t + 1]),
                                                        __uint_as_float(v[t + 2]), __uint_as_float(v[t + 3])));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&accempty[acc]);
        if (++acc == 2) {
          acc = 0;
          aph ^= 1u;
        }
        // window-relative values of this row, written straight to the CTA's
        // partial tile [128 rows][gw] | db[128] (each thread a contiguous row)
        const int pos = rt * 128 + i;
        const bool live = pos < a.c_out && u0 < u1;
        int j0 = 0;
        if (live) {
          j0 = __ldg(a.starts + row_oc(a, pos)) - a.rt_start8[rt];
          j0 += j0 < 0 ? a.c_in : 0;
        }
        float* dst = a.part + static_cast<int64_t>(sl) * a.elems +
                     static_cast<int64_t>(rt) * (128 * a.gw + 128);
        float wv[kMaxGw];
  #pragma unroll
        for (int sl = 0; sl < kMaxGw; ++sl) {
          int j = j0 + sl;
          j -= j >= a.c_in ? a.c_in : 0;
          wv[sl] = (live && sl < a.gw) ? prow[j] : 0.f;
        }
        if ((a.gw & 3) == 0) {
  #pragma unroll
          for (int sl = 0; sl < kMaxGw; sl += 4)
            if (sl < a.gw)
              *reinterpret_cast<float4*>(dst + i * a.gw + sl) = make_float4(wv[sl], wv[sl + 1], wv[sl + 2], wv[sl + 3]);
        } else {
  #pragma unroll
          for (int sl = 0; sl < kMaxGw; ++sl)
            if (sl < a.gw) dst[i * a.gw + sl] = wv[sl];
        }
        dst[128 * a.gw + i] = live ? prow[a.nx] : 0.f;
      }
    }
  }

  if (threadIdx.x == 0) W2CTA(2);
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// Fixed-order reduction of the per-slice partials (the kernel boundary with
// tc_wgrad2_kernel is the grid-wide sync; launched with programmatic stream
// serialization its CTAs are resident -- next to the big CTAs, it needs no
// shared memory -- and start the moment the partials are complete).
// 8 lanes per output: lane g sums slices g, g+8, ... in order, then a fixed
// shuffle tree combines the 8 group sums.  Bitwise reproducible.
__global__ void __launch_bounds__(256) tc_wgrad2_reduce(const __grid_constant__ W2Args a) {
  cudaGridDependencySynchronize();
  const int gtid = blockIdx.x * 256 + threadIdx.x;
  const int e = gtid >> 3, g = gtid & 7;
  float acc = 0.f;
  if (e < a.elems) {
    float v[10];
#pragma unroll
    for (int m = 0; m < 10; ++m) {
      const int k = g + 8 * m;
      v[m] = k < a.slices ? __ldcg(a.part + static_cast<int64_t>(k) * a.elems + e) : 0.f;
    }
#pragma unroll
    for (int m = 0; m < 10; ++m) acc += v[m];
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  if (g == 0 && e < a.elems) {
    const int tstride = 128 * a.gw + 128;  // one row tile's partial
    const int rt = e / tstride, rem = e - rt * tstride;
    const bool isb = rem >= 128 * a.gw;
    const int i = isb ? rem - 128 * a.gw : rem / a.gw;
    const int pos = rt * 128 + i;
    if (pos < a.c_out) {
      const int oc = row_oc(a, pos);
      if (!isb)
        a.dweight[static_cast<int64_t>(oc) * a.gw + (rem - i * a.gw)] = acc;
      else if (a.dbias != nullptr)
        a.dbias[oc] = acc;
    }
  }
}

int w2_stages(int xr) {
  int st = kMaxStages;
  while (st >= 2 && 1024 + WLayout(xr, st).total > kSmemLimit) --st;
  return st;
}

}  // namespace

// Supported when the tile's arc plus the ones row fits one MMA (N <= 128, so
// the accumulator and four TMEM A stages fit 512 columns) and the small tables
// fit the kernel parameters.
bool tc_wgrad2_supported(const TcWeightPlan& tw, int64_t n, int64_t plane, int32_t gw) {
  if (!tw.ok || plane % 4 != 0 || tw.n_rt > kMaxRt || tw.n_class > kMaxCls) return false;
  // Accumulation chain of a slice's TMEM accumulator (4 K = 8 steps per
  // 32-pixel block): each MMA rounds the running sum toward zero, a bias
  // linear in the chain (~6e-8 of max|dW| per step, scc_tc_wgrad.cu); larger
  // problems take the generation-1 kernel, which adds splits instead.
  if ((n * ((plane + 31) / 32) + kSlices - 1) / kSlices * 4 > 768) return false;
  int nx = 0;
  for (int rt = 0; rt < tw.n_rt; ++rt) nx = std::max(nx, tw.rt_info[2 * rt + 1]);
  const int xr = (nx + 1 + 15) / 16 * 16;
  if (xr > 128 || tw.rba < 8 || 32 % tw.rba != 0) return false;
  if (gw > kMaxGw || nx % tw.rbb != 0) return false;
  return w2_stages(xr) >= 3;
}

int tc_w2trace(unsigned long long* out, int n) {
  if (n > 64 + 3 * 256) n = 64 + 3 * 256;
  const int m = n < 64 ? n : 64;
  if (cudaMemcpyFromSymbol(out, g_w2trace, m * sizeof(unsigned long long)) != cudaSuccess) return -1;
  if (n > 64 && cudaMemcpyFromSymbol(out + 64, g_w2cta, (n - 64) * sizeof(unsigned long long)) != cudaSuccess)
    return -1;
  return n;
}

size_t tc_wgrad2_workspace_bytes(int32_t c_out, int32_t gw, int slices) {
  const size_t n_rt = (c_out + 127) / 128;
  return static_cast<size_t>(slices) * n_rt * (128 * static_cast<size_t>(gw) + 128) * sizeof(float);
}

cudaError_t launch_wgrad2(const TcWeightPlan& tw, const TcWeightCall& call, const int32_t* perm,
                          cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  static int nsm_cache[64] = {0};
  static bool attr_set[64] = {false};
  int nsm = 148;
  if (dev >= 0 && dev < 64 && nsm_cache[dev] > 0) {
    nsm = nsm_cache[dev];
  } else {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < 64) nsm_cache[dev] = nsm;
  }
  W2Args a{};
  int nx = 0;
  for (int rt = 0; rt < tw.n_rt; ++rt) {
    a.rt_start8[rt] = tw.rt_info[2 * rt];
    nx = std::max(nx, tw.rt_info[2 * rt + 1]);
  }
  for (size_t i = 0; i < tw.class_d.size(); ++i) a.class_d[i] = tw.class_d[i];
  a.n_rt = tw.n_rt;
  a.c_in = call.c_in;
  a.c_out = call.c_out;
  a.gw = call.gw;
  a.cls = tw.cls;
  a.nx = nx;
  a.xr = (nx + 1 + 15) / 16 * 16;
  a.rba = tw.rba;
  a.rbb = tw.rbb;
  a.n_class = tw.n_class;
  a.dybox = (tw.n_rt == 1 && call.c_out == tw.n_class * tw.cls && call.c_out <= 128 && tw.cls <= 256 &&
             tw.n_class <= 256) ? 1 : 0;
  a.xbox = 1;
  for (int rt = 0; rt < tw.n_rt; ++rt)
    if (tw.rt_info[2 * rt] + nx > call.c_in || nx > 256) a.xbox = 0;
  a.stages = w2_stages(a.xr);
  a.nbps = static_cast<int32_t>((call.plane + 31) / 32);
  const int64_t units = call.n * a.nbps;
  if (units > (1ll << 30)) return cudaErrorInvalidValue;
  a.units = static_cast<int32_t>(units);
  a.elems = tw.n_rt * (128 * call.gw + 128);
  a.slices = static_cast<int32_t>(std::min<int64_t>(units, kSlices));
  const int cap = call.max_ctas > 0 ? std::min(call.max_ctas, nsm) : nsm;
  const int grid = std::min(a.slices, cap);
  if (tc_wgrad2_workspace_bytes(call.c_out, call.gw, a.slices) > call.workspace_bytes) return cudaErrorInvalidValue;
  a.part = static_cast<float*>(call.workspace);
  a.dweight = call.dweight;
  a.dbias = call.dbias;
  a.perm = perm;
  a.starts = call.starts;

  const uint64_t P = static_cast<uint64_t>(call.plane);
  CUtensorMap tdy, tx;
  {
    // dy {P, cls, D, N} (row (d, j) = filter d + D*j), box {32 px, rba rows}
    const uint64_t dims[4] = {P, static_cast<uint64_t>(tw.cls), static_cast<uint64_t>(tw.n_class),
                              static_cast<uint64_t>(call.n)};
    const uint64_t strides[3] = {P * 4 * tw.n_class, P * 4, P * 4 * call.c_out};
    const uint32_t box[4] = {32, static_cast<uint32_t>(a.dybox ? tw.cls : tw.rba),
                             static_cast<uint32_t>(a.dybox ? tw.n_class : 1), 1};
    if (!encode_f32(&tdy, call.dy, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[3] = {P, static_cast<uint64_t>(call.c_in), static_cast<uint64_t>(call.n)};
    const uint64_t strides[2] = {P * 4, P * 4 * call.c_in};
    const uint32_t box[3] = {32, static_cast<uint32_t>(a.xbox ? nx : tw.rbb), 1};
    if (!encode_f32(&tx, call.x, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(tc_wgrad2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemLimit);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 1024 + WLayout(a.xr, a.stages).total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_wgrad2_kernel, tdy, tx, a);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t rc{};
  rc.gridDim = dim3(static_cast<unsigned>((a.elems * 8 + 255) / 256));
  rc.blockDim = dim3(256);
  rc.stream = s;
  rc.attrs = attr;
  rc.numAttrs = 1;
  e = cudaLaunchKernelEx(&rc, tc_wgrad2_reduce, a);
  if (e != cudaSuccess) return e;
  note_launches(2);
  return cudaSuccess;
}

}  // namespace scc
