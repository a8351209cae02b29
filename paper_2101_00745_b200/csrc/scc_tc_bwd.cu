// Fused tensor-core backward (tcgen05, 3xTF32), sm_100a: backward-data and
// backward-weight of one SCC layer from a single pass over dy
// (replaces scc_backward_input + scc_backward_params, kernel.cpp:100-189):
//
//   dx[n, ic, p]  = sum_oc  W^T[ic, oc] * dy[n, oc, p]          (W^T: window-relative W scattered)
//   dW[oc, ic]    = sum_{n,p} dy[n, oc, p] * x[n, ic, p]        (ic in the arc of the filters)
//   db[oc]        = sum_{n,p} dy[n, oc, p]                      (a ones row appended to x)
//
// Geometry: one row tile of filters (c_out <= 128, in the class-major order
// of a single {32 px, cls, D} dy box) and c_in <= 64 input channels.  The
// pipeline moves PAIRS of 32-pixel blocks (any two consecutive blocks of the
// CTA's pixel slice):
//   * dy [c_out rows][32 px] of each block lands by TMA in the
//     SWIZZLE_128B_BASE32B layout, which is at once an MN-major B operand of
//     the dx GEMM (D[ic][px] = W^T[ic][oc] * dy[oc][px], K = oc; the pair's two
//     blocks are the two 32-px atoms of an N = 64 operand) and row-readable by
//     the converter warps, which write its tf32 lo part to the lo buffers (dx
//     B lo) and its hi / lo rows to TMEM (A of the dW GEMM, lanes = filters);
//   * x [arc rows][32 px] (SWIZZLE_128B, K-major) plus a converted lo copy is
//     B of the dW GEMM (D[oc][ic] = dy[oc][px] * x[ic][px], K = px).
// W^T stays resident in TMEM, stacked: lanes 0-63 hold W_hi, lanes 64-127
// W_lo, so one M = 128 MMA yields W_hi*B and W_lo*B in the two lane halves
// (the epilogue adds them); 3xTF32 for dx is then two MMAs per k-step
// ([W_hi; W_lo] * dy and [W_hi; W_lo] * dy_lo, the lo*lo term included for
// free).  Every GEMM runs in TS mode (A from TMEM); shared memory only feeds
// B operands.  Per pair the MMAs that read the lo buffers go first, so the
// converters refill them while the rest of the pair's MMAs run.
//
// dW accumulates over the CTA's pixel slice in TMEM and is written as that
// slice's window-relative partial (db: the dy converters sum their rows on
// the CUDA cores, so the dW GEMM's N is exactly the x arc); a PDL-chained
// kernel sums the slice partials in a fixed order (the slice count is fixed
// per geometry, so the bits of dW do not depend on the grid).  dx is drained from TMEM per pair; the W_lo half of the stacked
// accumulator is exchanged through shared memory and the W_hi half adds it
// and stores straight to global.  The same kernel, with either GEMM switched
// off, serves scc_backward_input / scc_backward_params alone, so the fused
// and separate entry points agree bit for bit.
//
// Warp roles (384 threads, one CTA per SM, one slice per CTA):
//   warp 0      TMA producer
//   warp 1      TMEM allocator + MMA issuer
//   warps 2-3   x lo converters (+ the constant ones / zero rows)
//   warps 4-7   dy row converters (warp q: filter rows 32q..32q+31)
//   warps 8-11  W^T build (prologue), dx epilogue, dW slice epilogue
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

// Diagnostic timeline (build with -DSCC_TRACE): CTA-0 %globaltimer slots and
// per-CTA start / end stamps; scripts/bwd_timing.py reads them.
#if defined(SCC_TRACE)
__device__ unsigned long long g_trace3[64];
__device__ unsigned long long g_cta3[2 * 256];
#define TRACE3(slot)                                         \
  do {                                                       \
    if (blockIdx.x == 0) g_trace3[(slot)] = globaltimer();   \
  } while (0)
#define TRACE3K(base, k)                   \
  do {                                     \
    if ((k) < 8) TRACE3((base) + (k));     \
  } while (0)
#else
#define TRACE3(slot) \
  do {               \
  } while (0)
#define TRACE3K(base, k) \
  do {                   \
  } while (0)
#endif

constexpr int kThreads = 384;
constexpr int kSlots = 3;             // raw TMA pair slots (dy | x per block); x_lo is written in place
constexpr int kStages = 2;            // dy_lo pairs and TMEM dW A stages
constexpr int kSlices = 148;          // pixel slices (dW partials) per launch = CTAs (one per SM)
constexpr int kSmemLimit = 227 * 1024;
constexpr int kMaxGw = 32;
constexpr int kMaxXr = 64;            // dW accumulator columns
// TMEM columns (512 allocated)
constexpr uint32_t kWt = 0;          // W^T: [ic lane (hi) | 64 + ic lane (lo)][oc column]
constexpr uint32_t kDwAcc = 128;     // dW accumulator: [filter lane][x row column] (xr <= 64)
constexpr uint32_t kDxAcc = 192;     // dx accumulator: [ic lane (+64: lo part)][64 px]
constexpr uint32_t kDwA = 256;       // per stage: dy hi | lo of the pair's two blocks [filter lane][px]

struct BArgs {
  float* part;               // [slices][c_out*gw + c_out] partial dW | db (c_out <= 128)
  float* dweight;            // [c_out*gw]
  float* dx;                 // [n][c_in][plane]
  int32_t plane;
  float* dbias;              // [c_out] or nullptr
  const float* weight;       // [c_out*gw]
  const int32_t* starts;     // oc -> window start
  int32_t c_in, c_out, gw, cls, n_class;
  int32_t start8;            // first x row (input channel) of the filters' arc
  int32_t nx;                // x rows loaded (8-aligned arc)
  int32_t xr;                // x stage rows (nx rounded to 16) = dW MMA N
  int32_t rbb;               // x TMA box rows when the arc wraps
  int32_t xbox;              // 1: one x box {32 px, nx rows}
  int32_t nbps;              // 32-pixel blocks per sample
  int32_t units;             // n * nbps
  int32_t elems;             // per-slice partial floats: c_out*gw + c_out
  int32_t slices;
  int32_t do_dx, do_dw;
  int32_t w_bulk;            // 1: W staged by one bulk copy (16 B aligned, size % 16 == 0)
};


// Filter of class-major dy row `i` (row (d, j) = oc d + D*j).
__device__ __forceinline__ int row_oc(const BArgs& a, int i) {
  const int d = i / a.cls;
  return d + a.n_class * (i - d * a.cls);
}
// Slice `sl` owns blocks sl, sl + slices, sl + 2*slices, ... (interleaved: at
// any moment the CTAs fetch a contiguous window of blocks, i.e. whole channel
// planes, instead of 148 scattered 128 B pieces of them -- measured faster
// than contiguous slices); a pair is any two consecutive blocks of the slice.
__device__ __forceinline__ int slice_blocks(const BArgs& a, int sl) {
  return (a.units - sl + a.slices - 1) / a.slices;
}
__device__ __forceinline__ int blk_u(const BArgs& a, int sl, int m) { return sl + a.slices * m; }


__host__ __device__ constexpr int round1k(int b) { return (b + 1023) & ~1023; }

// Shared memory: kSlots raw TMA pair slots (per block: dy | x; x is turned
// into x_lo in place once the MMAs that read raw x are done), kStages dy_lo
// pairs (the dx GEMM's B lo), one dx exchange pair (the W_lo half of the
// accumulator, handed to the W_hi half), the per-filter (oc*gw - start,
// start) table.  The W staging of the prologue
// aliases the exchange pair when it fits (its first use follows the dx MMAs,
// which wait for W^T); the dW row dump of the epilogue aliases slot 0 (every
// MMA has completed by then).
struct BLayout {
  int blk, x, slot, dlo, dlob, stg, stgb, wst, kt, dump, bars, total;
  __host__ __device__ BLayout(int c_in, int c_out, int gw, int xr) {
    const int dyb = round1k(c_out * 128), xb = round1k(xr * 128);
    blk = dyb + xb;                       // one block: dy | x
    x = dyb;
    slot = 2 * blk;
    dlob = 2 * dyb;                       // one dy_lo pair
    dlo = kSlots * slot;
    stgb = round1k(c_in * 128);           // one block's dx [c_in rows][32 px] (SWIZZLE_128B)
    stg = dlo + kStages * dlob;
    int end = stg + 2 * stgb;
    const int wneed = c_out * gw * 4;
    if (wneed <= 2 * stgb) {
      wst = stg;
    } else {
      wst = end;
      end += round1k(wneed);
    }
    kt = end;                             // [c_out] int2
    end += round1k(c_out * 8);
    dump = 0;                             // [128][xr + 4] over slot 0
    bars = end;
    total = bars + 64 * 8;
  }
  __host__ __device__ bool dump_fits(int xr) const { return 128 * (xr + 4) * 4 <= slot; }
};

// Row `L` (this thread's TMEM lane) of the resident stacked W^T operand:
// lane ic (< 64) holds W_hi, lane 64 + ic holds W_lo, class-major filter
// columns, zero outside each filter's window; built from W and the
// (oc*gw - start, start) table staged in shared memory.
__device__ __forceinline__ void build_wt(const BArgs& a, uint32_t tmem, uint32_t lane_base, int L,
                                         const float* ws, const int2* kt) {
  const int ic = L & 63;
  const bool lo_lane = L >= 64;
  const bool live = ic < a.c_in;
  for (int c0 = 0; c0 < a.c_out; c0 += 32) {
    float v[32];
    if (a.cls % 32 == 0) {
      // the chunk is one window class: one start, filters D apart in W
      const int2 e = kt[c0];
      const int wrap = ic < e.y ? a.c_in : 0;
      const bool in = live && static_cast<unsigned>(ic - e.y + wrap) < static_cast<unsigned>(a.gw);
      const float* p = ws + (in ? e.x + ic + wrap : 0);
      const int stride = a.n_class * a.gw;
#pragma unroll
      for (int t = 0; t < 32; ++t) v[t] = in ? p[t * stride] : 0.f;
    } else {
      int idx[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const int2 e = kt[min(c0 + t, a.c_out - 1)];
        const int wrap = ic < e.y ? a.c_in : 0;
        const bool in = live && static_cast<unsigned>(ic - e.y + wrap) < static_cast<unsigned>(a.gw) &&
                        c0 + t < a.c_out;
        idx[t] = in ? e.x + ic + wrap : -1;
      }
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const float w = ws[max(idx[t], 0)];
        v[t] = idx[t] >= 0 ? w : 0.f;
      }
    }
    uint32_t r[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      const float h = tf32_hi(v[t]);
      r[t] = __float_as_uint(lo_lane ? v[t] - h : h);
    }
    tmem_st32(tmem + kWt + c0 + lane_base, r);
  }
  tmem_st_wait();
  tc_fence_before();
}

__device__ __forceinline__ float4 f4(const uint32_t* v) {
  return make_float4(__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]), __uint_as_float(v[3]));
}

// Pipeline (pair p: raw slot p % 3, dy_lo pair and TMEM dW A stage p % 2):
//   MMA  dW raw (dy_hi * x, dy_lo * x)  -> commit xraw   (x converters: x -> x_lo in place)
//        dx (W^T * dy, W^T * dy_lo)     -> commit dxfull (single accumulator; epilogue drains it)
//        dW lo (dy_hi * x_lo)           -> commit pfree (dy_lo pair + TMEM A), sfree (raw slot)
// so three pairs of raw data are in flight from the start (round 1 kept one
// lo pair and one TMEM A: conversion and MMA alternated, ~2 us per pair
// against 1.1 us of tensor work), the dy converters of pair p+1 run under the
// MMAs of pair p, and the in-place x_lo conversion runs under the dx MMAs.
// The first pair's dW MMAs do not need W^T, so they start while it is built.
__global__ void __launch_bounds__(kThreads, 1)
    tc_bwd_kernel(const __grid_constant__ CUtensorMap tdy, const __grid_constant__ CUtensorMap tx,
                  const __grid_constant__ BArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const BLayout L(a.c_in, a.c_out, a.gw, a.xr);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* full = bars;                       // [slot] TMA landed
  uint64_t* sfree = full + kSlots;             // [slot] MMA commit: raw slot consumed
  uint64_t* pfree = sfree + kSlots;            // [stage] MMA commit: dy_lo pair + TMEM A consumed
  uint64_t* conv = pfree + kStages;            // [stage] 4 dy converter warps: dy_lo + dW A written
  uint64_t* xraw = conv + kStages;             // [stage] MMA commit: raw x consumed
  uint64_t* xlo = xraw + kStages;              // [stage] 2 x warps: x_lo written in place
  uint64_t* dxfull = xlo + kStages;            // MMA commit
  uint64_t* dxempty = dxfull + 1;              // 4 epilogue warps
  uint64_t* accfull = dxempty + 1;             // MMA commit: the slice's dW done
  uint64_t* wt_ready = accfull + 1;            // 4 epilogue warps: W^T in TMEM
  uint64_t* w_bar = wt_ready + 1;              // W bulk copy landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_bar + 1);

  const uint32_t warp = warp_id();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
#if defined(SCC_TRACE)
    if (blockIdx.x == 0) g_trace3[59] = g_trace3[62];  // the previous call's reduce end
#endif
    TRACE3(48);
#if defined(SCC_TRACE)
    if (blockIdx.x < 256) g_cta3[2 * blockIdx.x] = globaltimer();
#endif
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sfree[s], 1);
    }
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&pfree[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&xraw[s], 1);
      mbar_init(&xlo[s], 2);
    }
    mbar_init(dxfull, 1);
    mbar_init(dxempty, 4);
    mbar_init(accfull, 1);
    mbar_init(wt_ready, 4);
    mbar_init(w_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tdy);
    if (a.do_dw) prefetch_tmap(&tx);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TRACE3(49);
  // the next kernel may start its prologue; it waits for this grid before
  // touching memory
  cudaTriggerProgrammaticLaunchCompletion();

  // this CTA's slice (exactly one, see the launch) and its block pairs
  const int sl = blockIdx.x;
  const int nblk = slice_blocks(a, sl);
  const int npairs = (nblk + 1) >> 1;

  if (warp == 0) {
    // ---------------- producer ----------------
    // A pair is 2 dy boxes + 2 x boxes (more when the x arc wraps); the lanes
    // issue them in parallel (one TMA instruction holds its thread ~0.1-0.3 us).
    cudaGridDependencySynchronize();
    if (a.do_dx && a.w_bulk && lane == 0) {
      // W first: the dx GEMM's operand is built from it
      const uint32_t wb = 4u * a.c_out * a.gw;
      mbar_expect_tx(w_bar, wb);
      bulk_load(smem + L.wst, a.weight, wb, w_bar);
    }
    const int nxb = a.do_dw ? (a.xbox ? 1 : a.nx / a.rbb) : 0;
    const int per_blk = 1 + nxb;
    const uint32_t bytes = a.c_out * 128 + (a.do_dw ? a.nx * 128 : 0);
    for (int p = 0; p < npairs; ++p) {
      const int s = p % kSlots;
      const int nb = min(2, nblk - 2 * p);
      if (p >= kSlots) mbar_wait(&sfree[s], (p / kSlots - 1) & 1);
      if (lane == 0) {
        TRACE3K(0, p);
        mbar_expect_tx(&full[s], bytes * nb);
      }
      __syncwarp();
      for (int bi = lane; bi < nb * per_blk; bi += 32) {
        const int k = bi / per_blk, j = bi - k * per_blk;
        const int u = blk_u(a, sl, 2 * p + k);
        const int n = u / a.nbps, px0 = (u - n * a.nbps) * 32;
        uint8_t* st = smem + s * L.slot + k * L.blk;
        if (j == 0) {
          tma_load_4d(st, &tdy, &full[s], px0, 0, 0, n);
        } else if (a.xbox) {
          tma_load_3d(st + L.x, &tx, &full[s], px0, a.start8, n);
        } else {
          const int r = (j - 1) * a.rbb;
          int ic = a.start8 + r;
          ic -= ic >= a.c_in ? a.c_in : 0;
          tma_load_3d(st + L.x + r * 128, &tx, &full[s], px0, ic, n);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idw = idesc_tf32(128, static_cast<uint32_t>(a.xr), 0, 0);
    const uint32_t idx = idesc_tf32(128, 64, 0, 1);  // B = dy of the pair, MN-major (pixels contiguous)
    const int ksteps = a.c_out >> 3;
    const uint32_t lbo = static_cast<uint32_t>(L.blk);   // the pair's second 32-px atom (raw)
    const uint32_t lbol = static_cast<uint32_t>(L.dlob / 2);  // ... (dy_lo)
    uint32_t dph = 0;
    for (int p = 0; p < npairs; ++p) {
      const int s = p % kSlots, e = p & 1;
      const uint32_t ph = (p >> 1) & 1;
      const int nb = min(2, nblk - 2 * p);
      mbar_wait(&conv[e], ph);
      tc_fence_after();
      const uint32_t st = smem_u32(smem + s * L.slot);
      const uint32_t lb = smem_u32(smem + L.dlo + e * L.dlob);
      const uint32_t aw = tmem + kDwA + 128 * e;
      if (a.do_dw) {
        // dW with raw x (x_hi): dy_hi * x, dy_lo * x
        if (elect_one()) {
          for (int k = 0; k < nb; ++k) {
            const uint32_t ah = aw + 64 * k, al = ah + 32;
            for (int q = 0; q < 4; ++q) {
              const uint64_t dbx = desc_sw128(st + k * L.blk + L.x + q * 32, 16, 1024);
              mma_tf32_ts(tmem + kDwAcc, ah + 8 * q, dbx, idw, (p == 0 && k == 0 && q == 0) ? 0u : 1u);
              mma_tf32_ts(tmem + kDwAcc, al + 8 * q, dbx, idw, 1);
            }
          }
          mma_commit(&xraw[e]);
          TRACE3K(16, p);
        }
        __syncwarp();
      }
      if (a.do_dx) {
        if (p == 0) mbar_wait(wt_ready, 0);
        mbar_wait(dxempty, dph ^ 1u);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t d = tmem + kDxAcc;
          for (int q = 0; q < ksteps; ++q) {
            mma_tf32_ts(d, tmem + kWt + 8 * q, desc_mn32(st + q * 1024, lbo, 512), idx, q == 0 ? 0u : 1u);
            mma_tf32_ts(d, tmem + kWt + 8 * q, desc_mn32(lb + q * 1024, lbol, 512), idx, 1);
          }
          mma_commit(dxfull);
          TRACE3K(24, p);
        }
        __syncwarp();
        dph ^= 1u;
      }
      if (a.do_dw) {
        // dW with x_lo (converted in place under the dx MMAs): dy_hi * x_lo
        mbar_wait(&xlo[e], ph);
        tc_fence_after();
        if (elect_one()) {
          for (int k = 0; k < nb; ++k) {
            const uint32_t ah = aw + 64 * k;
            for (int q = 0; q < 4; ++q)
              mma_tf32_ts(tmem + kDwAcc, ah + 8 * q, desc_sw128(st + k * L.blk + L.x + q * 32, 16, 1024), idw, 1);
          }
        }
        __syncwarp();
      }
      if (elect_one()) {
        mma_commit(&pfree[e]);
        mma_commit(&sfree[s]);
      }
      __syncwarp();
    }
    // (an empty slice accumulates nothing; the epilogue writes zeros)
    if (a.do_dw && elect_one()) mma_commit(accfull);
    __syncwarp();
  } else if (warp < 4) {
    // ---------------- x lo converters (in place) ----------------
    if (a.do_dw) {
      const int ct = threadIdx.x - 64;  // 0..63
      // padding rows [nx, xr) of every x block are zero (TMA never writes
      // them; lo of zero is zero)
      for (int b = 0; b < 2 * kSlots && a.xr > a.nx; ++b) {
        float* xs = reinterpret_cast<float*>(smem + (b >> 1) * L.slot + (b & 1) * L.blk + L.x);
        for (int i = ct; i < (a.xr - a.nx) * 32; i += 64) xs[a.nx * 32 + i] = 0.f;
      }
      fence_proxy_async_smem();
      const int words = a.nx * 8;  // float4 per x block
      for (int p = 0; p < npairs; ++p) {
        const int s = p % kSlots, e = p & 1;
        const int nb = min(2, nblk - 2 * p);
        // the MMAs that read raw x are done (and so the data had landed)
        mbar_wait(&xraw[e], (p >> 1) & 1);
        for (int k = 0; k < nb; ++k) {
          const uint32_t base = smem_u32(smem + s * L.slot + k * L.blk + L.x);
          for (int i0 = ct; i0 < words; i0 += 64 * 4) {
            float4 v[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) v[q] = lds_v4(base + min(i0 + 64 * q, words - 1) * 16);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (i0 + 64 * q < words) {
                float4 o;
                o.x = v[q].x - tf32_hi(v[q].x);
                o.y = v[q].y - tf32_hi(v[q].y);
                o.z = v[q].z - tf32_hi(v[q].z);
                o.w = v[q].w - tf32_hi(v[q].w);
                sts_v4(base + (i0 + 64 * q) * 16, o);
              }
            }
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&xlo[e]);
      }
    }
  } else if (warp < 8) {
    // ---------------- dy row converters ----------------
    // Row `row` of a block: 128 B, 32 B chunk c at physical chunk c ^ (row % 4)
    // (SWIZZLE_128B_BASE32B).  Writes the lo row to the stage's lo pair (dx B
    // lo) and, for dW, the hi / lo row to TMEM lane `row`.
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const int swp = (row >> 2) & 1;
    const bool live = row < a.c_out;
    const bool warp_live = q * 32 < a.c_out;  // tcgen05.st is warp-collective
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    // window start of filter row `row` (a plan table: no dependency wait)
    const int start_i = (a.do_dw && live) ? __ldg(a.starts + row_oc(a, row)) : 0;
    float dbsum = 0.f;  // db of this filter over the slice (fixed order: blocks, then pixels)
    for (int p = 0; p < npairs; ++p) {
      const int s = p % kSlots, e = p & 1;
      const int nb = min(2, nblk - 2 * p);
      mbar_wait(&full[s], (p / kSlots) & 1);
      if (p >= kStages) mbar_wait(&pfree[e], ((p >> 1) - 1) & 1);  // dy_lo pair + TMEM A of pair p-2
      tc_fence_after();
      for (int k = 0; k < nb; ++k) {
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) hi[c] = lo[c] = 0u;
        if (live) {
          const float4* rp = reinterpret_cast<const float4*>(smem + s * L.slot + k * L.blk + row * 128);
          float bs = 0.f;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            // 32 B atom j of the row sits at atom (j ^ row) & 3; rows 4 apart
            // share that position, so they take its two 16 B halves in the
            // opposite order: the 8 rows of a quarter warp hit 8 distinct
            // 16 B bank groups (no 2-way conflict).
            const int at = ((j ^ row) & 3) << 1;
            const float4 va = rp[at | swp], vb = rp[at | (swp ^ 1)];
            const float4 v0 = swp ? vb : va, v1 = swp ? va : vb;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const float4 v = hh ? v1 : v0;
              const int c = 2 * j + hh;
              const float e[4] = {v.x, v.y, v.z, v.w};
              bs += (e[0] + e[1]) + (e[2] + e[3]);
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const float h = tf32_hi(e[t]);
                hi[4 * c + t] = __float_as_uint(h);
                lo[4 * c + t] = __float_as_uint(e[t] - h);
              }
            }
          }
          dbsum += bs;
          const uint32_t lo_row = smem_u32(smem + L.dlo + e * L.dlob + k * (L.dlob / 2) + row * 128);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int at = ((j ^ row) & 3) << 1;
            const float4 l0 = f4(lo + 8 * j), l1 = f4(lo + 8 * j + 4);
            sts_v4(lo_row + (at | swp) * 16, swp ? l1 : l0);
            sts_v4(lo_row + (at | (swp ^ 1)) * 16, swp ? l0 : l1);
          }
        }
        if (a.do_dw && warp_live) {
          const uint32_t col = tmem + kDwA + 128 * e + 64 * k + lane_base;
          tmem_st32(col, hi);
          tmem_st32(col + 32, lo);
        }
      }
      fence_proxy_async_smem();
      if (a.do_dw) {
        tmem_st_wait();
        tc_fence_before();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[e]);
      if (row == 0) TRACE3K(8, p);
    }
    if (a.do_dw) {
      // dW slice epilogue (these warps are idle once the last pair is
      // converted; the epilogue warps may still be draining dx): TMEM row
      // `row` -> smem dump over slot 0 (every MMA has completed) -> the
      // window-relative values -> this slice's partial
      const int i = row;
      float* prow = reinterpret_cast<float*>(smem + L.dump) + i * (a.xr + 4);
      const uint32_t prow_a = smem_u32(prow);
      mbar_wait(accfull, 0);
      if (row == 0) TRACE3(51);
      tc_fence_after();
      for (int c0 = 0; c0 < a.xr; c0 += 32) {
        uint32_t v[32];
        tmem_ld32_nowait(tmem + kDwAcc + c0 + lane_base, v);
        tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < 32; t += 4)
          if (c0 + t < a.xr) sts_v4(prow_a + (c0 + t) * 4, f4(v + t));
      }
      __syncwarp();
      const bool wlive = i < a.c_out && nblk > 0;
      int j0 = 0;
      if (wlive) {
        j0 = start_i - a.start8;
        j0 += j0 < 0 ? a.c_in : 0;
      }
      float* dst = a.part + static_cast<int64_t>(sl) * a.elems;
      float wv[kMaxGw];
#pragma unroll
      for (int t = 0; t < kMaxGw; ++t) {
        int j = j0 + t;
        j -= j >= a.c_in ? a.c_in : 0;
        wv[t] = (wlive && t < a.gw) ? prow[j] : 0.f;
      }
      if (i < a.c_out) {
        if ((a.gw & 3) == 0) {
#pragma unroll
          for (int t = 0; t < kMaxGw; t += 4)
            if (t < a.gw)
              *reinterpret_cast<float4*>(dst + i * a.gw + t) = make_float4(wv[t], wv[t + 1], wv[t + 2], wv[t + 3]);
        } else {
#pragma unroll
          for (int t = 0; t < kMaxGw; ++t)
            if (t < a.gw) dst[i * a.gw + t] = wv[t];
        }
        dst[a.c_out * a.gw + i] = wlive ? dbsum : 0.f;
      }
    }
  } else {
    // ---------------- W^T build, dx epilogue, dW slice epilogue ----------------
    const int q = warp & 3;
    const int et = threadIdx.x - 256;  // 0..127
    const int i = q * 32 + lane;       // TMEM lane: input channel (+64: lo part) / filter row (dW)
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    float* wst = reinterpret_cast<float*>(smem + L.wst);
    int2* kt = reinterpret_cast<int2*>(smem + L.kt);
    // plan table, never written by a preceding kernel: loaded before the
    // dependency wait
    if (a.do_dx && et < a.c_out) {
      const int oc = row_oc(a, et);
      const int st = __ldg(a.starts + oc);
      kt[et] = make_int2(oc * a.gw - st, st);
    }
    cudaGridDependencySynchronize();
    if (et == 0) TRACE3(53);
    if (a.do_dx) {
      // W (bulk copy by the producer, or loads here, all in flight at once);
      // then this lane's row of W^T -> TMEM
      const int nw = a.c_out * a.gw;
      if (!a.w_bulk) {
        for (int k0 = 0; k0 < nw; k0 += 128 * 32) {
          float v[32];
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int k = k0 + t * 128 + et;
            v[t] = k < nw ? __ldg(a.weight + k) : 0.f;
          }
#pragma unroll
          for (int t = 0; t < 32; ++t) {
            const int k = k0 + t * 128 + et;
            if (k < nw) wst[k] = v[t];
          }
        }
      }
      named_bar_sync(1, 128);
      if (a.w_bulk) mbar_wait(w_bar, 0);
      if (et == 0) TRACE3(55);
      build_wt(a, tmem, lane_base, i, wst, kt);
      __syncwarp();
      if (lane == 0) mbar_arrive(wt_ready);
      if (et == 0) TRACE3(50);
    }
    // rows 0-63 of the dx accumulator hold W_hi * dy, rows 64-127 W_lo * dy
    const int dx_row = i & 63;
    const bool bottom = i >= 64;
    const bool dx_live = dx_row < a.c_in;
    const bool dx_warp = (q & 1) * 32 < a.c_in;
    const bool leader = et == 0;
    uint32_t dph = 0;
    if (a.do_dx) {
      for (int p = 0; p < npairs; ++p) {
        const int nb = min(2, nblk - 2 * p);
        mbar_wait(dxfull, dph);
        dph ^= 1u;
        if (et == 0) TRACE3K(32, p);
        tc_fence_after();
        uint32_t v0[32], v1[32];
        if (dx_warp) {
          tmem_ld32_nowait(tmem + kDxAcc + lane_base, v0);
          tmem_ld32_nowait(tmem + kDxAcc + 32 + lane_base, v1);
          tmem_ld_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(dxempty);
        // rows 64-127 (the W_lo part) -> exchange pair; rows 0-63 add theirs and
        // store the sum straight to global (each thread one input channel,
        // 32 contiguous pixels per block).  The first barrier orders this
        // pair's exchange writes after the previous pair's reads (and, on the
        // first pair, after every lane's last read of the W staging).
        named_bar_sync(1, 128);
        const uint32_t r0 = smem_u32(smem + L.stg + dx_row * 128), r1 = r0 + L.stgb;
        if (bottom && dx_warp && dx_live) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            sts_v4(r0 + ((j ^ (dx_row & 7)) << 4), f4(v0 + 4 * j));
            sts_v4(r1 + ((j ^ (dx_row & 7)) << 4), f4(v1 + 4 * j));
          }
        }
        named_bar_sync(1, 128);
        if (!bottom && dx_warp && dx_live) {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            if (k < nb) {
              const int u = blk_u(a, sl, 2 * p + k);
              const int n = u / a.nbps, px0 = (u - n * a.nbps) * 32;
              float* drow = a.dx + (static_cast<int64_t>(n) * a.c_in + dx_row) * a.plane + px0;
              const uint32_t* vv = k == 0 ? v0 : v1;
              const uint32_t rk = k == 0 ? r0 : r1;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 o = lds_v4(rk + ((j ^ (dx_row & 7)) << 4));
                const float4 m = f4(vv + 4 * j);
                if (px0 + 4 * j < a.plane)
                  __stcs(reinterpret_cast<float4*>(drow + 4 * j),
                         make_float4(m.x + o.x, m.y + o.y, m.z + o.z, m.w + o.w));
              }
            }
          }
        }
        if (leader) TRACE3K(40, p);
      }
    }
    if (leader) {
      TRACE3(52);
#if defined(SCC_TRACE)
      if (blockIdx.x < 256) g_cta3[2 * blockIdx.x + 1] = globaltimer();
#endif
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

// Fixed-order reduction of the per-slice partials, PDL-chained behind the main
// kernel (its CTAs launch while the main kernel runs and wait for it).  Block
// = 32 consecutive partial elements x 32 warps; warp w sums slices w, w+32,
// ... in order (each load a coalesced 128 B row piece; <= 5 loads per thread,
// all in flight at once -- 8 warps with 19 dependent-register loads each ran
// latency bound at 0.17 eligible warps), then warp 0 adds the 32 warp sums in
// order.  Bitwise reproducible.
constexpr int kRedWarps = 32;  // 1024 threads: <= 5 in-flight loads per thread (16 warps measured 0.7 us slower)
__global__ void __launch_bounds__(32 * kRedWarps) tc_bwd_reduce(const __grid_constant__ BArgs a) {
  __shared__ float red[kRedWarps][33];
  if (threadIdx.x == 0) TRACE3(60);
  cudaGridDependencySynchronize();
  if (threadIdx.x == 0) TRACE3(61);
  // the next kernel may start its prologue (it waits for this grid)
  cudaTriggerProgrammaticLaunchCompletion();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int e = blockIdx.x * 32 + l;
  float acc = 0.f;
  if (e < a.elems) {
    constexpr int kPer = (kSlices + kRedWarps - 1) / kRedWarps;
    float v[kPer];
#pragma unroll
    for (int m = 0; m < kPer; ++m) {
      const int k = w + kRedWarps * m;
      v[m] = k < a.slices ? __ldcg(a.part + static_cast<int64_t>(k) * a.elems + e) : 0.f;
    }
#pragma unroll
    for (int m = 0; m < kPer; ++m) acc += v[m];
  }
  red[w][l] = acc;
  __syncthreads();
  if (w == 0 && e < a.elems) {
    float t = red[0][l];
#pragma unroll
    for (int q = 1; q < kRedWarps; ++q) t += red[q][l];
    const int nw = a.c_out * a.gw;
    if (e < nw) {
      const int i = e / a.gw;
      a.dweight[static_cast<int64_t>(row_oc(a, i)) * a.gw + (e - i * a.gw)] = t;
    } else if (a.dbias != nullptr) {
      a.dbias[row_oc(a, e - nw)] = t;
    }
  }
  if (threadIdx.x == 0) TRACE3(62);
}

struct Geo {
  int nx = 0, xr = 0, start8 = 0;
  bool fits = false;
};

Geo geometry(const TcWeightPlan& tw, int32_t c_in, int32_t c_out, int32_t gw) {
  Geo g;
  g.start8 = tw.rt_info[0];
  g.nx = tw.rt_info[1];
  g.xr = (g.nx + 15) / 16 * 16;
  const BLayout L(c_in, c_out, gw, g.xr);
  g.fits = L.total <= kSmemLimit && L.dump_fits(g.xr) && g.xr <= kMaxXr;
  return g;
}

}  // namespace

int tc_bwd_trace(unsigned long long* out, int n) {
#if defined(SCC_TRACE)
  if (n > 64 + 512) n = 64 + 512;
  const int m = n < 64 ? n : 64;
  if (cudaMemcpyFromSymbol(out, g_trace3, m * sizeof(unsigned long long)) != cudaSuccess) return -1;
  if (n > 64 && cudaMemcpyFromSymbol(out + 64, g_cta3, (n - 64) * sizeof(unsigned long long)) != cudaSuccess)
    return -1;
  return n;
#else
  for (int i = 0; i < n; ++i) out[i] = 0;
  return n;
#endif
}

bool tc_bwd_supported(const TcWeightPlan& tw, int64_t plane, int32_t c_in, int32_t c_out, int32_t gw) {
  if (!tw.ok || plane % 4 != 0 || tw.n_rt != 1 || tw.rt_info.size() < 2) return false;
  if (c_out > 128 || c_out % 8 != 0 || c_out != tw.n_class * tw.cls || tw.cls > 256 || tw.n_class > 256)
    return false;
  if (c_in > 64 || gw > kMaxGw) return false;
  const Geo g = geometry(tw, c_in, c_out, gw);
  if (g.xr > 128 || g.nx % tw.rbb != 0) return false;
  return g.fits;
}

size_t tc_bwd_workspace_bytes(int32_t c_out, int32_t gw, int64_t n, int64_t plane) {
  const int64_t units = n * ((plane + 31) / 32);
  const int64_t slices = std::min<int64_t>(units, kSlices);
  return static_cast<size_t>(slices) * (static_cast<size_t>(c_out) * gw + c_out) * sizeof(float);
}

cudaError_t launch_tc_bwd(const TcWeightPlan& tw, const TcBwdCall& call, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  static bool attr_set[64] = {false};
  static int nsm_cache[64] = {0};
  int nsm = 148;
  if (dev >= 0 && dev < 64 && nsm_cache[dev] > 0) {
    nsm = nsm_cache[dev];
  } else {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < 64) nsm_cache[dev] = nsm;
  }
  if (!call.do_dx && !call.do_dw) return cudaSuccess;
  const Geo g = geometry(tw, call.c_in, call.c_out, call.gw);
  BArgs a{};
  a.c_in = call.c_in;
  a.c_out = call.c_out;
  a.gw = call.gw;
  a.cls = tw.cls;
  a.n_class = tw.n_class;
  a.start8 = g.start8;
  a.nx = g.nx;
  a.xr = g.xr;
  a.rbb = tw.rbb;
  a.xbox = (g.start8 + g.nx <= call.c_in && g.nx <= 256) ? 1 : 0;
  a.nbps = static_cast<int32_t>((call.plane + 31) / 32);
  const int64_t units = call.n * a.nbps;
  if (units > (1ll << 30) || units == 0) return units == 0 ? cudaSuccess : cudaErrorInvalidValue;
  a.units = static_cast<int32_t>(units);
  a.elems = call.c_out * call.gw + call.c_out;
  a.slices = static_cast<int32_t>(std::min<int64_t>(units, kSlices));
  a.do_dx = call.do_dx ? 1 : 0;
  a.do_dw = call.do_dw ? 1 : 0;
  a.w_bulk = (reinterpret_cast<uintptr_t>(call.weight) % 16 == 0 && (call.c_out * call.gw) % 4 == 0) ? 1 : 0;

  if (a.do_dw && tc_bwd_workspace_bytes(call.c_out, call.gw, call.n, call.plane) > call.workspace_bytes)
    return cudaErrorInvalidValue;
  a.part = static_cast<float*>(call.workspace);
  a.dweight = call.dweight;
  a.dx = call.dx;
  a.plane = static_cast<int32_t>(call.plane);
  a.dbias = call.dbias;
  a.weight = call.weight;
  a.starts = call.starts;
  // one slice per CTA (the dW dump aliases the lo pair, see BLayout)
  const int grid = a.slices;
  (void)nsm;

  const uint64_t P = static_cast<uint64_t>(call.plane);
  CUtensorMap tdy{}, tx{};
  {
    // dy {P, cls, D, N}: row (d, j) = filter d + D*j; one box per block
    const uint64_t dims[4] = {P, static_cast<uint64_t>(tw.cls), static_cast<uint64_t>(tw.n_class),
                              static_cast<uint64_t>(call.n)};
    const uint64_t strides[3] = {P * 4 * tw.n_class, P * 4, P * 4 * call.c_out};
    const uint32_t box[4] = {32, static_cast<uint32_t>(tw.cls), static_cast<uint32_t>(tw.n_class), 1};
    if (!encode_f32(&tdy, call.dy, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return cudaErrorInvalidValue;
  }
  const uint64_t dimx[3] = {P, static_cast<uint64_t>(call.c_in), static_cast<uint64_t>(call.n)};
  const uint64_t strx[2] = {P * 4, P * 4 * call.c_in};
  if (a.do_dw) {
    const uint32_t box[3] = {32, static_cast<uint32_t>(a.xbox ? g.nx : tw.rbb), 1};
    if (!encode_f32(&tx, call.x, 3, dimx, strx, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  }
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(tc_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = BLayout(a.c_in, a.c_out, a.gw, a.xr).total;
  cfg.stream = s;
  // PDL-chained to the neighbouring kernels; one CTA per SM.
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (grid > nsm) return cudaErrorInvalidConfiguration;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_bwd_kernel, tdy, tx, a);
  if (e != cudaSuccess) return e;
  int launches = 1;
  if (a.do_dw) {
    // the fixed-order partial reduction, PDL-chained (its CTAs launch while
    // this grid runs and wait on it).  Measured against alternatives without
    // a second launch (cooperative grid barrier; the last CTAs to arrive
    // reducing behind a ticket counter): +1.7 us for this kernel vs +2.5 /
    // +4.1 us for those (scripts/bwd_timing.py, config 1).
    cudaLaunchConfig_t rc{};
    rc.gridDim = dim3(static_cast<unsigned>((a.elems + 31) / 32));
    rc.blockDim = dim3(32 * kRedWarps);
    rc.stream = s;
    rc.attrs = attr;
    rc.numAttrs = 1;
    e = cudaLaunchKernelEx(&rc, tc_bwd_reduce, a);
    if (e != cudaSuccess) return e;
    ++launches;
  }
  note_launches(launches);
  return cudaSuccess;
}

}  // namespace scc
