// Fused tensor-core backward (tcgen05, bf16x3), sm_100a: backward-data and
// backward-weight of one SCC layer from a single pass over dy
// (replaces scc_backward_input + scc_backward_params, kernel.cpp:100-189):
//
//   dx[n, ic, p]  = sum_oc  W^T[ic, oc] * dy[n, oc, p]          (W^T: window-relative W scattered)
//   dW[oc, ic]    = sum_{n,p} dy[n, oc, p] * x[n, ic, p]        (ic in the arc of the filters)
//   db[oc]        = sum_{n,p} dy[n, oc, p]                      (CUDA cores, fp32)
//
// Precision: every operand is split into bf16 hi + lo (x = hi + lo + r, |r| <=
// 2^-18 |x|) and the MMAs (kind::f16, fp32 accumulate) take hi*hi + hi*lo +
// lo*hi (+ lo*lo for dx, free with the stacked W^T): ~1e-5 relative per
// product, inside the gradients' 1e-4 bar, at twice the rate of the 3xTF32
// kernels (K = 16 per instruction at the tf32 K = 8 cycle count).  The forward
// (1e-5 bar) stays 3xTF32.
//
// Geometry: one row tile of filters (c_out <= 128, in the class-major order
// of a single {32 px, cls, D} dy box) and c_in <= 64 input channels.  The
// pipeline moves PAIRS of 32-pixel blocks (any two consecutive blocks of the
// CTA's pixel slice); each pair lands raw by TMA and is rewritten in place:
//   * dy [c_out rows][64 px] -> bf16 hi | lo rows (SWIZZLE_128B, MN-major):
//     B of the dx GEMM (D[ic][px] = W^T[ic][oc] * dy[oc][px], K = oc); the same
//     hi | lo rows go to TMEM as A of the dW GEMM (lanes = filters, K = px);
//   * x [arc rows][64 px] -> bf16 hi | lo rows (SWIZZLE_128B, K-major): B of
//     the dW GEMM (D[oc][ic] = dy[oc][px] * x[ic][px]).
// W^T stays resident in TMEM, stacked: lanes 0-63 hold W_hi, lanes 64-127
// W_lo, so one M = 128 MMA yields W_hi*B and W_lo*B in the two lane halves
// (the epilogue adds them).  Every GEMM runs in TS mode (A from TMEM).
//
// dW accumulates over the CTA's pixel slice in TMEM and is written as that
// slice's window-relative partial (db: the dy converters sum their rows on
// the CUDA cores); a PDL-chained kernel sums the slice partials in a fixed
// order (the slice count is fixed per geometry, so the bits of dW do not
// depend on the grid).  dx is drained from TMEM per pair (two accumulators);
// the W_lo half of the stacked accumulator is staged in shared memory, the
// W_hi half adds itself in place and one TMA store per block writes dx.  The same kernel,
// with either GEMM switched off, serves scc_backward_input /
// scc_backward_params alone, so the fused and separate entry points agree bit
// for bit.
//
// Warp roles (384 threads, one CTA per SM, one slice per CTA):
//   warp 0      TMA producer
//   warp 1      TMEM allocator + MMA issuer
//   warps 2-3   x converters (thread = x row)
//   warps 4-7   dy converters (thread = filter row), db, dW slice epilogue
//   warps 8-11  W^T build (prologue), dx epilogue
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
__device__ unsigned long long g_trace3[128];
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
constexpr int kSlots = 4;             // pair slots: raw dy | x per block, overwritten in place by bf16 hi | lo
constexpr int kSlices = 148;          // pixel slices (dW partials) per launch = CTAs (one per SM)
constexpr int kSmemLimit = 227 * 1024;
constexpr int kMaxGw = 32;
constexpr int kMaxXr = 64;            // dW accumulator columns
// TMEM columns (512 allocated)
constexpr uint32_t kWt = 0;          // W^T bf16 pairs: [ic lane (hi) | 64 + ic lane (lo)][oc pair column]
constexpr uint32_t kDwAcc = 64;      // dW accumulator: [filter lane][x row column] (xr <= 64)
constexpr uint32_t kDxAcc = 128;     // dx accumulators (2): [ic lane (+64: lo part)][64 px]
constexpr uint32_t kDwA = 256;       // per slot: dy hi | lo bf16 pairs of the pair's 64 px [filter lane][32 | 32]
// MN-major bf16 B (the dx GEMM's dy): SWIZZLE_128B atoms of 8 K rows x 64 px,
// SBO = 1024 between 8-row K groups, LBO = stride between 64-px atoms (one
// atom: N = 64); verified by tests/cuda/bf16_probe.cu
constexpr uint32_t kMnLbo = 8192;

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
__host__ __device__ constexpr int round16(int v) { return (v + 15) & ~15; }

// Shared memory: kSlots pair slots of two blocks (dy | x each, as TMA lands
// them: [rows][32 px] fp32, SWIZZLE_128B); the converters overwrite a pair in
// place with its bf16 hi (block 0) and lo (block 1) parts, [rows][64 px]
// SWIZZLE_128B -- the same 128 B row span per row, so each converter thread
// only rewrites the rows it read.  Then two dx staging pairs (the W_lo half
// of the accumulator is written there, the W_hi half adds itself in place, one
// TMA store per block reads it), the per-filter (oc*gw - start, start) table.
// The W staging of the prologue aliases the dx staging (its first use follows
// the dx MMAs, which wait for W^T); the dW row dump of the epilogue aliases
// slot 0 (every MMA has completed by then).
struct BLayout {
  int blk, x, slot, stg, stgb, wst, kt, dump, bars, total;
  __host__ __device__ BLayout(int c_in, int c_out, int gw, int xr) {
    const int dyb = round1k(round16(c_out) * 128), xb = round1k(xr * 128);
    blk = dyb + xb;                       // one block: dy | x
    x = dyb;
    slot = 2 * blk;
    stgb = round1k(c_in * 128);           // one block's dx [c_in rows][32 px] (SWIZZLE_128B)
    stg = kSlots * slot;                  // 2 staging pairs (TMA-store sources)
    int end = stg + 4 * stgb;
    const int wneed = c_out * gw * 4;
    if (wneed <= 4 * stgb) {
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
// lane ic (< 64) holds bf16 W_hi, lane 64 + ic bf16 W_lo, class-major filter
// columns in bf16 pairs, zero outside each filter's window and past c_out;
// built from W and the (oc*gw - start, start) table staged in shared memory.
__device__ __forceinline__ void build_wt(const BArgs& a, uint32_t tmem, uint32_t lane_base, int L,
                                         const float* ws, const int2* kt) {
  // One 32-filter group (16 TMEM columns) per iteration, the group body
  // unrolled, the group loop not: the fully unrolled form (two code paths x
  // 128 filters) was ~2,100 instructions -- a third of the kernel's code,
  // fetched from L2 while the data loads; one column per store measured
  // 6 us slower (the W^T build is on the first dx MMA's path).
  const int ic = L & 63;
  const bool lo_lane = L >= 64;
  const bool live = ic < a.c_in;
  const int cpad = round16(a.c_out);
#pragma unroll 1
  for (int c0 = 0; c0 < cpad; c0 += 32) {
    float v[32];
    if (a.cls % 32 == 0 && c0 < a.c_out) {
      // the group is one window class: one start, filters D apart in W
      const int2 e = kt[c0];
      const int wrap = ic < e.y ? a.c_in : 0;
      const bool in = live && static_cast<unsigned>(ic - e.y + wrap) < static_cast<unsigned>(a.gw);
      const float* p = ws + (in ? e.x + ic + wrap : 0);
      const int stride = a.n_class * a.gw;
#pragma unroll
      for (int t = 0; t < 32; ++t) v[t] = in ? p[t * stride] : 0.f;
    } else {
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const int f = c0 + t;
        const int2 e = kt[min(f, a.c_out - 1)];
        const int wrap = ic < e.y ? a.c_in : 0;
        const bool in = live && f < a.c_out && static_cast<unsigned>(ic - e.y + wrap) < static_cast<unsigned>(a.gw);
        v[t] = ws[in ? e.x + ic + wrap : 0];
        v[t] = in ? v[t] : 0.f;
      }
    }
    uint32_t r[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      uint32_t hi, lo;
      bf16x2_split(v[2 * t], v[2 * t + 1], hi, lo);
      r[t] = lo_lane ? lo : hi;
    }
    tmem_st16(tmem + kWt + static_cast<uint32_t>(c0 / 2) + lane_base, r);
  }
  tmem_st_wait();
  tc_fence_before();
}

__device__ __forceinline__ float4 f4(const uint32_t* v) {
  return make_float4(__uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]), __uint_as_float(v[3]));
}
__device__ __forceinline__ void sts_u4(uint32_t addr, const uint32_t* v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]));
}

// One 128 B row of a pair (row r of block 0 and of block 1: 64 fp32 pixels,
// 16 B chunk j at physical chunk j ^ (r % 8)) -> bf16 hi | lo pairs (word c =
// pixels 2c, 2c+1), written back in place: hi over block 0's row, lo over block
// 1's (16 B chunk j = pixels 8j..8j+7 at j ^ (r % 8)).  The 8 rows of a
// quarter warp hit 8 distinct 16 B bank groups on every access.  Block 1 reads
// as zeros when the pair has one block.  Returns the fp32 sum of the row.
__device__ __forceinline__ float convert_row(uint32_t row0, uint32_t row1, int r, int nb, uint32_t (&hi)[32],
                                             uint32_t (&lo)[32]) {
  const int sw = r & 7;
  float sum = 0.f;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    float v[32];
    if (k == 0 || nb > 1) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float4 t = lds_v4((k ? row1 : row0) + ((j ^ sw) << 4));
        v[4 * j] = t.x, v[4 * j + 1] = t.y, v[4 * j + 2] = t.z, v[4 * j + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0.f;
    }
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int j = 0; j < 32; j += 2) s0 += v[j], s1 += v[j + 1];
    sum += s0 + s1;
#pragma unroll
    for (int c = 0; c < 16; ++c) bf16x2_split(v[2 * c], v[2 * c + 1], hi[16 * k + c], lo[16 * k + c]);
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    sts_u4(row0 + ((j ^ sw) << 4), hi + 4 * j);
    sts_u4(row1 + ((j ^ sw) << 4), lo + 4 * j);
  }
  return sum;
}

// Pipeline (pair p: slot and TMEM A stage p % kSlots, dx accumulator p % 2):
//   producer   TMA dy | x of both blocks into the slot
//   dy warps   rows -> bf16 hi | lo in place (dx GEMM B, MN-major) + TMEM A of
//              the dW GEMM (lanes = filters) + db on the CUDA cores
//   x warps    rows -> bf16 hi | lo in place (dW GEMM B, K-major)
//   MMA        dW: dy_hi*x_hi + dy_lo*x_hi + dy_hi*x_lo      (K = pair pixels)
//              dx: [W_hi; W_lo]*dy_hi + [W_hi; W_lo]*dy_lo   (K = filters)
//              -> commit dxfull[p % 2], sfree[slot]
//   epilogue   dx accumulator -> global (W_lo half added through smem)
// All of a CTA's slots are in flight from the start at config 1 (~3.5 pairs
// per CTA); the double-buffered dx accumulator lets the MMAs of pair p+1 run
// while pair p drains.  The first pair's dW MMAs do not need W^T, so they
// start while it is built.
__global__ void __launch_bounds__(kThreads, 1)
    tc_bwd_kernel(const __grid_constant__ CUtensorMap tdy, const __grid_constant__ CUtensorMap tx,
                  const __grid_constant__ CUtensorMap tdx, const __grid_constant__ BArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const BLayout L(a.c_in, a.c_out, a.gw, a.xr);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* full = bars;                       // [slot] TMA landed
  uint64_t* sfree = full + kSlots;             // [slot] MMA commit: slot + TMEM A stage consumed
  uint64_t* conv = sfree + kSlots;             // [slot] 4 dy converter warps: dy hi | lo + dW A written
  uint64_t* xconv = conv + kSlots;             // [slot] 2 x warps: x hi | lo written
  uint64_t* dxfull = xconv + kSlots;           // [2] MMA commit
  uint64_t* dxempty = dxfull + 2;              // [2] 4 epilogue warps
  uint64_t* accfull = dxempty + 2;             // MMA commit: the slice's dW done
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
    if (blockIdx.x < 256) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_cta3[2 * blockIdx.x] = (globaltimer() & ~0xFFull) | smid;  // start (256 ns) | SM id
    }
#endif
    for (int s = 0; s < kSlots; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&sfree[s], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&xconv[s], 2);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&dxfull[b], 1);
      mbar_init(&dxempty[b], 4);
    }
    mbar_init(accfull, 1);
    mbar_init(wt_ready, 4);
    mbar_init(w_bar, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tdy);
    if (a.do_dw) prefetch_tmap(&tx);
    if (a.do_dx) prefetch_tmap(&tdx);
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
    const uint32_t idw = idesc_bf16(128, static_cast<uint32_t>(a.xr), 0, 0);
    const uint32_t idx = idesc_bf16(128, 64, 0, 1);  // B = dy hi | lo of the pair, MN-major (pixels contiguous)
    const int kq = round16(a.c_out) >> 4;
    for (int p = 0; p < npairs; ++p) {
      const int s = p % kSlots, b = p & 1;
      const uint32_t ph = (p / kSlots) & 1;
      const int nb = min(2, nblk - 2 * p);
      const uint32_t st = smem_u32(smem + s * L.slot);
      mbar_wait(&conv[s], ph);
      // dx first: its accumulator drains (the exchange, TMA stores) while the
      // dW MMAs run, which shortens the tail after the last pair lands
      if (a.do_dx) {
        if (p == 0) mbar_wait(wt_ready, 0);
        if (p >= 2) mbar_wait(&dxempty[b], ((p >> 1) - 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t d = tmem + kDxAcc + 64 * b;
          for (int q = 0; q < kq; ++q) {
            mma_bf16_ts(d, tmem + kWt + 8 * q, desc_sw128(st + 2048 * q, kMnLbo, 1024), idx, q == 0 ? 0u : 1u);
            mma_bf16_ts(d, tmem + kWt + 8 * q, desc_sw128(st + L.blk + 2048 * q, kMnLbo, 1024), idx, 1);
          }
          mma_commit(&dxfull[b]);
          TRACE3K(24, p);
        }
        __syncwarp();
      }
      if (a.do_dw) {
        mbar_wait(&xconv[s], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t aw = tmem + kDwA + 64 * s;
          const uint32_t xh = st + L.x, xl = st + L.blk + L.x;
          for (int ks = 0; ks < 2 * nb; ++ks) {
            const uint64_t bh = desc_sw128(xh + 32 * ks, 16, 1024), bl = desc_sw128(xl + 32 * ks, 16, 1024);
            mma_bf16_ts(tmem + kDwAcc, aw + 8 * ks, bh, idw, (p == 0 && ks == 0) ? 0u : 1u);
            mma_bf16_ts(tmem + kDwAcc, aw + 32 + 8 * ks, bh, idw, 1);
            mma_bf16_ts(tmem + kDwAcc, aw + 8 * ks, bl, idw, 1);
          }
          TRACE3K(16, p);
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(&sfree[s]);
      __syncwarp();
    }
    // (an empty slice accumulates nothing; the epilogue writes zeros)
    if (a.do_dw && elect_one()) mma_commit(accfull);
    __syncwarp();
  } else if (warp < 4) {
    // ---------------- x converters (in place) ----------------
    // thread r: x row r of the pair (rows [nx, xr) are the MMA's zero padding)
    if (a.do_dw) {
      const int r = threadIdx.x - 64;  // 0..63
      for (int p = 0; p < npairs; ++p) {
        const int s = p % kSlots;
        const int nb = min(2, nblk - 2 * p);
        mbar_wait(&full[s], (p / kSlots) & 1);
        if (r < a.xr) {
          const uint32_t row0 = smem_u32(smem + s * L.slot + L.x + r * 128), row1 = row0 + L.blk;
          uint32_t hi[32], lo[32];
          if (r < a.nx) {
            convert_row(row0, row1, r, nb, hi, lo);
          } else {
            const uint32_t z[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              sts_u4(row0 + 16 * j, z);
              sts_u4(row1 + 16 * j, z);
            }
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&xconv[s]);
        if (r == 0 && p < 3) TRACE3(56 + p);
      }
    }
  } else if (warp < 8) {
    // ---------------- dy row converters ----------------
    // thread = filter row `row` of the pair: bf16 hi | lo in place (rows
    // [c_out, round16(c_out)) zero: the dx GEMM's K padding) and, for dW, the
    // hi | lo row to TMEM lane `row`; db summed from the fp32 values.
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const bool live = row < a.c_out;
    const bool pad = !live && row < round16(a.c_out);
    const bool warp_live = q * 32 < a.c_out;  // tcgen05.st is warp-collective
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    // window start of filter row `row` (a plan table: no dependency wait)
    const int start_i = (a.do_dw && live) ? __ldg(a.starts + row_oc(a, row)) : 0;
    float dbsum = 0.f;  // db of this filter over the slice (fixed order: pairs, then pixels)
    for (int p = 0; p < npairs; ++p) {
      const int s = p % kSlots;
      const int nb = min(2, nblk - 2 * p);
      mbar_wait(&full[s], (p / kSlots) & 1);
      tc_fence_after();
      uint32_t hi[32], lo[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) hi[c] = lo[c] = 0u;
      const uint32_t row0 = smem_u32(smem + s * L.slot + row * 128), row1 = row0 + L.blk;
      if (live) {
        dbsum += convert_row(row0, row1, row, nb, hi, lo);
      } else if (pad) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          sts_u4(row0 + 16 * j, hi);
          sts_u4(row1 + 16 * j, lo);
        }
      }
      if (a.do_dw && warp_live) {
        const uint32_t col = tmem + kDwA + 64 * s + lane_base;
        tmem_st32(col, hi);
        tmem_st32(col + 32, lo);
      }
      fence_proxy_async_smem();
      if (a.do_dw) {
        tmem_st_wait();
        tc_fence_before();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[s]);
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
      if (i < a.c_out) {
        // (compact loop: a fully unrolled gather was ~500 instructions)
        auto wat = [&](int t) {
          int j = j0 + t;
          j -= j >= a.c_in ? a.c_in : 0;
          return wlive ? prow[j] : 0.f;
        };
        if ((a.gw & 3) == 0) {
#pragma unroll 1
          for (int t = 0; t < a.gw; t += 4)
            *reinterpret_cast<float4*>(dst + i * a.gw + t) = make_float4(wat(t), wat(t + 1), wat(t + 2), wat(t + 3));
        } else {
#pragma unroll 1
          for (int t = 0; t < a.gw; ++t) dst[i * a.gw + t] = wat(t);
        }
        dst[a.c_out * a.gw + i] = wlive ? dbsum : 0.f;
      }
    }
  } else {
    // ---------------- W^T build, dx epilogue ----------------
    const int q = warp & 3;
    const int et = threadIdx.x - 256;  // 0..127
    const int i = q * 32 + lane;       // TMEM lane: input channel (+64: lo part)
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
    if (a.do_dx) {
      for (int p = 0; p < npairs; ++p) {
        const int nb = min(2, nblk - 2 * p), b = p & 1;
        mbar_wait(&dxfull[b], (p >> 1) & 1);
        if (et == 0) TRACE3K(32, p);
        tc_fence_after();
        uint32_t v0[32], v1[32];
        if (dx_warp) {
          tmem_ld32_nowait(tmem + kDxAcc + 64 * b + lane_base, v0);
          tmem_ld32_nowait(tmem + kDxAcc + 64 * b + 32 + lane_base, v1);
          tmem_ld_wait();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dxempty[b]);
        if (leader && p < 4) TRACE3(64 + p);
        // rows 64-127 (the W_lo part) -> staging buffer p % 2; rows 0-63 add
        // theirs in place (each thread one input channel: 32 pixels per
        // block, the row it alone touches) and one TMA store per block writes
        // the pair (the SWIZZLE_128B staging is the store's box).  Leader:
        // the stores of pair p-2 have finished reading buffer p % 2 before
        // the first barrier releases its writers.
        if (leader) bulk_wait_read<1>();
        if (leader && p < 4) TRACE3(68 + p);
        named_bar_sync(1, 128);
        if (leader && p < 4) TRACE3(72 + p);
        const uint32_t r0 = smem_u32(smem + L.stg + b * 2 * L.stgb + dx_row * 128), r1 = r0 + L.stgb;
        if (bottom && dx_warp && dx_live) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            sts_v4(r0 + ((j ^ (dx_row & 7)) << 4), f4(v0 + 4 * j));
            sts_v4(r1 + ((j ^ (dx_row & 7)) << 4), f4(v1 + 4 * j));
          }
        }
        named_bar_sync(1, 128);
        if (leader && p < 4) TRACE3(76 + p);
        if (!bottom) {
          if (dx_warp && dx_live) {
            // all 16 loads in flight before the first store (the shared-memory
            // accesses are volatile: load-store pairs serialise the round
            // trips, ~0.3-0.5 us each under the MMA / TMA traffic); the sums
            // overwrite the staged W_lo half in place
            float4 o[16];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              o[j] = lds_v4(r0 + ((j ^ (dx_row & 7)) << 4));
              o[8 + j] = lds_v4(r1 + ((j ^ (dx_row & 7)) << 4));
            }
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const uint32_t* vv = k == 0 ? v0 : v1;
              const uint32_t rk = k == 0 ? r0 : r1;
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 m = f4(vv + 4 * j), q4 = o[8 * k + j];
                sts_v4(rk + ((j ^ (dx_row & 7)) << 4), make_float4(m.x + q4.x, m.y + q4.y, m.z + q4.z, m.w + q4.w));
              }
            }
          }
          fence_proxy_async_smem();
          if (leader && p < 4) TRACE3(80 + p);
          named_bar_sync(2, 64);
          if (leader) {
            for (int k = 0; k < nb; ++k) {
              const int u = blk_u(a, sl, 2 * p + k);
              const int n = u / a.nbps, px0 = (u - n * a.nbps) * 32;
              tma_store_3d(&tdx, smem + L.stg + (2 * b + k) * L.stgb, px0, 0, n);
            }
            bulk_commit();
          }
        }
        if (leader) TRACE3K(40, p);
      }
    }
    if (leader) {
      bulk_wait<0>();
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
  if (n > 128 + 512) n = 128 + 512;
  const int m = n < 128 ? n : 128;
  if (cudaMemcpyFromSymbol(out, g_trace3, m * sizeof(unsigned long long)) != cudaSuccess) return -1;
  if (n > 128 && cudaMemcpyFromSymbol(out + 128, g_cta3, (n - 128) * sizeof(unsigned long long)) != cudaSuccess)
    return -1;
  return n;
#else
  for (int i = 0; i < n; ++i) out[i] = 0;
  return n;
#endif
}

bool tc_bwd_supported(const TcWeightPlan& tw, int64_t n, int64_t plane, int32_t c_in, int32_t c_out,
                      int32_t gw) {
  if (!tw.ok || plane % 4 != 0 || tw.n_rt != 1 || tw.rt_info.size() < 2) return false;
  // dW accumulation chain of a slice (2 K = 16 steps per 32-pixel block, one
  // slice per CTA): at most 768 steps, as the generation-1 weight kernel
  // bounds its splits (each MMA rounds the running sum toward zero); larger
  // problems take the two-kernel backward.
  if ((n * ((plane + 31) / 32) + kSlices - 1) / kSlices * 2 > 768) return false;
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
    if (!encode_f32(&tdy, call.dy, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  }
  const uint64_t dimx[3] = {P, static_cast<uint64_t>(call.c_in), static_cast<uint64_t>(call.n)};
  const uint64_t strx[2] = {P * 4, P * 4 * call.c_in};
  if (a.do_dw) {
    const uint32_t box[3] = {32, static_cast<uint32_t>(a.xbox ? g.nx : tw.rbb), 1};
    if (!encode_f32(&tx, call.x, 3, dimx, strx, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
  }
  CUtensorMap tdx{};
  if (a.do_dx) {
    const uint64_t dimd[3] = {P, static_cast<uint64_t>(call.c_in), static_cast<uint64_t>(call.n)};
    const uint32_t box[3] = {32, static_cast<uint32_t>(call.c_in), 1};
    if (!encode_f32(&tdx, call.dx, 3, dimd, strx, box, CU_TENSOR_MAP_SWIZZLE_128B)) return cudaErrorInvalidValue;
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_bwd_kernel, tdy, tx, tdx, a);
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
