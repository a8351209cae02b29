// Tensor-core band kernel, generation 2 (tcgen05, 3xTF32), sm_100a.
//
// Forward (kernel.cpp:29-69) and input-centric backward-data
// (kernel.cpp:98-138) as one banded GEMM per 128-pixel tile:
//     D[p, r] = sum_{k in arc(row tile)} A[k, p] * B[r, k]
//   forward:       A = x rows (ring = input channels),            B = W band
//   backward-data: A = dy rows (ring = filters, cycle-sorted),    B = W band^T
// M = 128 pixels (TMEM lanes), N = NT output rows (TMEM columns), K = the row
// tile's arc of the ring, 8 ring rows per MMA k-step.
//
// Design (measured on B200):
//   * The weight panel (hi/lo tf32 images, K-major SWIZZLE_128B) is built by
//     the CTA itself in shared memory from the [oc][k] weights: a call is ONE
//     launch, with no panel kernel and no panel scratch in HBM.
//   * Activations land by TMA as [ring row][32 px] 128 B rows; converter warps
//     split them into tf32 hi/lo and transpose them into TMEM ([pixel lane][ring
//     column]), so the MMAs run in TS mode (A from TMEM) and only the panel is
//     read from shared memory.  Every byte on the SM goes through the same
//     128 B/clk SRAM port (TMA writes, LDS/STS, the tensor core's smem operand
//     reads, TMA-store reads); SS-mode MMAs at N=128 alone would saturate it.
//   * Each CTA owns a contiguous run of 32-pixel blocks (balanced to one block
//     across the grid); runs are cut into tiles of up to 4 blocks.
//   * Small per-layer tables (row-tile arcs, TMA class coordinates) ride in the
//     kernel parameters, so the producer issues its first load as soon as the
//     grid dependency resolves.
//   * The epilogue drains TMEM and writes each warp's pixel block of the tile
//     with ONE TMA store (whole-tile box) when the row set allows.
//
// 3xTF32: the tensor core truncates raw fp32 operands to tf32
// (tests/test_tc_probe.py), so with A_hi = trunc(A), A_lo = A - A_hi and the
// panel holding B_hi / B_lo the three MMAs per k-step
//     A_hi*B_hi + A_lo*B_hi + A_hi*B_lo
// reproduce the fp32 product up to the dropped A_lo*B_lo term (~2^-22).
//
// Warp roles (one CTA per SM, 384 threads):
//   warp 0      TMA producer (raw activation ring)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2-7   build the weight panel (each 16 B panel word gathered once)
//   warps 4-7   then convert: raw stage -> TMEM A_hi / A_lo, warp q owns the
//               pixel block q (TMEM lanes 32q..32q+31)
//   warps 8-11  epilogue: TMEM lane quarter q = pixel block q of the tile
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
// per-CTA start / epilogue-end stamps; scripts/band_timing.py reads them.
#if defined(SCC_TRACE)
__device__ unsigned long long g_trace2[64];
__device__ unsigned long long g_cta2[2 * 1024];
#define TRACE2(slot)                                         \
  do {                                                       \
    if (blockIdx.x == 0) g_trace2[(slot)] = globaltimer();   \
  } while (0)
#define CTA_STAMP(k)                                                          \
  do {                                                                        \
    if (blockIdx.x < 1024) g_cta2[2 * blockIdx.x + (k)] = globaltimer();      \
  } while (0)
#else
#define TRACE2(slot) \
  do {               \
  } while (0)
#define CTA_STAMP(k) \
  do {               \
  } while (0)
#endif

constexpr int kThreads = 384;
// dsc_block fusion: the depthwise stage quadruples the converters' work, so
// a second converter set (warps 12..15, same TMEM lane quarters as 4..7)
// takes the upper 16 rows of every stage
constexpr int kDscThreads = 512;
constexpr int kDwStride = 12;                  // depthwise table row: 9 taps, bias, 2 pad (3 x 16 B)
constexpr int kBlkPx = 32;                     // pixels per block (one 128 B row)
constexpr int kStageBytes = 32 * 128 * 4;      // [32 ring rows][128 px]
constexpr int kMaxStages = 8;
constexpr int kTStages = 4;                    // TMEM A stages (hi + lo, 64 columns each)
constexpr int kWorkers = 192;                  // warps 2, 3, 8..11: panel builders
constexpr int kSmemLimit = 227 * 1024;
constexpr int kStoreBuf = 32 * 32 * 4;         // one [32 rows][32 px] TMA-store box
constexpr int kStoreBufs = 2;                  // per epilogue warp (32-row mode)
// Epilogue store modes.
enum : int32_t {
  kStoreStg = 0,    // plain per-row stores (ragged row sets)
  kStoreRows32 = 1, // [32 rows][32 px] boxes
};
constexpr int kMaxScratch = 32 * 1024;         // W + oc tables staged for the panel build
constexpr int kMaxRt = 16;                     // row tiles / classes carried in the params
constexpr int kMaxCls = 64;

__host__ __device__ inline int pad4(int v) { return (v + 3) & ~3; }

struct Band2Args {
  const float* weight;       // [c_out][gw]
  const float* bias;         // forward only (nullable)
  float* out;
  const int32_t* rows;       // [n_rt*NT] output channel per tile row, -1 = none
  const int32_t* perm;       // cycle-sorted position -> oc
  const int32_t* inv_perm;   // oc -> cycle-sorted position
  const int32_t* starts;     // oc -> window start
  int32_t rt_start8[kMaxRt], rt_nk8[kMaxRt], rt_cb[kMaxRt + 1];
  int32_t class_d[kMaxCls], out_class_d[kMaxCls];
  int32_t n_rt, ring, cls, rb;
  int32_t c_in, c_out, gw, c_out_t;
  int32_t store_mode, out_cls;  // kStore*; class run length of the output view
  int32_t w_staged;          // W + oc tables bulk-copied to smem for the panel build
  int32_t fwd4;              // forward panel words are whole-window or empty (build_panel_fwd4)
  int32_t nbps;              // 32-pixel blocks per sample
  int32_t stages;            // raw ring depth
  int32_t scratch;           // panel-build scratch bytes (W, starts, perm) in the staging area
  int32_t total_chunks;
  int32_t units;             // n * nbps
  int64_t plane;
  // fused dsc_block forward (DSC instantiation): stage rows carry a halo of
  // one image row (img_w px) before and after the tile's 128 px
  const float* dsc_w;        // [c_in][9]
  const float* dsc_b;        // [c_in] or nullptr
  float* dsc_t;              // [n][c_in][plane] or nullptr
  int32_t img_w;             // image width = halo
  int32_t stage_bytes;       // raw stage: 32 rows x (128 + 2 halo) px x 4 B
};

// This CTA's block range [u, u1) (see TileIter).  Not inlined: every warp
// role builds a TileIter, and four inlined copies of the division code were
// ~1,000 instructions of the kernel's ~3,900.
__device__ __noinline__ int2 tile_range(const Band2Args& a) {
  // Whole tiles, evenly: tile t = (sample t / tps, blocks 4 (t % tps) ..);
  // a CTA's run [t0, t1) maps to the block run TileIter cuts back into
  // exactly those tiles (tiles never straddle a sample).
  const int32_t tps = (a.nbps + 3) >> 2;  // tiles per sample
  const int32_t ns = a.nbps > 0 ? a.units / a.nbps : 0;
  const int64_t tiles = static_cast<int64_t>(ns) * tps;
  int64_t t0, t1;
  if (tiles < (1 << 22)) {
    // 32-bit division when the products fit (the 64-bit one is a slow call)
    t0 = (blockIdx.x * static_cast<uint32_t>(tiles)) / gridDim.x;
    t1 = ((blockIdx.x + 1) * static_cast<uint32_t>(tiles)) / gridDim.x;
  } else {
    t0 = (static_cast<int64_t>(blockIdx.x) * tiles) / gridDim.x;
    t1 = (static_cast<int64_t>(blockIdx.x + 1) * tiles) / gridDim.x;
  }
  const int32_t s0 = static_cast<int32_t>(t0 / tps), s1 = static_cast<int32_t>(t1 / tps);
  const int32_t j0 = static_cast<int32_t>(t0 - static_cast<int64_t>(s0) * tps);
  const int32_t j1 = static_cast<int32_t>(t1 - static_cast<int64_t>(s1) * tps);
  return make_int2(s0 * a.nbps + min(4 * j0, a.nbps), s1 * a.nbps + min(4 * j1, a.nbps));
}

// Contiguous run of blocks owned by this CTA, cut into tiles of <= 4 blocks
// that never straddle a sample.  A tile costs one pass of the load / convert /
// MMA / store pipeline whatever its width, so the runs are whole tiles,
// ceil(tiles / grid) at most per CTA: on config 1 every CTA has <= 2 tiles
// (an even split of the flat block range gave 22 % of the CTAs a run across a
// sample boundary and 3 tiles); at 64 -> 64, 32x32, N = 128, 7 (cutting runs
// inside samples, floor(grid / n) or one more per sample, gave 8).
struct TileIter {
  int32_t u, u1, nbps;
  int32_t n, b0, cnt;
  __device__ explicit TileIter(const Band2Args& a) {
    const int2 r = tile_range(a);
    u = r.x;
    u1 = r.y;
    nbps = a.nbps;
    n = b0 = cnt = 0;
  }
  __device__ bool next() {
    if (u >= u1) return false;
    n = u / nbps;
    b0 = u - n * nbps;
    cnt = min(min(4, nbps - b0), u1 - u);
    u += cnt;
    return true;
  }
};

__device__ __forceinline__ void advance(int& stage, uint32_t& phase, int stages) {
  if (++stage == stages) {
    stage = 0;
    phase ^= 1u;
  }
}

// Smem layout (host and device agree): panel | raw ring | store staging (also
// the panel-build scratch: W, starts, perm) | rows[n_rt*NT] | bias[n_rt*NT] |
// barriers.
template <int NT>
struct Layout {
  int panel, raw, st, st_warp, rows, bias, dwt, bars, total;
  // stage_bytes: one raw stage (kStageBytes, or more with the dsc halo);
  // dw_floats: the dsc_block's depthwise table (c_in x 10) or 0
  __host__ __device__ Layout(int total_chunks, int stages, int n_rt, int mode, int stage_bytes, int scratch,
                             int dw_floats = 0) {
    panel = 0;
    raw = panel + total_chunks * 2 * NT * 128;
    st = raw + stages * stage_bytes;
    st_warp = mode == kStoreRows32 ? kStoreBufs * kStoreBuf : 0;
    const int stb = 4 * st_warp > scratch ? 4 * st_warp : scratch;
    rows = st + ((stb + 1023) & ~1023);
    bias = rows + 4 * n_rt * NT;
    dwt = bias + 4 * n_rt * NT;
    bars = dwt + 4 * ((dw_floats + 3) & ~3);
    total = bars + (2 * kMaxStages + 2 * kTStages + 7) * 8 + 16;
  }
};

// Gather-build the band weight panel, hi and lo tf32 images in the K-major
// SWIZZLE_128B layout.  One lane owns one 16 B word (4 consecutive k of one
// row): 2 STS.128 per lane.  Work is processed in batches of kB warp items
// with every shared-memory load of the batch issued before its stores.
//   forward:        warp item = (chunk, 4 rows); lane = (row, word).  Each
//                   row is one filter: its window offset is per lane, the W
//                   reads are 4 consecutive slots.
//   backward-data:  warp item = (chunk, word, 32 rows); lane = row (input
//                   channel).  The 4 filters of the word are warp-uniform.
// W / starts / perm come from shared memory (staged) or global memory.
template <int NT, bool BWD, typename WP, typename IP>
__device__ __forceinline__ void build_panel(const Band2Args& a, uint8_t* panel, const int32_t* rows_s,
                                            WP wsrc, IP stt, IP prm, int ct) {
  constexpr int kPanelChunk = 2 * NT * 128;
  constexpr int kB = 4;
  constexpr int kWarps = kWorkers / 32;
  const int lane = ct & 31, wid = ct >> 5;
  const uint32_t pbase = smem_u32(panel);
  for (int rt = 0; rt < a.n_rt; ++rt) {
    const int cb = a.rt_cb[rt], nch = a.rt_cb[rt + 1] - cb;
    const int lim = 8 * a.rt_nk8[rt], start8 = a.rt_start8[rt];
    const int32_t* rrow = rows_s + rt * NT;
    if constexpr (!BWD) {
      const int items = nch * (NT / 4);
      const int rs = lane >> 3, q16 = lane & 7;
      for (int i0 = wid; i0 < items; i0 += kB * kWarps) {
        int ch[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int it = min(i0 + b * kWarps, items - 1);
          ch[b] = rrow[(it % (NT / 4)) * 4 + rs];
        }
        int st[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) st[b] = stt[ch[b] < 0 ? 0 : ch[b]];
        float w[kB][4];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int it = min(i0 + b * kWarps, items - 1);
          const int kk0 = 32 * (it / (NT / 4)) + 4 * q16;
          int ic = start8 + kk0;
          ic -= ic >= a.ring ? a.ring : 0;
          int sl0 = ic - st[b];
          sl0 += sl0 < 0 ? a.c_in : 0;
          const int base = (ch[b] < 0 ? 0 : ch[b]) * a.gw;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            int sl = sl0 + i;
            sl -= sl >= a.c_in ? a.c_in : 0;
            const bool ok = ch[b] >= 0 && kk0 + i < lim && sl < a.gw;
            const float v = wsrc[base + (ok ? sl : 0)];
            w[b][i] = ok ? v : 0.f;
          }
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int it = i0 + b * kWarps;
          if (it < items) {
            const int c = it / (NT / 4), r = (it - c * (NT / 4)) * 4 + rs;
            float4 h, l;
            h.x = tf32_hi(w[b][0]); l.x = w[b][0] - h.x;
            h.y = tf32_hi(w[b][1]); l.y = w[b][1] - h.y;
            h.z = tf32_hi(w[b][2]); l.z = w[b][2] - h.z;
            h.w = tf32_hi(w[b][3]); l.w = w[b][3] - h.w;
            const uint32_t img = pbase + (cb + c) * kPanelChunk;
            const uint32_t off = (r >> 3) * 1024 + (r & 7) * 128 + ((q16 ^ (r & 7)) << 4);
            sts_v4(img + off, h);
            sts_v4(img + NT * 128 + off, l);
          }
        }
      }
    } else {
      constexpr int kRb = NT / 32;  // 32-row blocks per tile
      const int items = nch * 8 * kRb;
      for (int i0 = wid; i0 < items; i0 += kB * kWarps) {
        int ic[kB], oc[kB][4];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int it = min(i0 + b * kWarps, items - 1);
          const int kw = it / kRb;  // chunk * 8 + word
          ic[b] = rrow[(it % kRb) * 32 + lane];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            int pos = start8 + 4 * kw + i;
            pos -= pos >= a.ring ? a.ring : 0;
            oc[b][i] = prm[pos < a.ring ? pos : 0];
          }
        }
        int st[kB][4];
#pragma unroll
        for (int b = 0; b < kB; ++b)
#pragma unroll
          for (int i = 0; i < 4; ++i) st[b][i] = stt[oc[b][i]];
        float w[kB][4];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int it = min(i0 + b * kWarps, items - 1);
          const int kw = it / kRb;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            int sl = (ic[b] < 0 ? 0 : ic[b]) - st[b][i];
            sl += sl < 0 ? a.c_in : 0;
            const bool ok = ic[b] >= 0 && 4 * kw + i < lim && sl < a.gw;
            const float v = wsrc[oc[b][i] * a.gw + (ok ? sl : 0)];
            w[b][i] = ok ? v : 0.f;
          }
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int it = i0 + b * kWarps;
          if (it < items) {
            const int kw = it / kRb, c = kw >> 3, q16 = kw & 7;
            const int r = (it % kRb) * 32 + lane;
            float4 h, l;
            h.x = tf32_hi(w[b][0]); l.x = w[b][0] - h.x;
            h.y = tf32_hi(w[b][1]); l.y = w[b][1] - h.y;
            h.z = tf32_hi(w[b][2]); l.z = w[b][2] - h.z;
            h.w = tf32_hi(w[b][3]); l.w = w[b][3] - h.w;
            const uint32_t img = pbase + (cb + c) * kPanelChunk;
            const uint32_t off = (r >> 3) * 1024 + (r & 7) * 128 + ((q16 ^ (r & 7)) << 4);
            sts_v4(img + off, h);
            sts_v4(img + NT * 128 + off, l);
          }
        }
      }
    }
  }
}

// Forward panel fast path: when every window start and gw are multiples of 4,
// each 16 B panel word (4 consecutive input channels) lies wholly inside or
// wholly outside its filter's window, so it is one 16 B load of W (staged in
// smem) or zero.  Lane = (row, word); a warp covers 4 rows of one chunk.
template <int NT>
__device__ __forceinline__ void build_panel_fwd4(const Band2Args& a, uint8_t* panel,
                                                 const int32_t* rows_s, const float* w_s,
                                                 const int32_t* start_s, int ct) {
  constexpr int kPanelChunk = 2 * NT * 128;
  constexpr int kWarps = kWorkers / 32;
  const int lane = ct & 31, wid = ct >> 5;
  const int rs = lane >> 3, q16 = lane & 7;
  const uint32_t pbase = smem_u32(panel);
  for (int rt = 0; rt < a.n_rt; ++rt) {
    const int cb = a.rt_cb[rt], nch = a.rt_cb[rt + 1] - cb;
    const int lim = 8 * a.rt_nk8[rt], start8 = a.rt_start8[rt];
    const int items = nch * (NT / 4);
#pragma unroll 4
    for (int it = wid; it < items; it += kWarps) {
      const int c = it / (NT / 4), r = (it - c * (NT / 4)) * 4 + rs;
      const int ch = rows_s[rt * NT + r];
      const int chs = ch < 0 ? 0 : ch;
      const int kk0 = 32 * c + 4 * q16;
      int sl0 = start8 + kk0 - start_s[chs];  // ring = c_in in the forward direction
      sl0 += sl0 < 0 ? a.c_in : 0;
      sl0 -= sl0 >= a.c_in ? a.c_in : 0;
      const bool ok = ch >= 0 && kk0 < lim && sl0 < a.gw;
      float4 v = *reinterpret_cast<const float4*>(w_s + chs * a.gw + (ok ? sl0 : 0));
      if (!ok) v = make_float4(0.f, 0.f, 0.f, 0.f);
      float4 h, l;
      h.x = tf32_hi(v.x); l.x = v.x - h.x;
      h.y = tf32_hi(v.y); l.y = v.y - h.y;
      h.z = tf32_hi(v.z); l.z = v.z - h.z;
      h.w = tf32_hi(v.w); l.w = v.w - h.w;
      const uint32_t img = pbase + (cb + c) * kPanelChunk;
      const uint32_t off = (r >> 3) * 1024 + (r & 7) * 128 + ((q16 ^ (r & 7)) << 4);
      sts_v4(img + off, h);
      sts_v4(img + NT * 128 + off, l);
    }
  }
}

template <int NT, bool BWD, bool DSC>
__global__ void __launch_bounds__(DSC ? kDscThreads : kThreads, 1)
    tc_band2_kernel(const __grid_constant__ CUtensorMap t1, const __grid_constant__ CUtensorMap tout,
                    const __grid_constant__ Band2Args a) {
  constexpr int kPanelChunk = 2 * NT * 128;  // hi + lo image of one 32-k chunk
  constexpr uint32_t kACol0 = 2 * NT;        // TMEM: [0, 2NT) accumulators, then A stages
  // No static shared memory in this kernel: the dynamic window starts
  // 1024-aligned and every derived pointer stays in the shared address space.
  extern __shared__ __align__(1024) uint8_t smem[];
  static_assert(!(BWD && DSC), "the dsc_block fusion is a forward");
  const int stage_bytes = DSC ? a.stage_bytes : kStageBytes;  // compile-time unless fused
  const Layout<NT> L(a.total_chunks, a.stages, a.n_rt, a.store_mode, stage_bytes, a.scratch,
                     DSC ? kDwStride * a.c_in : 0);
  uint8_t* panel = smem + L.panel;
  uint8_t* raw = smem + L.raw;
  uint8_t* stbuf = smem + L.st;
  int32_t* rows_s = reinterpret_cast<int32_t*>(smem + L.rows);
  float* bias_s = reinterpret_cast<float*>(smem + L.bias);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bars);
  uint64_t* full = bars;                   // raw stage landed (TMA)
  uint64_t* afree = bars + kMaxStages;     // 4 converter warps done reading it
  uint64_t* conv = afree + kMaxStages;     // TMEM A stage written (4 converter warps)
  uint64_t* tfree = conv + kTStages;       // MMAs done with the TMEM A stage
  uint64_t* tfull = tfree + kTStages;      // [2] accumulator complete
  uint64_t* tempty = tfull + 2;            // [2] accumulator drained (4 epilogue warps)
  uint64_t* panel_bar = tempty + 2;
  uint64_t* tab_bar = panel_bar + 1;
  uint64_t* w_bar = tab_bar + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(w_bar + 1);
  // Panel-build scratch in the store staging (dead until the first epilogue).
  float* w_s = reinterpret_cast<float*>(stbuf);
  int32_t* start_s = reinterpret_cast<int32_t*>(stbuf) + pad4(a.c_out * a.gw);
  int32_t* perm_s = start_s + pad4(a.c_out);

  const uint32_t warp = warp_id();
  const int lane = threadIdx.x & 31;
  // barrier init spread over the first warp (one mbarrier per lane)
  if (threadIdx.x < 32) {
    const int i = threadIdx.x;
    if (i < kMaxStages) {
      mbar_init(&full[i], 1);
      mbar_init(&afree[i], DSC ? 8 : 4);
    } else if (i < kMaxStages + kTStages) {
      mbar_init(&conv[i - kMaxStages], DSC ? 8 : 4);
      mbar_init(&tfree[i - kMaxStages], 1);
    } else if (i < kMaxStages + kTStages + 2) {
      mbar_init(&tfull[i - kMaxStages - kTStages], 1);
      mbar_init(&tempty[i - kMaxStages - kTStages], 4);
    } else if (i == 16) {
      mbar_init(panel_bar, 1);
    } else if (i == 17) {
      mbar_init(tab_bar, 1);
    } else if (i == 18) {
      mbar_init(w_bar, 1);
    }
    fence_mbar_init();
    __syncwarp();
  }
  if (threadIdx.x == 0) {
    TRACE2(0);
    CTA_STAMP(0);
    TRACE2(40);
    // Plan tables are constant per layer (never written by a preceding
    // kernel), so they load before the grid dependency wait.
    const uint32_t b_rows = 4u * a.n_rt * NT;
    const uint32_t b_oc = a.w_staged ? 4u * pad4(a.c_out) : 0u;
    const uint32_t b_perm = BWD ? b_oc : 0u;
    mbar_expect_tx(tab_bar, b_rows + b_oc + b_perm);
    bulk_load(rows_s, a.rows, b_rows, tab_bar);
    if (b_oc) bulk_load(start_s, a.starts, b_oc, tab_bar);
    if (b_perm) bulk_load(perm_s, a.perm, b_perm, tab_bar);
    TRACE2(41);
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&t1);
    prefetch_tmap(&tout);
  }
  if (warp == 1) {
    tmem_alloc<512>(tmem_slot);
    if (lane == 0) TRACE2(42);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 32) TRACE2(43);
  // Let the next kernel in the stream start its prologue; it waits for this
  // grid's completion before touching memory (griddepcontrol.wait).
  cudaTriggerProgrammaticLaunchCompletion();

  if (warp == 0) {
    // ---------------- producer ----------------
    // The lanes issue a stage's boxes in parallel (one TMA instruction holds
    // its issuing thread ~0.1-0.3 us under load; a stage is up to 4 boxes).
    {
      TileIter it(a);
      bool have = it.next();  // tile geometry needs no input data: before the wait
      if (lane == 0) TRACE2(44);
      cudaGridDependencySynchronize();
      if (lane == 0) TRACE2(1);
      int s = 0;
      uint32_t ph = 0;
      for (; have; have = it.next()) {
        for (int rt = 0; rt < a.n_rt; ++rt) {
          const int start8 = a.rt_start8[rt], nk8 = a.rt_nk8[rt];
          const int nch = (nk8 + 3) >> 2;
          for (int c = 0; c < nch; ++c) {
            mbar_wait(&afree[s], ph ^ 1u);
            const int rows = min(4, nk8 - 4 * c) * 8;
            // One box {128 px, rb rows} per rb rows: stage = [32 rows][128 px].
            // A partial tile over-reads the neighbour's pixels (or zero-fills
            // past the end of the sample); the epilogue never stores them.
            // (dsc: rows of 128 + 2 halo px from one image row before the
            // tile; out-of-sample pixels are zero-filled by TMA -- the
            // depthwise stage's top / bottom padding)
            const int rowb = stage_bytes / 32;
            if (lane == 0) mbar_expect_tx(&full[s], rows * rowb);
            __syncwarp();
            uint8_t* st = raw + s * stage_bytes;
            const int r = lane * a.rb;
            if (r < rows) {
              int pos = start8 + 32 * c + r;
              while (pos >= a.ring) pos -= a.ring;
              const int cl = pos / a.cls, j = pos - cl * a.cls;
              tma_load_4d(st + r * rowb, &t1, &full[s], it.b0 * kBlkPx - (DSC ? a.img_w : 0), j, a.class_d[cl],
                          it.n);
            }
            __syncwarp();
            if (c == 0 && lane == 0) TRACE2(2);
            advance(s, ph, a.stages);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (A from TMEM, B = panel from smem) ----------------
    constexpr uint32_t idesc = idesc_tf32(128, NT, 0, 0);
    int st = 0, acc = 0;
    uint32_t tph = 0, aph = 0;
    mbar_wait(panel_bar, 0);
    tc_fence_after();
    TileIter it(a);
    int ti = 0;
    while (it.next()) {
      for (int rt = 0; rt < a.n_rt; ++rt) {
        const int nk8 = a.rt_nk8[rt];
        const int nch = (nk8 + 3) >> 2;
        const int cb = a.rt_cb[rt];
        mbar_wait(&tempty[acc], aph ^ 1u);
        tc_fence_after();
        const uint32_t d_tmem = tmem + acc * NT;
        for (int c = 0; c < nch; ++c) {
          mbar_wait(&conv[st], tph);
          tc_fence_after();
          if (elect_one()) {
            const int steps = min(4, nk8 - 4 * c);
            const uint32_t a_hi = tmem + kACol0 + st * 64, a_lo = a_hi + 32;
            const uint32_t bh = smem_u32(panel + (cb + c) * kPanelChunk), bl = bh + NT * 128;
            for (int k = 0; k < steps; ++k) {
              const uint64_t dbh = desc_sw128(bh + k * 32, 16, 1024);
              const uint64_t dbl = desc_sw128(bl + k * 32, 16, 1024);
              mma_tf32_ts(d_tmem, a_hi + 8 * k, dbh, idesc, (c | k) != 0);
              mma_tf32_ts(d_tmem, a_lo + 8 * k, dbh, idesc, 1);
              mma_tf32_ts(d_tmem, a_hi + 8 * k, dbl, idesc, 1);
            }
            mma_commit(&tfree[st]);
            if (c == nch - 1) mma_commit(&tfull[acc]);
          }
          __syncwarp();
          advance(st, tph, kTStages);
        }
        if (ti < 8) TRACE2(6 + ti);
        ++ti;
        if (++acc == 2) {
          acc = 0;
          aph ^= 1u;
        }
      }
    }
  } else {
    if (warp < 4 || (warp >= 8 && (!DSC || warp < 12))) {
      // ---------------- panel build (warps 2, 3, 8..11; the converters start at once) ----------------
      const int ct = warp < 4 ? threadIdx.x - 64 : threadIdx.x - 192;  // 0..191
      cudaGridDependencySynchronize();  // W may come from the previous kernel
      if (ct == 0 && a.w_staged) {
        const uint32_t bytes = 4u * a.c_out * a.gw;
        mbar_expect_tx(w_bar, bytes);
        bulk_load(w_s, a.weight, bytes, w_bar);
      }
      mbar_wait(tab_bar, 0);
      if (a.w_staged) mbar_wait(w_bar, 0);
      if constexpr (BWD) {
        if (a.w_staged)
          build_panel<NT, true>(a, panel, rows_s, w_s, start_s, perm_s, ct);
        else
          build_panel<NT, true>(a, panel, rows_s, a.weight, a.starts, a.perm, ct);
      } else {
        if (a.fwd4)
          build_panel_fwd4<NT>(a, panel, rows_s, w_s, start_s, ct);
        else if (a.w_staged)
          build_panel<NT, false>(a, panel, rows_s, w_s, start_s, perm_s, ct);
        else
          build_panel<NT, false>(a, panel, rows_s, a.weight, a.starts, a.perm, ct);
      }
      if constexpr (DSC) {
        // the dsc_block's depthwise taps and bias, [c_in][12] (converters)
        float* dwt = reinterpret_cast<float*>(smem + L.dwt);
        for (int i = ct; i < kDwStride * a.c_in; i += kWorkers) {
          const int ch = i / kDwStride, k = i - kDwStride * ch;
          dwt[i] = k < 9 ? __ldg(a.dsc_w + 9 * ch + k) : (k == 9 && a.dsc_b != nullptr ? __ldg(a.dsc_b + ch) : 0.f);
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(1, kWorkers);
      if (ct == 0) {
        TRACE2(3);
        mbar_arrive(panel_bar);
      }
    }
    if ((warp >= 4 && warp < 8) || (DSC && warp >= 12)) {
      // ---------------- converters: raw [row][px] -> TMEM [px lane][row] hi / lo ----------------
      const int q = warp & 3;  // pixel block of the tile = TMEM lane quarter
      const int half = DSC && warp >= 12 ? 1 : 0;  // dsc: rows 16 * half .. + 15 of each stage
      const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
      int s = 0, st = 0;
      uint32_t ph = 0, tph = 0;
      const float* dwt = reinterpret_cast<const float*>(smem + L.dwt);
      if (DSC) mbar_wait(panel_bar, 0);  // the depthwise table is staged with the panel
      TileIter it(a);
      while (it.next()) {
        // dsc: this lane's pixel and its column masks (the depthwise stage's
        // left / right padding; rows come zero-filled from TMA)
        const int pix = it.b0 * kBlkPx + q * 32 + lane;
        const bool pv = q < it.cnt && pix < a.plane;
        const int col = DSC ? (pix & (a.img_w - 1)) : 0;
        // (selects, not weight x 0: the corner taps of the stage's first and
        // last pixel read outside the stage, and 0 x NaN is NaN)
        const bool ml = col > 0, mr = col < a.img_w - 1;
        for (int rt = 0; rt < a.n_rt; ++rt) {
          const int nk8 = a.rt_nk8[rt];
          const int nch = (nk8 + 3) >> 2;
          for (int c = 0; c < nch; ++c) {
            mbar_wait(&full[s], ph);
            // Element (row r, pixel 32q + lane) of the [32 rows][128 px] stage.
            // Rows past the chunk's k-steps hold stale data that lands in TMEM
            // columns the MMAs never read.
            if constexpr (DSC) {
              // t = DW3x3(x) for ring rows (channels, n_class == 1: channel =
              // ring position) 32c + 16 half.., from the haloed stage; t is
              // also the block's stored activation (the backward's SCC input)
              uint32_t hi[16], lo[16];
              const int W = a.img_w, SW = 128 + 2 * W;
              const float* src = reinterpret_cast<const float*>(raw + s * a.stage_bytes) + (16 * half) * SW + W +
                                 q * 32 + lane;
              const int ch0 = a.rt_start8[rt] + 32 * c + 16 * half;
              const int rows = min(4, nk8 - 4 * c) * 8 - 16 * half;
              float* tdst = a.dsc_t != nullptr ? a.dsc_t + (static_cast<int64_t>(it.n) * a.c_in + ch0) * a.plane + pix
                                               : nullptr;
#pragma unroll
              for (int r = 0; r < 16; ++r) {
                const float* x0 = src + r * SW;
                const float4* w4 = reinterpret_cast<const float4*>(dwt + kDwStride * min(ch0 + r, a.c_in - 1));
                const float4 wa = w4[0], wb = w4[1], wc = w4[2];
                float v = wc.y;
                v = fmaf(wa.x, ml ? x0[-W - 1] : 0.f, v);
                v = fmaf(wa.y, x0[-W], v);
                v = fmaf(wa.z, mr ? x0[-W + 1] : 0.f, v);
                v = fmaf(wa.w, ml ? x0[-1] : 0.f, v);
                v = fmaf(wb.x, x0[0], v);
                v = fmaf(wb.y, mr ? x0[1] : 0.f, v);
                v = fmaf(wb.z, ml ? x0[W - 1] : 0.f, v);
                v = fmaf(wb.w, x0[W], v);
                v = fmaf(wc.x, mr ? x0[W + 1] : 0.f, v);
                if (tdst != nullptr && pv && r < rows) __stcs(tdst + static_cast<int64_t>(r) * a.plane, v);
                const float h = tf32_hi(v);
                hi[r] = __float_as_uint(h);
                lo[r] = __float_as_uint(v - h);
              }
              __syncwarp();
              if (lane == 0) mbar_arrive(&afree[s]);
              mbar_wait(&tfree[st], tph ^ 1u);
              tc_fence_after();
              const uint32_t col = tmem + kACol0 + st * 64 + lane_base + 16 * half;
              tmem_st16(col, hi);
              tmem_st16(col + 32, lo);
            } else {
              uint32_t hi[32], lo[32];
              const float* src = reinterpret_cast<const float*>(raw + s * kStageBytes) + q * 32 + lane;
#pragma unroll
              for (int r = 0; r < 32; ++r) {
                const float v = src[r * 128];
                const float h = tf32_hi(v);
                hi[r] = __float_as_uint(h);
                lo[r] = __float_as_uint(v - h);
              }
              __syncwarp();
              if (lane == 0) mbar_arrive(&afree[s]);
              mbar_wait(&tfree[st], tph ^ 1u);
              tc_fence_after();
              const uint32_t col = tmem + kACol0 + st * 64 + lane_base;
              tmem_st32(col, hi);
              tmem_st32(col + 32, lo);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&conv[st]);
            advance(s, ph, a.stages);
            advance(st, tph, kTStages);
          }
        }
      }
    }
    if (warp >= 8 && (!DSC || warp < 12)) {
      // ---------------- epilogue (warps 8..11) ----------------
      const int et = threadIdx.x - 256;  // 0..127
      for (int i = et; i < a.n_rt * NT; i += 128) {
        const int row = rows_s[i];
        bias_s[i] = (!BWD && a.bias != nullptr && row >= 0) ? __ldg(a.bias + row) : 0.f;
      }
      named_bar_sync(2, 128);
      const int q = warp & 3;
      int acc = 0, sbuf = 0;
      uint32_t aph = 0;
      TileIter it(a);
      int ti = 0;
      uint8_t* wbuf = stbuf + q * L.st_warp;  // this warp's staging
      const uint32_t wbuf_a = smem_u32(wbuf);
      while (it.next()) {
        const int px = (it.b0 + q) * kBlkPx + lane;
        const bool valid = q < it.cnt && px < a.plane;
        float* obase = a.out + static_cast<int64_t>(it.n) * a.c_out_t * a.plane + px;
        for (int rt = 0; rt < a.n_rt; ++rt) {
          mbar_wait(&tfull[acc], aph);
          tc_fence_after();
          if (q < it.cnt) {
            const uint32_t taddr = tmem + acc * NT + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
            for (int c0 = 0; c0 < NT; c0 += 32) {
              const int g0 = rt * NT + c0;  // first tile row of this 32-row group
              uint32_t v[32];
              tmem_ld32_nowait(taddr + c0, v);
              tmem_ld_wait();
              float bb[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) bb[j] = bias_s[g0 + j];
              if (a.store_mode == kStoreRows32 && g0 + 32 <= a.c_out_t) {
                // Stage [32 rows][32 px] (lanes own consecutive words: no
                // conflicts) and write it with one TMA store; buffers rotate.
                // (A group past the last channel -- a tile wider than the
                // tensor -- takes the per-row path, which skips rows = -1;
                // its class coordinate would be outside the store view.)
                if (lane == 0) bulk_wait_read<kStoreBufs - 1>();
                __syncwarp();
                const uint32_t buf = wbuf_a + sbuf * kStoreBuf + lane * 4;
#pragma unroll
                for (int j = 0; j < 32; ++j) sts_f32(buf + j * 128, __uint_as_float(v[j]) + bb[j]);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                  const int cl = g0 / a.out_cls, jj = g0 - cl * a.out_cls;
                  tma_store_3d(&tout, wbuf + sbuf * kStoreBuf, (it.b0 + q) * kBlkPx, a.out_class_d[cl],
                               it.n * a.out_cls + jj);
                  bulk_commit();
                }
                sbuf = (sbuf + 1) & (kStoreBufs - 1);
              } else if (valid) {
                int32_t rr[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) rr[j] = rows_s[g0 + j];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                  if (rr[j] >= 0) obase[static_cast<int64_t>(rr[j]) * a.plane] = __uint_as_float(v[j]) + bb[j];
                }
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[acc]);
          if (ti < 8 && q == 0 && lane == 0) TRACE2(14 + ti);
          ++ti;
          if (++acc == 2) {
            acc = 0;
            aph ^= 1u;
          }
        }
      }
      if (lane == 0) bulk_wait<0>();
      if (lane == 0 && q == 0) CTA_STAMP(1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

template <int NT>
int band2_stages(const TcBandPlan& tp, int mode, int stage_bytes, int scratch, int dw_floats = 0) {
  int st = kMaxStages;
  while (st >= 2 &&
         1024 + Layout<NT>(tp.total_chunks, st, tp.n_rt, mode, stage_bytes, scratch, dw_floats).total > kSmemLimit)
    --st;
  return st;
}

template <int NT, bool BWD, bool DSC>
cudaError_t launch_tc2_nt(const TcBandPlan& tp, const TcDeviceTables& dt, const TcBandCall& call,
                          int64_t shift, int32_t c_out, cudaStream_t s) {
  const int64_t P = call.plane;
  const int32_t C = tp.cls * tp.n_class;  // channels of the activation tensor
  // Activations {P, cls, n_class, N}, box {128 px (+ 2 halo rows of the
  // image: dsc), rb rows}, no swizzle.
  const int halo = DSC ? call.img_w : 0;
  CUtensorMap t1;
  {
    const uint64_t dims[4] = {static_cast<uint64_t>(P), static_cast<uint64_t>(tp.cls),
                              static_cast<uint64_t>(tp.n_class), static_cast<uint64_t>(call.n)};
    const uint64_t strides[3] = {static_cast<uint64_t>(tp.n_class) * P * 4, static_cast<uint64_t>(P) * 4,
                                 static_cast<uint64_t>(C) * P * 4};
    const uint32_t box[4] = {static_cast<uint32_t>(128 + 2 * halo), static_cast<uint32_t>(tp.rb), 1, 1};
    if (!encode_f32(&t1, call.in, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE))
      return cudaErrorInvalidValue;
  }
  // Output view for TMA stores of 32-row groups: {P, D_out, N * out_cls}
  // (store_ok: every 32 consecutive tile rows are one equally strided class
  // run); otherwise plain per-row stores.
  const bool cls_ok = tp.store_ok && static_cast<int>(tp.out_class_d.size()) <= kMaxCls;
  // 32-row boxes stored as soon as they are staged.  (Whole-tile boxes,
  // one store per warp and tile, measured slower on config 1: 30.3 vs
  // 31.4 us per step -- the stores start a tile later -- and were dropped;
  // so was staging the warp's whole tile and issuing its 4 boxes from 4
  // lanes at once: 10.5 vs 9.6 us per forward.)
  const int32_t mode = cls_ok ? kStoreRows32 : kStoreStg;
  const bool cls_view = mode == kStoreRows32;
  CUtensorMap tout;
  {
    const int32_t ocls = cls_view ? tp.out_cls : call.c_out_t;
    const int32_t ond = cls_view ? tp.out_n_class : 1;
    const uint64_t dims[3] = {static_cast<uint64_t>(P), static_cast<uint64_t>(ond),
                              static_cast<uint64_t>(call.n) * ocls};
    const uint64_t strides[2] = {static_cast<uint64_t>(P) * 4, static_cast<uint64_t>(P) * 4 * ond};
    const uint32_t box[3] = {32, 1, 32};
    if (!encode_f32(&tout, call.out, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE))
      return cudaErrorInvalidValue;
  }
  Band2Args a{};
  a.weight = call.weight;
  a.bias = call.bias;
  a.out = call.out;
  a.rows = dt.rows;
  a.perm = dt.perm;
  a.inv_perm = dt.inv_perm;
  a.starts = dt.starts;
  for (int rt = 0; rt < tp.n_rt; ++rt) {
    a.rt_start8[rt] = tp.rt_info[4 * rt];
    a.rt_nk8[rt] = tp.rt_info[4 * rt + 1];
  }
  for (int rt = 0; rt <= tp.n_rt; ++rt) a.rt_cb[rt] = tp.chunk_base[rt];
  for (size_t i = 0; i < tp.class_d.size(); ++i) a.class_d[i] = tp.class_d[i];
  if (cls_ok)
    for (size_t i = 0; i < tp.out_class_d.size(); ++i) a.out_class_d[i] = tp.out_class_d[i];
  a.store_mode = mode;
  a.out_cls = tp.out_cls;
  a.n_rt = tp.n_rt;
  a.ring = tp.ring;
  a.cls = tp.cls;
  a.rb = tp.rb;
  a.c_in = call.c_in;
  a.c_out = c_out;
  a.gw = call.gw;
  a.c_out_t = call.c_out_t;
  a.nbps = static_cast<int32_t>((P + 31) / 32);
  a.total_chunks = tp.total_chunks;
  // W + starts (+ perm) go to the staging area by bulk copy when they fit and
  // the weight pointer/size suit cp.async.bulk.
  {
    const int64_t wbytes = 4ll * c_out * call.gw;
    const int64_t need = 4ll * (pad4(c_out * call.gw) + 2 * pad4(c_out));
    a.w_staged = (need <= kMaxScratch && wbytes % 16 == 0 &&
                  reinterpret_cast<uintptr_t>(call.weight) % 16 == 0) ? 1 : 0;
    a.scratch = a.w_staged ? static_cast<int32_t>(need) : 0;
    // window starts (oc * shift mod c_in) and arc starts (multiples of 8) are
    // multiples of 4 when shift and c_in are
    a.fwd4 = (!BWD && a.w_staged && call.gw % 4 == 0 && call.c_in % 4 == 0 && shift % 4 == 0) ? 1 : 0;
  }
  a.stage_bytes = 32 * (128 + 2 * halo) * 4;
  a.dsc_w = call.dsc_w;
  a.dsc_b = call.dsc_b;
  a.dsc_t = call.dsc_t;
  a.img_w = call.img_w;
  const int dw_floats = DSC ? kDwStride * call.c_in : 0;
  a.stages = band2_stages<NT>(tp, a.store_mode, a.stage_bytes, a.scratch, dw_floats);
  if (a.stages < 3) return cudaErrorInvalidValue;
  a.plane = P;
  const int64_t units = call.n * a.nbps;
  if (units > (1ll << 30)) return cudaErrorInvalidValue;
  a.units = static_cast<int32_t>(units);
  const int smem =
      1024 + Layout<NT>(a.total_chunks, a.stages, a.n_rt, a.store_mode, a.stage_bytes, a.scratch, dw_floats).total;

  static int nsm_cache[64] = {0};
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  int nsm = 148;
  if (dev >= 0 && dev < 64 && nsm_cache[dev] > 0) {
    nsm = nsm_cache[dev];
  } else {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < 64) nsm_cache[dev] = nsm;
  }
  if (dev < 0 || dev >= 64 || !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(tc_band2_kernel<NT, BWD, DSC>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit);
    if (e != cudaSuccess) return e;
    if (dev >= 0 && dev < 64) attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg{};
  const int64_t cap = call.max_ctas > 0 ? std::min(call.max_ctas, nsm) : nsm;
  cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(a.units, cap)));
  cfg.blockDim = dim3(DSC ? kDscThreads : kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_band2_kernel<NT, BWD, DSC>, t1, tout, a);
  if (e != cudaSuccess) return e;
  note_launches(1);
  return cudaSuccess;
}

}  // namespace

bool tc_band2_supported(const TcBandPlan& tp, int64_t plane, int32_t c_out) {
  (void)c_out;
  if (!tp.ok || plane % 4 != 0 || plane < 4) return false;
  if (tp.rb % 8 != 0 || tp.n_rt > kMaxRt || tp.n_class > kMaxCls) return false;
  // The whole panel stays resident next to >= 4 raw stages.
  const int st = tp.nt == 128 ? band2_stages<128>(tp, kStoreRows32, kStageBytes, kMaxScratch)
                               : band2_stages<64>(tp, kStoreRows32, kStageBytes, kMaxScratch);
  return st >= 4;
}

bool tc_dsc2_supported(const TcBandPlan& tp, int64_t plane, int64_t img_w, int32_t c_in, int32_t c_out) {
  if (!tc_band2_supported(tp, plane, c_out)) return false;
  // (widths 16 and 32: every tile starts at an image column 0 and ends at
  // column w - 1, so a halo of exactly one image row covers every tap)
  if (!(img_w == 16 || img_w == 32) || plane % 128 != 0 || plane % img_w != 0) return false;
  // one row tile whose arc is every input channel once, ring position =
  // channel (the converters index the depthwise table by it).  Several row
  // tiles would each convert their own (overlapping) arc: measured slower
  // than the depthwise kernel + SCC forward pair (128 -> 128 at 16x16,
  // N = 128: 32.3 vs 29.0 us, the converters redoing 1.5x the depthwise work)
  if (tp.n_rt != 1 || tp.n_class != 1 || tp.rt_info.size() < 2 || tp.rt_info[0] != 0 ||
      tp.rt_info[1] * 8 != c_in || tp.ring != c_in)
    return false;
  const int halo_stage = 32 * (128 + 2 * static_cast<int>(img_w)) * 4;
  const int st = tp.nt == 128 ? band2_stages<128>(tp, kStoreRows32, halo_stage, kMaxScratch, kDwStride * c_in)
                               : band2_stages<64>(tp, kStoreRows32, halo_stage, kMaxScratch, kDwStride * c_in);
  return st >= 3;
}

cudaError_t launch_band_tc2(const TcBandPlan& tp, const TcDeviceTables& dt, const TcBandCall& call,
                            int64_t shift, int32_t c_out, cudaStream_t s) {
  const bool bwd = call.backward_data, dsc = call.dsc_w != nullptr;
  if (dsc && bwd) return cudaErrorInvalidValue;
  switch (tp.nt) {
    case 64:
      return bwd ? launch_tc2_nt<64, true, false>(tp, dt, call, shift, c_out, s)
                 : (dsc ? launch_tc2_nt<64, false, true>(tp, dt, call, shift, c_out, s)
                        : launch_tc2_nt<64, false, false>(tp, dt, call, shift, c_out, s));
    case 128:
      return bwd ? launch_tc2_nt<128, true, false>(tp, dt, call, shift, c_out, s)
                 : (dsc ? launch_tc2_nt<128, false, true>(tp, dt, call, shift, c_out, s)
                        : launch_tc2_nt<128, false, false>(tp, dt, call, shift, c_out, s));
    default:
      return cudaErrorInvalidValue;
  }
}

int tc2_trace(unsigned long long* out, int n) {
#if defined(SCC_TRACE)
  if (n > 64 + 2048) n = 64 + 2048;
  const int a = n < 64 ? n : 64;
  if (cudaMemcpyFromSymbol(out, g_trace2, a * sizeof(unsigned long long)) != cudaSuccess) return -1;
  if (n > 64 && cudaMemcpyFromSymbol(out + 64, g_cta2, (n - 64) * sizeof(unsigned long long)) != cudaSuccess)
    return -1;
  return n;
#else
  for (int i = 0; i < n; ++i) out[i] = 0;
  return n;
#endif
}

}  // namespace scc
