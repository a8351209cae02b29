// Tensor-core (tcgen05, 3xTF32) family of the SCC operator, sm_100a.
//
// tc_band_kernel — forward (kernel.cpp:29-69) and input-centric backward-data
// (kernel.cpp:98-138) as one banded GEMM per 128-pixel tile:
//     D[p, r] = sum_{k in arc(r-tile)} A[p, k] * B[k, r]
//   forward:       A = x rows (ring = input channels),      B = W band^T
//   backward-data: A = dy rows (ring = filters, cycle-sorted), B = W band
// M = 128 pixels (TMEM lanes), N = NT rows (TMEM columns), K = the row tile's
// arc of the ring in 8-row steps.  Activations arrive by TMA; the band
// weights arrive pre-split (hi/lo) and pre-swizzled (K-major SWIZZLE_128B) by
// a bulk copy.  fp32 accuracy from three tf32 MMAs per step:
//     A_hi*B_hi + A_lo*B_hi + A_hi*B_lo,  A_hi = A with the low 13 bits dropped
// (the tensor core reads raw fp32 operands that way; tests/test_tc_probe.py).
//
// kind::tf32 only accepts K-major operands (an MN-major A silently yields
// zeros; tests/cuda/tc_layout_probe.cu), and activations are pixel-contiguous,
// so the converter warps transpose each staged [ring][pixel] tile into TMEM
// ([pixel lane][ring column]) as hi/lo parts and the MMA runs in TS mode.
//
// Warp roles (persistent CTA, one per SM):
//   warp 0      TMA / bulk-copy producer
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  converters: smem [k][p] -> TMEM A_hi, A_lo
//   warps 6..9  epilogue: TMEM -> registers -> coalesced NCHW stores (+ bias)
// Accumulators are double-buffered in TMEM so the epilogue of tile i overlaps
// the MMAs of tile i+1.  Every output element is written exactly once.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>

#include "scc_kernels.hpp"
#include "scc_plan.hpp"
#include "sm100.cuh"
#include "tmap.hpp"

namespace scc {
namespace {

using namespace sm100;

// Diagnostic timeline of the last tensor-core band launch (CTA 0 only; ns,
// %globaltimer).  Slots: 0 start, 1 setup done, 2 producer first TMA issued,
// 3 producer dependency satisfied, 4 converter first stage landed,
// 5 MMA first stage converted, 6.. per tile (up to 8): MMA commit of tile i
// at 6+2i, epilogue done with tile i at 7+2i, 30 end.
__device__ unsigned long long g_trace[32];
#if defined(SCC_TRACE)
#define TRACE(slot)                                           \
  do {                                                        \
    if (blockIdx.x == 0) g_trace[(slot)] = globaltimer();     \
  } while (0)
#else
#define TRACE(slot) \
  do {              \
  } while (0)
#endif

constexpr int kTcThreads = 352;  // 11 warps: + a streamed-panel producer
constexpr int KC = 32;          // ring positions per pipeline stage (4 k-steps of 8)
constexpr int TM = 128;         // pixels per tile
constexpr int kABytes = TM * KC * 4;  // 16 KB per A buffer

// BF: bf16x3 (backward-data): the weight image of a chunk is one [NT rows][hi 32
// | lo 32] bf16 K-major SWIZZLE_128B block and a TMEM A stage holds bf16 pairs
// (KC columns instead of 2 KC); the forward (1e-5 bar) stays 3xTF32.
template <int NT, bool BF = false>
struct TcCfg {
  static_assert(NT == 64 || NT == 128, "row tile must be 64 or 128");
  static constexpr int kBBytes = (BF ? 1 : 2) * NT * KC * 4;  // hi + lo weight image of one chunk
  static constexpr int kAStageCols = BF ? KC : 2 * KC;       // TMEM columns of one A stage
  static constexpr int kTStages = NT == 128 ? 3 : 4;  // TMEM A stages
  static constexpr int kAccCols = NT;               // per accumulator buffer
  static constexpr int kACol0 = 2 * NT;             // first TMEM column of A stages
  static constexpr int kTmemCols = 512;
  static_assert(kACol0 + kTStages * 2 * KC <= kTmemCols, "TMEM budget");
  static constexpr int kStoreBytes = 4 * 2 * 32 * 32 * 4;  // 4 warps x 2 bufs x [32 rows][32 px]
  static constexpr int kMaxAStages = 8;
  static constexpr int kMaxBStages = 8;
};

// Shared-memory plan of one launch (host computes, kernel re-derives).
struct BandSmem {
  int a_stages;     // raw activation ring depth (16 KB each)
  int b_resident;   // 1: whole panel in smem, loaded once; 2: this CTA's row tile's panel
  int b_stages;     // streamed panel ring depth
  int b_bytes;      // resident panel bytes, or one chunk image
  int total;        // dynamic smem bytes
};

struct TcBandArgs {
  const float* panel;        // B images: per row tile, per chunk: hi[NT][32], lo[NT][32] (swizzled)
  const int32_t* rt_info;    // per row tile: start8 (ring pos), nk8, panel offset (floats), chunks
  const int32_t* rows;       // [n_rt * NT] output channel per tile row, -1 = none
  const int32_t* class_d;    // ring class -> TMA coordinate d
  const int32_t* out_class_d;  // output view class -> d (TMA stores)
  const float* bias;         // forward only
  float* out;
  int32_t n_rt;              // row tiles
  int32_t ring;              // ring length (c_in fwd / c_out bwd)
  int32_t cls;               // ring positions per class (c_in fwd / c_out/D bwd)
  int32_t rb;                // activation box rows
  int32_t c_out_t;           // channels of the output tensor
  int32_t rows_total;        // valid tile rows (c_out fwd / c_in bwd)
  int32_t rows_per_sample_3d;  // TMA dim-2 rows per sample (c_in fwd / c_out/D bwd)
  int32_t out_cls;           // output view rows per class
  int32_t store_ok;          // TMA-store epilogue usable
  int32_t ptiles;            // pixel tiles per sample
  int32_t spt;               // > 1: a tile packs spt = 128 / plane whole samples (planes that divide 128)
  int32_t panel_floats;      // whole panel size (resident mode)
  BandSmem sm;
  int64_t plane;
  int64_t n;
};

__device__ __forceinline__ void advance(int& stage, uint32_t& phase, int stages) {
  if (++stage == stages) {
    stage = 0;
    phase ^= 1u;
  }
}

// Tile t -> (row tile, sample, first pixel).
struct TileCoord {
  int rt;
  int n;
  int p0;
};
// Packed tiles (spt > 1): tile pt covers samples [pt*spt, pt*spt + spt), the
// 128 TMEM lanes are (sample, pixel) in that order, p0 = 0.
template <bool PACK>
__device__ __forceinline__ TileCoord tile_coord(const TcBandArgs& a, int64_t t) {
  TileCoord c;
  c.rt = static_cast<int>(t % a.n_rt);
  const int64_t pt = t / a.n_rt;
  if (PACK) {
    c.n = static_cast<int>(pt * a.spt);
    c.p0 = 0;
    return c;
  }
  c.n = static_cast<int>(pt / a.ptiles);
  c.p0 = static_cast<int>(pt - static_cast<int64_t>(c.n) * a.ptiles) * TM;
  return c;
}

template <bool PACK>
__device__ __forceinline__ int64_t band_tiles(const TcBandArgs& a) {
  return (PACK ? (a.n + a.spt - 1) / a.spt : a.n * a.ptiles) * a.n_rt;
}

__device__ __forceinline__ int chunks_of(const TcBandArgs& a, int rt) {
  return (a.rt_info[4 * rt + 1] + 3) / 4;
}

template <int NT, bool PACK, bool BF>
__global__ void __launch_bounds__(kTcThreads, 1)
    tc_band_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tout,
                   const TcBandArgs a) {
  using C = TcCfg<NT, BF>;
  // panel offset (floats) of a row tile: rt_info holds the 3xTF32 layout's
  // (two fp32 images per chunk); a bf16 chunk image is half that size
  auto pofs = [&](int rt) { return BF ? a.rt_info[4 * rt + 2] / 2 : a.rt_info[4 * rt + 2]; };
  constexpr int ST = C::kTStages;
  const int SA = a.sm.a_stages;
  const int SB = a.sm.b_stages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  // [A ring: SA x ([32 rows][128 px] = 16 KB)] [B: resident panel or SB chunk
  // images] [store staging 32 KB] [barriers]
  uint8_t* a_ring = smem;
  uint8_t* b_base = a_ring + SA * kABytes;
  uint8_t* store_buf = b_base + (a.sm.b_resident ? a.sm.b_bytes : SB * C::kBBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(store_buf + C::kStoreBytes);
  uint64_t* a_full = bars;                              // [8]
  uint64_t* a_free = bars + C::kMaxAStages;             // [8] 4 converter warps read it
  uint64_t* b_full = bars + 2 * C::kMaxAStages;         // [2]
  uint64_t* b_free = b_full + C::kMaxBStages;           // [2]
  uint64_t* conv = b_free + C::kMaxBStages;             // [ST] TMEM A stage written
  uint64_t* t_free = conv + ST;                         // [ST] MMAs done with TMEM stage
  uint64_t* tfull = t_free + ST;                        // [2]
  uint64_t* tempty = tfull + 2;                         // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const uint32_t warp = warp_id();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    TRACE(0);
    for (int s = 0; s < C::kMaxAStages; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_free[s], 4);
    }
    for (int s = 0; s < C::kMaxBStages; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_free[s], 1);
    }
    for (int s = 0; s < ST; ++s) {
      mbar_init(&conv[s], 4);
      mbar_init(&t_free[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmap);
    prefetch_tmap(&tout);
  }
  if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) TRACE(1);

  const int64_t total = band_tiles<PACK>(a);

  if (warp == 0) {
    // ---------------- producer: activation ring (+ streamed weight panel) ----------------
    // The lanes issue a stage's boxes in parallel (one box each): a TMA
    // instruction holds its issuing thread ~0.1-0.3 us and short class runs
    // cut a stage into up to 4 boxes.
    {
      const int lane = threadIdx.x & 31;
      int sa = 0;
      uint32_t pa = 0;
      int sb = 0;
      uint32_t pb = 0;
      bool dep_synced = false;
      auto panel_ready = [&]() {
        if (!dep_synced) {
          TRACE(2);
          cudaGridDependencySynchronize();  // the panel-build kernel (PDL)
          TRACE(3);
          dep_synced = true;
        }
      };
      for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
        const TileCoord tc = tile_coord<PACK>(a, t);
        const int start8 = a.rt_info[4 * tc.rt], nk8 = a.rt_info[4 * tc.rt + 1];
        const int nch = (nk8 + 3) / 4;
        for (int c = 0; c < nch; ++c) {
          // activations: [32 ring rows][128 px], boxes of rb rows
          mbar_wait_tag(&a_free[sa], pa ^ 1u, 1);
          const int steps = min(4, nk8 - 4 * c);
          if (lane == 0) mbar_expect_tx(&a_full[sa], steps * 8 * TM * 4);
          __syncwarp();
          {
            const int r = lane * a.rb;
            if (r < steps * 8) {
              int pos = start8 + 32 * c + r;
              while (pos >= a.ring) pos -= a.ring;
              const int cl = pos / a.cls, j = pos - cl * a.cls;
              if (PACK)  // 4-D view {P, N, rows, D}: box {P, spt, rb, 1} = [rb rows][128 px]
                tma_load_4d(a_ring + sa * kABytes + r * (TM * 4), &tmap, &a_full[sa], 0, tc.n, j,
                            __ldg(a.class_d + cl));
              else
                tma_load_3d(a_ring + sa * kABytes + r * (TM * 4), &tmap, &a_full[sa], tc.p0,
                            __ldg(a.class_d + cl), tc.n * a.rows_per_sample_3d + j);
            }
          }
          __syncwarp();
          advance(sa, pa, SA);
          if (lane != 0) continue;
          if (a.sm.b_resident == 1 && t == blockIdx.x && c == 0) {
            panel_ready();
            mbar_expect_tx(&b_full[0], a.panel_floats * 4);
            bulk_load(b_base, a.panel, a.panel_floats * 4, &b_full[0]);
          } else if (a.sm.b_resident == 2 && t == blockIdx.x && c == 0) {
            // every tile of this CTA has row tile blockIdx.x % n_rt (the grid
            // is a multiple of n_rt): only that row tile's panel is resident
            panel_ready();
            const uint32_t bytes = static_cast<uint32_t>(nch) * C::kBBytes;
            mbar_expect_tx(&b_full[0], bytes);
            bulk_load(b_base, a.panel + pofs(tc.rt), bytes, &b_full[0]);
          }
        }
      }
      (void)sb;
      (void)pb;
    }
  } else if (warp == 10) {
    // ---------------- streamed panel producer ----------------
    // Its own warp, so the activation ring runs SA stages ahead of the MMAs
    // instead of being throttled by the panel ring's b_free waits.
    if (!a.sm.b_resident && elect_one()) {
      cudaGridDependencySynchronize();  // the panel-build kernel (PDL)
      int sb = 0;
      uint32_t pb = 0;
      for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
        const int rt = static_cast<int>(t % a.n_rt);
        const int nch = chunks_of(a, rt);
        const float* prow = a.panel + pofs(rt);
        for (int c = 0; c < nch; ++c) {
          mbar_wait_tag(&b_free[sb], pb ^ 1u, 2);
          mbar_expect_tx(&b_full[sb], C::kBBytes);
          bulk_load(b_base + sb * C::kBBytes,
                    prow + static_cast<int64_t>(c) * (C::kBBytes / 4),
                    C::kBBytes, &b_full[sb]);
          advance(sb, pb, SB);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (A from TMEM, B from SMEM) ----------------
    constexpr uint32_t idesc = BF ? idesc_bf16(TM, NT, 0, 0) : idesc_tf32(TM, NT, 0, 0);
    int st = 0;
    uint32_t ps = 0;
    int sb = 0;
    uint32_t pb = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    if (a.sm.b_resident) mbar_wait_tag(&b_full[0], 0, 3);
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      const int rt = static_cast<int>(t % a.n_rt);
      const int nk8 = a.rt_info[4 * rt + 1];
      const int nch = (nk8 + 3) / 4;
      const int prt = a.sm.b_resident == 1 ? pofs(rt) : 0;  // (global loads once per tile)
      mbar_wait_tag(&tempty[acc], acc_phase ^ 1u, 4);
      tc_fence_after();
      const uint32_t d_tmem = tmem + acc * C::kAccCols;
      for (int c = 0; c < nch; ++c) {
        mbar_wait_tag(&conv[st], ps, 5);
        uint8_t* bimg;
        if (a.sm.b_resident == 1) {
          bimg = b_base + (prt + c * (C::kBBytes / 4)) * 4;
        } else if (a.sm.b_resident == 2) {
          bimg = b_base + c * C::kBBytes;
        } else {
          mbar_wait_tag(&b_full[sb], pb, 6);
          bimg = b_base + sb * C::kBBytes;
        }
        tc_fence_after();
        if (t == blockIdx.x && c == 0 && lane == 0) TRACE(5);
        const int steps = min(4, nk8 - 4 * c);
        if (elect_one()) {
          const uint32_t a_hi = tmem + C::kACol0 + st * C::kAStageCols;
          if (BF) {
            // [hi pairs 16 cols | lo pairs 16 cols]; B row = [hi 32 | lo 32] bf16
            const uint32_t a_lo = a_hi + KC / 2;
            const uint32_t bh = smem_u32(bimg);
            for (int k = 0; k < (steps + 1) / 2; ++k) {
              const uint64_t dbh = desc_sw128(bh + k * 32, 16, 1024);
              const uint64_t dbl = desc_sw128(bh + 64 + k * 32, 16, 1024);
              mma_bf16_ts(d_tmem, a_hi + 8 * k, dbh, idesc, (c | k) != 0);
              mma_bf16_ts(d_tmem, a_lo + 8 * k, dbh, idesc, 1);
              mma_bf16_ts(d_tmem, a_hi + 8 * k, dbl, idesc, 1);
            }
          } else {
            const uint32_t a_lo = a_hi + KC;
            const uint32_t bh = smem_u32(bimg), bl = bh + NT * KC * 4;
            for (int k = 0; k < steps; ++k) {
              const uint64_t dbh = desc_sw128(bh + k * 32, 16, 1024);
              const uint64_t dbl = desc_sw128(bl + k * 32, 16, 1024);
              mma_tf32_ts(d_tmem, a_hi + 8 * k, dbh, idesc, (c | k) != 0);
              mma_tf32_ts(d_tmem, a_lo + 8 * k, dbh, idesc, 1);
              mma_tf32_ts(d_tmem, a_hi + 8 * k, dbl, idesc, 1);
            }
          }
          mma_commit(&t_free[st]);
          if (!a.sm.b_resident) mma_commit(&b_free[sb]);
          if (c == nch - 1) {
            mma_commit(&tfull[acc]);
            const int64_t ti = (t - blockIdx.x) / gridDim.x;
            if (ti < 8) TRACE(6 + 2 * ti);
          }
        }
        __syncwarp();
        advance(st, ps, ST);
        if (!a.sm.b_resident) advance(sb, pb, SB);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  } else if (warp < 6) {
    // ---------------- converters: smem [k][p] -> TMEM [p][k] hi / lo ----------------
    // Warp q transposes pixels 32q..32q+31 (TMEM lanes 32q..32q+31).
    const int q = warp & 3;
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    int sa = 0;
    uint32_t pa = 0;
    int st = 0;
    uint32_t ps = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      const int nk8 = a.rt_info[4 * static_cast<int>(t % a.n_rt) + 1];  // once per tile
      const int nch = (nk8 + 3) / 4;
      for (int c = 0; c < nch; ++c) {
        mbar_wait_tag(&a_full[sa], pa, 7);
        if (t == blockIdx.x && c == 0 && q == 0 && lane == 0) TRACE(4);
        const uint32_t src = smem_u32(a_ring + sa * kABytes) + 4u * (q * 32 + lane);
        uint32_t hi[KC], lo[KC];
        if (BF) {
          // bf16 pairs (ring rows 2i, 2i+1); rows past the chunk's last k8 step
          // are zero (an odd step count leaves half a K = 16 step)
          const int rows = 8 * min(4, nk8 - 4 * c);
          float v[KC];
#pragma unroll
          for (int k = 0; k < KC; ++k) v[k] = lds_f32(src + 4u * k * TM);
#pragma unroll
          for (int k = 0; k < KC; ++k) v[k] = k < rows ? v[k] : 0.f;
#pragma unroll
          for (int i = 0; i < KC / 2; ++i) bf16x2_split(v[2 * i], v[2 * i + 1], hi[i], lo[i]);
        } else {
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const float v = lds_f32(src + 4u * k * TM);
            const float h = tf32_hi(v);
            hi[k] = __float_as_uint(h);
            lo[k] = __float_as_uint(v - h);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_free[sa]);
        advance(sa, pa, SA);
        mbar_wait_tag(&t_free[st], ps ^ 1u, 8);
        tc_fence_after();
        const uint32_t col = tmem + C::kACol0 + st * C::kAStageCols + lane_base;
        if (BF) {
          uint32_t h16[16], l16[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) h16[i] = hi[i], l16[i] = lo[i];
          tmem_st16(col, h16);
          tmem_st16(col + KC / 2, l16);
        } else {
          tmem_st32(col, hi);
          tmem_st32(col + KC, lo);
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[st]);
        advance(st, ps, ST);
      }
    }
  } else {
    // ---------------- epilogue ----------------
    // Warp q drains TMEM lanes 32q..32q+31 (its pixel quarter) 32 columns at a
    // time, adds the bias and either stages a [32 rows][32 px] block in smem
    // for one TMA store, or (ragged rows / no contiguous output view) stores
    // each channel row directly (128 B per warp store).
    __shared__ int32_t row_s[NT];
    __shared__ float bias_s[NT];
    const int et = threadIdx.x - 192;  // 0..127
    const int q = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    int cur_rt = -1;
    int sbuf = 0;
    for (int64_t t = blockIdx.x; t < total; t += gridDim.x) {
      const TileCoord tc = tile_coord<PACK>(a, t);
      const int rt = tc.rt;
      if (rt != cur_rt) {
        named_bar_sync(1, 128);
        for (int i = et; i < NT; i += 128) {
          const int row = __ldg(a.rows + rt * NT + i);
          row_s[i] = row;
          bias_s[i] = (a.bias != nullptr && row >= 0) ? __ldg(a.bias + row) : 0.f;
        }
        named_bar_sync(1, 128);
        cur_rt = rt;
      }
      mbar_wait_tag(&tfull[acc], acc_phase, 9);
      tc_fence_after();
      // this lane's pixel: (sample n_l, pixel p) -- packed tiles hold spt samples
      int n_l = tc.n;
      int64_t p = tc.p0 + q * 32 + lane;
      if (PACK) {
        n_l = tc.n + static_cast<int>(p / a.plane);
        p -= static_cast<int64_t>(n_l - tc.n) * a.plane;
      }
      const bool pv = p < a.plane && (!PACK || n_l < a.n);
      const uint32_t taddr = tmem + acc * C::kAccCols + (static_cast<uint32_t>(q * 32) << 16);
#pragma unroll 1
      for (int c0 = 0; c0 < NT; c0 += 32) {
        uint32_t v[32];
        tmem_ld32_nowait(taddr + c0, v);
        float bb[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) bb[j] = bias_s[c0 + j];
        const int g0 = rt * NT + c0;  // first tile row of this group
        const bool tma_group = a.store_ok && g0 + 32 <= a.rows_total;
        tmem_ld_wait();
        if (tma_group) {
          float* buf = reinterpret_cast<float*>(store_buf + (q * 2 + sbuf) * 4096);
          const uint32_t bufa = smem_u32(buf) + 4u * lane;
          if (lane == 0) bulk_wait_read<1>();  // this buffer's previous store has read it
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 32; ++j) sts_f32(bufa + 128u * j, __uint_as_float(v[j]) + bb[j]);
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int cl = g0 / a.out_cls, jj = g0 - cl * a.out_cls;
            if (PACK) {
              // 4-D view {P, N, out_cls, D_out}: box {min(P,32), max(32/P,1), 32, 1}
              const int px0 = 32 * q;
              tma_store_4d(&tout, buf, static_cast<int>(px0 % a.plane), tc.n + static_cast<int>(px0 / a.plane), jj,
                           __ldg(a.out_class_d + cl));
            } else {
              tma_store_3d(&tout, buf, tc.p0 + 32 * q, __ldg(a.out_class_d + cl),
                           tc.n * a.out_cls + jj);
            }
            bulk_commit();
          }
          sbuf ^= 1;
        } else if (pv) {
          float* __restrict__ obase = a.out + static_cast<int64_t>(n_l) * a.c_out_t * a.plane + p;
          int32_t rr[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) rr[j] = row_s[c0 + j];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            if (rr[j] >= 0) obase[static_cast<int64_t>(rr[j]) * a.plane] = __uint_as_float(v[j]) + bb[j];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      {
        const int64_t ti = (t - blockIdx.x) / gridDim.x;
        if (ti < 8 && et == 0) TRACE(7 + 2 * ti);
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TRACE(30);
  if (warp == 1) tmem_dealloc<C::kTmemCols>(tmem);
}

// Band weight panel: per row tile and chunk, hi and lo images of the K-major
// SWIZZLE_128B layout the MMA reads ([NT rows][32 k], 8-row groups of 1 KB).
struct PanelArgs {
  const float* weight;
  const int32_t* rt_info;
  const int32_t* rows;     // output row channel per tile row (-1 none)
  const int32_t* starts;   // oc -> window start
  const int32_t* ring_map; // bwd: ring pos -> oc; fwd: nullptr
  float* panel;
  int32_t n_rt, ring, c_in, gw;
  int32_t backward_data;
  int64_t total;           // number of (rt, chunk, row, k) entries
  const int32_t* chunk_base;  // prefix sum of chunks per row tile (entries / (NT*32))
};

template <int NT, bool BF>
__global__ void __launch_bounds__(256) tc_panel_kernel(const PanelArgs a) {
  // Let the dependent band kernel get scheduled now; it waits for this grid's
  // completion (griddepcontrol.wait) before it reads the panel.
  cudaTriggerProgrammaticLaunchCompletion();
  for (int64_t e = blockIdx.x * 256ll + threadIdx.x; e < a.total; e += gridDim.x * 256ll) {
    const int k = static_cast<int>(e & 31);
    const int r = static_cast<int>((e >> 5) % NT);
    const int64_t gc = e / (32 * NT);  // global chunk index
    int rt = 0;
    while (rt + 1 < a.n_rt && a.chunk_base[rt + 1] <= gc) ++rt;
    const int c = static_cast<int>(gc - a.chunk_base[rt]);
    const int start8 = a.rt_info[4 * rt], nk8 = a.rt_info[4 * rt + 1];
    const int kk = 32 * c + k;
    float v = 0.f;
    const int row = a.rows[rt * NT + r];
    if (kk < 8 * nk8 && row >= 0) {
      int pos = start8 + kk;
      while (pos >= a.ring) pos -= a.ring;
      const int oc = a.backward_data ? a.ring_map[pos] : row;
      const int ic = a.backward_data ? row : pos;
      int s = ic - a.starts[oc];
      if (s < 0) s += a.c_in;
      if (s < a.gw) v = a.weight[static_cast<int64_t>(oc) * a.gw + s];
    }
    if (BF) {
      // row r = [hi 32 | lo 32] bf16, 16 B chunk j at j ^ (r % 8)
      const __nv_bfloat16 h = __float2bfloat16_rn(v);
      const __nv_bfloat16 l = __float2bfloat16_rn(v - __bfloat162float(h));
      uint8_t* img = reinterpret_cast<uint8_t*>(a.panel + gc * (NT * 32));
      const int rb = (r >> 3) * 1024 + (r & 7) * 128;
      *reinterpret_cast<__nv_bfloat16*>(img + rb + (((k >> 3) ^ (r & 7)) << 4) + (k & 7) * 2) = h;
      *reinterpret_cast<__nv_bfloat16*>(img + rb + ((((k >> 3) + 4) ^ (r & 7)) << 4) + (k & 7) * 2) = l;
    } else {
      const float hi = tf32_hi(v);
      float* img = a.panel + gc * (2 * NT * 32);
      const int off = (r >> 3) * 256 + (r & 7) * 32 + (((k >> 2) ^ (r & 7)) << 2) + (k & 3);
      img[off] = hi;
      img[NT * 32 + off] = v - hi;
    }
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// host side

bool tc_band_supported(const TcBandPlan& tp, int64_t plane) {
  return tp.ok && plane % 4 == 0 && plane >= 4;
}

template <int NT, bool BF>
static cudaError_t launch_tc_nt(const TcBandPlan& tp, const TcDeviceTables& dt,
                                const TcBandCall& call, cudaStream_t s) {
  using C = TcCfg<NT, BF>;
  // --- panel ---
  const int64_t entries = static_cast<int64_t>(tp.total_chunks) * NT * 32;
  float* panel = call.panel;
  cudaError_t e = cudaSuccess;
  PanelArgs pa{};
  pa.weight = call.weight;
  pa.rt_info = dt.rt_info;
  pa.rows = dt.rows;
  pa.starts = dt.starts;
  pa.ring_map = call.backward_data ? dt.perm : nullptr;
  pa.panel = panel;
  pa.n_rt = tp.n_rt;
  pa.ring = tp.ring;
  pa.c_in = call.c_in;
  pa.gw = call.gw;
  pa.backward_data = call.backward_data ? 1 : 0;
  pa.total = entries;
  pa.chunk_base = dt.chunk_base;
  const int pgrid = static_cast<int>(std::min<int64_t>((entries + 255) / 256, 148 * 8));
  tc_panel_kernel<NT, BF><<<pgrid, 256, 0, s>>>(pa);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;

  // Planes that divide the 128-pixel tile pack spt = 128 / P samples per tile
  // (4-D views with a sample dimension); otherwise one sample per tile.
  const int64_t P = call.plane;
  const int32_t spt = (P < TM && TM % P == 0 && P % 4 == 0) ? static_cast<int32_t>(TM / P) : 1;
  CUtensorMap tm, tout;
  if (spt > 1) {
    const uint64_t C = static_cast<uint64_t>(tp.n_class) * tp.rows_per_sample_3d;
    const uint64_t dims[4] = {static_cast<uint64_t>(P), static_cast<uint64_t>(call.n),
                              static_cast<uint64_t>(tp.rows_per_sample_3d), static_cast<uint64_t>(tp.n_class)};
    const uint64_t strides[3] = {C * P * 4, static_cast<uint64_t>(tp.n_class) * P * 4, static_cast<uint64_t>(P) * 4};
    const uint32_t box[4] = {static_cast<uint32_t>(P), static_cast<uint32_t>(spt), static_cast<uint32_t>(tp.rb), 1};
    if (!encode_f32(&tm, call.in, 4, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
    const int32_t ocls = tp.store_ok ? tp.out_cls : call.c_out_t;
    const int32_t ond = tp.store_ok ? tp.out_n_class : 1;
    const uint64_t odims[4] = {static_cast<uint64_t>(P), static_cast<uint64_t>(call.n), static_cast<uint64_t>(ocls),
                               static_cast<uint64_t>(ond)};
    const uint64_t ostr[3] = {static_cast<uint64_t>(call.c_out_t) * P * 4, static_cast<uint64_t>(ond) * P * 4,
                              static_cast<uint64_t>(P) * 4};
    const uint32_t obox[4] = {static_cast<uint32_t>(std::min<int64_t>(P, 32)),
                              static_cast<uint32_t>(std::max<int64_t>(32 / P, 1)), 32, 1};
    if (!encode_f32(&tout, call.out, 4, odims, ostr, obox, CU_TENSOR_MAP_SWIZZLE_NONE)) return cudaErrorInvalidValue;
  }
  // --- activations: {P, D, N * rows_per_sample} fp32, no swizzle, box {32, 1, rb}
  if (spt == 1) {
    const uint64_t dims[3] = {static_cast<uint64_t>(call.plane), static_cast<uint64_t>(tp.n_class),
                              static_cast<uint64_t>(call.n) * tp.rows_per_sample_3d};
    const uint64_t strides[2] = {static_cast<uint64_t>(call.plane) * 4,
                                 static_cast<uint64_t>(call.plane) * 4 * tp.n_class};
    const uint32_t box[3] = {TM, 1, static_cast<uint32_t>(tp.rb)};
    if (!encode_f32(&tm, call.in, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE))
      return cudaErrorInvalidValue;
  }
  // --- output view for TMA stores: {P, D_out, N * out_cls}, box {32, 1, 32}
  if (spt == 1) {
    const int32_t ocls = tp.store_ok ? tp.out_cls : call.c_out_t;
    const int32_t ond = tp.store_ok ? tp.out_n_class : 1;
    const uint64_t dims[3] = {static_cast<uint64_t>(call.plane), static_cast<uint64_t>(ond),
                              static_cast<uint64_t>(call.n) * ocls};
    const uint64_t strides[2] = {static_cast<uint64_t>(call.plane) * 4,
                                 static_cast<uint64_t>(call.plane) * 4 * ond};
    const uint32_t box[3] = {32, 1, 32};
    if (!encode_f32(&tout, call.out, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_NONE))
      return cudaErrorInvalidValue;
  }

  TcBandArgs ka{};
  ka.panel = panel;
  ka.rt_info = dt.rt_info;
  ka.rows = dt.rows;
  ka.class_d = dt.class_d;
  ka.out_class_d = dt.out_class_d;
  ka.bias = call.bias;
  ka.out = call.out;
  ka.n_rt = tp.n_rt;
  ka.ring = tp.ring;
  ka.cls = tp.cls;
  ka.rb = tp.rb;
  ka.c_out_t = call.c_out_t;
  ka.rows_total = call.c_out_t;
  ka.out_cls = tp.out_cls;
  ka.store_ok = tp.store_ok && call.plane % 4 == 0;
  ka.rows_per_sample_3d = tp.rows_per_sample_3d;
  ka.ptiles = static_cast<int32_t>((call.plane + TM - 1) / TM);
  ka.spt = spt;
  ka.plane = call.plane;
  ka.n = call.n;
  const int64_t tiles = (spt > 1 ? (call.n + spt - 1) / spt : call.n * ka.ptiles) * tp.n_rt;
  int nsm = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  int64_t grid = std::min<int64_t>(tiles, call.max_ctas > 0 ? std::min(call.max_ctas, nsm) : nsm);
  // Shared memory: resident weight panel when it fits next to a >= 5-deep
  // activation ring; else, when a grid that is a multiple of n_rt gives each
  // CTA a single row tile, that row tile's panel resident; else a streamed
  // panel ring on its own producer warp.
  {
    constexpr int kBudget = 227 * 1024 - 1024 /*align*/ - 2048 /*barriers + static*/;
    const int panel_bytes = static_cast<int>(tc_panel_bytes(tp) / (BF ? 2 : 1));
    BandSmem& sm = ka.sm;
    const int rest = kBudget - C::kStoreBytes;
    if (panel_bytes + 5 * kABytes <= rest) {
      sm.b_resident = 1;
      sm.b_bytes = panel_bytes;
      sm.b_stages = 1;
    } else {
      int max_rt = 0;
      for (int rt = 0; rt < tp.n_rt; ++rt) max_rt = std::max(max_rt, tp.rt_info[4 * rt + 3]);
      const int64_t grid_rt = grid / tp.n_rt * tp.n_rt;
      if (grid_rt >= tp.n_rt && grid_rt >= grid - grid / 16 &&
          max_rt * C::kBBytes + 5 * kABytes <= rest) {
        sm.b_resident = 2;
        sm.b_bytes = max_rt * C::kBBytes;
        sm.b_stages = 1;
        grid = grid_rt;
      } else {
        // Streamed panel ring: one chunk image per MMA stage from L2, so its
        // depth x (L2 latency) bounds the MMA rate.  bf16 chunk images are
        // half the bytes: twice the depth in the same shared memory (3 tf32
        // stages kept the tensor pipe ~52 % busy at C=1024 cg=2 56x56).
        sm.b_resident = 0;
        sm.b_bytes = C::kBBytes;
        sm.b_stages = BF ? 6 : 3;
      }
    }
    const int b_total = sm.b_resident ? sm.b_bytes : sm.b_stages * C::kBBytes;
    sm.a_stages = std::min(C::kMaxAStages, (rest - b_total) / kABytes);
    sm.total = sm.a_stages * kABytes + b_total + C::kStoreBytes + 1024 + 512;
  }
  ka.panel_floats = static_cast<int32_t>(tc_panel_bytes(tp) / (BF ? 8 : 4));
  // packed tiles are a separate instantiation: the unpacked kernel keeps its
  // register allocation (the sample arithmetic cost 20 registers and ~25 %
  // at C256 cg8 56x56 when it was a runtime branch)
  auto kern = spt > 1 ? tc_band_kernel<NT, true, BF> : tc_band_kernel<NT, false, BF>;
  {
    static bool attr_set[2][64] = {{false}};  // per packing, device (one table per template instance)
    int dev = 0;
    cudaGetDevice(&dev);
    const int pk = spt > 1 ? 1 : 0;
    if (dev < 0 || dev >= 64 || !attr_set[pk][dev]) {
      e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 1024);
      if (e != cudaSuccess) return e;
      if (dev >= 0 && dev < 64) attr_set[pk][dev] = true;
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kTcThreads);
  cfg.dynamicSmemBytes = ka.sm.total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, tm, tout, ka);
  if (e != cudaSuccess) return e;
  note_launches(2);
  return cudaSuccess;
}

int tc_hang(unsigned int* out) {
#if defined(SCC_WATCHDOG)
  return cudaMemcpyFromSymbol(out, sm100::g_hang, 64 * sizeof(unsigned int)) == cudaSuccess ? 64 : -1;
#else
  (void)out;
  return 0;
#endif
}

int tc_trace(unsigned long long* out, int n) {
  if (n > 32) n = 32;
  return cudaMemcpyFromSymbol(out, g_trace, n * sizeof(unsigned long long)) == cudaSuccess ? n : -1;
}

size_t tc_panel_bytes(const TcBandPlan& tp) {
  return static_cast<size_t>(tp.total_chunks) * 2 * tp.nt * 32 * sizeof(float);
}

// bf16x3 for backward-data only (1e-4 bar).  The forward stays 3xTF32: a
// bf16x3 forward measured <= 6e-6 norm-relative on every C5 shape (within the
// 1e-5 bar; 3xTF32: 0.9-5.8e-6) and 1.2-1.5x faster at gw >= 128, but through
// a network its larger errors flip ReLU masks of near-zero activations: the
// reference harness's mobilenet_like gradients moved from ~1e-5 to 5e-3
// (scripts/probes/harness_prec.py).  -DSCC_FWD_BF16 builds that variant for
// scripts/probes/precision_probe.py.
static bool bf16x3_band(const TcBandCall& call) {
#if defined(SCC_FWD_BF16)
  (void)call;
  return true;
#else
  return call.backward_data;
#endif
}

cudaError_t launch_band_tc(const TcBandPlan& tp, const TcDeviceTables& dt, const TcBandCall& call,
                           cudaStream_t s) {
  switch (tp.nt) {
    case 64:
      return bf16x3_band(call) ? launch_tc_nt<64, true>(tp, dt, call, s) : launch_tc_nt<64, false>(tp, dt, call, s);
    case 128:
      return bf16x3_band(call) ? launch_tc_nt<128, true>(tp, dt, call, s) : launch_tc_nt<128, false>(tp, dt, call, s);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace scc
