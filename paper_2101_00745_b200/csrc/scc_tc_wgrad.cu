// Tensor-core (tcgen05, 3xTF32) backward-weight of the SCC operator, sm_100a
// (replaces scc_backward_params, kernel.cpp:140-181).
//
//   dWband[oc, ic] = sum_{n,p} dy[n, oc, p] * x[n, ic, p]      (ic in the arc of oc's tile)
//   db[oc]         = sum_{n,p} dy[n, oc, p]
//
// GEMM with M = 128 filters (cycle-sorted order, TMEM lanes), N = the tile's
// input-channel arc (<= 256 columns per chunk), K = pixels.  Both operands are
// pixel-contiguous, i.e. K-major:
//   * dy goes through a deep shared-memory ring (SWIZZLE_128B boxes, 64 pixels
//     per stage) into TMEM as tf32 hi/lo columns (TS-mode MMA).  The swizzle
//     makes the row-per-thread reads bank-conflict free, and the ring slot is
//     released as soon as it is converted, so loads run far ahead;
//   * x stays in shared memory in the canonical SWIZZLE_128B K-major layout,
//     plus a converted lo copy (SS-mode operand).
// Loaded bytes in flight, not TMA issue slots, bound the kernel, so boxes are
// as wide as the geometry allows (4-D boxes cover two 32-pixel atoms).
// The pixel range is split across CTAs; each writes an fp32 partial tile and a
// second kernel reduces the partials in a fixed order (warp per output, fixed
// lane assignment and shuffle tree) into the window-relative [oc][k] layout.
// No atomics: results are bitwise reproducible.
#include <algorithm>

#include "scc_kernels.hpp"
#include "scc_plan.hpp"
#include "sm100.cuh"
#include "tmap.hpp"

namespace scc {
namespace {

using namespace sm100;

// Diagnostic timeline (CTA 0, ns): 0 start, 1 setup, 2+i chunk i issued
// (i<8), 10+i converter done with chunk i, 18+i MMA committed chunk i,
// 26 epilogue done.
__device__ unsigned long long g_wtrace[32];
#if defined(SCC_TRACE)
#define WTRACE(slot)                                            \
  do {                                                          \
    if (blockIdx.x == 0) g_wtrace[(slot)] = globaltimer();      \
  } while (0)
#else
#define WTRACE(slot) \
  do {               \
  } while (0)
#endif

constexpr int kThreads = 352;  // 11 warps: dy loads from warp 0, x loads from warp 10
constexpr int kAtom = 32;              // pixels per SWIZZLE_128B atom (128 B)
constexpr int kMaxA = 8;               // dy ring depth cap
constexpr int kMaxT = 3;               // TMEM / x stage depth cap

struct WArgs {
  const int32_t* rt_info;  // per row tile: start8, ncols
  const int32_t* class_d;
  const int32_t* perm;     // sorted position -> oc
  const int32_t* starts;   // oc -> window start
  float* part;             // [split][rt][nc][128][nw] (only each row's window columns are written)
  float* pbias;            // [split][rt][128]
  int32_t n_rt, n_nc, nw, cls, c_in, c_out, gw;
  int32_t rba, rbb;        // TMA box rows (dy, x)
  int32_t blk;             // 32-pixel atoms per stage (1 or 2)
  int32_t a_stages, t_stages;
  int32_t acol0;           // first TMEM column of the A stages
  int32_t dy4d;            // dy boxes are 4-D (both atoms in one box)
  int32_t has_bias;
  int64_t pcs;             // pixel chunks (of blk atoms) per sample
  int64_t total_chunks, chunks_per_split;
  int64_t plane;
};

__device__ __forceinline__ void advance(int& stage, uint32_t& phase, int stages) {
  if (++stage == stages) {
    stage = 0;
    phase ^= 1u;
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    tc_weight_kernel(const __grid_constant__ CUtensorMap tdy, const __grid_constant__ CUtensorMap tx,
                     const WArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int SA = a.a_stages, ST = a.t_stages, NB = a.blk;
  const int a_stage_bytes = 128 * NB * kAtom * 4;     // 128 rows x NB atoms
  const int b_blk_bytes = a.nw * kAtom * 4;           // one atom of x rows
  const int b_stage_bytes = NB * b_blk_bytes;         // raw, converted in place to bf16 [hi 32 | lo 32] rows
  uint8_t* a_ring = smem;
  uint8_t* b_ring = a_ring + SA * a_stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_ring + ST * b_stage_bytes);
  uint64_t* a_full = bars;                 // [kMaxA]
  uint64_t* a_free = bars + kMaxA;         // [kMaxA] 4 converter warps
  uint64_t* b_full = bars + 2 * kMaxA;     // [kMaxT]
  uint64_t* conv = b_full + kMaxT;         // [kMaxT] 4 converter warps
  uint64_t* t_free = conv + kMaxT;         // [kMaxT] MMA done (TMEM A + x stage)
  uint64_t* tfull = t_free + kMaxT;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

  const int nc = static_cast<int>(blockIdx.x % a.n_nc);
  const int rest = static_cast<int>(blockIdx.x / a.n_nc);
  const int rt = rest % a.n_rt;
  const int split = rest / a.n_rt;
  const int64_t q_begin = static_cast<int64_t>(split) * a.chunks_per_split;
  const int64_t q_end = min(a.total_chunks, q_begin + a.chunks_per_split);
  const int nchunks = q_end > q_begin ? static_cast<int>(q_end - q_begin) : 0;
  const int start8 = a.rt_info[2 * rt], ncols = a.rt_info[2 * rt + 1];
  const int kpix = NB * kAtom;

  const uint32_t warp = warp_id();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    WTRACE(0);
    for (int s = 0; s < kMaxA; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_free[s], 4);
    }
    for (int s = 0; s < kMaxT; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&conv[s], 8);  // 4 dy converter warps + 4 x-lo converter warps
      mbar_init(&t_free[s], 1);
    }
    mbar_init(tfull, 1);
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
  if (threadIdx.x == 0) WTRACE(1);
  // PDL: the prologue above overlaps the previous kernel's tail; every global
  // read (dy, x) and write (the partials, which a previous call's finalize
  // may still read) comes after its completion.
  cudaGridDependencySynchronize();
  cudaTriggerProgrammaticLaunchCompletion();

  // Row r (0..127) of a dy stage: quarter q = r/32 holds boxes of rba rows,
  // each box [NB atoms][rba rows][128 B].
  auto a_row_off = [&](int r, int b) {
    const int q = r >> 5, l = r & 31;
    return q * (32 * NB * 128) + (l / a.rba) * (a.rba * NB * 128) + b * (a.rba * 128) +
           (l % a.rba) * 128;
  };

  // Producers.  A TMA instruction occupies its issuing thread for ~0.1-0.4 us,
  // so dy and x loads are issued from two warps (one elected thread each),
  // each running ahead on its own ring.  (Dealing a side's boxes over two
  // issuers measured slower: the interleaved prefetches delay the boxes the
  // MMA needs first.)
  const bool dy_role = warp == 0;
  const bool x_role = warp == 10;
  if (dy_role) {
    // All 32 lanes issue the stage's boxes (one box per lane): a TMA
    // instruction holds its issuing thread ~0.1-0.3 us, and short class runs
    // (co = 25 / 75 %, cg = 8) give up to 16 boxes per stage.  (All lanes
    // poll the ring barrier: polling from one lane measured slower.)
    int sa = 0;
    uint32_t pa = 0;
    const int rows_a = min(128, a.c_out - rt * 128);
    const int a_boxes_rows = (rows_a + a.rba - 1) / a.rba * a.rba;
    const int nbox = a_boxes_rows / a.rba;
    for (int64_t qc = q_begin; qc < q_end; ++qc) {
      const int n = static_cast<int>(qc / a.pcs);
      const int p0 = static_cast<int>(qc - static_cast<int64_t>(n) * a.pcs) * kpix;
      if (lane == 0 && qc - q_begin == 1) WTRACE(27);
      mbar_wait_tag(&a_free[sa], pa ^ 1u, 20);
      if (lane == 0) {
        if (qc - q_begin == 1) WTRACE(28);
        mbar_expect_tx(&a_full[sa], a_boxes_rows * NB * 128);
      }
      __syncwarp();
      uint8_t* ad = a_ring + sa * a_stage_bytes;
      for (int bi = lane; bi < nbox; bi += 32) {
        const int r = bi * a.rba;
        const int i0 = rt * 128 + r;
        const int cl = i0 / a.cls, j = i0 - cl * a.cls;
        const int d = __ldg(a.class_d + cl);
        if (a.dy4d) {
          tma_load_4d(ad + a_row_off(r, 0), &tdy, &a_full[sa], 0, d, n * a.cls + j, p0 / kAtom);
        } else {
          for (int b = 0; b < NB; ++b) {
            tma_load_3d(ad + a_row_off(r, b), &tdy, &a_full[sa], p0 + b * kAtom, d, n * a.cls + j);
          }
        }
      }
      __syncwarp();
      advance(sa, pa, SA);
      if (lane == 0) {
        if (qc - q_begin == 1) WTRACE(29);
        if (qc - q_begin < 8) WTRACE(2 + (qc - q_begin));
      }
    }
  } else if (x_role) {
    int sb = 0;
    uint32_t pb = 0;
    const int cols_b = min(a.nw, ncols - nc * a.nw);
    const int b_boxes_rows = (cols_b + a.rbb - 1) / a.rbb * a.rbb;
    const int nbr = b_boxes_rows / a.rbb;
    for (int64_t qc = q_begin; qc < q_end; ++qc) {
      const int n = static_cast<int>(qc / a.pcs);
      const int p0 = static_cast<int>(qc - static_cast<int64_t>(n) * a.pcs) * kpix;
      mbar_wait_tag(&t_free[sb], pb ^ 1u, 21);
      if (lane == 0) {
        if (qc - q_begin == 1) WTRACE(30);
        mbar_expect_tx(&b_full[sb], b_boxes_rows * NB * 128);
      }
      __syncwarp();
      uint8_t* bd = b_ring + sb * b_stage_bytes;
      for (int bi = lane; bi < NB * nbr; bi += 32) {
        const int b = bi / nbr, r = (bi - b * nbr) * a.rbb;
        int pos = start8 + nc * a.nw + r;
        while (pos >= a.c_in) pos -= a.c_in;
        tma_load_3d(bd + b * b_blk_bytes + r * 128, &tx, &b_full[sb], p0 + b * kAtom, 0, n * a.c_in + pos);
      }
      __syncwarp();
      if (lane == 0 && qc - q_begin == 1) WTRACE(31);
      advance(sb, pb, ST);
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (dy hi/lo from TMEM, x from SMEM) ----------------
    // N in at most two parts: an MMA's N is <= 256 (columns [256, nw) of a
    // 257-384-column chunk are a second MMA on the B rows past 256)
    const int n1 = min(a.nw, 256), n2 = a.nw - n1;
    const uint32_t idesc = idesc_bf16(128, n1, 0, 0);
    const uint32_t idesc2 = idesc_bf16(128, n2 > 0 ? n2 : 16, 0, 0);
    int st = 0;
    uint32_t ps = 0;
    for (int c = 0; c < nchunks; ++c) {
      mbar_wait_tag(&conv[st], ps, 22);
      tc_fence_after();
      if (elect_one()) {
        // A stage: [hi pairs: kpix/2 cols][lo pairs: kpix/2 cols]; an x atom
        // row holds [hi 32 px | lo 32 px] bf16 (128 B, K-major SWIZZLE_128B)
        const uint32_t ahi = tmem + a.acol0 + st * kpix;
        const uint32_t alo = ahi + kpix / 2;
        const uint32_t braw = smem_u32(b_ring + st * b_stage_bytes);
        for (int k = 0; k < kpix / 16; ++k) {
          const int b = k >> 1, kk = k & 1;
          const uint64_t dbh = desc_sw128(braw + b * b_blk_bytes + kk * 32, 16, 1024);
          const uint64_t dbl = desc_sw128(braw + b * b_blk_bytes + 64 + kk * 32, 16, 1024);
          mma_bf16_ts(tmem, ahi + 8 * k, dbh, idesc, (c | k) != 0);
          mma_bf16_ts(tmem, alo + 8 * k, dbh, idesc, 1);
          mma_bf16_ts(tmem, ahi + 8 * k, dbl, idesc, 1);
          if (n2 > 0) {
            const uint32_t off = static_cast<uint32_t>(n1) * 128u;  // B rows past 256 (1 KB-aligned 8-row groups)
            const uint64_t dbh2 = desc_sw128(braw + b * b_blk_bytes + off + kk * 32, 16, 1024);
            const uint64_t dbl2 = desc_sw128(braw + b * b_blk_bytes + off + 64 + kk * 32, 16, 1024);
            mma_bf16_ts(tmem + n1, ahi + 8 * k, dbh2, idesc2, (c | k) != 0);
            mma_bf16_ts(tmem + n1, alo + 8 * k, dbh2, idesc2, 1);
            mma_bf16_ts(tmem + n1, ahi + 8 * k, dbl2, idesc2, 1);
          }
        }
        mma_commit(&t_free[st]);
        if (c == nchunks - 1) mma_commit(tfull);
        if (c < 8) WTRACE(18 + c);
      }
      __syncwarp();
      advance(st, ps, ST);
    }
  } else if (warp < 6) {
    // ---------------- converters (+ bias row sums) ----------------
    const int q = warp & 3;
    const int t = q * 32 + lane;  // filter row of the tile == TMEM lane
    const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
    float bsum = 0.f;
    int sa = 0, st = 0;
    uint32_t pa = 0, ps = 0;
    for (int c = 0; c < nchunks; ++c) {
      mbar_wait_tag(&a_full[sa], pa, 23);
      const uint8_t* ab = a_ring + sa * a_stage_bytes;
      uint32_t hi[2][16], lo[2][16];
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        if (b < NB) {
          const uint32_t src = smem_u32(ab + a_row_off(t, b));
          float4 v[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            // 16 B chunk k of the row sits at chunk index (k ^ row%8): undo the
            // swizzle so columns come out in pixel order.
            v[k] = lds_v4(src + 16 * (k ^ (t & 7)));
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            bf16x2_split(v[k].x, v[k].y, hi[b][2 * k], lo[b][2 * k]);
            bf16x2_split(v[k].z, v[k].w, hi[b][2 * k + 1], lo[b][2 * k + 1]);
            bsum += ((v[k].x + v[k].y) + v[k].z) + v[k].w;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&a_free[sa]);
      advance(sa, pa, SA);
      // TMEM A stage st is free once the MMAs of its previous use completed
      // (the same commit that lets the producer refill x stage st).
      mbar_wait_tag(&t_free[st], ps ^ 1u, 24);
      tc_fence_after();
      const uint32_t col = tmem + a.acol0 + st * kpix + lane_base;
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        if (b < NB) {
          tmem_st16(col + b * (kAtom / 2), hi[b]);
          tmem_st16(col + kpix / 2 + b * (kAtom / 2), lo[b]);
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[st]);
      if (c < 8 && t == 0) WTRACE(10 + c);
      advance(st, ps, ST);
    }
    if (a.has_bias && nc == 0) {
      a.pbias[(static_cast<int64_t>(split) * a.n_rt + rt) * 128 + t] = bsum;
    }
  } else {
    // ---------------- x converters, then the epilogue ----------------
    // Each x atom row (32 px fp32, 128 B) becomes [hi 32 | lo 32] bf16 in
    // place (thread = row: it alone reads and writes that 128 B, 16 B chunk j
    // at j ^ (row % 8) both ways, conflict-free), once x has landed (the
    // producer refills a stage only after the MMAs of its previous use), in
    // parallel with the dy converters.
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    {
      const int rows = NB * a.nw;  // atom rows per stage
      int st = 0;
      uint32_t ps = 0;
      for (int c = 0; c < nchunks; ++c) {
        mbar_wait_tag(&b_full[st], ps, 24);
        const uint32_t base = smem_u32(b_ring + st * b_stage_bytes);
        for (int r = quarter * 32 + lane; r < rows; r += 128) {
          const uint32_t row = base + 128u * r;
          const int sw = r & 7;
          float4 v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) v[j] = lds_v4(row + ((j ^ sw) << 4));
          uint32_t hi[16], lo[16];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            bf16x2_split(v[j].x, v[j].y, hi[2 * j], lo[2 * j]);
            bf16x2_split(v[j].z, v[j].w, hi[2 * j + 1], lo[2 * j + 1]);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + ((j ^ sw) << 4)), "r"(hi[4 * j]),
                         "r"(hi[4 * j + 1]), "r"(hi[4 * j + 2]), "r"(hi[4 * j + 3]));
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + (((4 + j) ^ sw) << 4)),
                         "r"(lo[4 * j]), "r"(lo[4 * j + 1]), "r"(lo[4 * j + 2]), "r"(lo[4 * j + 3]));
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&conv[st]);
        advance(st, ps, ST);
      }
    }
    // ---------------- epilogue: accumulator -> partial tile ----------------
    const int row = quarter * 32 + lane;
    float* dst = a.part + ((static_cast<int64_t>(split) * a.n_rt + rt) * a.n_nc + nc) * 128 * a.nw +
                 static_cast<int64_t>(row) * a.nw;
    // Only the float4 groups that overlap this filter's window are written:
    // the finalize reads nothing else (the band is gw of the tile's nw
    // columns, so this cuts the partial traffic by nw / gw).
    // (window start in tile columns; a tile spanning the whole ring starts at
    // column 0 and its windows may wrap)
    int j0 = -1;
    const int pos = rt * 128 + row;
    if (pos < a.c_out) {
      j0 = __ldg(a.starts + __ldg(a.perm + pos)) - start8;
      j0 += j0 < 0 ? a.c_in : 0;
    }
    auto in_window = [&](int c4) {  // float4 group at chunk column c4 touches the window
      if (j0 < 0) return false;
      const int col = nc * a.nw + c4;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        int d = col + t - j0;
        d += d < 0 ? a.c_in : 0;
        if (d < a.gw) return true;
      }
      return false;
    };
    if (nchunks > 0) {
      mbar_wait_tag(tfull, 0, 25);
      tc_fence_after();
      const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
      for (int c0 = 0; c0 < a.nw; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          if (in_window(c0 + j))
            *reinterpret_cast<float4*>(dst + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
      }
    } else {
      for (int c0 = 0; c0 < a.nw; c0 += 4)
        if (in_window(c0)) *reinterpret_cast<float4*>(dst + c0) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (row == 0) WTRACE(26);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

struct FArgs {
  const float* part;
  const float* pbias;
  const int32_t* rt_info;
  const int32_t* starts;
  const int32_t* inv_perm;
  float* dweight;
  float* dbias;
  int32_t splits, n_rt, n_nc, nw, c_in, c_out, gw;
};

// Partial-tile location of window slot k of filter oc.
__device__ __forceinline__ int64_t fin_base(const FArgs& a, int oc, int k) {
  const int pos = a.inv_perm[oc];
  const int rt = pos >> 7, row = pos & 127;
  int col = a.starts[oc] + k - a.rt_info[2 * rt];
  while (col < 0) col += a.c_in;
  while (col >= a.c_in) col -= a.c_in;
  const int nc = col / a.nw, c = col - nc * a.nw;
  return ((static_cast<int64_t>(rt) * a.n_nc + nc) * 128 + row) * a.nw + c;
}

// Thread per output (many outputs, few splits): the split partials are summed
// in ascending order; neighbouring threads read neighbouring window slots, so
// every split plane is read coalesced.
__global__ void __launch_bounds__(256) tc_weight_finalize_wide(const FArgs a) {
  cudaGridDependencySynchronize();
  cudaTriggerProgrammaticLaunchCompletion();
  const int64_t nw_out = static_cast<int64_t>(a.c_out) * a.gw;
  const int64_t total = nw_out + (a.dbias ? a.c_out : 0);
  const int64_t stride = static_cast<int64_t>(a.n_rt) * a.n_nc * 128 * a.nw;
  for (int64_t o = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; o < total;
       o += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float s = 0.f;
    if (o < nw_out) {
      const int oc = static_cast<int>(o / a.gw);
      const int64_t base = fin_base(a, oc, static_cast<int>(o - static_cast<int64_t>(oc) * a.gw));
#pragma unroll 8
      for (int sp = 0; sp < a.splits; ++sp) s += a.part[base + sp * stride];
      a.dweight[o] = s;
    } else {
      const int oc = static_cast<int>(o - nw_out);
      const int pos = a.inv_perm[oc];
      const int rt = pos >> 7, row = pos & 127;
      for (int sp = 0; sp < a.splits; ++sp) s += a.pbias[(static_cast<int64_t>(sp) * a.n_rt + rt) * 128 + row];
      a.dbias[oc] = s;
    }
  }
}

// Few outputs, many splits: block = 32 consecutive outputs x W warps; warp w
// sums splits w, w+W, ... in order (each load a coalesced row piece of one
// split plane -- the former warp-per-output scheme touched 32 split planes per
// load, ~8x the sectors), then warp 0 adds the W warp sums in order.  W is
// chosen from the output count so the grid is one resident wave (round 1
// used W = 32 everywhere: 1032 blocks of 1024 threads, one load each, at
// C256 cg2 14x14 -- 19.8 us cold for 4.2 MB).  The order depends on W, which
// depends on the geometry only.
template <int W>
__global__ void __launch_bounds__(32 * W) tc_weight_finalize(const FArgs a) {
  __shared__ float red[W][33];
  cudaGridDependencySynchronize();
  cudaTriggerProgrammaticLaunchCompletion();
  const int64_t nw_out = static_cast<int64_t>(a.c_out) * a.gw;
  const int64_t total = nw_out + (a.dbias ? a.c_out : 0);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int64_t o = blockIdx.x * 32ll + l;
  float s = 0.f;
  if (o < nw_out) {
    const int oc = static_cast<int>(o / a.gw);
    const int64_t base = fin_base(a, oc, static_cast<int>(o - static_cast<int64_t>(oc) * a.gw));
    const int64_t stride = static_cast<int64_t>(a.n_rt) * a.n_nc * 128 * a.nw;
#pragma unroll 8
    for (int sp = w; sp < a.splits; sp += W) s += a.part[base + sp * stride];
  } else if (o < total) {
    const int oc = static_cast<int>(o - nw_out);
    const int pos = a.inv_perm[oc];
    const int rt = pos >> 7, row = pos & 127;
#pragma unroll 8
    for (int sp = w; sp < a.splits; sp += W) s += a.pbias[(static_cast<int64_t>(sp) * a.n_rt + rt) * 128 + row];
  }
  if (W == 1) {
    if (o < total) {
      if (o < nw_out) a.dweight[o] = s;
      else a.dbias[o - nw_out] = s;
    }
    return;
  }
  red[w][l] = s;
  __syncthreads();
  if (w == 0 && o < total) {
    float t = red[0][l];
#pragma unroll
    for (int q = 1; q < W; ++q) t += red[q][l];
    if (o < nw_out) a.dweight[o] = t;
    else a.dbias[o - nw_out] = t;
  }
}

// Warps per finalize block: the largest W in {32, 16, 8, 4, 2, 1} whose grid
// (one block per 32 outputs) fits in one wave of 148 SMs x 2048 threads.
int fin_warps(int64_t outs) {
  const int64_t blocks = (outs + 31) / 32;
  for (int w : {32, 16, 8, 4, 2}) {
    if (blocks * 32 * w <= 148ll * 2048) return w;
  }
  return 1;
}

struct WGrid {
  int blk, a_stages, t_stages, acol0, smem;
  int64_t pcs, total_chunks, chunks_per_split;
  int32_t splits;
};

WGrid weight_grid(const TcWeightPlan& tw, int64_t n, int64_t plane) {
  WGrid g{};
  g.blk = tw.nw <= 128 ? 2 : 1;
  g.acol0 = tw.nw <= 128 ? 128 : (tw.nw <= 256 ? 256 : 384);
  constexpr int kBudget = 227 * 1024 - 1024 - 1024;
  // Keep >= 2 dy stages: shed x/TMEM stages first, then halve the stage width
  // (nw = 128 with 2-atom stages needs 64 KB per x stage).
  int kpix = 0, a_stage = 0, b_stage = 0;
  for (;;) {
    kpix = g.blk * kAtom;
    g.t_stages = std::min(kMaxT, (512 - g.acol0) / kpix);  // bf16 hi | lo pairs: kpix columns per stage
    a_stage = 128 * kpix * 4;
    b_stage = tw.nw * kpix * 4;                             // raw x, converted in place
    while (g.t_stages > 1 && (kBudget - g.t_stages * b_stage) / a_stage < 2) --g.t_stages;
    g.a_stages = std::min(kMaxA, (kBudget - g.t_stages * b_stage) / a_stage);
    // A single x stage serialises load -> lo convert -> MMA per chunk
    // (measured ~4x slower at nw = 192), so halve the stage width instead.
    if ((g.a_stages >= 2 && g.t_stages >= 2) || g.blk == 1) break;
    g.blk = 1;
  }
  g.smem = g.a_stages * a_stage + g.t_stages * b_stage + 1024 + 512;
  g.pcs = (plane + kpix - 1) / kpix;
  g.total_chunks = n * g.pcs;
  const int64_t items = static_cast<int64_t>(tw.n_rt) * tw.n_nc;
  // One CTA per SM (shared memory): a grid just over 148 runs a second,
  // nearly empty wave, so round the split count down.  Small problems
  // (latency bound) get half the SMs: scc_backward then runs backward-data
  // beside this kernel on the other half (tc_weight_small); the rule depends
  // on the geometry only, so every entry point sums in the same order.
  const int64_t cap = tc_weight_small(n, plane, std::max(tw.c_in, tw.c_out)) ? 74 : 148;
  int64_t splits = std::max<int64_t>(1, cap / items);
  // Bound the accumulation chain of each split's TMEM accumulator: every MMA
  // rounds the running fp32 sum toward zero, a bias that grows linearly with
  // the chain (measured ~6e-8 of max|dW| per K = 16 step: 4.0e-5 at the
  // 697-step chains of C=1024 cg=2 56x56, N=32).  At most kMaxChain steps per
  // split keeps dW within ~4.5e-5 of the 1e-4 bar at any N * plane; extra
  // splits come in whole waves.
  constexpr int64_t kMaxChain = 768;
  const int64_t steps = g.total_chunks * (kpix / 16);
  if (steps > splits * kMaxChain) {
    const int64_t wave = splits;
    splits = (steps + kMaxChain - 1) / kMaxChain;
    splits = (splits + wave - 1) / wave * wave;
  }
  splits = std::min(splits, g.total_chunks);
  g.chunks_per_split = (g.total_chunks + splits - 1) / splits;
  g.splits = static_cast<int32_t>((g.total_chunks + g.chunks_per_split - 1) / g.chunks_per_split);
  return g;
}

}  // namespace

int tc_wtrace(unsigned long long* out, int n) {
  if (n > 32) n = 32;
  return cudaMemcpyFromSymbol(out, g_wtrace, n * sizeof(unsigned long long)) == cudaSuccess ? n : -1;
}

// latency bound: little work per SM even on half the SMs (measured on the C5
// 14x14 rows and the SCC-ResNet-18 8x8 / 4x4 layers: a win up to ~2 M
// pixel-channels, a loss from C=512 at 14x14 on, where the MMAs dominate)
bool tc_weight_small(int64_t n, int64_t plane, int64_t channels) {
  return n * plane <= 16384 && n * plane * channels <= (int64_t{1} << 21);
}

bool tc_weight_supported(const TcWeightPlan& tw, int64_t plane) {
  return tw.ok && plane % 4 == 0;
}

size_t tc_weight_workspace_bytes(const TcWeightPlan& tw, int64_t n, int64_t plane) {
  const WGrid g = weight_grid(tw, n, plane);
  return static_cast<size_t>(g.splits) * tw.n_rt * (static_cast<size_t>(tw.n_nc) * 128 * tw.nw + 128) *
             sizeof(float) + 256;
}

cudaError_t launch_weight_tc(const TcWeightPlan& tw, const TcWeightCall& call, cudaStream_t s) {
  const WGrid g = weight_grid(tw, call.n, call.plane);
  if (g.a_stages < 2 || g.t_stages < 1) return cudaErrorInvalidValue;
  if (tc_weight_workspace_bytes(tw, call.n, call.plane) > call.workspace_bytes) return cudaErrorInvalidValue;
  float* part = static_cast<float*>(call.workspace);
  float* pbias = part + static_cast<size_t>(g.splits) * tw.n_rt * tw.n_nc * 128 * tw.nw;

  const uint64_t P = static_cast<uint64_t>(call.plane);
  CUtensorMap tdy, tx;
  bool dy4d = false;
  if (call.plane % kAtom == 0 && g.blk > 1) {
    // dy as {32 px, D, N*cls rows, P/32 atoms}: one box = [atoms][rows][128 B]
    const uint64_t dims[4] = {static_cast<uint64_t>(kAtom), static_cast<uint64_t>(tw.n_class),
                              static_cast<uint64_t>(call.n) * tw.cls, P / kAtom};
    const uint64_t strides[3] = {P * 4, P * 4 * tw.n_class, kAtom * 4};
    const uint32_t box[4] = {kAtom, 1, static_cast<uint32_t>(tw.rba), static_cast<uint32_t>(g.blk)};
    dy4d = encode_f32_sw128(&tdy, call.dy, 4, dims, strides, box);
  }
  // With one atom per stage the dy stage is plain [128 rows][128 B], so a box
  // may span every row of one class run (up to the whole tile): fewer TMA
  // instructions per chunk (each one holds its issuing thread ~0.3 us).
  int rba = tw.rba;
  if (!dy4d && g.blk == 1) {
    for (int rb : {128, 64}) {
      if (rb > rba && tw.cls % rb == 0) {
        rba = rb;
        break;
      }
    }
  }
  if (!dy4d) {
    const uint64_t dims[3] = {P, static_cast<uint64_t>(tw.n_class),
                              static_cast<uint64_t>(call.n) * tw.cls};
    const uint64_t strides[2] = {P * 4, P * 4 * tw.n_class};
    const uint32_t box[3] = {kAtom, 1, static_cast<uint32_t>(rba)};
    if (!encode_f32_sw128(&tdy, call.dy, 3, dims, strides, box)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[3] = {P, 1, static_cast<uint64_t>(call.n) * call.c_in};
    const uint64_t strides[2] = {P * 4, P * 4};
    const uint32_t box[3] = {kAtom, 1, static_cast<uint32_t>(tw.rbb1)};
    if (!encode_f32_sw128(&tx, call.x, 3, dims, strides, box)) return cudaErrorInvalidValue;
  }
  WArgs a{};
  a.rt_info = call.rt_info;
  a.class_d = call.class_d;
  a.perm = call.perm;
  a.starts = call.starts;
  a.gw = call.gw;
  a.part = part;
  a.pbias = pbias;
  a.n_rt = tw.n_rt;
  a.n_nc = tw.n_nc;
  a.nw = tw.nw;
  a.cls = tw.cls;
  a.c_in = call.c_in;
  a.c_out = call.c_out;
  a.rba = rba;
  a.rbb = tw.rbb1;
  a.blk = g.blk;
  a.a_stages = g.a_stages;
  a.t_stages = g.t_stages;
  a.acol0 = g.acol0;
  a.dy4d = dy4d ? 1 : 0;
  a.has_bias = call.dbias != nullptr;
  a.pcs = g.pcs;
  a.total_chunks = g.total_chunks;
  a.chunks_per_split = g.chunks_per_split;
  a.plane = call.plane;
  {
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
      cudaError_t e = cudaFuncSetAttribute(tc_weight_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           227 * 1024 - 1024);
      if (e != cudaSuccess) return e;
      if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
  }
  const unsigned grid = static_cast<unsigned>(g.splits) * tw.n_rt * tw.n_nc;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = g.smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, tc_weight_kernel, tdy, tx, a);
  if (e != cudaSuccess) return e;
  FArgs f{};
  f.part = part;
  f.pbias = pbias;
  f.rt_info = call.rt_info;
  f.starts = call.starts;
  f.inv_perm = call.inv_perm;
  f.dweight = call.dweight;
  f.dbias = call.dbias;
  f.splits = g.splits;
  f.n_rt = tw.n_rt;
  f.n_nc = tw.n_nc;
  f.nw = tw.nw;
  f.c_in = call.c_in;
  f.c_out = call.c_out;
  f.gw = call.gw;
  const int64_t outs = static_cast<int64_t>(call.c_out) * call.gw + (call.dbias ? call.c_out : 0);
  cudaLaunchConfig_t fc{};
  fc.stream = s;
  fc.attrs = attr;
  fc.numAttrs = 1;
  if (outs >= 65536) {
    fc.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>((outs + 255) / 256, 148 * 8)));
    fc.blockDim = dim3(256);
    e = cudaLaunchKernelEx(&fc, tc_weight_finalize_wide, f);
  } else {
    const int wf = fin_warps(outs);
    fc.gridDim = dim3(static_cast<unsigned>((outs + 31) / 32));
    fc.blockDim = dim3(32 * wf);
    switch (wf) {
      case 32: e = cudaLaunchKernelEx(&fc, tc_weight_finalize<32>, f); break;
      case 16: e = cudaLaunchKernelEx(&fc, tc_weight_finalize<16>, f); break;
      case 8: e = cudaLaunchKernelEx(&fc, tc_weight_finalize<8>, f); break;
      case 4: e = cudaLaunchKernelEx(&fc, tc_weight_finalize<4>, f); break;
      case 2: e = cudaLaunchKernelEx(&fc, tc_weight_finalize<2>, f); break;
      default: e = cudaLaunchKernelEx(&fc, tc_weight_finalize<1>, f); break;
    }
  }
  note_launches(2);
  return e;
}

}  // namespace scc
