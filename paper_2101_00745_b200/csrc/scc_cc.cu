// CUDA-core (fp32 FFMA) family of the SCC operator, sm_100a.
//
// band_cc_kernel  — forward (kernel.cpp:29-69) AND input-centric backward-data
//                   (kernel.cpp:98-138).  Both are the same "banded channel
//                   mix": every output row (a filter, or an input channel)
//                   reduces a cyclic arc of the other side's channels.  A CTA
//                   owns 128 pixels and a group of 8 row-blocks (8 rows each,
//                   one per warp); it stages the group's arc of input rows in
//                   shared memory chunk by chunk, so each input row is read
//                   once per group and reused by every filter whose window
//                   covers it (the paper's channel-cyclic reuse).  Writes are
//                   disjoint per output element: no atomics anywhere.
// weight_cc_kernel — backward-weight (kernel.cpp:140-181): per row-block and
//                   arc tile, outer products over pixel tiles staged in smem,
//                   fixed-order reduction across lanes, then a fixed-order
//                   reduction across pixel splits in weight_finalize_kernel.
//                   Deterministic: bitwise identical from run to run.
#include <algorithm>

#include "scc_kernels.hpp"
#include "scc_plan.hpp"

namespace scc {
namespace {

constexpr int kThreads = 256;
constexpr int KC = 32;   // ring positions per staged chunk
constexpr int TQ = 128;  // pixels per CTA in the band kernel (32 lanes x 4)

__device__ __forceinline__ int wrap(int v, int n) { return v >= n ? v - n : v; }

// w[oc][(ic - start(oc)) mod c_in] inside the window, else 0.
__device__ __forceinline__ float band_weight(const BandLaunch& a, int oc, int ic) {
  int s = ic - __ldg(a.starts + oc);
  if (s < 0) s += a.c_in;
  return s < a.gw ? __ldg(a.weight + static_cast<int64_t>(oc) * a.gw + s) : 0.f;
}

// Pixel q -> (sample n, in-plane p); 32-bit division when it fits.
__device__ __forceinline__ void pix_np(int64_t q, int64_t plane, int64_t& n, int64_t& p) {
  if (q < 0x7fffffffLL && plane < 0x7fffffffLL) {
    const uint32_t qq = static_cast<uint32_t>(q), pl = static_cast<uint32_t>(plane);
    const uint32_t nn = qq / pl;
    n = nn;
    p = qq - nn * pl;
  } else {
    n = q / plane;
    p = q - n * plane;
  }
}

// Pixel q -> element offset of (n, channel 0, p) in an [N][C][P] tensor.
__device__ __forceinline__ int64_t pix_offset(int64_t q, int64_t plane, int64_t c_t) {
  int64_t n, p;
  pix_np(q, plane, n, p);
  return n * c_t * plane + p;
}

// Fused depthwise prologue.  A staging thread owns 4 fixed DW-output pixels
// for the whole chunk loop, so their input offsets and 3x3 tap masks are
// computed once (DwPix); each staged element is then 9 predicated loads and
// 9 FMAs in the order of conv_forward_impl (bias, then taps i, j ascending,
// reference.cpp:94-106; out-of-plane taps contribute nothing where the
// reference multiplies an explicit 0.0, reference.cpp:67-72).
struct DwPix {
  int64_t base;   // element offset of (n, channel 0, iy0, ix0) in x, iy0 = oy*s - 1
  uint32_t mask;  // bit 3i+j: tap (i, j) inside the input plane
};

__device__ __forceinline__ DwPix dw_pix(const BandLaunch& a, int64_t q, bool valid) {
  DwPix d{0, 0u};
  if (!valid) return d;
  int64_t n, p;
  pix_np(q, a.plane, n, p);
  const int oy = static_cast<int>(p / a.w_out), ox = static_cast<int>(p - static_cast<int64_t>(oy) * a.w_out);
  const int iy0 = oy * a.dw_stride - 1, ix0 = ox * a.dw_stride - 1;
  d.base = n * a.c_in_t * static_cast<int64_t>(a.h_in) * a.w_in + static_cast<int64_t>(iy0) * a.w_in + ix0;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      if (iy0 + i >= 0 && iy0 + i < a.h_in && ix0 + j >= 0 && ix0 + j < a.w_in) d.mask |= 1u << (3 * i + j);
  return d;
}

__device__ __forceinline__ float dw_value(const BandLaunch& a, const float (&wk)[9], float b,
                                          const float* chan, const DwPix& d) {
  float sum = b;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const float v = (d.mask >> (3 * i + j)) & 1u ? __ldg(chan + d.base + i * a.w_in + j) : 0.f;
      sum = fmaf(wk[3 * i + j], v, sum);
    }
  return sum;
}

template <bool VEC, bool DW = false>
__global__ void __launch_bounds__(kThreads) band_cc_kernel(const BandLaunch a) {
  __shared__ __align__(16) float xs[KC][TQ];
  __shared__ __align__(16) float ws[kBlocksPerGroup][KC][kRowsPerBlock];

  const int g = static_cast<int>(blockIdx.x % a.ngrp);
  const int64_t q0 = static_cast<int64_t>(blockIdx.x / a.ngrp) * TQ;
  const int first = a.groups[4 * g + 0];
  const int nb = a.groups[4 * g + 1];
  const int gstart = a.groups[4 * g + 2];
  const int glen = a.groups[4 * g + 3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t qend = a.n * a.plane;

  const bool active = warp < nb;
  int boff = 0, blen = 0;
  int orow[kRowsPerBlock];
  float4 acc[kRowsPerBlock];
  if (active) {
    const int blk = first + warp;
    blen = a.blocks[2 * blk + 1];
    boff = a.blocks[2 * blk] - gstart;
    if (boff < 0) boff += a.ring;
#pragma unroll
    for (int j = 0; j < kRowsPerBlock; ++j) {
      orow[j] = a.rows[blk * kRowsPerBlock + j];
      const float b = (a.bias != nullptr && orow[j] >= 0) ? __ldg(a.bias + orow[j]) : 0.f;
      acc[j] = make_float4(b, b, b, b);
    }
  }
  // The block's arc in group coordinates: [boff, boff+blen), which can wrap
  // past glen only when the group arc is the whole ring.
  const int i1_lo = boff, i1_hi = min(boff + blen, glen);
  const int i2_hi = max(0, boff + blen - glen);

  // Staging role of this thread: pixel column c4 (fixed), rows warp+8k.
  const int c4 = threadIdx.x & (TQ / 4 - 1);
  const int64_t qv = q0 + c4 * 4;
  int64_t poff[4];
  bool pval[4];
  if (VEC) {
    pval[0] = qv < qend;
    poff[0] = pval[0] ? pix_offset(qv, a.plane, a.c_in_t) : 0;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      pval[e] = qv + e < qend;
      poff[e] = pval[e] ? pix_offset(qv + e, a.plane, a.c_in_t) : 0;
    }
  }
  DwPix dwp[4];
  if (DW) {
#pragma unroll
    for (int e = 0; e < 4; ++e) dwp[e] = dw_pix(a, qv + e, qv + e < qend);
  }
  // Weight-staging role: (r, j) fixed, one entry per block of the group.
  const int wr = threadIdx.x >> 3, wj = threadIdx.x & 7;

  for (int c0 = 0; c0 < glen; c0 += KC) {
    const int kc = min(KC, glen - c0);
#pragma unroll
    for (int k = 0; k < KC / (kThreads / (TQ / 4)); ++k) {
      const int r = (threadIdx.x >> 5) + k * (kThreads / (TQ / 4));
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < kc && DW) {
        // fused dsc_block: stage DW3x3(x) rows instead of x rows; the DW
        // output never goes to HBM (forward ring = input channels)
        const int ch = wrap(gstart + c0 + r, a.ring);
        const float* chan = a.in + static_cast<int64_t>(ch) * a.h_in * a.w_in;
        float wk[9];
#pragma unroll
        for (int t = 0; t < 9; ++t) wk[t] = __ldg(a.dw_w + ch * 9 + t);
        const float b = a.dw_b != nullptr ? __ldg(a.dw_b + ch) : 0.f;
        v.x = dw_value(a, wk, b, chan, dwp[0]);
        v.y = dw_value(a, wk, b, chan, dwp[1]);
        v.z = dw_value(a, wk, b, chan, dwp[2]);
        v.w = dw_value(a, wk, b, chan, dwp[3]);
      } else if (r < kc) {
        const int pos = wrap(gstart + c0 + r, a.ring);
        const int ch = a.ring_map ? __ldg(a.ring_map + pos) : pos;
        const float* src = a.in + static_cast<int64_t>(ch) * a.plane;
        if (VEC) {
          if (pval[0]) v = __ldg(reinterpret_cast<const float4*>(src + poff[0]));
        } else {
          v.x = pval[0] ? __ldg(src + poff[0]) : 0.f;
          v.y = pval[1] ? __ldg(src + poff[1]) : 0.f;
          v.z = pval[2] ? __ldg(src + poff[2]) : 0.f;
          v.w = pval[3] ? __ldg(src + poff[3]) : 0.f;
        }
      }
      *reinterpret_cast<float4*>(&xs[r][c4 * 4]) = v;
    }
    for (int wb = 0; wb < nb; ++wb) {
      float v = 0.f;
      if (wr < kc) {
        const int blk = first + wb;
        int off = a.blocks[2 * blk] - gstart;
        if (off < 0) off += a.ring;
        int u = c0 + wr - off;
        if (u < 0) u += a.ring;
        const int row = a.rows[blk * kRowsPerBlock + wj];
        if (u < a.blocks[2 * blk + 1] && row >= 0) {
          const int pos = wrap(gstart + c0 + wr, a.ring);
          v = a.backward_data ? band_weight(a, __ldg(a.ring_map + pos), row)
                              : band_weight(a, row, pos);
        }
      }
      ws[wb][wr][wj] = v;
    }
    __syncthreads();
    if (active) {
      // Two sub-ranges of this chunk that lie inside the block arc.
      const int ra0 = max(i1_lo - c0, 0), ra1 = min(i1_hi - c0, kc);
      const int rb0 = 0, rb1 = min(i2_hi - c0, kc);
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        const int r0 = pass == 0 ? ra0 : rb0;
        const int r1 = pass == 0 ? ra1 : rb1;
#pragma unroll 4
        for (int r = r0; r < r1; ++r) {
          const float4 xv = *reinterpret_cast<const float4*>(&xs[r][lane * 4]);
          const float4 w0 = *reinterpret_cast<const float4*>(&ws[warp][r][0]);
          const float4 w1 = *reinterpret_cast<const float4*>(&ws[warp][r][4]);
          const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
          for (int j = 0; j < kRowsPerBlock; ++j) {
            acc[j].x = fmaf(wv[j], xv.x, acc[j].x);
            acc[j].y = fmaf(wv[j], xv.y, acc[j].y);
            acc[j].z = fmaf(wv[j], xv.z, acc[j].z);
            acc[j].w = fmaf(wv[j], xv.w, acc[j].w);
          }
        }
      }
    }
    __syncthreads();
  }
  if (active) {
    const int64_t qo = q0 + lane * 4;
    int64_t ooff[4];
    bool oval[4];
    if (VEC) {
      oval[0] = qo < qend;
      ooff[0] = oval[0] ? pix_offset(qo, a.plane, a.c_out_t) : 0;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        oval[e] = qo + e < qend;
        ooff[e] = oval[e] ? pix_offset(qo + e, a.plane, a.c_out_t) : 0;
      }
    }
#pragma unroll
    for (int j = 0; j < kRowsPerBlock; ++j) {
      if (orow[j] < 0) continue;
      float* dst = a.out + static_cast<int64_t>(orow[j]) * a.plane;
      if (VEC) {
        if (oval[0]) *reinterpret_cast<float4*>(dst + ooff[0]) = acc[j];
      } else {
        if (oval[0]) dst[ooff[0]] = acc[j].x;
        if (oval[1]) dst[ooff[1]] = acc[j].y;
        if (oval[2]) dst[ooff[2]] = acc[j].z;
        if (oval[3]) dst[ooff[3]] = acc[j].w;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// backward-weight

struct WeightGrid {
  int kt_size;      // 32 or 64 arc positions per CTA
  int nkt;          // arc tiles per block
  int splits;       // pixel splits (reduced in finalize)
  int64_t qchunk;   // pixels per split (multiple of the pixel tile)
  int64_t blk_stride;   // floats per block in one split's partial slab
  int64_t split_stride; // floats per split
};

WeightGrid weight_grid(int32_t nblk, int32_t max_block_len, int64_t n, int64_t plane) {
  WeightGrid g{};
  g.kt_size = max_block_len <= 32 ? 32 : 64;
  g.nkt = std::max(1, (max_block_len + g.kt_size - 1) / g.kt_size);
  const int tqw = (kThreads / (g.kt_size / 4)) * 4;
  const int64_t q = n * plane;
  const int64_t tiles = std::max<int64_t>(1, (q + tqw - 1) / tqw);
  const int64_t want = (148 * 6 + static_cast<int64_t>(nblk) * g.nkt - 1) /
                       (static_cast<int64_t>(nblk) * g.nkt);
  g.splits = static_cast<int>(std::clamp<int64_t>(want, 1, std::max<int64_t>(1, tiles / 2)));
  const int64_t tiles_per = (tiles + g.splits - 1) / g.splits;
  g.qchunk = tiles_per * tqw;
  g.splits = static_cast<int>((q + g.qchunk - 1) / g.qchunk);
  if (g.splits < 1) g.splits = 1;
  g.blk_stride = static_cast<int64_t>(g.nkt) * g.kt_size * kRowsPerBlock + kRowsPerBlock;
  g.split_stride = g.blk_stride * nblk;
  return g;
}

template <int KT, bool VEC>
__global__ void __launch_bounds__(kThreads) weight_cc_kernel(const WeightLaunch a, WeightGrid gr) {
  constexpr int NKG = KT / 4;          // arc-position groups (4 positions each, strided)
  constexpr int NQL = kThreads / NKG;  // pixel lanes
  constexpr int TQW = NQL * 4;         // pixels per staged tile
  constexpr int XS = TQW + 4;          // padded row stride (bank-conflict free)
  constexpr int kStage = kRowsPerBlock * TQW + KT * XS;
  constexpr int kRed = NQL * kRowsPerBlock * KT;
  constexpr int kSmem = (kStage > kRed ? kStage : kRed) + NQL * kRowsPerBlock;
  __shared__ __align__(16) float smem[kSmem];
  float* gs = smem;                       // [8][TQW]
  float* xs = smem + kRowsPerBlock * TQW; // [KT][XS]
  float* red = smem;                      // [NQL][8][KT] (after the main loop)
  float* bred = smem + (kStage > kRed ? kStage : kRed);  // [NQL][8]

  const int blk = static_cast<int>(blockIdx.x % a.nblk);
  const int rest = static_cast<int>(blockIdx.x / a.nblk);
  const int kt = rest % gr.nkt;
  const int split = rest / gr.nkt;
  const int bstart = a.blocks[2 * blk], blen = a.blocks[2 * blk + 1];
  const int k0 = kt * KT;
  if (k0 >= blen && kt > 0) return;  // uniform across the CTA
  const int tid = threadIdx.x;
  const int kg = tid % NKG, ql = tid / NKG;
  const int64_t qend_all = a.n * a.plane;
  const int64_t qs = static_cast<int64_t>(split) * gr.qchunk;
  const int64_t qe = min(qend_all, qs + gr.qchunk);
  const bool bias_lane = (a.dbias != nullptr) && kt == 0 && kg == 0;

  int rows[kRowsPerBlock];
#pragma unroll
  for (int j = 0; j < kRowsPerBlock; ++j) rows[j] = a.rows[blk * kRowsPerBlock + j];

  float acc[kRowsPerBlock][4];
  float bacc[kRowsPerBlock];
#pragma unroll
  for (int j = 0; j < kRowsPerBlock; ++j) {
    bacc[j] = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[j][i] = 0.f;
  }

  // Staging role: pixel column sc4 (fixed per thread), rows (tid / (TQW/4)) + step*k.
  constexpr int kCols = TQW / 4;
  constexpr int kRowStep = kThreads / kCols;
  const int sc4 = tid % kCols;
  const int srow = tid / kCols;
  for (int64_t q0 = qs; q0 < qe; q0 += TQW) {
    const int64_t qv = q0 + sc4 * 4;
    int64_t offx[4], offg[4];
    bool val[4];
    if (VEC) {
      val[0] = qv < qe;
      if (val[0]) {
        int64_t n, p;
        pix_np(qv, a.plane, n, p);
        offx[0] = n * a.c_in * a.plane + p;
        offg[0] = n * a.c_out * a.plane + p;
      } else {
        offx[0] = offg[0] = 0;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        val[e] = qv + e < qe;
        offx[e] = val[e] ? pix_offset(qv + e, a.plane, a.c_in) : 0;
        offg[e] = val[e] ? pix_offset(qv + e, a.plane, a.c_out) : 0;
      }
    }
    for (int j = srow; j < kRowsPerBlock; j += kRowStep) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (rows[j] >= 0) {
        const float* src = a.dy + static_cast<int64_t>(rows[j]) * a.plane;
        if (VEC) {
          if (val[0]) v = __ldg(reinterpret_cast<const float4*>(src + offg[0]));
        } else {
          v.x = val[0] ? __ldg(src + offg[0]) : 0.f;
          v.y = val[1] ? __ldg(src + offg[1]) : 0.f;
          v.z = val[2] ? __ldg(src + offg[2]) : 0.f;
          v.w = val[3] ? __ldg(src + offg[3]) : 0.f;
        }
      }
      *reinterpret_cast<float4*>(gs + j * TQW + sc4 * 4) = v;
    }
#pragma unroll
    for (int r = srow; r < KT; r += kRowStep) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k0 + r < blen) {
        const int ch = wrap(bstart + k0 + r, a.c_in);
        const float* src = a.x + static_cast<int64_t>(ch) * a.plane;
        if (VEC) {
          if (val[0]) v = __ldg(reinterpret_cast<const float4*>(src + offx[0]));
        } else {
          v.x = val[0] ? __ldg(src + offx[0]) : 0.f;
          v.y = val[1] ? __ldg(src + offx[1]) : 0.f;
          v.z = val[2] ? __ldg(src + offx[2]) : 0.f;
          v.w = val[3] ? __ldg(src + offx[3]) : 0.f;
        }
      }
      *reinterpret_cast<float4*>(xs + r * XS + sc4 * 4) = v;
    }
    __syncthreads();
    float4 xv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) xv[i] = *reinterpret_cast<const float4*>(xs + (kg + NKG * i) * XS + ql * 4);
#pragma unroll
    for (int j = 0; j < kRowsPerBlock; ++j) {
      const float4 g4 = *reinterpret_cast<const float4*>(gs + j * TQW + ql * 4);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float t = acc[j][i];
        t = fmaf(g4.x, xv[i].x, t);
        t = fmaf(g4.y, xv[i].y, t);
        t = fmaf(g4.z, xv[i].z, t);
        t = fmaf(g4.w, xv[i].w, t);
        acc[j][i] = t;
      }
      if (bias_lane) bacc[j] += ((g4.x + g4.y) + g4.z) + g4.w;
    }
    __syncthreads();
  }

  // Fixed-order reduction across the pixel lanes.
#pragma unroll
  for (int j = 0; j < kRowsPerBlock; ++j) {
#pragma unroll
    for (int i = 0; i < 4; ++i) red[(ql * kRowsPerBlock + j) * KT + kg + NKG * i] = acc[j][i];
  }
  if (kt == 0 && kg == 0) {
#pragma unroll
    for (int j = 0; j < kRowsPerBlock; ++j) bred[ql * kRowsPerBlock + j] = bacc[j];
  }
  __syncthreads();
  float* part = a.partial + split * gr.split_stride + blk * gr.blk_stride;
  for (int o = tid; o < kRowsPerBlock * KT; o += kThreads) {
    const int j = o / KT, k = o - j * KT;
    float s = 0.f;
#pragma unroll 4
    for (int l = 0; l < NQL; ++l) s += red[(l * kRowsPerBlock + j) * KT + k];
    part[(k0 + k) * kRowsPerBlock + j] = s;
  }
  if (kt == 0 && tid < kRowsPerBlock) {
    float s = 0.f;
    for (int l = 0; l < NQL; ++l) s += bred[l * kRowsPerBlock + tid];
    part[gr.nkt * KT * kRowsPerBlock + tid] = s;
  }
}

__global__ void __launch_bounds__(kThreads) weight_finalize_kernel(const WeightLaunch a, WeightGrid gr) {
  const int64_t nw = static_cast<int64_t>(a.c_out) * a.gw;
  const int64_t total = nw + (a.dbias != nullptr ? a.c_out : 0);
  for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (idx < nw) {
      const int oc = static_cast<int>(idx / a.gw);
      const int slot = static_cast<int>(idx - static_cast<int64_t>(oc) * a.gw);
      const int pos = a.inv_perm[oc];
      const int blk = pos / kRowsPerBlock, j = pos - blk * kRowsPerBlock;
      int k = a.starts[oc] + slot - a.blocks[2 * blk];
      if (k < 0) k += a.c_in;
      if (k >= a.c_in) k -= a.c_in;
      const float* p = a.partial + blk * gr.blk_stride + k * kRowsPerBlock + j;
      float s = 0.f;
      for (int sp = 0; sp < gr.splits; ++sp) s += p[sp * gr.split_stride];
      a.dweight[idx] = s;
    } else {
      const int oc = static_cast<int>(idx - nw);
      const int pos = a.inv_perm[oc];
      const int blk = pos / kRowsPerBlock, j = pos - blk * kRowsPerBlock;
      const float* p = a.partial + blk * gr.blk_stride + gr.nkt * gr.kt_size * kRowsPerBlock + j;
      float s = 0.f;
      for (int sp = 0; sp < gr.splits; ++sp) s += p[sp * gr.split_stride];
      a.dbias[oc] = s;
    }
  }
}

// Plane padding for the tensor-core path on planes with P % 4 != 0 (TMA
// strides must be 16 B multiples): out[r][p] = p < P ? in[r][p] : 0 over
// P4 = P rounded up to 4 (pad), or the inverse copy (unpad).
__global__ void __launch_bounds__(256) pad_planes_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                         int64_t rows, int32_t P, int32_t P4, int32_t unpad) {
  const int32_t src_w = unpad ? P4 : P, dst_w = unpad ? P : P4;
  const int64_t total = rows * dst_w;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / dst_w;
    const int32_t c = static_cast<int32_t>(i - r * dst_w);
    out[i] = c < P ? __ldg(in + r * src_w + c) : 0.f;
  }
}

}  // namespace

cudaError_t launch_pad_planes(const float* in, float* out, int64_t rows, int32_t P, int32_t P4, bool unpad,
                              cudaStream_t s) {
  const int64_t total = rows * (unpad ? P : P4);
  if (total <= 0) return cudaSuccess;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16));
  pad_planes_kernel<<<grid, 256, 0, s>>>(in, out, rows, P, P4, unpad ? 1 : 0);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_band_cc(const BandLaunch& a, cudaStream_t s) {
  const int64_t q = a.n * a.plane;
  const int64_t tiles = (q + TQ - 1) / TQ;
  const int64_t grid = tiles * a.ngrp;
  if (grid <= 0) return cudaSuccess;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  if (a.dw_w != nullptr) {
    band_cc_kernel<false, true><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(a);
  } else if (a.plane % 4 == 0 && aligned16(a.in) && aligned16(a.out)) {
    band_cc_kernel<true><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(a);
  } else {
    band_cc_kernel<false><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(a);
  }
  note_launches(1);
  return cudaGetLastError();
}

size_t weight_cc_workspace_bytes(int32_t nblk, int32_t max_block_len, int64_t n,
                                 int64_t plane) {
  const WeightGrid g = weight_grid(nblk, max_block_len, n, plane);
  return static_cast<size_t>(g.split_stride) * g.splits * sizeof(float);
}

cudaError_t launch_weight_cc(const WeightLaunch& a, size_t ws_bytes, cudaStream_t s) {
  const WeightGrid g = weight_grid(a.nblk, a.max_block_len, a.n, a.plane);
  if (static_cast<size_t>(g.split_stride) * g.splits * sizeof(float) > ws_bytes)
    return cudaErrorInvalidValue;
  const int64_t grid = static_cast<int64_t>(a.nblk) * g.nkt * g.splits;
  const bool vec = a.plane % 4 == 0 && aligned16(a.dy) && aligned16(a.x);
  if (g.kt_size == 32) {
    if (vec) weight_cc_kernel<32, true><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(a, g);
    else weight_cc_kernel<32, false><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(a, g);
  } else {
    if (vec) weight_cc_kernel<64, true><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(a, g);
    else weight_cc_kernel<64, false><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(a, g);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t total = static_cast<int64_t>(a.c_out) * a.gw + (a.dbias ? a.c_out : 0);
  const int fgrid = static_cast<int>(std::min<int64_t>((total + kThreads - 1) / kThreads, 148 * 8));
  weight_finalize_kernel<<<fgrid, kThreads, 0, s>>>(a, g);
  note_launches(2);
  return cudaGetLastError();
}

}  // namespace scc
