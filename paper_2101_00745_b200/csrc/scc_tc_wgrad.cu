// Tensor-core (tcgen05, 3xTF32) backward-weight of the SCC operator, sm_100a
// (replaces scc_backward_params, kernel.cpp:140-181).
//
//   dWband[oc, ic] = sum_{n,p} dy[n, oc, p] * x[n, ic, p]      (ic in the arc of oc's tile)
//   db[oc]         = sum_{n,p} dy[n, oc, p]
//
// GEMM with M = 128 filters (cycle-sorted order), N = the tile's input-channel
// arc (<= 256 columns per chunk), K = pixels.  Both operands are pixel-
// contiguous, i.e. K-major, so TMA drops them straight into the canonical
// SWIZZLE_128B layout (box {32 pixels, 8 rows}); converter warps add the tf32
// "lo" copies (and the bias row sums) in shared memory.  The pixel range is
// split across CTAs; every CTA writes its fp32 partial tile, and a second
// kernel reduces the partials in a fixed order (warp per output, fixed lane
// assignment and shuffle tree) and scatters the band entries into the
// window-relative [oc][k] layout.  No atomics: results are bitwise
// reproducible.
#include <algorithm>

#include "scc_kernels.hpp"
#include "scc_plan.hpp"
#include "sm100.cuh"
#include "tmap.hpp"

namespace scc {
namespace {

using namespace sm100;

// Diagnostic timeline (CTA 0, ns): 0 start, 1 setup, 2+i refill of chunk
// i issued (i<8), 10+i converter done with chunk i, 18+i MMA committed chunk
// i, 26 epilogue done.
__device__ unsigned long long g_wtrace[32];
#define WTRACE(slot)                                            \
  do {                                                          \
    if (blockIdx.x == 0) g_wtrace[(slot)] = globaltimer();      \
  } while (0)

constexpr int kThreads = 320;
constexpr int kPix = 32;             // pixels (K) per stage
constexpr int kABytes = 128 * kPix * 4;  // 16 KB: 128 filter rows x 32 pixels
constexpr int kMaxStages = 4;

struct WArgs {
  const int32_t* rt_info;  // per row tile: start8, ncols
  const int32_t* class_d;
  float* part;             // [split][rt][nc][128][nw]
  float* pbias;            // [split][rt][128]
  int32_t n_rt, n_nc, nw, cls, c_in, c_out, stages;
  int32_t rba, rbb;        // TMA box rows (dy per quarter, x)
  int32_t has_bias;
  int64_t pcs;             // pixel chunks per sample
  int64_t total_chunks, chunks_per_split;
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
  const int S = a.stages;
  const int bbytes = a.nw * kPix * 4;
  const int stage_bytes = 2 * kABytes + 2 * bbytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + S * stage_bytes);
  uint64_t* full = bars;                       // [kMaxStages][4] one per loader warp
  uint64_t* conv = bars + 4 * kMaxStages;      // [kMaxStages] 4 warp arrivals
  uint64_t* empty = bars + 5 * kMaxStages;     // [kMaxStages] MMA done with the stage
  uint64_t* tfull = bars + 6 * kMaxStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 6 * kMaxStages + 1);
  auto a_hi = [&](int s) { return smem + s * stage_bytes; };
  auto a_lo = [&](int s) { return smem + s * stage_bytes + kABytes; };
  auto b_hi = [&](int s) { return smem + s * stage_bytes + 2 * kABytes; };
  auto b_lo = [&](int s) { return smem + s * stage_bytes + 2 * kABytes + bbytes; };

  const int nc = static_cast<int>(blockIdx.x % a.n_nc);
  const int rest = static_cast<int>(blockIdx.x / a.n_nc);
  const int rt = rest % a.n_rt;
  const int split = rest / a.n_rt;
  const int64_t q_begin = static_cast<int64_t>(split) * a.chunks_per_split;
  const int64_t q_end = min(a.total_chunks, q_begin + a.chunks_per_split);
  const int nchunks = q_end > q_begin ? static_cast<int>(q_end - q_begin) : 0;
  const int start8 = a.rt_info[2 * rt], ncols = a.rt_info[2 * rt + 1];

  const uint32_t warp = warp_id();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    WTRACE(0);
    for (int s = 0; s < S; ++s) {
      for (int q = 0; q < 4; ++q) mbar_init(&full[4 * s + q], 1);
      mbar_init(&conv[s], 4);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_mbar_init();
  }
  if (warp == 2 && lane == 0) {
    prefetch_tmap(&tdy);
    prefetch_tmap(&tx);
  }
  if (warp == 1) tmem_alloc<256>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) WTRACE(1);

  if (warp == 0) {
    // (loads are issued by the four converter warps, see below)
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = idesc_tf32(128, a.nw, 0, 0);
    int stage = 0;
    uint32_t phase = 0;
    for (int c = 0; c < nchunks; ++c) {
      mbar_wait_tag(&conv[stage], phase, 10);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t ah = smem_u32(a_hi(stage)), al = smem_u32(a_lo(stage));
        const uint32_t bh = smem_u32(b_hi(stage)), bl = smem_u32(b_lo(stage));
#pragma unroll
        for (int ks = 0; ks < kPix / 8; ++ks) {
          const uint64_t dah = desc_sw128(ah + ks * 32, 16, 1024);
          const uint64_t dal = desc_sw128(al + ks * 32, 16, 1024);
          const uint64_t dbh = desc_sw128(bh + ks * 32, 16, 1024);
          const uint64_t dbl = desc_sw128(bl + ks * 32, 16, 1024);
          mma_tf32(tmem, dah, dbh, idesc, (c | ks) != 0);
          mma_tf32(tmem, dal, dbh, idesc, 1);
          mma_tf32(tmem, dah, dbl, idesc, 1);
        }
        mma_commit(&empty[stage]);
        if (c == nchunks - 1) mma_commit(tfull);
        if (c < 8) WTRACE(18 + c);
      }
      __syncwarp();
      advance(stage, phase, S);
    }
  } else if (warp < 6) {
    // ---------------- loaders + converters (+ bias row sums) ----------------
    // Warp q loads and converts filter rows 32q..32q+31 of the tile and x
    // rows [q*nw/4, (q+1)*nw/4) of the column chunk: the TMA issue cost is
    // spread over four warps and nobody waits for another warp's loads.
    const int q = warp & 3;
    const int t = q * 32 + lane;  // filter row of the tile owned by this thread
    const int bq = a.nw / 4;      // x rows per warp
    float bsum = 0.f;
    int a_rows = 0, b_rows = 0;
    {
      const int i0 = rt * 128 + 32 * q;
      a_rows = min(32, max(0, a.c_out - i0));
      const int r0 = nc * a.nw + q * bq;
      b_rows = min(bq, max(0, ncols - r0));
      a_rows = (a_rows + a.rba - 1) / a.rba * a.rba;  // boxes are issued whole
      b_rows = (b_rows + a.rbb - 1) / a.rbb * a.rbb;
    }
    auto issue = [&](int s, int64_t qc) {
      if (lane != 0) return;
      const int n = static_cast<int>(qc / a.pcs);
      const int p0 = static_cast<int>(qc - static_cast<int64_t>(n) * a.pcs) * kPix;
      mbar_expect_tx(&full[4 * s + q], (a_rows + b_rows) * 128);
      for (int r = 0; r < a_rows; r += a.rba) {
        const int i0 = rt * 128 + 32 * q + r;
        const int cl = i0 / a.cls, j = i0 - cl * a.cls;
        tma_load_3d(a_hi(s) + (32 * q + r) * 128, &tdy, &full[4 * s + q], p0, __ldg(a.class_d + cl),
                    n * a.cls + j);
      }
      for (int r = 0; r < b_rows; r += a.rbb) {
        int pos = start8 + nc * a.nw + q * bq + r;
        while (pos >= a.c_in) pos -= a.c_in;
        tma_load_3d(b_hi(s) + (q * bq + r) * 128, &tx, &full[4 * s + q], p0, 0, n * a.c_in + pos);
      }
    };
    for (int c = 0; c < min(S, nchunks); ++c) issue(c, q_begin + c);
    int stage = 0;
    uint32_t phase = 0;
    int prev_stage = 0;
    uint32_t prev_phase = 0;
    for (int c = 0; c < nchunks; ++c) {
      mbar_wait_tag(&full[4 * stage + q], phase, 11);
      {
        // row t occupies the 128 B at (t/8)*1024 + (t%8)*128 (16 B chunks swizzled)
        const float4* src = reinterpret_cast<const float4*>(a_hi(stage) + (t >> 3) * 1024 + (t & 7) * 128);
        float4* dst = reinterpret_cast<float4*>(a_lo(stage) + (t >> 3) * 1024 + (t & 7) * 128);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float4 v = src[k];
          float4 lo;
          lo.x = v.x - tf32_hi(v.x);
          lo.y = v.y - tf32_hi(v.y);
          lo.z = v.z - tf32_hi(v.z);
          lo.w = v.w - tf32_hi(v.w);
          dst[k] = lo;
          bsum += ((v.x + v.y) + v.z) + v.w;
        }
      }
      {
        const float4* src = reinterpret_cast<const float4*>(b_hi(stage) + q * bq * 128);
        float4* dst = reinterpret_cast<float4*>(b_lo(stage) + q * bq * 128);
        for (int i = lane; i < bq * 8; i += 32) {
          const float4 v = src[i];
          float4 lo;
          lo.x = v.x - tf32_hi(v.x);
          lo.y = v.y - tf32_hi(v.y);
          lo.z = v.z - tf32_hi(v.z);
          lo.w = v.w - tf32_hi(v.w);
          dst[i] = lo;
        }
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[stage]);
      if (c < 8 && t == 0) WTRACE(10 + c);
      // Refill the previous stage once the MMAs of its chunk are done.
      if (c >= 1 && c - 1 + S < nchunks) {
        mbar_wait_tag(&empty[prev_stage], prev_phase, 12);
        issue(prev_stage, q_begin + c - 1 + S);
        if (c - 1 < 8 && t == 0) WTRACE(2 + (c - 1));
      }
      prev_stage = stage;
      prev_phase = phase;
      advance(stage, phase, S);
    }
    if (a.has_bias && nc == 0) {
      a.pbias[(static_cast<int64_t>(split) * a.n_rt + rt) * 128 + t] = bsum;
    }
  } else {
    // ---------------- epilogue: accumulator -> partial tile ----------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    float* dst = a.part + ((static_cast<int64_t>(split) * a.n_rt + rt) * a.n_nc + nc) * 128 * a.nw +
                 static_cast<int64_t>(row) * a.nw;
    if (nchunks > 0) {
      mbar_wait_tag(tfull, 0, 13);
      tc_fence_after();
      const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
      for (int c0 = 0; c0 < a.nw; c0 += 16) {
        float v[16];
        tmem_ld16(taddr + c0, v);
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          *reinterpret_cast<float4*>(dst + c0 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
        }
      }
    } else {
      for (int c0 = 0; c0 < a.nw; c0 += 4) *reinterpret_cast<float4*>(dst + c0) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (row == 0) WTRACE(26);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<256>(tmem);
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

// Warp per output: lane l sums splits l, l+32, ... in order, then a fixed
// butterfly combines the lanes.
__global__ void __launch_bounds__(256) tc_weight_finalize(const FArgs a) {
  const int64_t nw_out = static_cast<int64_t>(a.c_out) * a.gw;
  const int64_t total = nw_out + (a.dbias ? a.c_out : 0);
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x / 32);
  for (int64_t o = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + (threadIdx.x >> 5); o < total;
       o += warps) {
    float s = 0.f;
    if (o < nw_out) {
      const int oc = static_cast<int>(o / a.gw);
      const int k = static_cast<int>(o - static_cast<int64_t>(oc) * a.gw);
      const int pos = a.inv_perm[oc];
      const int rt = pos >> 7, row = pos & 127;
      int col = a.starts[oc] + k - a.rt_info[2 * rt];
      while (col < 0) col += a.c_in;
      while (col >= a.c_in) col -= a.c_in;
      const int nc = col / a.nw, c = col - nc * a.nw;
      const int64_t base = ((static_cast<int64_t>(rt) * a.n_nc + nc) * 128 + row) * a.nw + c;
      const int64_t stride = static_cast<int64_t>(a.n_rt) * a.n_nc * 128 * a.nw;
      for (int sp = lane; sp < a.splits; sp += 32) s += a.part[base + sp * stride];
    } else {
      const int oc = static_cast<int>(o - nw_out);
      const int pos = a.inv_perm[oc];
      const int rt = pos >> 7, row = pos & 127;
      for (int sp = lane; sp < a.splits; sp += 32) s += a.pbias[(static_cast<int64_t>(sp) * a.n_rt + rt) * 128 + row];
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
    if (lane == 0) {
      if (o < nw_out) a.dweight[o] = s;
      else a.dbias[o - nw_out] = s;
    }
  }
}

struct WGrid {
  int64_t pcs, total_chunks, chunks_per_split;
  int32_t splits, stages;
  int smem;
};

WGrid weight_grid(const TcWeightPlan& tw, int64_t n, int64_t plane) {
  WGrid g{};
  g.pcs = (plane + kPix - 1) / kPix;
  g.total_chunks = n * g.pcs;
  const int64_t items = static_cast<int64_t>(tw.n_rt) * tw.n_nc;
  int64_t splits = std::max<int64_t>(1, (148 + items - 1) / items);
  splits = std::min(splits, g.total_chunks);
  g.chunks_per_split = (g.total_chunks + splits - 1) / splits;
  g.splits = static_cast<int32_t>((g.total_chunks + g.chunks_per_split - 1) / g.chunks_per_split);
  const int stage_bytes = 2 * kABytes + 2 * tw.nw * kPix * 4;
  g.stages = std::min(kMaxStages, (200 * 1024) / stage_bytes);
  g.smem = g.stages * stage_bytes + 1024 + 256;
  return g;
}

}  // namespace

int tc_wtrace(unsigned long long* out, int n) {
  if (n > 32) n = 32;
  return cudaMemcpyFromSymbol(out, g_wtrace, n * sizeof(unsigned long long)) == cudaSuccess ? n : -1;
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
  if (tc_weight_workspace_bytes(tw, call.n, call.plane) > call.workspace_bytes) return cudaErrorInvalidValue;
  float* part = static_cast<float*>(call.workspace);
  float* pbias = part + static_cast<size_t>(g.splits) * tw.n_rt * tw.n_nc * 128 * tw.nw;

  CUtensorMap tdy, tx;
  {
    const uint64_t dims[3] = {static_cast<uint64_t>(call.plane), static_cast<uint64_t>(tw.n_class),
                              static_cast<uint64_t>(call.n) * tw.cls};
    const uint64_t strides[2] = {static_cast<uint64_t>(call.plane) * 4,
                                 static_cast<uint64_t>(call.plane) * 4 * tw.n_class};
    const uint32_t box[3] = {kPix, 1, static_cast<uint32_t>(tw.rba)};
    if (!encode_f32_sw128(&tdy, call.dy, 3, dims, strides, box)) return cudaErrorInvalidValue;
  }
  {
    const uint64_t dims[3] = {static_cast<uint64_t>(call.plane), 1,
                              static_cast<uint64_t>(call.n) * call.c_in};
    const uint64_t strides[2] = {static_cast<uint64_t>(call.plane) * 4,
                                 static_cast<uint64_t>(call.plane) * 4};
    const uint32_t box[3] = {kPix, 1, static_cast<uint32_t>(tw.rbb)};
    if (!encode_f32_sw128(&tx, call.x, 3, dims, strides, box)) return cudaErrorInvalidValue;
  }
  WArgs a{};
  a.rt_info = call.rt_info;
  a.class_d = call.class_d;
  a.part = part;
  a.pbias = pbias;
  a.n_rt = tw.n_rt;
  a.n_nc = tw.n_nc;
  a.nw = tw.nw;
  a.cls = tw.cls;
  a.c_in = call.c_in;
  a.c_out = call.c_out;
  a.stages = g.stages;
  a.rba = tw.rba;
  a.rbb = tw.rbb;
  a.has_bias = call.dbias != nullptr;
  a.pcs = g.pcs;
  a.total_chunks = g.total_chunks;
  a.chunks_per_split = g.chunks_per_split;
  {
    static bool attr_set[64] = {false};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64 || !attr_set[dev]) {
      cudaError_t e = cudaFuncSetAttribute(tc_weight_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           227 * 1024);
      if (e != cudaSuccess) return e;
      if (dev >= 0 && dev < 64) attr_set[dev] = true;
    }
  }
  const unsigned grid = static_cast<unsigned>(g.splits) * tw.n_rt * tw.n_nc;
  tc_weight_kernel<<<grid, kThreads, g.smem, s>>>(tdy, tx, a);
  cudaError_t e = cudaGetLastError();
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
  const int fgrid = static_cast<int>(std::min<int64_t>((outs + 7) / 8, 148 * 16));
  tc_weight_finalize<<<fgrid, 256, 0, s>>>(f);
  note_launches(2);
  return cudaGetLastError();
}

}  // namespace scc
