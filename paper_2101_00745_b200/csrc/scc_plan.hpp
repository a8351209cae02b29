// Host-side plan for the B200 SCC operator.
//
// Replaces the reference's per-call geometry work (config.cpp:62-83,
// cycle.cpp:9-40, the pull table of kernel.cpp:109-118) with tables built once
// per layer configuration and uploaded once per device:
//   * the window start of every filter, start(oc) = (oc*shift) mod c_in, which
//     equals windows[oc mod cyclic_dist] of compute_channel_cycle
//     (cycle_test.cpp:104-106, asserted in build());
//   * a "cycle-sorted" permutation of the output channels (by window start,
//     then oc), under which every input channel's covering filters form one
//     contiguous arc (the inverse map covering_filters walks, cycle.cpp:28-40);
//   * band tiles: runs of kRowsPerBlock consecutive output rows (forward) or
//     input rows (backward-data) together with the smallest cyclic arc of the
//     other side's channels that feeds them.  The CUDA kernels iterate over
//     exactly that arc, so no kernel ever touches channels outside the band.
#pragma once

#include <atomic>
#include <cstdint>
#include <deque>
#include <mutex>
#include <string>
#include <vector>

#include "scc_b200.h"

namespace scc {

constexpr int kRowsPerBlock = 8;    // output rows owned by one warp
constexpr int kBlocksPerGroup = 8;  // warps (blocks) per CTA in the band kernels

// Thrown inside the library and mapped to scc_status_t at the C boundary.
struct Error {
  scc_status_t code;
  std::string msg;
};

// A cyclic arc [start, start+len) over a ring of `ring` positions.
struct Arc {
  int32_t start = 0;
  int32_t len = 0;
};

// Smallest arc covering every (non-empty) arc of `parts` on a ring of size n.
Arc cover_arcs(const std::vector<Arc>& parts, int32_t n);

// Band tiling of one operator direction.
struct BandSide {
  int32_t ring = 0;                  // positions on the reduction ring
  std::vector<int32_t> ring_map;     // ring position -> channel (empty = identity)
  std::vector<int32_t> rows;         // nblk*8 output channels (-1 = padding)
  std::vector<Arc> blocks;           // per block: arc on the ring
  std::vector<int32_t> groups;       // per group: first_blk, nblk, arc.start, arc.len
  int32_t max_block_len = 0;
  int nblk() const { return static_cast<int>(blocks.size()); }
  int ngrp() const { return static_cast<int>(groups.size() / 4); }
};

// Tensor-core band tiling of one direction (see scc_tc.cu): row tiles of nt
// output rows, each with an 8-aligned arc of the ring in 8-position k-steps.
struct TcBandPlan {
  bool ok = false;
  std::string why;                  // reason when !ok
  int32_t nt = 0, n_rt = 0, ring = 0;
  int32_t cls = 0;                  // ring positions per class (TMA dim 2 run)
  int32_t n_class = 1;              // TMA dim 1 extent (D for backward-data)
  int32_t rows_per_sample_3d = 0;   // TMA dim-2 rows per sample
  int32_t total_chunks = 0;
  int32_t rb = 8;                   // TMA box rows for the activations (8, 16 or 32)
  // Output tensor view for TMA stores of 32-row groups (store_ok == false:
  // the epilogue uses plain stores).
  bool store_ok = false;
  int32_t out_cls = 0, out_n_class = 1;
  std::vector<int32_t> out_class_d;
  std::vector<int32_t> rt_info;     // per row tile: start8, nk8, panel offset (floats), chunks
  std::vector<int32_t> rows;        // n_rt * nt
  std::vector<int32_t> class_d;     // class -> d coordinate
  std::vector<int32_t> chunk_base;  // n_rt + 1 prefix sums of chunks
};

// Tensor-core backward-weight tiling: row tiles of 128 filters (sorted order)
// x N-chunks (<= 256 columns) of the tile's input-channel arc; K = pixels.
struct TcWeightPlan {
  bool ok = false;
  std::string why;
  int32_t n_rt = 0, n_nc = 0, nw = 0;  // row tiles, column chunks per tile, chunk width
  int32_t c_in = 0, c_out = 0;
  int32_t cls = 0, n_class = 1;        // dy 3-D view (as backward-data)
  int32_t rba = 8, rbb = 8;            // TMA box rows for dy (per warp quarter) and x
  int32_t rbb1 = 8;                    // x box rows of the generation-1 kernel (no quarter rule)
  std::vector<int32_t> rt_info;        // per row tile: start8 (ic ring), ncols (8-aligned)
  std::vector<int32_t> class_d;
};

struct TcDeviceTables {
  const int32_t* rt_info = nullptr;
  const int32_t* rows = nullptr;
  const int32_t* class_d = nullptr;
  const int32_t* chunk_base = nullptr;
  const int32_t* starts = nullptr;
  const int32_t* perm = nullptr;
  const int32_t* out_class_d = nullptr;
  const int32_t* inv_perm = nullptr;
};

// Device copy of the tables (one per CUDA device).
struct DeviceTables {
  int device = -1;
  void* base = nullptr;  // single allocation
  const int32_t* fwd_rows = nullptr;
  const int32_t* fwd_blocks = nullptr;  // [nblk][2]
  const int32_t* fwd_groups = nullptr;  // [ngrp][4]
  const int32_t* bwd_rows = nullptr;
  const int32_t* bwd_blocks = nullptr;
  const int32_t* bwd_groups = nullptr;
  const int32_t* perm = nullptr;      // sorted position -> oc
  const int32_t* inv_perm = nullptr;  // oc -> sorted position
  const int32_t* starts = nullptr;    // oc -> window start
  TcDeviceTables tc_fwd, tc_bwd;
  const int32_t* tcw_rt_info = nullptr;
  const int32_t* tcw_class_d = nullptr;
};

// Device staging for the host-buffer entry points.
// Host-buffer entry points pipeline over batch chunks: copy-in stream,
// compute stream, copy-out stream, one event pair per chunk.
constexpr int kMaxHostChunks = 16;
struct HostStaging {
  int device = -1;
  void* buf = nullptr;
  size_t bytes = 0;
  void* stream = nullptr;     // cudaStream_t: compute
  void* stream_in = nullptr;  // cudaStream_t: H2D copies
  void* stream_out = nullptr; // cudaStream_t: D2H copies
  void* ev_in[kMaxHostChunks] = {};    // cudaEvent_t: chunk inputs resident
  void* ev_done[kMaxHostChunks] = {};  // cudaEvent_t: chunk outputs written
  void* ev_out = nullptr;              // cudaEvent_t: all D2H issued
  void* ev_fork = nullptr;             // cudaEvent_t: fork of the copy streams off the compute stream
};

// Per (device, stream, direction) scratch for the tensor-core weight panels,
// so concurrent calls on different streams never share one.
struct PanelBuf {
  int device = -1;
  void* stream = nullptr;
  int dir = 0;
  void* ptr = nullptr;
  size_t bytes = 0;
};

// Fork/join resources of the concurrent backward (backward-data on the caller
// stream, backward-weight on a side stream), per (device, caller stream).
struct ForkJoin {
  int device = -1;
  void* stream = nullptr;  // caller stream
  void* side = nullptr;    // cudaStream_t
  void* ev_fork = nullptr; // cudaEvent_t
  void* ev_join = nullptr;
};

// Scratch for the padded-plane tensor-core path, per (device, stream).
// Grown on demand; outgrown buffers are kept until the plan is destroyed
// (work queued earlier on the stream may still reference them).
struct PadBuf {
  int device = -1;
  void* stream = nullptr;
  void* ptr = nullptr;
  size_t bytes = 0;
  std::vector<void*> retired;
};

struct Plan {
  scc_config_t cfg{};
  std::vector<int64_t> cycle_starts;  // compute_channel_cycle order
  std::vector<int32_t> perm, inv_perm, starts;
  BandSide fwd, bwd;
  std::vector<Arc> ic_arcs;          // covering arc of each input channel (sorted order)
  TcBandPlan tc_fwd, tc_bwd;
  TcWeightPlan tc_wgt;
  // forced kernel family (scc_plan_set_path); atomic so a concurrent set_path
  // is not a data race (calls already in flight may still see either value)
  std::atomic<int32_t> path{SCC_PATH_AUTO};

  std::mutex dev_mu;
  std::deque<DeviceTables> dev;  // deque: references stay valid
  std::mutex panel_mu;
  std::deque<PanelBuf> panels;
  std::mutex host_mu;
  std::deque<HostStaging> staging;
  std::deque<ForkJoin> forks;  // guarded by panel_mu
  std::deque<PadBuf> pads;     // guarded by panel_mu

  int64_t start_of(int64_t oc) const { return (oc * cfg.shift) % cfg.c_in; }
  // Forward-band weight of output channel oc on input channel ic (0 outside
  // the window); slot index into the [oc][k] weight array, or -1.
  int64_t slot_of(int64_t oc, int64_t ic) const {
    const int64_t s = ((ic - start_of(oc)) % cfg.c_in + cfg.c_in) % cfg.c_in;
    return s < cfg.group_width ? oc * cfg.group_width + s : -1;
  }
};

// Validates like scc_config_new and builds every table (throws Error).
void build_plan(Plan& p, int64_t c_in, int64_t c_out, int64_t cg, int32_t kind,
                double ratio, int64_t count, int32_t has_bias);

// Overlap::resolve semantics (config.cpp:39-53).
int64_t resolve_overlap(int32_t kind, double ratio, int64_t count, int64_t gw);

// Overlap::parse semantics (config.cpp:15-37).
void parse_overlap(const char* text, int32_t* kind, double* ratio, int64_t* count);

}  // namespace scc
