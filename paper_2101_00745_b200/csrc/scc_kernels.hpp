// Launch interface of the SCC device kernels (CUDA-core and tcgen05 families).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace scc {

// Vector (float4) and TMA paths need 16-byte aligned activation pointers; a
// caller's view with an odd storage offset takes the scalar CUDA-core path.
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Geometry + tables one band launch needs (all device pointers).
struct BandLaunch {
  const float* in;          // [N][c_in_t][P]  (x for forward, dy for backward-data)
  float* out;               // [N][c_out_t][P]
  const float* weight;      // [c_out*gw], window-relative
  const float* bias;        // [c_out] or nullptr (forward only)
  const int32_t* rows;      // [nblk*8] output channel per row, -1 = pad
  const int32_t* ring_map;  // ring position -> input channel, nullptr = identity
  const int32_t* starts;    // oc -> window start
  const int32_t* blocks;    // [nblk][2] arc on the ring
  const int32_t* groups;    // [ngrp][4]
  int32_t ngrp;
  int32_t ring;
  int32_t c_in_t, c_out_t;  // channel counts of in / out tensors
  int32_t c_in, gw;         // operator geometry (weight lookup)
  int64_t shift;
  int64_t n, plane;         // batch, H*W
  bool backward_data;       // weight lookup orientation
  // Fused depthwise prologue (dsc_block, model.cpp:213-220): when dw_w is set
  // the staged "input" rows are DW3x3(x) computed on the fly from x of
  // [N][c_in][h_in][w_in] (stride dw_stride, padding 1); `plane` is then the
  // DW output plane h_out * w_out.
  const float* dw_w = nullptr;  // [c_in][3][3]
  const float* dw_b = nullptr;  // [c_in] or nullptr
  int32_t dw_stride = 1, h_in = 0, w_in = 0, w_out = 0;
};

struct WeightLaunch {
  const float* dy;          // [N][c_out][P]
  const float* x;           // [N][c_in][P]
  float* dweight;           // [c_out*gw]
  float* dbias;             // [c_out] or nullptr
  float* partial;           // workspace
  const int32_t* rows;      // forward rows (sorted filters), [nblk*8]
  const int32_t* blocks;    // forward block arcs
  const int32_t* inv_perm;  // oc -> sorted position
  const int32_t* starts;    // oc -> window start
  int32_t nblk;
  int32_t max_block_len;
  int32_t c_in, c_out, gw;
  int64_t shift;
  int64_t n, plane;
};

struct TcBandPlan;
struct TcDeviceTables;

// One tensor-core band call (forward or backward-data).
struct TcBandCall {
  const float* in;      // x (forward) / dy (backward-data)
  float* out;           // y / dx
  const float* weight;
  const float* bias;    // forward only
  int64_t n, plane;
  int32_t c_in, gw;     // operator geometry
  int32_t c_out_t;      // channels of the output tensor
  bool backward_data;
  float* panel;         // scratch for the band weight images (tc_panel_bytes)
  int32_t max_ctas = 0; // grid cap (0 = one CTA per SM); the concurrent backward splits the SMs
  // fused dsc_block forward (generation-2 kernel only): `in` is the block
  // input x, the converters compute t = DW3x3(x) (stride 1, padding 1) from a
  // haloed stage, feed it to the SCC GEMM and (if dsc_t) store it
  const float* dsc_w = nullptr;  // [c_in][3][3], nullptr: plain SCC forward
  const float* dsc_b = nullptr;  // [c_in] or nullptr
  float* dsc_t = nullptr;        // [n][c_in][plane] or nullptr
  int32_t img_w = 0;             // image width (the plane is img_w wide)
};
// The fused dsc_block forward on the generation-2 kernel: stride 1, image
// width 16 / 32 (planes a multiple of 128 px), one row tile whose arc is
// every input channel exactly once.
bool tc_dsc2_supported(const TcBandPlan& tp, int64_t plane, int64_t img_w, int32_t c_in, int32_t c_out);

size_t tc_panel_bytes(const TcBandPlan& tp);

struct TcWeightPlan;
struct TcWeightCall {
  const float* dy;
  const float* x;
  float* dweight;
  float* dbias;          // nullptr when the layer has no bias
  void* workspace;
  size_t workspace_bytes;
  int64_t n, plane;
  int32_t c_in, c_out, gw;
  const int32_t* starts;    // oc -> window start
  const int32_t* inv_perm;  // oc -> sorted position
  const int32_t* perm = nullptr;  // sorted position -> oc
  const int32_t* rt_info;   // TcWeightPlan::rt_info (device)
  const int32_t* class_d;
  int32_t max_ctas = 0;     // grid cap (0 = one CTA per SM)
};
bool tc_weight_supported(const TcWeightPlan& tw, int64_t plane);
size_t tc_weight_workspace_bytes(const TcWeightPlan& tw, int64_t n, int64_t plane);
cudaError_t launch_weight_tc(const TcWeightPlan& tw, const TcWeightCall& call, cudaStream_t s);
int tc_trace(unsigned long long* out, int n);
int tc_hang(unsigned int* out);
int tc_wtrace(unsigned long long* out, int n);

// Counter of kernels launched by this library (scc_launch_count()).
void note_launches(uint64_t k);

// CUDA-core family -----------------------------------------------------------
cudaError_t launch_band_cc(const BandLaunch& a, cudaStream_t s);
// Zero-padded copy [rows][P] -> [rows][P4] (or back, unpad) for the
// tensor-core path on planes with P % 4 != 0.
cudaError_t launch_pad_planes(const float* in, float* out, int64_t rows, int32_t P, int32_t P4, bool unpad,
                              cudaStream_t s);
size_t weight_cc_workspace_bytes(int32_t nblk, int32_t max_block_len, int64_t n,
                                 int64_t plane);
cudaError_t launch_weight_cc(const WeightLaunch& a, size_t ws_bytes, cudaStream_t s);

// Tensor-core family -----------------------------------------------------------
bool tc_band_supported(const TcBandPlan& tp, int64_t plane);
// Generation 2 (scc_tc2.cu): MN-major TMA operands, in-kernel weight panel.
bool tc_band2_supported(const TcBandPlan& tp, int64_t plane, int32_t c_out);
cudaError_t launch_band_tc2(const TcBandPlan& tp, const TcDeviceTables& dt, const TcBandCall& call,
                            int64_t shift, int32_t c_out, cudaStream_t s);
int tc2_trace(unsigned long long* out, int n);
// Backward-weight generation 2 (scc_tc_wgrad2.cu): TS-mode MMAs, per-slice
// partials reduced in a fixed order by a PDL-chained second kernel.
bool tc_wgrad2_supported(const TcWeightPlan& tw, int64_t n, int64_t plane, int32_t gw);
size_t tc_wgrad2_workspace_bytes(int32_t c_out, int32_t gw, int nsm);
int tc_w2trace(unsigned long long* out, int n);
cudaError_t launch_wgrad2(const TcWeightPlan& tw, const TcWeightCall& call, const int32_t* perm,
                          cudaStream_t s);
cudaError_t launch_band_tc(const TcBandPlan& tp, const TcDeviceTables& dt, const TcBandCall& call,
                           cudaStream_t s);
// Small (latency-bound) problems: the generation-1 backward-weight kernel
// takes half the SMs so scc_backward can run backward-data beside it.
bool tc_weight_small(int64_t n, int64_t plane, int64_t channels);

// Fused backward (scc_tc_bwd.cu): backward-data and backward-weight from one
// pass over dy (either half can be switched off; the arithmetic of each half
// does not depend on the other, so fused and separate calls agree bitwise).
struct TcBwdCall {
  const float* dy;
  const float* x;        // backward-weight only
  const float* weight;   // backward-data only
  float* dx;
  float* dweight;
  float* dbias;          // nullptr when the layer has no bias
  void* workspace;
  size_t workspace_bytes;
  int64_t n, plane;
  int32_t c_in, c_out, gw;
  const int32_t* starts;  // oc -> window start
  bool do_dx = false, do_dw = false;
  int32_t max_ctas = 0;
};
bool tc_bwd_supported(const TcWeightPlan& tw, int64_t n, int64_t plane, int32_t c_in, int32_t c_out, int32_t gw);
size_t tc_bwd_workspace_bytes(int32_t c_out, int32_t gw, int64_t n, int64_t plane);
cudaError_t launch_tc_bwd(const TcWeightPlan& tw, const TcBwdCall& call, cudaStream_t s);
int tc_bwd_trace(unsigned long long* out, int n);

// Depthwise 3x3 stage of a dsc_block (scc_dw.cu).  op 0 forward, 1
// backward-data, 2 backward-weight (+ bias; part = workspace partials).
struct DwArgs {
  const float* x = nullptr;   // [n][c][h][w]
  const float* wt = nullptr;  // [c][3][3]
  const float* b = nullptr;   // [c] or nullptr (forward)
  float* y = nullptr;         // [n][c][ho][wo]
  const float* dy = nullptr;  // [n][c][ho][wo]
  float* dx = nullptr;        // [n][c][h][w]
  float* dw = nullptr;        // [c][3][3]
  float* db = nullptr;        // [c] or nullptr
  float* part = nullptr;      // workspace
  int64_t n = 0, c = 0;
  int32_t h = 0, w = 0, ho = 0, wo = 0, stride = 1;
  int32_t staged = 0;
};
size_t dw_workspace_bytes(int64_t c);
cudaError_t launch_dw(DwArgs a, int op, cudaStream_t s);

}  // namespace scc
