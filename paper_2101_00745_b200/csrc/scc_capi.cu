// extern "C" boundary of libscc_b200.so (include/scc_b200.h).
//
// Maps the reference's exception taxonomy (errors.hpp:9-55) onto status codes,
// validates arguments the way kernel.cpp:14-25,32-35,100-103,142-146 do, keeps
// the per-device plan tables, and dispatches to the kernel families.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <vector>
#include <cmath>

#include "scc_b200.h"
#include "scc_kernels.hpp"
#include "scc_plan.hpp"

struct scc_plan : scc::Plan {};

namespace scc {

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

[[noreturn]] void fail(scc_status_t code, std::string msg) { throw Error{code, std::move(msg)}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    fail(SCC_ERR_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" +
                           cudaGetErrorString(e) + ")");
  }
}

template <class F>
scc_status_t guard(F&& f) {
  try {
    f();
    g_err.clear();
    return SCC_OK;
  } catch (const Error& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SCC_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SCC_ERR_INTERNAL;
  }
}

// One-time check that the current device is a B200-class sm_100 part: the
// fat binary only carries sm_100a code, so anything else must fail loudly.
int current_device() {
  int dev = -1;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  static std::mutex mu;
  static int checked[64] = {0};  // 0 unknown, 1 ok, 2 bad
  std::lock_guard<std::mutex> lk(mu);
  if (dev >= 0 && dev < 64 && checked[dev] == 0) {
    cudaDeviceProp prop{};
    cuda_check(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
    checked[dev] = (prop.major == 10 && prop.minor == 0) ? 1 : 2;
  }
  if (dev < 0 || dev >= 64 || checked[dev] != 1) {
    fail(SCC_ERR_CUDA, "libscc_b200 carries sm_100a code only; current device is not sm_100");
  }
  return dev;
}

const DeviceTables& tables(Plan& p) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(p.dev_mu);
  for (const DeviceTables& t : p.dev) {
    if (t.device == dev) return t;
  }
  // Pack every table into one int32 buffer.
  std::vector<int32_t> h;
  auto put = [&](const std::vector<int32_t>& v) {
    const size_t off = h.size();
    h.insert(h.end(), v.begin(), v.end());
    while (h.size() % 4) h.push_back(0);  // 16-byte alignment of every table
    return off;
  };
  auto arcs = [](const std::vector<Arc>& v) {
    std::vector<int32_t> o;
    for (const Arc& a : v) {
      o.push_back(a.start);
      o.push_back(a.len);
    }
    return o;
  };
  const size_t o_fr = put(p.fwd.rows), o_fb = put(arcs(p.fwd.blocks)), o_fg = put(p.fwd.groups);
  const size_t o_br = put(p.bwd.rows), o_bb = put(arcs(p.bwd.blocks)), o_bg = put(p.bwd.groups);
  const size_t o_pm = put(p.perm), o_ip = put(p.inv_perm), o_st = put(p.starts);
  const size_t o_tf[5] = {put(p.tc_fwd.rt_info), put(p.tc_fwd.rows), put(p.tc_fwd.class_d),
                          put(p.tc_fwd.chunk_base), put(p.tc_fwd.out_class_d)};
  const size_t o_tb[5] = {put(p.tc_bwd.rt_info), put(p.tc_bwd.rows), put(p.tc_bwd.class_d),
                          put(p.tc_bwd.chunk_base), put(p.tc_bwd.out_class_d)};
  const size_t o_tw[2] = {put(p.tc_wgt.rt_info), put(p.tc_wgt.class_d)};
  if (h.empty()) h.push_back(0);
  DeviceTables t;
  t.device = dev;
  cuda_check(cudaMalloc(&t.base, h.size() * sizeof(int32_t)), "cudaMalloc(plan tables)");
  cuda_check(cudaMemcpy(t.base, h.data(), h.size() * sizeof(int32_t), cudaMemcpyHostToDevice),
             "cudaMemcpy(plan tables)");
  const int32_t* b = static_cast<const int32_t*>(t.base);
  t.fwd_rows = b + o_fr;
  t.fwd_blocks = b + o_fb;
  t.fwd_groups = b + o_fg;
  t.bwd_rows = b + o_br;
  t.bwd_blocks = b + o_bb;
  t.bwd_groups = b + o_bg;
  t.perm = b + o_pm;
  t.inv_perm = b + o_ip;
  t.starts = b + o_st;
  for (int k = 0; k < 2; ++k) {
    TcDeviceTables& d = k == 0 ? t.tc_fwd : t.tc_bwd;
    const size_t* o = k == 0 ? o_tf : o_tb;
    d.rt_info = b + o[0];
    d.rows = b + o[1];
    d.class_d = b + o[2];
    d.chunk_base = b + o[3];
    d.out_class_d = b + o[4];
    d.starts = t.starts;
    d.perm = t.perm;
    d.inv_perm = t.inv_perm;
  }
  t.tcw_rt_info = b + o_tw[0];
  t.tcw_class_d = b + o_tw[1];
  p.dev.push_back(t);
  return p.dev.back();
}

void check_extents(int64_t n, int64_t h, int64_t w) {
  // Tensor4 requires every extent >= 1 (tensor.cpp:11-18).
  if (n < 1 || h < 1 || w < 1) {
    fail(SCC_ERR_SHAPE, "tensor extents must all be >= 1, got n=" + std::to_string(n) +
                            " h=" + std::to_string(h) + " w=" + std::to_string(w));
  }
}

void check_ptr(const void* p, const char* name) {
  if (p == nullptr) fail(SCC_ERR_ARGUMENT, std::string(name) + " is null");
}

// check_weights (kernel.cpp:14-25): bias present exactly when has_bias.
void check_bias(const Plan& p, const void* bias, const char* name) {
  if (p.cfg.has_bias && bias == nullptr) {
    fail(SCC_ERR_SHAPE, std::string(name) + " array has 0 entries, config needs " +
                            std::to_string(p.cfg.c_out));
  }
  if (!p.cfg.has_bias && bias != nullptr) {
    fail(SCC_ERR_SHAPE, std::string(name) + " given but config has no bias");
  }
}

// Kernel family for one direction (0 forward, 1 backward-data).  A forced
// tensor path falls back to CUDA cores for directions the band GEMM cannot
// express (ring not a multiple of 8, plane not a multiple of 4, ...).
int32_t choose_path(const Plan& p, int64_t /*n*/, int64_t h, int64_t w, int dir = 0) {
  const bool tc_ok = dir == 2 ? tc_weight_supported(p.tc_wgt, h * w)
                              : tc_band_supported(dir == 0 ? p.tc_fwd : p.tc_bwd, h * w);
  if (p.path == SCC_PATH_CUDA_CORE) return SCC_PATH_CUDA_CORE;
  // AUTO: the tensor-core kernels win on every shape they can express
  // (profiles/README.md); CUDA cores take the rest (ragged planes, rings
  // that are not multiples of 8, uneven window classes).
  return tc_ok ? SCC_PATH_TENSOR : SCC_PATH_CUDA_CORE;
}

float* panel_buffer(Plan& p, int dir, cudaStream_t s) {
  const int dev = current_device();
  const TcBandPlan& tp = dir == 0 ? p.tc_fwd : p.tc_bwd;
  const size_t bytes = tc_panel_bytes(tp);
  std::lock_guard<std::mutex> lk(p.panel_mu);
  for (PanelBuf& b : p.panels) {
    if (b.device == dev && b.stream == static_cast<void*>(s) && b.dir == dir) return static_cast<float*>(b.ptr);
  }
  PanelBuf b;
  b.device = dev;
  b.stream = s;
  b.dir = dir;
  b.bytes = bytes;
  cuda_check(cudaMalloc(&b.ptr, bytes), "cudaMalloc(panel)");
  p.panels.push_back(b);
  return static_cast<float*>(b.ptr);
}

int device_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

TcBandCall tc_call(const Plan& p, bool bwd, int64_t n, int64_t plane, const float* in, float* out,
                   const float* weight, const float* bias) {
  TcBandCall c{};
  c.in = in;
  c.out = out;
  c.weight = weight;
  c.bias = bias;
  c.n = n;
  c.plane = plane;
  c.c_in = static_cast<int32_t>(p.cfg.c_in);
  c.gw = static_cast<int32_t>(p.cfg.group_width);
  c.c_out_t = static_cast<int32_t>(bwd ? p.cfg.c_in : p.cfg.c_out);
  c.backward_data = bwd;
  return c;
}

BandLaunch band_args(const Plan& p, const DeviceTables& t, bool bwd, int64_t n, int64_t plane,
                     const float* in, float* out, const float* weight, const float* bias) {
  const BandSide& side = bwd ? p.bwd : p.fwd;
  BandLaunch a{};
  a.in = in;
  a.out = out;
  a.weight = weight;
  a.bias = bias;
  a.rows = bwd ? t.bwd_rows : t.fwd_rows;
  a.ring_map = bwd ? t.perm : nullptr;
  a.starts = t.starts;
  a.blocks = bwd ? t.bwd_blocks : t.fwd_blocks;
  a.groups = bwd ? t.bwd_groups : t.fwd_groups;
  a.ngrp = side.ngrp();
  a.ring = side.ring;
  a.c_in_t = static_cast<int32_t>(bwd ? p.cfg.c_out : p.cfg.c_in);
  a.c_out_t = static_cast<int32_t>(bwd ? p.cfg.c_in : p.cfg.c_out);
  a.c_in = static_cast<int32_t>(p.cfg.c_in);
  a.gw = static_cast<int32_t>(p.cfg.group_width);
  a.shift = p.cfg.shift;
  a.n = n;
  a.plane = plane;
  a.backward_data = bwd;
  return a;
}

WeightLaunch weight_args(const Plan& p, const DeviceTables& t, int64_t n, int64_t plane,
                         const float* dy, const float* x, float* dw, float* db, void* ws) {
  WeightLaunch a{};
  a.dy = dy;
  a.x = x;
  a.dweight = dw;
  a.dbias = db;
  a.partial = static_cast<float*>(ws);
  a.rows = t.fwd_rows;
  a.blocks = t.fwd_blocks;
  a.inv_perm = t.inv_perm;
  a.starts = t.starts;
  a.nblk = p.fwd.nblk();
  a.max_block_len = p.fwd.max_block_len;
  a.c_in = static_cast<int32_t>(p.cfg.c_in);
  a.c_out = static_cast<int32_t>(p.cfg.c_out);
  a.gw = static_cast<int32_t>(p.cfg.group_width);
  a.shift = p.cfg.shift;
  a.n = n;
  a.plane = plane;
  return a;
}

// The fused backward kernel (scc_tc_bwd.cu) serves scc_backward and, so
// that fused and separate calls agree bitwise, the separate backward-data and
// backward-weight entry points too, whenever its geometry fits.
bool fused_bwd_supported(const Plan& p, int64_t n, int64_t plane) {
  if (p.path == SCC_PATH_TENSOR_STREAMED || p.path == SCC_PATH_CUDA_CORE) return false;
  return tc_bwd_supported(p.tc_wgt, n, plane, static_cast<int32_t>(p.cfg.c_in), static_cast<int32_t>(p.cfg.c_out),
                          static_cast<int32_t>(p.cfg.group_width));
}

size_t weight_ws_bytes_plane(const Plan& p, int64_t n, int64_t plane);
size_t weight_ws_bytes(const Plan& p, int64_t n, int64_t plane) {
  // the padded-plane path (do_forward_padded) runs the kernels on P4 planes
  size_t b = weight_ws_bytes_plane(p, n, plane);
  if (plane % 4 != 0) b = std::max(b, weight_ws_bytes_plane(p, n, (plane + 3) & ~int64_t(3)));
  return b;
}
size_t weight_ws_bytes_plane(const Plan& p, int64_t n, int64_t plane) {
  const size_t cc = weight_cc_workspace_bytes(p.fwd.nblk(), p.fwd.max_block_len, n, plane);
  const size_t tc = tc_weight_supported(p.tc_wgt, plane) ? tc_weight_workspace_bytes(p.tc_wgt, n, plane) : 0;
  const size_t tc2 = tc_wgrad2_supported(p.tc_wgt, n, plane, static_cast<int32_t>(p.cfg.group_width))
                         ? tc_wgrad2_workspace_bytes(static_cast<int32_t>(p.cfg.c_out),
                                                     static_cast<int32_t>(p.cfg.group_width), 74)
                         : 0;
  // (independent of the forced path, so a size queried before set_path stays
  // large enough after it)
  const size_t tc3 = tc_bwd_supported(p.tc_wgt, n, plane, static_cast<int32_t>(p.cfg.c_in),
                                      static_cast<int32_t>(p.cfg.c_out), static_cast<int32_t>(p.cfg.group_width))
                         ? tc_bwd_workspace_bytes(static_cast<int32_t>(p.cfg.c_out),
                                                  static_cast<int32_t>(p.cfg.group_width), n, plane)
                         : 0;
  return std::max(std::max(cc, tc), std::max(tc2, tc3));
}

// Planes with P % 4 != 0 (7x7 in ResNet-50 stage 4, ...) cannot be described
// to TMA (16 B strides).  For windows wide enough that the CUDA-core kernels
// are compute-bound (gw >= 64), the operands are copied into zero-padded
// [rows][P4] planes and the tensor-core kernels run on those: a 1x1
// convolution does not care about the spatial shape, the padded pixels are
// zeros (they add nothing to dW / db) and their outputs are dropped.
constexpr int64_t kPadMinGw = 64;
int64_t round4(int64_t v) { return (v + 3) & ~int64_t(3); }

bool pad_tc(const Plan& p, int64_t n, int64_t h, int64_t w, int dir) {
  const int64_t P = h * w;
  if (P % 4 == 0 || p.path == SCC_PATH_CUDA_CORE || p.cfg.group_width < kPadMinGw) return false;
  if (round4(P) > (int64_t(1) << 30)) return false;
  return choose_path(p, n, 1, round4(P), dir) == SCC_PATH_TENSOR;
}

float* pad_buffer(Plan& p, cudaStream_t s, size_t bytes) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(p.panel_mu);
  PadBuf* b = nullptr;
  for (PadBuf& e : p.pads) {
    if (e.device == dev && e.stream == static_cast<void*>(s)) b = &e;
  }
  if (b == nullptr) {
    p.pads.push_back(PadBuf{});
    b = &p.pads.back();
    b->device = dev;
    b->stream = s;
  }
  if (b->bytes < bytes) {
    if (b->ptr) b->retired.push_back(b->ptr);
    b->ptr = nullptr;
    cuda_check(cudaMalloc(&b->ptr, bytes), "cudaMalloc(pad scratch)");
    b->bytes = bytes;
  }
  return static_cast<float*>(b->ptr);
}

void pad(const float* in, float* out, int64_t rows, int64_t P, cudaStream_t s) {
  cuda_check(launch_pad_planes(in, out, rows, static_cast<int32_t>(P), static_cast<int32_t>(round4(P)), false, s),
             "pad launch");
}
void unpad(const float* in, float* out, int64_t rows, int64_t P, cudaStream_t s) {
  cuda_check(launch_pad_planes(in, out, rows, static_cast<int32_t>(P), static_cast<int32_t>(round4(P)), true, s),
             "unpad launch");
}

void do_forward(Plan& p, int64_t n, int64_t h, int64_t w, const float* x, const float* wt,
                const float* b, float* y, cudaStream_t s);

void do_forward_padded(Plan& p, int64_t n, int64_t h, int64_t w, const float* x, const float* wt,
                       const float* b, float* y, cudaStream_t s) {
  const int64_t P = h * w, P4 = round4(P);
  const int64_t ci = p.cfg.c_in, co = p.cfg.c_out;
  float* xp = pad_buffer(p, s, static_cast<size_t>(n * (ci + co) * P4) * sizeof(float));
  float* yp = xp + n * ci * P4;
  pad(x, xp, n * ci, P, s);
  do_forward(p, n, 1, P4, xp, wt, b, yp, s);
  unpad(yp, y, n * co, P, s);
}

void do_forward(Plan& p, int64_t n, int64_t h, int64_t w, const float* x, const float* wt,
                const float* b, float* y, cudaStream_t s) {
  check_extents(n, h, w);
  check_ptr(x, "x");
  check_ptr(wt, "weight");
  check_ptr(y, "y");
  check_bias(p, b, "bias");
  if (pad_tc(p, n, h, w, 0)) {
    do_forward_padded(p, n, h, w, x, wt, b, y, s);
    return;
  }
  const DeviceTables& t = tables(p);
  if (aligned16(x) && aligned16(y) && choose_path(p, n, h, w, 0) == SCC_PATH_TENSOR) {
    TcBandCall c = tc_call(p, false, n, h * w, x, y, wt, b);
    if (p.path != SCC_PATH_TENSOR_STREAMED && tc_band2_supported(p.tc_fwd, h * w, static_cast<int32_t>(p.cfg.c_out))) {
      cuda_check(launch_band_tc2(p.tc_fwd, t.tc_fwd, c, p.cfg.shift, static_cast<int32_t>(p.cfg.c_out), s),
                 "forward (tensor) launch");
      return;
    }
    c.panel = panel_buffer(p, 0, s);
    cuda_check(launch_band_tc(p.tc_fwd, t.tc_fwd, c, s), "forward (tensor) launch");
    return;
  }
  cuda_check(launch_band_cc(band_args(p, t, false, n, h * w, x, y, wt, b), s), "forward launch");
}

bool use_fused(Plan& p, int64_t n, int64_t h, int64_t w, std::initializer_list<const void*> ptrs) {
  for (const void* q : ptrs)
    if (q != nullptr && !aligned16(q)) return false;
  return choose_path(p, n, h, w, 2) == SCC_PATH_TENSOR && fused_bwd_supported(p, n, h * w);
}

void launch_fused(Plan& p, int64_t n, int64_t h, int64_t w, const float* dy, const float* x, const float* wt,
                  float* dx, float* dw, float* db, void* ws, size_t ws_bytes, cudaStream_t s) {
  const DeviceTables& t = tables(p);
  TcBwdCall c{};
  c.dy = dy;
  c.x = x;
  c.weight = wt;
  c.dx = dx;
  c.dweight = dw;
  c.dbias = db;
  c.workspace = ws;
  c.workspace_bytes = ws_bytes;
  c.n = n;
  c.plane = h * w;
  c.c_in = static_cast<int32_t>(p.cfg.c_in);
  c.c_out = static_cast<int32_t>(p.cfg.c_out);
  c.gw = static_cast<int32_t>(p.cfg.group_width);
  c.starts = t.starts;
  c.do_dx = dx != nullptr;
  c.do_dw = dw != nullptr;
  cuda_check(launch_tc_bwd(p.tc_wgt, c, s), "backward (fused tensor) launch");
}

void do_backward_data(Plan& p, int64_t n, int64_t h, int64_t w, const float* dy, const float* wt,
                      float* dx, cudaStream_t s, int32_t max_ctas = 0) {
  check_extents(n, h, w);
  check_ptr(dy, "dy");
  check_ptr(wt, "weight");
  check_ptr(dx, "dx");
  if (pad_tc(p, n, h, w, 1)) {
    const int64_t P = h * w, P4 = round4(P), ci = p.cfg.c_in, co = p.cfg.c_out;
    float* dyp = pad_buffer(p, s, static_cast<size_t>(n * (ci + co) * P4) * sizeof(float));
    float* dxp = dyp + n * co * P4;
    pad(dy, dyp, n * co, P, s);
    do_backward_data(p, n, 1, P4, dyp, wt, dxp, s, max_ctas);
    unpad(dxp, dx, n * ci, P, s);
    return;
  }
  if (use_fused(p, n, h, w, {dy, dx})) {
    launch_fused(p, n, h, w, dy, nullptr, wt, dx, nullptr, nullptr, nullptr, 0, s);
    return;
  }
  const DeviceTables& t = tables(p);
  if (aligned16(dy) && aligned16(dx) && choose_path(p, n, h, w, 1) == SCC_PATH_TENSOR) {
    TcBandCall c = tc_call(p, true, n, h * w, dy, dx, wt, nullptr);
    c.max_ctas = max_ctas;
    if (p.path != SCC_PATH_TENSOR_STREAMED && tc_band2_supported(p.tc_bwd, h * w, static_cast<int32_t>(p.cfg.c_out))) {
      cuda_check(launch_band_tc2(p.tc_bwd, t.tc_bwd, c, p.cfg.shift, static_cast<int32_t>(p.cfg.c_out), s),
                 "backward-data (tensor) launch");
      return;
    }
    c.panel = panel_buffer(p, 1, s);
    cuda_check(launch_band_tc(p.tc_bwd, t.tc_bwd, c, s), "backward-data (tensor) launch");
    return;
  }
  cuda_check(launch_band_cc(band_args(p, t, true, n, h * w, dy, dx, wt, nullptr), s),
             "backward-data launch");
}

void do_backward_weight(Plan& p, int64_t n, int64_t h, int64_t w, const float* dy, const float* x,
                        float* dw, float* db, void* ws, size_t ws_bytes, cudaStream_t s,
                        int32_t max_ctas = 0) {
  check_extents(n, h, w);
  check_ptr(dy, "dy");
  check_ptr(x, "x");
  check_ptr(dw, "dweight");
  check_bias(p, db, "dbias");
  const size_t need = weight_ws_bytes(p, n, h * w);
  if (ws_bytes < need || (need > 0 && ws == nullptr)) {
    fail(SCC_ERR_ARGUMENT, "workspace too small: need " + std::to_string(need) + " bytes");
  }
  if (pad_tc(p, n, h, w, 2)) {
    const int64_t P = h * w, P4 = round4(P), ci = p.cfg.c_in, co = p.cfg.c_out;
    float* dyp = pad_buffer(p, s, static_cast<size_t>(n * (ci + co) * P4) * sizeof(float));
    float* xp = dyp + n * co * P4;
    pad(dy, dyp, n * co, P, s);
    pad(x, xp, n * ci, P, s);
    do_backward_weight(p, n, 1, P4, dyp, xp, dw, db, ws, ws_bytes, s, max_ctas);
    return;
  }
  if (use_fused(p, n, h, w, {dy, x})) {
    launch_fused(p, n, h, w, dy, x, nullptr, nullptr, dw, db, ws, ws_bytes, s);
    return;
  }
  const DeviceTables& t = tables(p);
  if (aligned16(dy) && aligned16(x) && choose_path(p, n, h, w, 2) == SCC_PATH_TENSOR) {
    TcWeightCall c{};
    c.dy = dy;
    c.x = x;
    c.dweight = dw;
    c.dbias = db;
    c.workspace = ws;
    c.workspace_bytes = ws_bytes;
    c.n = n;
    c.plane = h * w;
    c.c_in = static_cast<int32_t>(p.cfg.c_in);
    c.c_out = static_cast<int32_t>(p.cfg.c_out);
    c.gw = static_cast<int32_t>(p.cfg.group_width);
    c.starts = t.starts;
    c.inv_perm = t.inv_perm;
    c.perm = t.perm;
    c.rt_info = t.tcw_rt_info;
    c.class_d = t.tcw_class_d;
    c.max_ctas = max_ctas;
    if (p.path != SCC_PATH_TENSOR_STREAMED && tc_wgrad2_supported(p.tc_wgt, n, h * w, c.gw)) {
      cuda_check(launch_wgrad2(p.tc_wgt, c, t.perm, s), "backward-weight (tensor) launch");
      return;
    }
    cuda_check(launch_weight_tc(p.tc_wgt, c, s), "backward-weight (tensor) launch");
    return;
  }
  cuda_check(launch_weight_cc(weight_args(p, t, n, h * w, dy, x, dw, db, ws), ws_bytes, s),
             "backward-weight launch");
}

ForkJoin& fork_join(Plan& p, cudaStream_t s) {
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(p.panel_mu);
  for (ForkJoin& f : p.forks) {
    if (f.device == dev && f.stream == static_cast<void*>(s)) return f;
  }
  ForkJoin f;
  f.device = dev;
  f.stream = s;
  cudaStream_t side;
  cudaEvent_t a, b;
  cuda_check(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking), "cudaStreamCreate(side)");
  cuda_check(cudaEventCreateWithFlags(&a, cudaEventDisableTiming), "cudaEventCreate");
  cuda_check(cudaEventCreateWithFlags(&b, cudaEventDisableTiming), "cudaEventCreate");
  f.side = side;
  f.ev_fork = a;
  f.ev_join = b;
  p.forks.push_back(f);
  return p.forks.back();
}

// scc_backward (kernel.cpp:183-189): backward-data and backward-weight read
// the same dy but are otherwise independent.  When both run the generation-2
// tensor-core kernels, they run concurrently on disjoint halves of the SMs
// (backward-weight on a side stream, joined back into the caller's stream),
// so each one's start-up and tail overlap the other's streaming.
void do_backward(Plan& p, int64_t n, int64_t h, int64_t w, const float* dy, const float* x,
                 const float* wt, float* dx, float* dw, float* db, void* ws, size_t ws_bytes,
                 cudaStream_t s) {
  const int64_t plane = h * w;
  if (pad_tc(p, n, h, w, 1) && pad_tc(p, n, h, w, 2)) {
    check_extents(n, h, w);
    check_ptr(dy, "dy");
    check_ptr(x, "x");
    check_ptr(dx, "dx");
    const int64_t P4 = round4(plane), ci = p.cfg.c_in, co = p.cfg.c_out;
    float* dyp = pad_buffer(p, s, static_cast<size_t>(n * (2 * ci + co) * P4) * sizeof(float));
    float* xp = dyp + n * co * P4;
    float* dxp = xp + n * ci * P4;
    pad(dy, dyp, n * co, plane, s);
    pad(x, xp, n * ci, plane, s);
    do_backward(p, n, 1, P4, dyp, xp, wt, dxp, dw, db, ws, ws_bytes, s);
    unpad(dxp, dx, n * ci, plane, s);
    return;
  }
  if (use_fused(p, n, h, w, {dy, x, dx})) {
    check_extents(n, h, w);
    check_ptr(dy, "dy");
    check_ptr(x, "x");
    check_ptr(wt, "weight");
    check_ptr(dx, "dx");
    check_ptr(dw, "dweight");
    check_bias(p, db, "dbias");
    const size_t need = weight_ws_bytes(p, n, plane);
    if (ws_bytes < need || (need > 0 && ws == nullptr)) {
      fail(SCC_ERR_ARGUMENT, "workspace too small: need " + std::to_string(need) + " bytes");
    }
    launch_fused(p, n, h, w, dy, x, wt, dx, dw, db, ws, ws_bytes, s);
    return;
  }
  const bool both2 = aligned16(dy) && aligned16(x) && aligned16(dx) &&
                     p.path != SCC_PATH_TENSOR_STREAMED && p.path != SCC_PATH_CUDA_CORE &&
                     choose_path(p, n, h, w, 1) == SCC_PATH_TENSOR &&
                     choose_path(p, n, h, w, 2) == SCC_PATH_TENSOR &&
                     tc_band2_supported(p.tc_bwd, plane, static_cast<int32_t>(p.cfg.c_out)) &&
                     tc_wgrad2_supported(p.tc_wgt, n, plane, static_cast<int32_t>(p.cfg.group_width));
  // Generation-1 pair on a small (latency-bound) problem: the weight kernel
  // is sized to half the SMs (tc_weight_small), backward-data takes the rest.
  const bool both1 = !both2 && aligned16(dy) && aligned16(x) && aligned16(dx) &&
                     p.path != SCC_PATH_CUDA_CORE &&
                     tc_weight_small(n, plane, std::max(p.cfg.c_in, p.cfg.c_out)) &&
                     choose_path(p, n, h, w, 1) == SCC_PATH_TENSOR &&
                     choose_path(p, n, h, w, 2) == SCC_PATH_TENSOR &&
                     tc_weight_supported(p.tc_wgt, plane) &&
                     (p.path == SCC_PATH_TENSOR_STREAMED ||
                      !tc_wgrad2_supported(p.tc_wgt, n, plane, static_cast<int32_t>(p.cfg.group_width)));
  if (!both2 && !both1) {
    do_backward_data(p, n, h, w, dy, wt, dx, s);
    do_backward_weight(p, n, h, w, dy, x, dw, db, ws, ws_bytes, s);
    return;
  }
  const int nsm = device_sms();
  const int32_t half = nsm / 2;
  ForkJoin& f = fork_join(p, s);
  cudaStream_t side = static_cast<cudaStream_t>(f.side);
  cuda_check(cudaEventRecord(static_cast<cudaEvent_t>(f.ev_fork), s), "cudaEventRecord(fork)");
  cuda_check(cudaStreamWaitEvent(side, static_cast<cudaEvent_t>(f.ev_fork), 0), "cudaStreamWaitEvent(fork)");
  // backward-data first: the kernel enqueued second starts ~1 us later, and
  // backward-data has the longer critical path
  do_backward_data(p, n, h, w, dy, wt, dx, s, half);
  do_backward_weight(p, n, h, w, dy, x, dw, db, ws, ws_bytes, side, nsm - half);
  cuda_check(cudaEventRecord(static_cast<cudaEvent_t>(f.ev_join), side), "cudaEventRecord(join)");
  cuda_check(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(f.ev_join), 0), "cudaStreamWaitEvent(join)");
}

// Host-buffer staging ------------------------------------------------------

struct Staged {
  float *x, *w, *b, *dy, *y, *dx, *dw, *db;
  void* ws;
  size_t ws_bytes;
  cudaStream_t s, s_in, s_out;
  HostStaging* st;
};

Staged stage(Plan& p, int64_t n, int64_t h, int64_t wd) {
  const int dev = current_device();
  const scc_config_t& c = p.cfg;
  const size_t nx = static_cast<size_t>(n * c.c_in * h * wd);
  const size_t ny = static_cast<size_t>(n * c.c_out * h * wd);
  const size_t nw = static_cast<size_t>(c.c_out * c.group_width);
  const size_t nb = static_cast<size_t>(c.c_out);
  const size_t wsb = weight_ws_bytes(p, n, h * wd);
  auto al = [](size_t bytes) { return (bytes + 255) & ~size_t(255); };
  const size_t total = al(nx * 4) * 2 + al(ny * 4) * 2 + al(nw * 4) * 2 + al(nb * 4) * 2 + al(wsb);
  HostStaging* st = nullptr;
  for (HostStaging& e : p.staging) {
    if (e.device == dev) st = &e;
  }
  if (st == nullptr) {
    p.staging.push_back(HostStaging{});
    st = &p.staging.back();
    st->device = dev;
    cudaStream_t s;
    cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    st->stream = s;
    cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    st->stream_in = s;
    cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    st->stream_out = s;
    auto mk = [](void** e) {
      cudaEvent_t ev;
      cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
      *e = ev;
    };
    for (int i = 0; i < kMaxHostChunks; ++i) {
      mk(&st->ev_in[i]);
      mk(&st->ev_done[i]);
    }
    mk(&st->ev_out);
    mk(&st->ev_fork);
  }
  if (st->bytes < total) {
    if (st->buf) cuda_check(cudaFree(st->buf), "cudaFree(staging)");
    st->buf = nullptr;
    cuda_check(cudaMalloc(&st->buf, total), "cudaMalloc(staging)");
    st->bytes = total;
  }
  char* q = static_cast<char*>(st->buf);
  Staged g{};
  auto take = [&](size_t bytes) {
    char* r = q;
    q += al(bytes);
    return r;
  };
  g.x = reinterpret_cast<float*>(take(nx * 4));
  g.dx = reinterpret_cast<float*>(take(nx * 4));
  g.y = reinterpret_cast<float*>(take(ny * 4));
  g.dy = reinterpret_cast<float*>(take(ny * 4));
  g.w = reinterpret_cast<float*>(take(nw * 4));
  g.dw = reinterpret_cast<float*>(take(nw * 4));
  g.b = reinterpret_cast<float*>(take(nb * 4));
  g.db = reinterpret_cast<float*>(take(nb * 4));
  g.ws = take(wsb);
  g.ws_bytes = wsb;
  g.s = static_cast<cudaStream_t>(st->stream);
  g.s_in = static_cast<cudaStream_t>(st->stream_in);
  g.s_out = static_cast<cudaStream_t>(st->stream_out);
  g.st = st;
  return g;
}

void h2d(void* d, const void* h, size_t bytes, cudaStream_t s) {
  cuda_check(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync H2D");
}
void d2h(void* h, const void* d, size_t bytes, cudaStream_t s) {
  cuda_check(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync D2H");
}

// Host-buffer operator, pipelined over batch chunks so PCIe H2D, the kernels
// and PCIe D2H overlap (the link is full duplex).  All x chunks go first, so
// the forward and the y read-back start after one x chunk has landed and y
// (the largest output) drains while dy comes in; dx trails dy by one chunk:
//   copy-in stream : w, b, x_0..x_k-1 (-> ev_in[c]), dy_0..dy_k-1 (-> ev_in[8+c])
//   compute stream : forward of chunk c after x_c (-> ev_done[c]); backward-data
//                    of chunk c after dy_c (-> ev_done[8+c]); then
//                    backward-weight over the whole batch (it reduces over n,
//                    so its bits equal the device entry point's)
//   copy-out stream: y_0..y_k-1, dx_0..dx_k-1; dW / db last (compute stream)
// Forward and backward-data are per sample (kernel.cpp:45-60, :107-137) and
// the kernels' per-element arithmetic does not depend on n, so chunked
// results are bitwise equal to one full-batch call.  Any subset of the three
// passes runs (y: forward, dx: backward-data, dw: backward-weight), so the
// reference's separate scc_backward_input / scc_backward_params calls move
// only their own bytes.
struct HostIo {
  const float *x = nullptr, *w = nullptr, *b = nullptr, *dy = nullptr;
  float *y = nullptr, *dx = nullptr, *dw = nullptr, *db = nullptr;
};

// Chunk boundaries (sample counts) of one pipelined pass.  The schedule may
// differ between the x pass and the dy pass (SCC_HOST_XCH / SCC_HOST_DYCH:
// comma-separated relative weights, for the sweep in scripts/host_sweep.py).
int host_split(int64_t n, int k, const char* env, int64_t* bounds) {
  std::vector<double> wts;
  if (const char* e = getenv(env)) {
    for (const char* q = e; *q;) {
      wts.push_back(atof(q));
      while (*q && *q != ',') ++q;
      if (*q == ',') ++q;
    }
  }
  if (wts.empty()) {
    // measured best at config 1 (scripts/host_sweep.py, profiles/r02_host_sweep.txt):
    // x in a quarter then three quarters (y -- twice x -- starts draining
    // early), dy in three equal chunks
    // (an explicit SCC_HOST_CHUNKS asks for k equal chunks instead)
    const bool tuned = k >= 3 && getenv("SCC_HOST_CHUNKS") == nullptr;
    if (tuned && std::strcmp(env, "SCC_HOST_XCH") == 0) wts = {1.0, 3.0};
    else if (tuned) wts = {1.0, 1.0, 1.0};
    else wts.assign(static_cast<size_t>(k), 1.0);
  }
  int m = static_cast<int>(std::min<size_t>(wts.size(), static_cast<size_t>(std::min<int64_t>(n, kMaxHostChunks / 2))));
  double tot = 0;
  for (int i = 0; i < m; ++i) tot += wts[i];
  bounds[0] = 0;
  double acc = 0;
  int c = 0;
  for (int i = 0; i < m; ++i) {
    acc += wts[i];
    int64_t b = i == m - 1 ? n : static_cast<int64_t>(std::llround(acc / tot * static_cast<double>(n)));
    b = std::max<int64_t>(b, bounds[c] + 1);
    b = std::min<int64_t>(b, n - (m - 1 - i));
    if (b > bounds[c]) bounds[++c] = b;
  }
  return c;
}

int host_chunks(int64_t n, size_t bytes_per_sample) {
  // >= ~1 MB of traffic per chunk keeps each copy near full PCIe speed
  // (scripts/host_sweep.py sweeps the depth)
  const int64_t by_size = static_cast<int64_t>(bytes_per_sample * n / (1u << 20));
  int64_t k = std::min<int64_t>({n, 4, std::max<int64_t>(by_size, 1)});
  if (const char* e = getenv("SCC_HOST_CHUNKS")) k = std::max<int64_t>(1, std::min<int64_t>({atoi(e), n, kMaxHostChunks / 2}));
  return static_cast<int>(k);
}

void issue_host(Plan& p, int64_t n, int64_t h, int64_t wd, const HostIo& io, const Staged& g, int k) {
  const scc_config_t& c = p.cfg;
  const int64_t P = h * wd;
  const bool fwd = io.y != nullptr, bdata = io.dx != nullptr, bwt = io.dw != nullptr;
  const bool need_x = fwd || bwt, need_dy = bdata || bwt;
  const size_t sx = static_cast<size_t>(c.c_in * P) * 4, sy = static_cast<size_t>(c.c_out * P) * 4;
  const size_t nw = static_cast<size_t>(c.c_out * c.group_width) * 4, nb = static_cast<size_t>(c.c_out) * 4;
  constexpr int kHalf = kMaxHostChunks / 2;
  auto ev = [](void* e) { return static_cast<cudaEvent_t>(e); };
  auto rec = [](cudaEvent_t e, cudaStream_t s) { cuda_check(cudaEventRecord(e, s), "cudaEventRecord"); };
  auto wait = [](cudaStream_t s, cudaEvent_t e) { cuda_check(cudaStreamWaitEvent(s, e, 0), "cudaStreamWaitEvent"); };
  int64_t xb[kHalf + 1], yb[kHalf + 1];
  const int kx = host_split(n, k, "SCC_HOST_XCH", xb);
  const int ky = host_split(n, k, "SCC_HOST_DYCH", yb);
  // fork the copy streams off the compute stream (also makes the sequence capturable)
  rec(ev(g.st->ev_fork), g.s);
  wait(g.s_in, ev(g.st->ev_fork));
  wait(g.s_out, ev(g.st->ev_fork));
  if (fwd || bdata) h2d(g.w, io.w, nw, g.s_in);
  if (fwd && io.b) h2d(g.b, io.b, nb, g.s_in);
  if (need_x) {
    for (int i = 0; i < kx; ++i) {
      const int64_t m = xb[i + 1] - xb[i];
      const size_t ox = static_cast<size_t>(xb[i]) * sx / 4, oy = static_cast<size_t>(xb[i]) * sy / 4;
      h2d(g.x + ox, io.x + ox, m * sx, g.s_in);
      rec(ev(g.st->ev_in[i]), g.s_in);
      if (!fwd) continue;
      wait(g.s, ev(g.st->ev_in[i]));
      do_forward(p, m, h, wd, g.x + ox, g.w, io.b ? g.b : nullptr, g.y + oy, g.s);
      rec(ev(g.st->ev_done[i]), g.s);
      wait(g.s_out, ev(g.st->ev_done[i]));
      d2h(io.y + oy, g.y + oy, m * sy, g.s_out);
    }
  }
  if (need_dy) {
    for (int i = 0; i < ky; ++i) {
      const int64_t m = yb[i + 1] - yb[i];
      const size_t ox = static_cast<size_t>(yb[i]) * sx / 4, oy = static_cast<size_t>(yb[i]) * sy / 4;
      h2d(g.dy + oy, io.dy + oy, m * sy, g.s_in);
      rec(ev(g.st->ev_in[kHalf + i]), g.s_in);
      wait(g.s, ev(g.st->ev_in[kHalf + i]));
      if (!bdata) continue;
      do_backward_data(p, m, h, wd, g.dy + oy, g.w, g.dx + ox, g.s);
      rec(ev(g.st->ev_done[kHalf + i]), g.s);
      wait(g.s_out, ev(g.st->ev_done[kHalf + i]));
      d2h(io.dx + ox, g.dx + ox, m * sx, g.s_out);
    }
  }
  if (bwt) {
    // after the last x and dy chunk (the compute stream waited for both)
    do_backward_weight(p, n, h, wd, g.dy, g.x, g.dw, io.db ? g.db : nullptr, g.ws, g.ws_bytes, g.s);
    d2h(io.dw, g.dw, nw, g.s);
    if (io.db) d2h(io.db, g.db, nb, g.s);
  }
  rec(ev(g.st->ev_out), g.s_out);
  wait(g.s, ev(g.st->ev_out));
}

void run_host(Plan& p, int64_t n, int64_t h, int64_t wd, const HostIo& io) {
  const scc_config_t& c = p.cfg;
  const int64_t P = h * wd;
  Staged g = stage(p, n, h, wd);
  const bool fwd = io.y != nullptr, bdata = io.dx != nullptr, bwt = io.dw != nullptr;
  const size_t sx = static_cast<size_t>(c.c_in * P) * 4, sy = static_cast<size_t>(c.c_out * P) * 4;
  const size_t per_sample = ((fwd || bwt) ? sx : 0) + ((bdata || bwt) ? sy : 0) + (fwd ? sy : 0) + (bdata ? sx : 0);
  issue_host(p, n, h, wd, io, g, host_chunks(n, per_sample));
  cuda_check(cudaStreamSynchronize(g.s), "cudaStreamSynchronize");
}

}  // namespace

void note_launches(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

}  // namespace scc

using scc::guard;

extern "C" {

const char* scc_last_error(void) { return scc::g_err.c_str(); }
int scc_abi_version(void) { return SCC_B200_ABI_VERSION; }
uint64_t scc_launch_count(void) { return scc::g_launches.load(); }

int scc_debug_trace(uint64_t* out, int n) {
  // slots [0, 32): band kernel; [32, 64): backward-weight kernel
  int k = scc::tc_trace(reinterpret_cast<unsigned long long*>(out), n < 32 ? n : 32);
  if (k < 0 || n <= 32) return k;
  const int m = scc::tc_wtrace(reinterpret_cast<unsigned long long*>(out) + 32, n < 64 ? n - 32 : 32);
  if (m < 0) return -1;
  if (n < 128) return 32 + m;
  unsigned int hang[64];
  if (scc::tc_hang(hang) < 0) return -1;
  for (int i = 0; i < 64; ++i) out[64 + i] = hang[i];  // watchdog builds only
  if (n < 192) return 128;
  // slots [128, 192): generation-2 band kernel; [192, 192 + 2*1024): per-CTA
  // start / epilogue-end timestamps of that kernel
  if (n >= 128 + 64 + 2048 + 64) {
    // slots [128, 192 + 2048): band gen 2; then 64 + 3*256 slots of backward-weight gen 2
    if (scc::tc2_trace(reinterpret_cast<unsigned long long*>(out) + 128, 64 + 2048) < 0) return -1;
    const int m = n - (128 + 64 + 2048);
    return scc::tc_w2trace(reinterpret_cast<unsigned long long*>(out) + 128 + 64 + 2048, m) < 0
               ? -1
               : 128 + 64 + 2048 + m;
  }
  const int m2 = n - 128 < 64 + 2048 ? n - 128 : 64 + 2048;
  return scc::tc2_trace(reinterpret_cast<unsigned long long*>(out) + 128, m2) < 0 ? -1 : 128 + m2;
}

int scc_debug_trace_fused(uint64_t* out, int n) {
  return scc::tc_bwd_trace(reinterpret_cast<unsigned long long*>(out), n);
}

scc_status_t scc_overlap_parse(const char* text, int32_t* kind, double* ratio, int64_t* count) {
  return guard([&] {
    scc::check_ptr(kind, "kind");
    scc::check_ptr(ratio, "ratio");
    scc::check_ptr(count, "count");
    scc::parse_overlap(text, kind, ratio, count);
  });
}

scc_status_t scc_overlap_resolve(int32_t kind, double ratio, int64_t count, int64_t gw,
                                 int64_t* channels) {
  return guard([&] {
    scc::check_ptr(channels, "channels");
    *channels = scc::resolve_overlap(kind, ratio, count, gw);
  });
}

scc_status_t scc_plan_create(int64_t c_in, int64_t c_out, int64_t cg, int32_t kind, double ratio,
                             int64_t count, int32_t has_bias, scc_plan_t** plan) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    *plan = nullptr;
    auto* p = new scc_plan;
    try {
      scc::build_plan(*p, c_in, c_out, cg, kind, ratio, count, has_bias);
    } catch (...) {
      delete p;
      throw;
    }
    *plan = p;
  });
}

scc_status_t scc_plan_destroy(scc_plan_t* plan) {
  return guard([&] {
    if (plan == nullptr) return;
    int prev = -1;
    cudaGetDevice(&prev);
    for (const scc::DeviceTables& t : plan->dev) {
      cudaSetDevice(t.device);
      cudaFree(t.base);
    }
    for (const scc::PanelBuf& b : plan->panels) {
      cudaSetDevice(b.device);
      cudaFree(b.ptr);
    }
    for (const scc::HostStaging& s : plan->staging) {
      cudaSetDevice(s.device);
      if (s.buf) cudaFree(s.buf);
      for (void* q : {s.stream, s.stream_in, s.stream_out}) {
        if (q) cudaStreamDestroy(static_cast<cudaStream_t>(q));
      }
      for (int i = 0; i < scc::kMaxHostChunks; ++i) {
        if (s.ev_in[i]) cudaEventDestroy(static_cast<cudaEvent_t>(s.ev_in[i]));
        if (s.ev_done[i]) cudaEventDestroy(static_cast<cudaEvent_t>(s.ev_done[i]));
      }
      if (s.ev_out) cudaEventDestroy(static_cast<cudaEvent_t>(s.ev_out));
      if (s.ev_fork) cudaEventDestroy(static_cast<cudaEvent_t>(s.ev_fork));
    }
    for (const scc::PadBuf& b : plan->pads) {
      cudaSetDevice(b.device);
      cudaStreamSynchronize(static_cast<cudaStream_t>(b.stream));
      if (b.ptr) cudaFree(b.ptr);
      for (void* q : b.retired) cudaFree(q);
    }
    for (const scc::ForkJoin& f : plan->forks) {
      cudaSetDevice(f.device);
      cudaStreamSynchronize(static_cast<cudaStream_t>(f.side));
      cudaStreamDestroy(static_cast<cudaStream_t>(f.side));
      cudaEventDestroy(static_cast<cudaEvent_t>(f.ev_fork));
      cudaEventDestroy(static_cast<cudaEvent_t>(f.ev_join));
    }
    if (prev >= 0) cudaSetDevice(prev);
    delete plan;
  });
}

scc_status_t scc_plan_config(const scc_plan_t* plan, scc_config_t* out) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_ptr(out, "out");
    *out = plan->cfg;
  });
}

scc_status_t scc_plan_cycle_starts(const scc_plan_t* plan, int64_t* starts, int64_t capacity,
                                   int64_t* count) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_ptr(count, "count");
    const auto& cs = plan->cycle_starts;
    *count = static_cast<int64_t>(cs.size());
    for (int64_t i = 0; i < capacity && i < static_cast<int64_t>(cs.size()); ++i) starts[i] = cs[i];
  });
}

scc_status_t scc_plan_window_of(const scc_plan_t* plan, int64_t oc, int64_t* start,
                                int64_t* length) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    // window_of (cycle.cpp:23-26) throws IndexError for oc < 0 and wraps the
    // cycle for oc >= c_out.
    if (oc < 0) scc::fail(SCC_ERR_INDEX, "output channel must be >= 0, got " + std::to_string(oc));
    const auto& cs = plan->cycle_starts;
    if (start) *start = cs[static_cast<size_t>(oc % static_cast<int64_t>(cs.size()))];
    if (length) *length = plan->cfg.group_width;
  });
}

scc_status_t scc_plan_covering_filters(const scc_plan_t* plan, int64_t ic, int64_t* filters,
                                       int64_t capacity, int64_t* count) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_ptr(count, "count");
    const scc_config_t& c = plan->cfg;
    if (ic < 0 || ic >= c.c_in) {
      scc::fail(SCC_ERR_INDEX, "input channel " + std::to_string(ic) + " out of range [0, " +
                                   std::to_string(c.c_in) + ")");
    }
    int64_t k = 0;
    for (int64_t oc = 0; oc < c.c_out; ++oc) {
      if (plan->slot_of(oc, ic) >= 0) {
        if (filters && k < capacity) filters[k] = oc;
        ++k;
      }
    }
    *count = k;
  });
}

scc_status_t scc_forward_macs(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                              uint64_t* macs) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_ptr(macs, "macs");
    scc::check_extents(n, h, w);
    *macs = static_cast<uint64_t>(n * plan->cfg.c_out * h * w * plan->cfg.group_width);
  });
}

scc_status_t scc_plan_set_path(scc_plan_t* plan, int32_t path) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    if (path != SCC_PATH_AUTO && path != SCC_PATH_CUDA_CORE && path != SCC_PATH_TENSOR &&
        path != SCC_PATH_TENSOR_STREAMED) {
      scc::fail(SCC_ERR_ARGUMENT, "unknown path " + std::to_string(path));
    }
    plan->path = path;
  });
}

scc_status_t scc_plan_get_path(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                               int32_t* path) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_ptr(path, "path");
    *path = scc::pad_tc(*plan, n, h, w, 0) ? SCC_PATH_TENSOR : scc::choose_path(*plan, n, h, w);
  });
}

scc_status_t scc_forward_f32(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                             const float* x, const float* weight, const float* bias, float* y,
                             void* stream) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::do_forward(*const_cast<scc_plan_t*>(plan), n, h, w, x, weight, bias, y,
                    static_cast<cudaStream_t>(stream));
  });
}

scc_status_t scc_backward_data_f32(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                   const float* dy, const float* weight, float* dx, void* stream) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::do_backward_data(*const_cast<scc_plan_t*>(plan), n, h, w, dy, weight, dx,
                          static_cast<cudaStream_t>(stream));
  });
}

scc_status_t scc_backward_weight_workspace_size(const scc_plan_t* plan, int64_t n, int64_t h,
                                                int64_t w, size_t* bytes) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_ptr(bytes, "bytes");
    scc::check_extents(n, h, w);
    *bytes = scc::weight_ws_bytes(*plan, n, h * w);
  });
}

scc_status_t scc_backward_weight_f32(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                     const float* dy, const float* x, float* dweight,
                                     float* dbias, void* workspace, size_t workspace_bytes,
                                     void* stream) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::do_backward_weight(*const_cast<scc_plan_t*>(plan), n, h, w, dy, x, dweight, dbias,
                            workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  });
}

scc_status_t scc_backward_f32(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                              const float* dy, const float* x, const float* weight, float* dx,
                              float* dweight, float* dbias, void* workspace,
                              size_t workspace_bytes, void* stream) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    auto& p = *const_cast<scc_plan_t*>(plan);
    const auto s = static_cast<cudaStream_t>(stream);
    scc::do_backward(p, n, h, w, dy, x, weight, dx, dweight, dbias, workspace, workspace_bytes, s);
  });
}

scc_status_t scc_dsc_forward_f32(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                 int64_t stride, const float* x, const float* dw_weight,
                                 const float* dw_bias, const float* weight, const float* bias,
                                 float* y, void* stream) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_extents(n, h, w);
    scc::check_ptr(x, "x");
    scc::check_ptr(dw_weight, "dw_weight");
    scc::check_ptr(weight, "weight");
    scc::check_ptr(y, "y");
    auto& p = *const_cast<scc_plan_t*>(plan);
    scc::check_bias(p, bias, "bias");
    if (stride != 1 && stride != 2) {
      scc::fail(SCC_ERR_ARGUMENT, "depthwise stride must be 1 or 2, got " + std::to_string(stride));
    }
    const int64_t ho = (h - 1) / stride + 1, wo = (w - 1) / stride + 1;
    if (n * p.cfg.c_in * h * w >= (int64_t(1) << 31) || n * ho * wo >= (int64_t(1) << 31)) {
      scc::fail(SCC_ERR_SHAPE, "dsc forward: tensor too large for 32-bit plane indexing");
    }
    const scc::DeviceTables& t = scc::tables(p);
    scc::BandLaunch a = scc::band_args(p, t, false, n, ho * wo, x, y, weight, bias);
    a.dw_w = dw_weight;
    a.dw_b = dw_bias;
    a.dw_stride = static_cast<int32_t>(stride);
    a.h_in = static_cast<int32_t>(h);
    a.w_in = static_cast<int32_t>(w);
    a.w_out = static_cast<int32_t>(wo);
    scc::cuda_check(scc::launch_band_cc(a, static_cast<cudaStream_t>(stream)), "dsc forward launch");
  });
}

scc_status_t scc_dsc_forward_t_f32(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                   int64_t stride, const float* x, const float* dw_weight,
                                   const float* dw_bias, const float* weight, const float* bias,
                                   float* y, float* t, void* stream) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_extents(n, h, w);
    scc::check_ptr(x, "x");
    scc::check_ptr(dw_weight, "dw_weight");
    scc::check_ptr(weight, "weight");
    scc::check_ptr(y, "y");
    scc::check_ptr(t, "t");
    auto& p = *const_cast<scc_plan_t*>(plan);
    scc::check_bias(p, bias, "bias");
    if (stride != 1 && stride != 2) {
      scc::fail(SCC_ERR_ARGUMENT, "depthwise stride must be 1 or 2, got " + std::to_string(stride));
    }
    const int64_t ho = (h - 1) / stride + 1, wo = (w - 1) / stride + 1;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int32_t ci = static_cast<int32_t>(p.cfg.c_in), co = static_cast<int32_t>(p.cfg.c_out);
    // One tensor-core kernel when the geometry allows (stride 1, 16- or
    // 32-wide images, one row tile over every channel): the depthwise stage
    // runs in the SCC kernel's converters and t is stored on the way.
    if (stride == 1 && p.path != SCC_PATH_CUDA_CORE && p.path != SCC_PATH_TENSOR_STREAMED &&
        scc::aligned16(x) && scc::aligned16(y) && scc::aligned16(t) &&
        scc::choose_path(p, n, h, w, 0) == SCC_PATH_TENSOR &&
        scc::tc_dsc2_supported(p.tc_fwd, h * w, w, ci, co) && n * ci * h * w < (int64_t(1) << 31)) {
      const scc::DeviceTables& tb = scc::tables(p);
      scc::TcBandCall c = scc::tc_call(p, false, n, h * w, x, y, weight, bias);
      c.dsc_w = dw_weight;
      c.dsc_b = dw_bias;
      c.dsc_t = t;
      c.img_w = static_cast<int32_t>(w);
      scc::cuda_check(scc::launch_band_tc2(p.tc_fwd, tb.tc_fwd, c, p.cfg.shift, co, s), "dsc forward (tensor) launch");
      return;
    }
    // otherwise the pair: depthwise kernel into t, then the SCC forward on t
    const scc_status_t st = scc_dw3x3_forward_f32(n, ci, h, w, stride, x, dw_weight, dw_bias, t, stream);
    if (st != SCC_OK) scc::fail(st, scc::g_err);
    scc::do_forward(p, n, ho, wo, t, weight, bias, y, s);
  });
}

namespace scc {
namespace {
DwArgs dw_args(int64_t n, int64_t c, int64_t h, int64_t w, int64_t stride) {
  check_extents(n, h, w);
  if (c < 1) fail(SCC_ERR_SHAPE, "depthwise channel count must be >= 1, got " + std::to_string(c));
  if (stride != 1 && stride != 2) {
    fail(SCC_ERR_ARGUMENT, "depthwise stride must be 1 or 2, got " + std::to_string(stride));
  }
  if (n * c * h * w >= (int64_t(1) << 31)) fail(SCC_ERR_SHAPE, "depthwise tensor too large (>= 2^31 elements)");
  current_device();
  DwArgs a;
  a.n = n;
  a.c = c;
  a.h = static_cast<int32_t>(h);
  a.w = static_cast<int32_t>(w);
  a.ho = static_cast<int32_t>((h - 1) / stride + 1);
  a.wo = static_cast<int32_t>((w - 1) / stride + 1);
  a.stride = static_cast<int32_t>(stride);
  return a;
}
}  // namespace
}  // namespace scc

scc_status_t scc_dw3x3_forward_f32(int64_t n, int64_t c, int64_t h, int64_t w, int64_t stride,
                                   const float* x, const float* weight, const float* bias,
                                   float* y, void* stream) {
  return guard([&] {
    scc::DwArgs a = scc::dw_args(n, c, h, w, stride);
    scc::check_ptr(x, "x");
    scc::check_ptr(weight, "weight");
    scc::check_ptr(y, "y");
    a.x = x;
    a.wt = weight;
    a.b = bias;
    a.y = y;
    scc::cuda_check(scc::launch_dw(a, 0, static_cast<cudaStream_t>(stream)), "depthwise forward launch");
  });
}

scc_status_t scc_dw3x3_backward_data_f32(int64_t n, int64_t c, int64_t h, int64_t w,
                                         int64_t stride, const float* dy, const float* weight,
                                         float* dx, void* stream) {
  return guard([&] {
    scc::DwArgs a = scc::dw_args(n, c, h, w, stride);
    scc::check_ptr(dy, "dy");
    scc::check_ptr(weight, "weight");
    scc::check_ptr(dx, "dx");
    a.dy = dy;
    a.wt = weight;
    a.dx = dx;
    scc::cuda_check(scc::launch_dw(a, 1, static_cast<cudaStream_t>(stream)),
                    "depthwise backward-data launch");
  });
}

scc_status_t scc_dw3x3_workspace_size(int64_t c, size_t* bytes) {
  return guard([&] {
    scc::check_ptr(bytes, "bytes");
    *bytes = scc::dw_workspace_bytes(c);
  });
}

scc_status_t scc_dw3x3_backward_weight_f32(int64_t n, int64_t c, int64_t h, int64_t w,
                                           int64_t stride, const float* dy, const float* x,
                                           float* dweight, float* dbias, void* workspace,
                                           size_t workspace_bytes, void* stream) {
  return guard([&] {
    scc::DwArgs a = scc::dw_args(n, c, h, w, stride);
    scc::check_ptr(dy, "dy");
    scc::check_ptr(x, "x");
    scc::check_ptr(dweight, "dweight");
    if (workspace == nullptr || workspace_bytes < scc::dw_workspace_bytes(c)) {
      scc::fail(SCC_ERR_ARGUMENT, "workspace too small: need " + std::to_string(scc::dw_workspace_bytes(c)) + " bytes");
    }
    a.dy = dy;
    a.x = x;
    a.dw = dweight;
    a.db = dbias;
    a.part = static_cast<float*>(workspace);
    scc::cuda_check(scc::launch_dw(a, 2, static_cast<cudaStream_t>(stream)),
                    "depthwise backward-weight launch");
  });
}

scc_status_t scc_dw3x3_backward_f32(int64_t n, int64_t c, int64_t h, int64_t w, int64_t stride,
                                    const float* dy, const float* x, const float* weight, float* dx,
                                    float* dweight, float* dbias, void* workspace, size_t workspace_bytes,
                                    void* stream) {
  return guard([&] {
    scc::DwArgs a = scc::dw_args(n, c, h, w, stride);
    scc::check_ptr(dy, "dy");
    scc::check_ptr(x, "x");
    scc::check_ptr(weight, "weight");
    scc::check_ptr(dx, "dx");
    scc::check_ptr(dweight, "dweight");
    if (workspace == nullptr || workspace_bytes < scc::dw_workspace_bytes(c)) {
      scc::fail(SCC_ERR_ARGUMENT, "workspace too small: need " + std::to_string(scc::dw_workspace_bytes(c)) + " bytes");
    }
    a.dy = dy;
    a.x = x;
    a.wt = weight;
    a.dx = dx;
    a.dw = dweight;
    a.db = dbias;
    a.part = static_cast<float*>(workspace);
    scc::cuda_check(scc::launch_dw(a, 3, static_cast<cudaStream_t>(stream)), "depthwise backward launch");
  });
}

scc_status_t scc_forward_host_f32(scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                  const float* x, const float* weight, const float* bias,
                                  float* y) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_extents(n, h, w);
    scc::check_ptr(x, "x");
    scc::check_ptr(weight, "weight");
    scc::check_ptr(y, "y");
    scc::check_bias(*plan, bias, "bias");
    std::lock_guard<std::mutex> lk(plan->host_mu);
    scc::HostIo io;
    io.x = x;
    io.w = weight;
    io.b = bias;
    io.y = y;
    scc::run_host(*plan, n, h, w, io);
  });
}

scc_status_t scc_backward_host_f32(scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                   const float* dy, const float* x, const float* weight,
                                   float* dx, float* dweight, float* dbias) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_extents(n, h, w);
    scc::check_ptr(dy, "dy");
    scc::check_ptr(x, "x");
    scc::check_ptr(weight, "weight");
    scc::check_ptr(dx, "dx");
    scc::check_ptr(dweight, "dweight");
    scc::check_bias(*plan, dbias, "dbias");
    std::lock_guard<std::mutex> lk(plan->host_mu);
    scc::HostIo io;
    io.x = x;
    io.w = weight;
    io.dy = dy;
    io.dx = dx;
    io.dw = dweight;
    io.db = dbias;
    scc::run_host(*plan, n, h, w, io);
  });
}

scc_status_t scc_backward_data_host_f32(scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                        const float* dy, const float* weight, float* dx) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_extents(n, h, w);
    scc::check_ptr(dy, "dy");
    scc::check_ptr(weight, "weight");
    scc::check_ptr(dx, "dx");
    std::lock_guard<std::mutex> lk(plan->host_mu);
    scc::HostIo io;
    io.w = weight;
    io.dy = dy;
    io.dx = dx;
    scc::run_host(*plan, n, h, w, io);
  });
}

scc_status_t scc_backward_weight_host_f32(scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                          const float* dy, const float* x, float* dweight,
                                          float* dbias) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_extents(n, h, w);
    scc::check_ptr(dy, "dy");
    scc::check_ptr(x, "x");
    scc::check_ptr(dweight, "dweight");
    scc::check_bias(*plan, dbias, "dbias");
    std::lock_guard<std::mutex> lk(plan->host_mu);
    scc::HostIo io;
    io.x = x;
    io.dy = dy;
    io.dw = dweight;
    io.db = dbias;
    scc::run_host(*plan, n, h, w, io);
  });
}

scc_status_t scc_fwd_bwd_host_f32(scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                  const float* x, const float* weight, const float* bias,
                                  const float* dy, float* y, float* dx, float* dweight,
                                  float* dbias) {
  return guard([&] {
    scc::check_ptr(plan, "plan");
    scc::check_extents(n, h, w);
    for (const void* p : {static_cast<const void*>(x), static_cast<const void*>(weight),
                          static_cast<const void*>(dy), static_cast<const void*>(y),
                          static_cast<const void*>(dx), static_cast<const void*>(dweight)}) {
      scc::check_ptr(p, "buffer");
    }
    scc::check_bias(*plan, bias, "bias");
    scc::check_bias(*plan, dbias, "dbias");
    std::lock_guard<std::mutex> lk(plan->host_mu);
    scc::HostIo io;
    io.x = x;
    io.w = weight;
    io.b = bias;
    io.dy = dy;
    io.y = y;
    io.dx = dx;
    io.dw = dweight;
    io.db = dbias;
    scc::run_host(*plan, n, h, w, io);
  });
}

}  // extern "C"
