/*
 * scc_b200.h — C ABI of the B200-native sliding-channel convolution (SCC).
 *
 * Drop-in boundary for the reference operator library proj/core
 * (/root/reference/proj/core/include/sccl/*.hpp).  The reference exposes a C++
 * API over host fp64 tensors; this ABI exposes the same operator over
 * caller-owned fp32 NCHW device buffers (plus a host-buffer convenience layer),
 * with plain pointers, sizes and status codes only (no torch or C++ types).
 * include/sccl_b200.hpp restores the reference's C++ names on top of it, and
 * INTEGRATION.md shows the binding a maintainer adds on the reference side.
 *
 * Semantics (identical to the reference):
 *   gw     = c_in / cg                         (config.cpp:78)
 *   ov     = llround(ratio * gw) | count       (config.cpp:39-53)
 *   shift  = gw - ov                           (config.cpp:80)
 *   start(oc) = (oc * shift) mod c_in          (cycle.cpp:9-26, cycle_test.cpp:104-106)
 *   y[n,oc,p]  = b[oc] + sum_k w[oc*gw+k] * x[n,(start(oc)+k) mod c_in,p]
 *   dx[n,ic,p] = sum_{oc covers ic} w[oc*gw+(ic-start(oc)) mod c_in] * dy[n,oc,p]
 *   dw[oc*gw+k] = sum_{n,p} dy[n,oc,p] * x[n,(start(oc)+k) mod c_in,p]
 *   db[oc]      = sum_{n,p} dy[n,oc,p]
 *
 * Threading: every device entry point is asynchronous on the caller's stream
 * (a cudaStream_t passed as void*; NULL = legacy default stream), re-entrant
 * across streams and plans, and deterministic (no floating-point atomics), so
 * repeated calls are bitwise identical — the GPU analogue of the reference's
 * thread-count invariance (kernel.hpp:43-48, kernel_test.cpp:209-241).
 *
 * Activation pointers should be 16-byte aligned: the vector / TMA kernels
 * need it, and a misaligned buffer takes the scalar CUDA-core kernels.
 * Non-finite activations: the banded tensor-core kernels multiply explicit
 * zero weights outside each window, so an Inf/NaN input reaches every output
 * sharing its pixel and row tile -- a superset of the outputs the reference
 * makes non-finite (kernel.cpp:45-60 only touches in-window channels);
 * finite inputs are unaffected.
 */
#ifndef SCC_B200_H_
#define SCC_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCC_B200_ABI_VERSION 1

/* Status codes, 1:1 with the reference's exception classes
 * (proj/core/include/sccl/errors.hpp:9-55) plus device failures. */
typedef enum {
  SCC_OK = 0,
  SCC_ERR_SHAPE = 1,    /* sccl::ShapeError    */
  SCC_ERR_INDEX = 2,    /* sccl::IndexError    */
  SCC_ERR_CONFIG = 3,   /* sccl::ConfigError   */
  SCC_ERR_ARGUMENT = 4, /* sccl::ArgumentError */
  SCC_ERR_NUMERIC = 5,  /* sccl::NumericError  */
  SCC_ERR_CUDA = 6,     /* CUDA runtime / launch failure, or no sm_100a device */
  SCC_ERR_INTERNAL = 7
} scc_status_t;

/* Overlap flavour (config.hpp:12-38): a fraction of the window, or a count. */
typedef enum { SCC_OVERLAP_CHANNELS = 0, SCC_OVERLAP_RATIO = 1 } scc_overlap_kind_t;

/* Kernel family selection.  AUTO picks per shape. */
typedef enum {
  SCC_PATH_AUTO = 0,
  SCC_PATH_CUDA_CORE = 1,       /* fp32 FFMA banded kernels                                */
  SCC_PATH_TENSOR = 2,          /* tcgen05 banded-GEMM kernels (AUTO): 3xTF32 forward, bf16x3 fused /
                                   generation-1 backward (gradient bar 1e-4)                   */
  SCC_PATH_TENSOR_STREAMED = 3  /* tcgen05 kernels that stream the weight panel from L2: the
                                   family AUTO uses for layers whose panel does not fit in
                                   shared memory; forcing it on small layers is for tests  */
} scc_path_t;

typedef struct scc_plan scc_plan_t;

/* Mirrors sccl::SccConfig (config.hpp:43-55) + ChannelCycle::cyclic_dist. */
typedef struct {
  int64_t c_in, c_out, cg, overlap_channels, group_width, shift;
  int32_t has_bias;
  int32_t fully_overlapped; /* SccConfig::fully_overlapped() (config.hpp:54) */
  int64_t cyclic_dist;      /* ChannelCycle::cyclic_dist (cycle.hpp:30-33)  */
} scc_config_t;

/* Message of the last failing call on this thread ("" if none). */
const char* scc_last_error(void);
int scc_abi_version(void);

/* Number of CUDA kernels this library has launched in this process (all
 * threads); used by bench.py to report gpu_launches. */
uint64_t scc_launch_count(void);

/* Diagnostic: per-phase %globaltimer stamps (ns) of CTA 0 of the last
 * tensor-core band launch (slots 0..31, map in scc_tc.cu) and of the last
 * backward-weight launch (slots 32..63, map in scc_tc_wgrad.cu) on the
 * current device.  Copies min(n, 64) values; returns the count or -1. */
int scc_debug_trace(uint64_t* out, int n);
/* Diagnostic: the same for the fused backward kernel (scc_tc_bwd.cu; 64
 * CTA-0 slots, then start / end stamps of up to 256 CTAs).  Zeros unless the
 * library was built with -DSCC_TRACE. */
int scc_debug_trace_fused(uint64_t* out, int n);

/* ---- geometry (host only; replaces config.cpp / cycle.cpp) --------------- */

/* Overlap::parse (config.cpp:15-37): "50%", "0.5" -> ratio; "3" -> count.
 * SCC_ERR_ARGUMENT on unparseable text. */
scc_status_t scc_overlap_parse(const char* text, int32_t* kind, double* ratio,
                               int64_t* count);

/* Overlap::resolve (config.cpp:39-53). SCC_ERR_CONFIG when out of range. */
scc_status_t scc_overlap_resolve(int32_t kind, double ratio, int64_t count,
                                 int64_t group_width, int64_t* channels);

/* scc_config_new (config.cpp:62-83) + plan tables.  SCC_ERR_CONFIG on invalid
 * geometry.  The plan is immutable after creation (device tables are uploaded
 * lazily, once per device, under a lock). */
scc_status_t scc_plan_create(int64_t c_in, int64_t c_out, int64_t cg,
                             int32_t overlap_kind, double ratio, int64_t count,
                             int32_t has_bias, scc_plan_t** plan);
scc_status_t scc_plan_destroy(scc_plan_t* plan);
scc_status_t scc_plan_config(const scc_plan_t* plan, scc_config_t* out);

/* compute_channel_cycle (cycle.cpp:9-21): distinct window starts in walk
 * order.  *count = cyclic_dist; at most `capacity` entries are written. */
scc_status_t scc_plan_cycle_starts(const scc_plan_t* plan, int64_t* starts,
                                   int64_t capacity, int64_t* count);

/* window_of (cycle.cpp:23-26): SCC_ERR_INDEX when oc < 0. */
scc_status_t scc_plan_window_of(const scc_plan_t* plan, int64_t oc, int64_t* start,
                                int64_t* length);

/* covering_filters (cycle.cpp:28-40): ascending oc covering ic.
 * SCC_ERR_INDEX when ic is outside [0, c_in). */
scc_status_t scc_plan_covering_filters(const scc_plan_t* plan, int64_t ic,
                                       int64_t* filters, int64_t capacity,
                                       int64_t* count);

/* MACs of one forward, the count scc_forward_counted reports
 * (kernel.hpp:51-54, kernel.cpp:59): n * c_out * h * w * gw. */
scc_status_t scc_forward_macs(const scc_plan_t* plan, int64_t n, int64_t h,
                              int64_t w, uint64_t* macs);

/* Force a kernel family for this plan (tests/bench); AUTO by default.
 * Set it before issuing work: calls already in flight on other threads may
 * run with either the old or the new family.
 * SCC_PATH_TENSOR is a preference: directions (or calls) the tensor-core
 * band GEMM cannot express run on the CUDA-core kernels.  SCC_ERR_ARGUMENT for
 * an unknown value. */
scc_status_t scc_plan_set_path(scc_plan_t* plan, int32_t path);
/* The family AUTO would pick (or the forced one) for n*h*w pixels. */
scc_status_t scc_plan_get_path(const scc_plan_t* plan, int64_t n, int64_t h,
                               int64_t w, int32_t* path);

/* ---- device operator (fp32 NCHW, caller-owned device memory) ------------- */

/* scc_forward (kernel.hpp:43-49 / kernel.cpp:89-91).
 * x: [n, c_in, h, w]; weight: [c_out * gw] window-relative ([oc][k],
 * kernel.hpp:13-17); bias: [c_out] or NULL iff !has_bias; y: [n, c_out, h, w]. */
scc_status_t scc_forward_f32(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                             const float* x, const float* weight, const float* bias,
                             float* y, void* stream);

/* scc_backward_input (kernel.hpp:56-61 / kernel.cpp:98-138).  Input-centric,
 * no atomics; channels no filter covers are written as zero. */
scc_status_t scc_backward_data_f32(const scc_plan_t* plan, int64_t n, int64_t h,
                                   int64_t w, const float* dy, const float* weight,
                                   float* dx, void* stream);

/* Workspace for the deterministic split reduction of the parameter gradients. */
scc_status_t scc_backward_weight_workspace_size(const scc_plan_t* plan, int64_t n,
                                                int64_t h, int64_t w, size_t* bytes);

/* scc_backward_params (kernel.hpp:62-68 / kernel.cpp:140-181).
 * dweight: [c_out * gw]; dbias: [c_out] or NULL iff !has_bias. */
scc_status_t scc_backward_weight_f32(const scc_plan_t* plan, int64_t n, int64_t h,
                                     int64_t w, const float* dy, const float* x,
                                     float* dweight, float* dbias, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* scc_backward (kernel.hpp:70-72 / kernel.cpp:183-189): both passes; may fuse
 * them into one pass over dy/x.  Workspace as scc_backward_weight_f32. */
scc_status_t scc_backward_f32(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                              const float* dy, const float* x, const float* weight,
                              float* dx, float* dweight, float* dbias, void* workspace,
                              size_t workspace_bytes, void* stream);

/* ---- host-buffer operator (what a host caller of proj/core links) -------- */
/* Synchronous.  Buffers live in host memory (pinned for full PCIe speed);
 * device staging is owned by the plan (grown on demand, per device) so
 * concurrent host calls on one plan are serialised. */
scc_status_t scc_forward_host_f32(scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                  const float* x, const float* weight,
                                  const float* bias, float* y);
scc_status_t scc_backward_host_f32(scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                   const float* dy, const float* x, const float* weight,
                                   float* dx, float* dweight, float* dbias);
/* scc_backward_input (kernel.hpp:56-61) with host buffers: moves dy in and dx
 * out only (backward-data never sees x, kernel.cpp:98-138). */
scc_status_t scc_backward_data_host_f32(scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                        const float* dy, const float* weight, float* dx);
/* scc_backward_params (kernel.hpp:62-68) with host buffers: dy and x in,
 * dweight / dbias out (dbias NULL iff !has_bias). */
scc_status_t scc_backward_weight_host_f32(scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                          const float* dy, const float* x, float* dweight,
                                          float* dbias);
/* One training step of the layer (forward then backward) with host buffers.
 * All host entry points pipeline H2D / kernels / D2H over batch chunks. */
scc_status_t scc_fwd_bwd_host_f32(scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                  const float* x, const float* weight, const float* bias,
                                  const float* dy, float* y, float* dx, float* dweight,
                                  float* dbias);

/* ---- fused dsc_block forward (model.cpp:213-220) ------------------------- */
/* y = SCC(DW3x3(x)): the depthwise 3x3 stage (groups = c_in, padding 1,
 * stride 1 or 2; conv_forward_impl, reference.cpp:74-123) computed inside the
 * SCC kernel's staging step, so the DW output never goes to HBM.
 * x: [n][c_in][h][w]; dw_weight: [c_in][3][3]; dw_bias: [c_in] or NULL;
 * weight / bias: the SCC layer's (as scc_forward_f32);
 * y: [n][c_out][h_out][w_out], h_out = (h - 1) / stride + 1 (same for w). */
scc_status_t scc_dsc_forward_f32(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                 int64_t stride, const float* x, const float* dw_weight,
                                 const float* dw_bias, const float* weight, const float* bias,
                                 float* y, void* stream);

/* dsc_block forward that also returns t = DW3x3(x) (the SCC stage's input,
 * which the block's backward needs): y = SCC(t).  For stride 1 on 16- or
 * 32-wide images (planes a multiple of 128 px) whose SCC layer is one
 * tensor-core row tile over every input channel, one kernel computes t in
 * its staging step (the depthwise output goes to HBM once, as t, and is
 * never read back); otherwise the depthwise kernel then
 * scc_forward_f32.  t: [n][c_in][h_out][w_out]. */
scc_status_t scc_dsc_forward_t_f32(const scc_plan_t* plan, int64_t n, int64_t h, int64_t w,
                                   int64_t stride, const float* x, const float* dw_weight,
                                   const float* dw_bias, const float* weight, const float* bias,
                                   float* y, float* t, void* stream);

/* ---- depthwise 3x3 stage of a dsc_block (model.cpp:213-220) -------------- */
/* groups = c, kernel 3, padding 1, stride 1 or 2 (conv_forward_impl,
 * reference.cpp:74-123).  x: [n][c][h][w]; weight: [c][3][3]; bias: [c] or
 * NULL; y / dy: [n][c][h_out][w_out] with h_out = (h - 1) / stride + 1.
 * Backward-weight needs scc_dw3x3_workspace_size() bytes of workspace and is
 * deterministic (fixed-order reduction, no atomics). */
scc_status_t scc_dw3x3_forward_f32(int64_t n, int64_t c, int64_t h, int64_t w, int64_t stride,
                                   const float* x, const float* weight, const float* bias,
                                   float* y, void* stream);
scc_status_t scc_dw3x3_backward_data_f32(int64_t n, int64_t c, int64_t h, int64_t w,
                                         int64_t stride, const float* dy, const float* weight,
                                         float* dx, void* stream);
scc_status_t scc_dw3x3_workspace_size(int64_t c, size_t* bytes);
scc_status_t scc_dw3x3_backward_weight_f32(int64_t n, int64_t c, int64_t h, int64_t w,
                                           int64_t stride, const float* dy, const float* x,
                                           float* dweight, float* dbias, void* workspace,
                                           size_t workspace_bytes, void* stream);
/* The whole depthwise backward (grouped_conv_backward, reference.cpp:155-247):
 * dx, dweight and dbias (NULL: skipped) from one pass over dy and x at
 * stride 1 (bitwise the two calls above); stride 2 runs those two calls. */
scc_status_t scc_dw3x3_backward_f32(int64_t n, int64_t c, int64_t h, int64_t w, int64_t stride,
                                    const float* dy, const float* x, const float* weight, float* dx,
                                    float* dweight, float* dbias, void* workspace, size_t workspace_bytes,
                                    void* stream);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* SCC_B200_H_ */
