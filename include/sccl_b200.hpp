// sccl_b200.hpp — header-only C++ layer over the C ABI (scc_b200.h) that
// restores the reference operator API of proj/core (namespace sccl):
//
//   reference (proj/core/include/sccl/...)         here (namespace sccl_b200)
//   Overlap::ratio/channels/parse/resolve/str      same          config.hpp:12-38
//   SccConfig, scc_config_new                      same          config.hpp:43-61
//   ChannelWindow, ChannelCycle,                   same          cycle.hpp:13-48
//     compute_channel_cycle, window_of,
//     covering_filters
//   SccWeights / SccParamGradients / SccGradients  same names    kernel.hpp:18-33
//   scc_forward / scc_backward_input /             same names    kernel.hpp:43-72
//     scc_backward_params / scc_backward
//   Error, ShapeError, IndexError, ConfigError,    same names    errors.hpp:9-55
//     ArgumentError, NumericError (+ CudaError)
//
// Two tensor flavours:
//   * HostTensor4 (fp64 NCHW, like sccl::Tensor4) -> host-buffer entry points;
//     values are rounded to fp32 for the device and widened back.  This is the
//     literal drop-in for callers of the reference (model.cpp:266,372,
//     gradcheck.cpp, bench.cpp).
//   * DeviceTensor4 (fp32 NCHW view of device memory) -> asynchronous device
//     entry points on a caller stream.
#pragma once

#include <cstdint>
#include <cstdio>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "scc_b200.h"

namespace sccl_b200 {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class ShapeError : public Error {
 public:
  using Error::Error;
};
class IndexError : public Error {
 public:
  using Error::Error;
};
class ConfigError : public Error {
 public:
  using Error::Error;
};
class ArgumentError : public Error {
 public:
  using Error::Error;
};
class NumericError : public Error {
 public:
  using Error::Error;
};
class CudaError : public Error {
 public:
  using Error::Error;
};

inline void check(scc_status_t s) {
  if (s == SCC_OK) return;
  const std::string msg = scc_last_error();
  switch (s) {
    case SCC_ERR_SHAPE: throw ShapeError(msg);
    case SCC_ERR_INDEX: throw IndexError(msg);
    case SCC_ERR_CONFIG: throw ConfigError(msg);
    case SCC_ERR_ARGUMENT: throw ArgumentError(msg);
    case SCC_ERR_NUMERIC: throw NumericError(msg);
    case SCC_ERR_CUDA: throw CudaError(msg);
    default: throw Error(msg);
  }
}

class Overlap {
 public:
  static Overlap ratio(double r) { return Overlap(SCC_OVERLAP_RATIO, r, 0); }
  static Overlap channels(std::int64_t count) { return Overlap(SCC_OVERLAP_CHANNELS, 0.0, count); }
  static Overlap parse(const std::string& text) {
    int32_t kind = 0;
    double r = 0;
    int64_t c = 0;
    check(scc_overlap_parse(text.c_str(), &kind, &r, &c));
    return Overlap(kind, r, c);
  }
  bool is_ratio() const { return kind_ == SCC_OVERLAP_RATIO; }
  std::int64_t resolve(std::int64_t group_width) const {
    int64_t out = 0;
    check(scc_overlap_resolve(kind_, ratio_, count_, group_width, &out));
    return out;
  }
  std::string str() const {
    if (!is_ratio()) return std::to_string(count_);
    char buf[32];
    std::snprintf(buf, sizeof(buf), "%g%%", ratio_ * 100.0);
    return buf;
  }
  int32_t kind() const { return kind_; }
  double ratio_value() const { return ratio_; }
  std::int64_t count_value() const { return count_; }

 private:
  Overlap(int32_t k, double r, std::int64_t c) : kind_(k), ratio_(r), count_(c) {}
  int32_t kind_;
  double ratio_;
  std::int64_t count_;
};

// sccl::SccConfig plus the native plan that carries the device tables.
struct SccConfig {
  std::int64_t c_in = 0, c_out = 0, cg = 0, overlap_channels = 0, group_width = 0, shift = 0;
  bool has_bias = true;
  bool fully_overlapped() const { return shift == 0 && cg > 1; }
  scc_plan_t* plan() const { return plan_.get(); }

  std::shared_ptr<scc_plan_t> plan_;
};

inline SccConfig scc_config_new(std::int64_t c_in, std::int64_t c_out, std::int64_t cg,
                                const Overlap& co, bool has_bias) {
  scc_plan_t* p = nullptr;
  check(scc_plan_create(c_in, c_out, cg, co.kind(), co.ratio_value(), co.count_value(),
                        has_bias ? 1 : 0, &p));
  SccConfig cfg;
  cfg.plan_ = std::shared_ptr<scc_plan_t>(p, [](scc_plan_t* q) { scc_plan_destroy(q); });
  scc_config_t c{};
  check(scc_plan_config(p, &c));
  cfg.c_in = c.c_in;
  cfg.c_out = c.c_out;
  cfg.cg = c.cg;
  cfg.overlap_channels = c.overlap_channels;
  cfg.group_width = c.group_width;
  cfg.shift = c.shift;
  cfg.has_bias = c.has_bias != 0;
  return cfg;
}

struct ChannelWindow {
  std::int64_t start = 0, length = 0;
  bool contains(std::int64_t ch, std::int64_t c_in) const { return (ch - start + c_in) % c_in < length; }
  std::int64_t last(std::int64_t c_in) const { return (start + length - 1) % c_in; }
  bool operator==(const ChannelWindow&) const = default;
};

struct ChannelCycle {
  std::vector<ChannelWindow> windows;
  std::int64_t cyclic_dist = 0;
};

inline ChannelCycle compute_channel_cycle(const SccConfig& cfg) {
  int64_t n = 0;
  check(scc_plan_cycle_starts(cfg.plan(), nullptr, 0, &n));
  std::vector<int64_t> starts(static_cast<size_t>(n));
  check(scc_plan_cycle_starts(cfg.plan(), starts.data(), n, &n));
  ChannelCycle cyc;
  for (int64_t s : starts) cyc.windows.push_back({s, cfg.group_width});
  cyc.cyclic_dist = n;
  return cyc;
}

inline const ChannelWindow& window_of(const ChannelCycle& cycle, std::int64_t oc) {
  if (oc < 0) throw IndexError("output channel must be >= 0, got " + std::to_string(oc));
  return cycle.windows[static_cast<size_t>(oc % cycle.cyclic_dist)];
}

inline std::vector<std::int64_t> covering_filters(const SccConfig& cfg, const ChannelCycle&,
                                                  std::int64_t ic) {
  int64_t n = 0;
  check(scc_plan_covering_filters(cfg.plan(), ic, nullptr, 0, &n));
  std::vector<std::int64_t> out(static_cast<size_t>(n));
  check(scc_plan_covering_filters(cfg.plan(), ic, out.data(), n, &n));
  return out;
}

// ---- host fp64 tensors (the reference's Tensor4 contract, tensor.hpp:15-48) ----
class HostTensor4 {
 public:
  HostTensor4() = default;
  HostTensor4(std::int64_t n, std::int64_t c, std::int64_t h, std::int64_t w)
      : n_(n), c_(c), h_(h), w_(w) {
    if (n < 1 || c < 1 || h < 1 || w < 1) throw ShapeError("tensor extents must all be >= 1");
    data_.assign(static_cast<size_t>(n * c * h * w), 0.0);
  }
  std::int64_t n() const { return n_; }
  std::int64_t c() const { return c_; }
  std::int64_t h() const { return h_; }
  std::int64_t w() const { return w_; }
  std::int64_t size() const { return static_cast<std::int64_t>(data_.size()); }
  std::int64_t index(std::int64_t n, std::int64_t c, std::int64_t y, std::int64_t x) const {
    return ((n * c_ + c) * h_ + y) * w_ + x;
  }
  double& at(std::int64_t n, std::int64_t c, std::int64_t y, std::int64_t x) {
    return data_[static_cast<size_t>(index(n, c, y, x))];
  }
  double at(std::int64_t n, std::int64_t c, std::int64_t y, std::int64_t x) const {
    return data_[static_cast<size_t>(index(n, c, y, x))];
  }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }

 private:
  std::int64_t n_ = 0, c_ = 0, h_ = 0, w_ = 0;
  std::vector<double> data_;
};

struct SccWeights {
  std::vector<double> weight;
  std::vector<double> bias;
};
struct SccParamGradients {
  std::vector<double> grad_weight;
  std::vector<double> grad_bias;
};
struct SccGradients {
  HostTensor4 grad_input;
  SccParamGradients params;
};

inline SccWeights scc_weights_filled(const SccConfig& cfg, double w, double b = 0.0) {
  SccWeights s;
  s.weight.assign(static_cast<size_t>(cfg.c_out * cfg.group_width), w);
  if (cfg.has_bias) s.bias.assign(static_cast<size_t>(cfg.c_out), b);
  return s;
}

namespace detail {
inline std::vector<float> narrow(const double* p, std::int64_t n) {
  std::vector<float> v(static_cast<size_t>(n));
  for (std::int64_t i = 0; i < n; ++i) v[static_cast<size_t>(i)] = static_cast<float>(p[i]);
  return v;
}
inline void widen(const std::vector<float>& v, double* p) {
  for (size_t i = 0; i < v.size(); ++i) p[i] = v[i];
}
inline void check_weights(const SccWeights& wts, const SccConfig& cfg) {  // kernel.cpp:14-25
  if (static_cast<std::int64_t>(wts.weight.size()) != cfg.c_out * cfg.group_width)
    throw ShapeError("weight array has " + std::to_string(wts.weight.size()) + " entries");
  if (static_cast<std::int64_t>(wts.bias.size()) != (cfg.has_bias ? cfg.c_out : 0))
    throw ShapeError("bias array has " + std::to_string(wts.bias.size()) + " entries");
}
}  // namespace detail

// scc_forward (kernel.hpp:43-49), host fp64 in / out, fp32 on the device.
inline HostTensor4 scc_forward(const HostTensor4& input, const SccWeights& wts, const SccConfig& cfg) {
  if (input.c() != cfg.c_in)
    throw ShapeError("input has " + std::to_string(input.c()) + " channels, config expects " +
                     std::to_string(cfg.c_in));
  detail::check_weights(wts, cfg);
  const auto x = detail::narrow(input.data(), input.size());
  const auto w = detail::narrow(wts.weight.data(), static_cast<std::int64_t>(wts.weight.size()));
  const auto b = detail::narrow(wts.bias.data(), static_cast<std::int64_t>(wts.bias.size()));
  HostTensor4 out(input.n(), cfg.c_out, input.h(), input.w());
  std::vector<float> y(static_cast<size_t>(out.size()));
  check(scc_forward_host_f32(cfg.plan(), input.n(), input.h(), input.w(), x.data(), w.data(),
                             cfg.has_bias ? b.data() : nullptr, y.data()));
  detail::widen(y, out.data());
  return out;
}

// scc_backward (kernel.hpp:70-72): both passes in one host call.
inline SccGradients scc_backward(const HostTensor4& grad_out, const HostTensor4& input,
                                 const SccWeights& wts, const SccConfig& cfg) {
  if (grad_out.c() != cfg.c_out || input.c() != cfg.c_in || grad_out.n() != input.n() ||
      grad_out.h() != input.h() || grad_out.w() != input.w())
    throw ShapeError("grad_out/input shapes inconsistent with config");
  detail::check_weights(wts, cfg);
  const auto g = detail::narrow(grad_out.data(), grad_out.size());
  const auto x = detail::narrow(input.data(), input.size());
  const auto w = detail::narrow(wts.weight.data(), static_cast<std::int64_t>(wts.weight.size()));
  std::vector<float> dx(static_cast<size_t>(input.size())), dw(wts.weight.size()),
      db(static_cast<size_t>(cfg.has_bias ? cfg.c_out : 0));
  check(scc_backward_host_f32(cfg.plan(), input.n(), input.h(), input.w(), g.data(), x.data(),
                              w.data(), dx.data(), dw.data(), cfg.has_bias ? db.data() : nullptr));
  SccGradients out;
  out.grad_input = HostTensor4(input.n(), cfg.c_in, input.h(), input.w());
  detail::widen(dx, out.grad_input.data());
  out.params.grad_weight.assign(dw.begin(), dw.end());
  out.params.grad_bias.assign(db.begin(), db.end());
  return out;
}

// scc_backward_input (kernel.hpp:56-61): dy in, dx out (backward-data never
// sees x, kernel.cpp:98-138).
inline HostTensor4 scc_backward_input(const HostTensor4& grad_out, const SccWeights& wts,
                                      const SccConfig& cfg) {
  if (grad_out.c() != cfg.c_out)
    throw ShapeError("grad_out has " + std::to_string(grad_out.c()) + " channels, config expects " +
                     std::to_string(cfg.c_out));
  detail::check_weights(wts, cfg);
  const auto g = detail::narrow(grad_out.data(), grad_out.size());
  const auto w = detail::narrow(wts.weight.data(), static_cast<std::int64_t>(wts.weight.size()));
  HostTensor4 out(grad_out.n(), cfg.c_in, grad_out.h(), grad_out.w());
  std::vector<float> dx(static_cast<size_t>(out.size()));
  check(scc_backward_data_host_f32(cfg.plan(), grad_out.n(), grad_out.h(), grad_out.w(), g.data(),
                                   w.data(), dx.data()));
  detail::widen(dx, out.data());
  return out;
}

// scc_backward_params (kernel.hpp:62-68): dy and x in, dW / db out.
inline SccParamGradients scc_backward_params(const HostTensor4& grad_out, const HostTensor4& input,
                                             const SccConfig& cfg) {
  if (grad_out.c() != cfg.c_out || input.c() != cfg.c_in || grad_out.n() != input.n() ||
      grad_out.h() != input.h() || grad_out.w() != input.w())
    throw ShapeError("grad_out/input shapes inconsistent with config");
  const auto g = detail::narrow(grad_out.data(), grad_out.size());
  const auto x = detail::narrow(input.data(), input.size());
  std::vector<float> dw(static_cast<size_t>(cfg.c_out * cfg.group_width)),
      db(static_cast<size_t>(cfg.has_bias ? cfg.c_out : 0));
  check(scc_backward_weight_host_f32(cfg.plan(), input.n(), input.h(), input.w(), g.data(), x.data(),
                                     dw.data(), cfg.has_bias ? db.data() : nullptr));
  SccParamGradients out;
  out.grad_weight.assign(dw.begin(), dw.end());
  out.grad_bias.assign(db.begin(), db.end());
  return out;
}

// ---- device fp32 views (asynchronous on a caller stream) ----
struct DeviceTensor4 {
  float* data = nullptr;
  std::int64_t n = 0, c = 0, h = 0, w = 0;
};

inline void scc_forward(const DeviceTensor4& x, const float* weight, const float* bias,
                        const SccConfig& cfg, DeviceTensor4& y, void* stream = nullptr) {
  if (x.c != cfg.c_in || y.c != cfg.c_out || y.n != x.n || y.h != x.h || y.w != x.w)
    throw ShapeError("forward tensor shapes inconsistent with config");
  check(scc_forward_f32(cfg.plan(), x.n, x.h, x.w, x.data, weight, bias, y.data, stream));
}

}  // namespace sccl_b200
