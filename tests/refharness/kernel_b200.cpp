// Link-level drop-in for proj/core/src/kernel.cpp: every function declared in
// the reference's sccl/kernel.hpp (kernel.hpp:37-72), implemented over the
// B200 C ABI (include/scc_b200.h).  Linking this file instead of kernel.cpp
// runs the reference's own model / training code (model.cpp:266 forward,
// model.cpp:372 backward, train.cpp) with every SCC layer on the GPU.
//
// Values cross the boundary as fp32 (the device arithmetic type): the fp64
// Tensor4 is rounded to fp32 on the way in and widened on the way out.
// Geometry, validation order and exception types follow the reference:
// ShapeError for channel / weight-size mismatches (kernel.cpp:14-25,32-35,
// 100-103,142-146); device failures surface as sccl::NumericError.
//
// Plans (one per distinct SccConfig) are cached for the process lifetime.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "scc_b200.h"
#include "sccl/errors.hpp"
#include "sccl/kernel.hpp"

namespace sccl {

namespace {

void check_weights(const SccWeights& wts, const SccConfig& cfg) {
  const std::size_t want_w = static_cast<std::size_t>(cfg.c_out * cfg.group_width);
  if (wts.weight.size() != want_w) {
    throw ShapeError("weight array has " + std::to_string(wts.weight.size()) +
                     " entries, config needs " + std::to_string(want_w));
  }
  const std::size_t want_b = cfg.has_bias ? static_cast<std::size_t>(cfg.c_out) : 0;
  if (wts.bias.size() != want_b) {
    throw ShapeError("bias array has " + std::to_string(wts.bias.size()) +
                     " entries, config needs " + std::to_string(want_b));
  }
}

void check(scc_status_t st) {
  if (st == SCC_OK) return;
  const std::string msg = std::string("libscc_b200: ") + scc_last_error();
  switch (st) {
    case SCC_ERR_SHAPE: throw ShapeError(msg);
    case SCC_ERR_CONFIG: throw ConfigError(msg);
    case SCC_ERR_INDEX: throw IndexError(msg);
    case SCC_ERR_ARGUMENT: throw ArgumentError(msg);
    default: throw NumericError(msg);
  }
}

scc_plan_t* plan_for(const SccConfig& cfg) {
  using Key = std::tuple<int64_t, int64_t, int64_t, int64_t, bool>;
  static std::mutex mu;
  static std::map<Key, scc_plan_t*> plans;
  const Key k{cfg.c_in, cfg.c_out, cfg.cg, cfg.overlap_channels, cfg.has_bias};
  std::lock_guard<std::mutex> lk(mu);
  auto it = plans.find(k);
  if (it != plans.end()) return it->second;
  scc_plan_t* p = nullptr;
  check(scc_plan_create(cfg.c_in, cfg.c_out, cfg.cg, SCC_OVERLAP_CHANNELS, 0.0,
                        cfg.overlap_channels, cfg.has_bias ? 1 : 0, &p));
  plans.emplace(k, p);
  return p;
}

std::vector<float> narrow(const double* src, std::size_t n) {
  std::vector<float> out(n);
  for (std::size_t i = 0; i < n; ++i) out[i] = static_cast<float>(src[i]);
  return out;
}

void widen(const std::vector<float>& src, double* dst) {
  for (std::size_t i = 0; i < src.size(); ++i) dst[i] = static_cast<double>(src[i]);
}

}  // namespace

SccWeights scc_weights_filled(const SccConfig& cfg, double weight_value, double bias_value) {
  SccWeights wts;
  wts.weight.assign(static_cast<std::size_t>(cfg.c_out * cfg.group_width), weight_value);
  if (cfg.has_bias) wts.bias.assign(static_cast<std::size_t>(cfg.c_out), bias_value);
  return wts;
}

// Same draw order as kernel.cpp:82-87 (weights in [oc][k] order, bias zero),
// so a network built over this file starts from the reference's weights.
SccWeights scc_weights_init(const SccConfig& cfg, Rng& rng) {
  SccWeights wts = scc_weights_filled(cfg, 0.0, 0.0);
  const double bound = std::sqrt(1.0 / static_cast<double>(cfg.group_width));
  for (double& w : wts.weight) w = rng.uniform(-bound, bound);
  return wts;
}

Tensor4 scc_forward(const Tensor4& input, const SccWeights& wts, const SccConfig& cfg) {
  if (input.c() != cfg.c_in) {
    throw ShapeError("input has " + std::to_string(input.c()) + " channels, config expects " +
                     std::to_string(cfg.c_in));
  }
  check_weights(wts, cfg);
  Tensor4 out(input.n(), cfg.c_out, input.h(), input.w());
  const std::vector<float> x = narrow(input.data(), static_cast<std::size_t>(input.size()));
  const std::vector<float> w = narrow(wts.weight.data(), wts.weight.size());
  const std::vector<float> b = narrow(wts.bias.data(), wts.bias.size());
  std::vector<float> y(static_cast<std::size_t>(out.size()));
  check(scc_forward_host_f32(plan_for(cfg), input.n(), input.h(), input.w(), x.data(), w.data(),
                             cfg.has_bias ? b.data() : nullptr, y.data()));
  widen(y, out.data());
  return out;
}

Tensor4 scc_forward_counted(const Tensor4& input, const SccWeights& wts, const SccConfig& cfg,
                            std::uint64_t* mac_count) {
  Tensor4 out = scc_forward(input, wts, cfg);
  if (mac_count) {
    // Every multiply of the reference loop (kernel.cpp:52-58): N*Co*H*W*gw.
    *mac_count = static_cast<std::uint64_t>(input.n() * cfg.c_out * input.h() * input.w() *
                                            cfg.group_width);
  }
  return out;
}

SccGradients scc_backward(const Tensor4& grad_out, const Tensor4& input, const SccWeights& wts,
                          const SccConfig& cfg) {
  if (grad_out.c() != cfg.c_out) {
    throw ShapeError("grad_out has " + std::to_string(grad_out.c()) +
                     " channels, config expects " + std::to_string(cfg.c_out));
  }
  if (input.c() != cfg.c_in) {
    throw ShapeError("input has " + std::to_string(input.c()) + " channels, config expects " +
                     std::to_string(cfg.c_in));
  }
  if (grad_out.n() != input.n() || grad_out.h() != input.h() || grad_out.w() != input.w()) {
    throw ShapeError("grad_out and input disagree on batch or spatial extents");
  }
  check_weights(wts, cfg);
  SccGradients g;
  g.grad_input = Tensor4(input.n(), cfg.c_in, input.h(), input.w());
  const std::vector<float> dy = narrow(grad_out.data(), static_cast<std::size_t>(grad_out.size()));
  const std::vector<float> x = narrow(input.data(), static_cast<std::size_t>(input.size()));
  const std::vector<float> w = narrow(wts.weight.data(), wts.weight.size());
  std::vector<float> dx(static_cast<std::size_t>(input.size()));
  std::vector<float> dw(wts.weight.size()), db(static_cast<std::size_t>(cfg.has_bias ? cfg.c_out : 0));
  check(scc_backward_host_f32(plan_for(cfg), input.n(), input.h(), input.w(), dy.data(), x.data(),
                              w.data(), dx.data(), dw.data(), cfg.has_bias ? db.data() : nullptr));
  widen(dx, g.grad_input.data());
  g.params.grad_weight.assign(dw.begin(), dw.end());
  g.params.grad_bias.assign(db.begin(), db.end());
  return g;
}

Tensor4 scc_backward_input(const Tensor4& grad_out, const SccWeights& wts, const SccConfig& cfg) {
  if (grad_out.c() != cfg.c_out) {
    throw ShapeError("grad_out has " + std::to_string(grad_out.c()) +
                     " channels, config expects " + std::to_string(cfg.c_out));
  }
  check_weights(wts, cfg);
  // backward-data never sees X (kernel.cpp:120): dy in, dx out
  Tensor4 dx(grad_out.n(), cfg.c_in, grad_out.h(), grad_out.w());
  const std::vector<float> dy = narrow(grad_out.data(), static_cast<std::size_t>(grad_out.size()));
  const std::vector<float> w = narrow(wts.weight.data(), wts.weight.size());
  std::vector<float> out(static_cast<std::size_t>(dx.size()));
  check(scc_backward_data_host_f32(plan_for(cfg), grad_out.n(), grad_out.h(), grad_out.w(), dy.data(),
                                   w.data(), out.data()));
  widen(out, dx.data());
  return dx;
}

SccParamGradients scc_backward_params(const Tensor4& grad_out, const Tensor4& input,
                                      const SccConfig& cfg) {
  if (grad_out.c() != cfg.c_out) {
    throw ShapeError("grad_out has " + std::to_string(grad_out.c()) +
                     " channels, config expects " + std::to_string(cfg.c_out));
  }
  if (input.c() != cfg.c_in) {
    throw ShapeError("input has " + std::to_string(input.c()) + " channels, config expects " +
                     std::to_string(cfg.c_in));
  }
  if (grad_out.n() != input.n() || grad_out.h() != input.h() || grad_out.w() != input.w()) {
    throw ShapeError("grad_out and input disagree on batch or spatial extents");
  }
  const std::vector<float> dy = narrow(grad_out.data(), static_cast<std::size_t>(grad_out.size()));
  const std::vector<float> x = narrow(input.data(), static_cast<std::size_t>(input.size()));
  std::vector<float> dw(static_cast<std::size_t>(cfg.c_out * cfg.group_width));
  std::vector<float> db(static_cast<std::size_t>(cfg.has_bias ? cfg.c_out : 0));
  check(scc_backward_weight_host_f32(plan_for(cfg), input.n(), input.h(), input.w(), dy.data(), x.data(),
                                     dw.data(), cfg.has_bias ? db.data() : nullptr));
  SccParamGradients g;
  g.grad_weight.assign(dw.begin(), dw.end());
  g.grad_bias.assign(db.begin(), db.end());
  return g;
}

}  // namespace sccl
