// The reference's own known-answer tests (proj/tests/kernel_test.cpp:33-106,
// cycle_test.cpp:32-88, config_test.cpp) written against the drop-in C++
// layer include/sccl_b200.hpp -- i.e. reference-style code, B200 kernels.
#include <cmath>
#include <cstdio>
#include <vector>

#include "sccl_b200.hpp"

using namespace sccl_b200;

static int failures = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (!(cond)) {                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
      ++failures;                                                          \
    }                                                                      \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static HostTensor4 column_input(const std::vector<double>& ch) {
  HostTensor4 t(1, static_cast<std::int64_t>(ch.size()), 1, 1);
  for (std::int64_t c = 0; c < t.c(); ++c) t.at(0, c, 0, 0) = ch[static_cast<size_t>(c)];
  return t;
}

int main() {
  // config_test.cpp
  CHECK(Overlap::parse("50%").resolve(2) == 1);
  CHECK(Overlap::parse("33%").resolve(3) == 1);
  CHECK(throws<ArgumentError>([] { Overlap::parse("abc"); }));
  CHECK(throws<ConfigError>([] { scc_config_new(4, 4, 3, Overlap::channels(0), true); }));
  // cycle_test.cpp
  {
    const SccConfig cfg = scc_config_new(4, 4, 2, Overlap::channels(1), true);
    const ChannelCycle cyc = compute_channel_cycle(cfg);
    CHECK(cyc.cyclic_dist == 4);
    CHECK(window_of(cyc, 7) == window_of(cyc, 3));
    CHECK((covering_filters(cfg, cyc, 1) == std::vector<std::int64_t>{0, 1}));
    CHECK(throws<IndexError>([&] { covering_filters(cfg, cyc, 4); }));
    const SccConfig wide = scc_config_new(4, 8, 2, Overlap::channels(1), true);
    CHECK((covering_filters(wide, compute_channel_cycle(wide), 3) ==
           std::vector<std::int64_t>{2, 3, 6, 7}));
  }
  // kernel_test.cpp: forward worked example
  {
    const SccConfig cfg = scc_config_new(4, 4, 2, Overlap::channels(1), false);
    const SccWeights wts = scc_weights_filled(cfg, 1.0);
    const HostTensor4 out = scc_forward(column_input({1, 2, 3, 4}), wts, cfg);
    CHECK(out.at(0, 0, 0, 0) == 3.0 && out.at(0, 1, 0, 0) == 5.0);
    CHECK(out.at(0, 2, 0, 0) == 7.0 && out.at(0, 3, 0, 0) == 5.0);
    // backward input / params worked examples
    HostTensor4 ones(1, 4, 1, 1);
    for (std::int64_t c = 0; c < 4; ++c) ones.at(0, c, 0, 0) = 1.0;
    const HostTensor4 gi = scc_backward_input(ones, wts, cfg);
    for (std::int64_t c = 0; c < 4; ++c) CHECK(gi.at(0, c, 0, 0) == 2.0);
    const SccParamGradients gp = scc_backward_params(ones, column_input({1, 2, 3, 4}), cfg);
    CHECK(gp.grad_weight[0] == 1.0 && gp.grad_weight[1] == 2.0);
    CHECK(gp.grad_weight[6] == 4.0 && gp.grad_weight[7] == 1.0);
    // shape validation (kernel_test.cpp:243-253)
    CHECK(throws<ShapeError>([&] { scc_forward(HostTensor4(1, 6, 2, 2), wts, cfg); }));
  }
  // bias gradient (kernel_test.cpp:85-93)
  {
    const SccConfig cfg = scc_config_new(4, 4, 2, Overlap::channels(1), true);
    HostTensor4 x(1, 4, 2, 2), g(1, 4, 2, 2);
    for (std::int64_t i = 0; i < x.size(); ++i) {
      x.data()[i] = 0.5;
      g.data()[i] = 1.0;
    }
    const SccParamGradients p = scc_backward_params(g, x, cfg);
    for (double b : p.grad_bias) CHECK(b == 4.0);
  }
  std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
  return failures ? 1 : 0;
}
