// Training driver over the reference's own model / dataset / SGD code
// (proj/core/src/model.cpp, dataset.cpp, train.cpp), mirroring `scc train`
// (tools/scc/main.cpp:164-190, whose CLI11 dependency is absent here).
// Linked twice by the Makefile: with the reference's kernel.cpp (CPU, fp64)
// and with kernel_b200.cpp (every SCC layer on the B200 through the C ABI).
//
//   usage: train_main MODEL.json EPOCHS LR BATCH SAMPLES CLASSES SPATIAL [SEED]
//          prints "epoch E loss L accuracy A" per epoch;
//          train_main MODEL.json grad BATCH SPATIAL [SEED]
//          one forward + backward of the whole network (Network::forward /
//          Network::backward, model.cpp:243-304, :306-380) on seeded N(0,1)
//          images, printing the logits and every stage's parameter gradients
//          as one JSON object.
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>
#include <variant>
#include <vector>

#include "sccl/dataset.hpp"
#include "sccl/rng.hpp"
#include "sccl/model.hpp"
#include "sccl/train.hpp"

static void print_vec(const char* name, const std::vector<double>& v, bool comma) {
  std::printf("\"%s\": [", name);
  for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
  std::printf("]%s", comma ? ", " : "");
}

static int run_grad(const std::string& model, std::int64_t batch, std::int64_t spatial, std::uint64_t seed) {
  const sccl::ModelSpec spec = sccl::parse_model_spec_file(model);
  const sccl::Network net = sccl::build_network(spec, seed);
  sccl::Tensor4 x(batch, net.input_channels(), spatial, spatial);
  sccl::Rng rng(seed + 1000);
  for (std::int64_t i = 0; i < x.size(); ++i) x.data()[i] = rng.uniform(-1.0, 1.0);
  sccl::NetworkTrace trace;
  const std::vector<double> logits = net.forward(x, &trace);
  std::vector<std::int64_t> labels(static_cast<std::size_t>(batch));
  for (std::int64_t i = 0; i < batch; ++i) labels[static_cast<std::size_t>(i)] = i % net.classes();
  std::vector<double> grad;
  const double loss = sccl::softmax_cross_entropy(logits, labels, net.classes(), &grad);
  const sccl::NetworkGradients g = net.backward(trace, grad);
  std::printf("{\"loss\": %.17g, ", loss);
  print_vec("logits", logits, true);
  std::printf("\"stages\": [");
  for (std::size_t i = 0; i < g.stages.size(); ++i) {
    const bool scc = std::holds_alternative<sccl::SccStage>(net.stages[i].op);
    std::printf("%s{\"scc\": %s, ", i ? ", " : "", scc ? "true" : "false");
    print_vec("weight", g.stages[i].weight, true);
    print_vec("bias", g.stages[i].bias, false);
    std::printf("}");
  }
  std::printf("], ");
  print_vec("head_weight", g.head.weight, false);
  std::printf("}\n");
  return 0;
}

int main(int argc, char** argv) {
  if (argc >= 5 && std::string(argv[2]) == "grad") {
    try {
      return run_grad(argv[1], std::atoll(argv[3]), std::atoll(argv[4]),
                      argc > 5 ? std::strtoull(argv[5], nullptr, 10) : 1);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 1;
    }
  }
  if (argc < 8) {
    std::fprintf(stderr, "usage: %s MODEL.json EPOCHS LR BATCH SAMPLES CLASSES SPATIAL [SEED]\n", argv[0]);
    return 2;
  }
  try {
    const std::string model = argv[1];
    const std::int64_t epochs = std::atoll(argv[2]);
    const double lr = std::atof(argv[3]);
    const std::int64_t batch = std::atoll(argv[4]);
    const std::int64_t samples = std::atoll(argv[5]);
    const std::int64_t classes = std::atoll(argv[6]);
    const std::int64_t spatial = std::atoll(argv[7]);
    const std::uint64_t seed = argc > 8 ? std::strtoull(argv[8], nullptr, 10) : 1;
    const sccl::ModelSpec spec = sccl::parse_model_spec_file(model);
    sccl::Network net = sccl::build_network(spec, seed);
    sccl::LabeledDataset data =
        sccl::synth_dataset(seed, samples, classes, net.input_channels(), spatial);
    sccl::TrainConfig cfg;
    cfg.epochs = epochs;
    cfg.batch_size = batch;
    cfg.learning_rate = lr;
    cfg.seed = seed;
    for (const sccl::EpochStats& e : sccl::train(net, data, cfg)) {
      std::printf("epoch %" PRId64 " loss %.9f accuracy %.6f\n", e.epoch, e.loss, e.accuracy);
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
