// oracle/ckpt_golden.cpp -- TEST INFRASTRUCTURE (never shipped, never on the product path).
//
// Writes golden QFTC v1 checkpoints with the UNMODIFIED reference: the reference headers
// plus proj/src/checkpoint.cpp (save_checkpoint, checkpoint.cpp:100-140), compiled by
// oracle/Makefile target `ckpt` into oracle/_ref/ckpt_golden.  For each case it
//   1. builds a Model (Model::build, network.hpp:162-175) and LionState::init
//      (optimizer.hpp:57-66),
//   2. runs two lion_step_quantized steps (optimizer.hpp:86-120) on seeded quantized
//      gradients so the momentum has real codes -> writes <name>_a.qftc,
//   3. writes the third step's gradients (per layer: scale f32[rows], zero_point
//      i32[rows], codes u8[rows*cols]) -> <name>_g.bin,
//   4. runs that third step -> writes <name>_b.qftc.
// tests/golden/make_golden_ckpt.sh runs it; the files are committed under tests/golden.
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "qft/gradflow.hpp"
#include "qft/network.hpp"
#include "qft/optimizer.hpp"
#include "qft/quantize.hpp"
#include "qft/trainer.hpp"

namespace {

// splitmix64 -> uniform doubles -> Box-Muller normals (seeded, platform independent)
struct Rng {
  std::uint64_t s;
  std::uint64_t next() {
    std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return ((next() >> 11) + 0.5) * (1.0 / 9007199254740992.0); }
};

qft::GradientStack<float> grads(const qft::Model<float>& m, std::uint64_t seed, float sigma) {
  Rng rng{seed};
  qft::GradientStack<float> st;
  const int L = m.config().num_layers();
  std::vector<qft::QuantizedTensor<float>> qs;
  for (int l = 0; l < L; ++l) {
    const auto& w = m.layers()[l].weight;
    qft::Tensor<float> g(w.rows(), w.cols());
    for (int i = 0; i < w.rows() * w.cols(); ++i)
      g.data()[i] = static_cast<float>(sigma * (2.0 * rng.uniform() - 1.0));
    qs.push_back(qft::quantize_state(g, m.config().bit_width, m.config().quant_mode));
  }
  for (int l = L; l >= 1; --l) st.push(l, qs[l - 1]);  // FILO: layer 1 on top
  return st;
}

void write_grads(const qft::GradientStack<float>& st0, int L, const std::string& path) {
  qft::GradientStack<float> st = st0;
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  for (int l = 1; l <= L; ++l) {
    auto e = st.pop();
    const auto& q = e.grad;
    f.write(reinterpret_cast<const char*>(q.params.scale.data()), 4 * q.params.scale.size());
    f.write(reinterpret_cast<const char*>(q.params.zero_point.data()),
            4 * q.params.zero_point.size());
    f.write(reinterpret_cast<const char*>(q.data.data()), q.data.size());
  }
}

void run_case(const std::string& dir, const std::string& name, std::vector<int> dims, int bw,
              qft::ThresholdKind kind, qft::LossKind loss, std::vector<qft::Activation> junc,
              double frac, float lr, float wd, std::uint64_t seed) {
  qft::ModelConfig cfg;
  cfg.layer_dims = dims;
  cfg.junctions = junc;
  cfg.loss = loss;
  cfg.seed = seed;
  cfg.outlier_fraction = frac;
  cfg.bit_width = bw;
  cfg.threshold_kind = kind;
  cfg.init_outlier_fraction = 0.01;
  auto model = qft::Model<float>::build(cfg);
  auto state = qft::LionState<float>::init(model);
  qft::LionHyper<float> h;
  h.lr = lr;
  h.weight_decay = wd;
  for (int s = 0; s < 2; ++s) {
    auto st = grads(model, seed * 31 + s, 0.05f);
    qft::lion_step_quantized(model, state, st, h);
  }
  qft::save_checkpoint(model, state, dir + "/" + name + "_a.qftc");
  auto g3 = grads(model, seed * 31 + 7, 0.05f);
  write_grads(g3, cfg.num_layers(), dir + "/" + name + "_g.bin");
  qft::lion_step_quantized(model, state, g3, h);
  qft::save_checkpoint(model, state, dir + "/" + name + "_b.qftc");
  std::printf("%s: %d layers\n", name.c_str(), cfg.num_layers());
}

}  // namespace

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  using A = qft::Activation;
  run_case(dir, "ckpt_b8", {48, 64, 40, 17}, 8, qft::ThresholdKind::percentile,
           qft::LossKind::mse, {}, 0.01, 1e-3f, 0.0f, 11);
  run_case(dir, "ckpt_b4", {33, 96, 24}, 4, qft::ThresholdKind::range_fraction,
           qft::LossKind::softmax_cross_entropy, {A::none}, 0.0045, 2e-3f, 0.01f, 12);
  run_case(dir, "ckpt_b3", {16, 8}, 3, qft::ThresholdKind::percentile, qft::LossKind::mse, {},
           0.05, 5e-3f, 0.0f, 13);
  return 0;
}
