// oracle/dropin_test.cpp -- TEST INFRASTRUCTURE (built into oracle/_ref/, run by
// tests/test_gpu_dropin_cpp.py on the GPU box).
//
// The C++ drop-in proof: the reference's own types and functions (its headers, compiled
// unmodified from /root/reference/proj/include) side by side with qft_b200:: (the shim
// over the sm_100a C-ABI, include/qft_b200/qft.hpp), called with the SAME source text
// -- only the namespace differs.  Every output is compared byte for byte:
//   * quantizer surface: quantize_state (affine + pass-through), dequantize,
//     compute_outlier_thresholds, decompose_weight (both threshold kinds),
//     requantize_weight, reconstruct (quantize.hpp:189-338);
//   * lion_step_quantized on a qft::Model / LionState / GradientStack for several steps,
//     with and without a LionStepTrace (optimizer.hpp:85-120), at 8 and 4 bits, and the
//     pass-through model (test_optimizer.cpp:160-187);
//   * stack validation (test_optimizer.cpp:296-328): wrong depth, order, shape, momentum
//     count -> std::invalid_argument from both, and the same partially-updated state
//     when the bad entry sits below a good one.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "qft/gradflow.hpp"
#include "qft/network.hpp"
#include "qft/optimizer.hpp"
#include "qft/quantize.hpp"
#include "qft_b200/qft.hpp"

namespace {

int g_fail = 0;
int g_checks = 0;

void expect(bool ok, const std::string& what) {
  ++g_checks;
  if (!ok) {
    ++g_fail;
    std::fprintf(stderr, "FAIL: %s\n", what.c_str());
  }
}

template <class A>
bool same_bytes(const std::vector<A>& a, const std::vector<A>& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), sizeof(A) * a.size()) == 0);
}

bool same_tensor(const qft::Tensor<float>& a, const qft::Tensor<float>& b) {
  return a.rows() == b.rows() && a.cols() == b.cols() &&
         std::memcmp(a.data(), b.data(), sizeof(float) * a.size()) == 0;
}

bool same_qt(const qft::QuantizedTensor<float>& a, const qft::QuantizedTensor<float>& b) {
  return a.rows == b.rows && a.cols == b.cols && a.mode == b.mode && same_bytes(a.data, b.data) &&
         same_bytes(a.raw, b.raw) && same_bytes(a.params.scale, b.params.scale) &&
         same_bytes(a.params.zero_point, b.params.zero_point) &&
         (a.mode == qft::QuantMode::passthrough || a.params.bit_width == b.params.bit_width);
}

bool same_dsw(const qft::DenseSparseWeight<float>& a, const qft::DenseSparseWeight<float>& b) {
  return same_qt(a.dense, b.dense) && same_bytes(a.sparse.row_ptr, b.sparse.row_ptr) &&
         same_bytes(a.sparse.col_idx, b.sparse.col_idx) &&
         same_bytes(a.sparse.values, b.sparse.values) && same_bytes(a.t_min, b.t_min) &&
         same_bytes(a.t_max, b.t_max) && a.outlier_fraction == b.outlier_fraction;
}

bool same_model(const qft::Model<float>& a, const qft::Model<float>& b) {
  if (a.layers().size() != b.layers().size()) return false;
  for (size_t l = 0; l < a.layers().size(); ++l)
    if (!same_dsw(a.layers()[l].weight, b.layers()[l].weight)) return false;
  return true;
}

bool same_state(const qft::LionState<float>& a, const qft::LionState<float>& b) {
  if (a.momentum.size() != b.momentum.size()) return false;
  for (size_t l = 0; l < a.momentum.size(); ++l)
    if (!same_qt(a.momentum[l], b.momentum[l])) return false;
  return true;
}

bool same_trace(const qft::LionStepTrace<float>& a, const qft::LionStepTrace<float>& b) {
  auto eq = [](const std::vector<qft::Tensor<float>>& x, const std::vector<qft::Tensor<float>>& y) {
    if (x.size() != y.size()) return false;
    for (size_t i = 0; i < x.size(); ++i)
      if (!same_tensor(x[i], y[i])) return false;
    return true;
  };
  return eq(a.weights_in, b.weights_in) && eq(a.gradients, b.gradients) &&
         eq(a.momentum_in, b.momentum_in) && eq(a.weights_updated, b.weights_updated) &&
         eq(a.momentum_updated, b.momentum_updated);
}

// explicit generator (std::*_distribution output is implementation-defined)
struct Rng {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
};

qft::Tensor<float> random_tensor(int r, int c, uint64_t seed, double scale, double spike_p) {
  Rng g{seed};
  qft::Tensor<float> t(r, c);
  for (size_t i = 0; i < t.size(); ++i) {
    double v = (g.uniform() * 2.0 - 1.0) * scale;
    if (g.uniform() < spike_p) v *= 200.0;
    t.data()[i] = static_cast<float>(v);
  }
  return t;
}

qft::GradientStack<float> make_stack(const qft::Model<float>& m, uint64_t seed, double gscale) {
  qft::GradientStack<float> st;
  const int L = m.config().num_layers();
  for (int l = L; l >= 1; --l) {  // backward pushes L..1 (gradflow.hpp:15-16)
    const auto& w = m.layers()[l - 1].weight;
    st.push(l, qft::quantize_state(random_tensor(w.rows(), w.cols(), seed + l, gscale, 0.0),
                                   m.config().bit_width, m.config().quant_mode));
  }
  return st;
}

void quantizer_surface() {
  for (int bw : {2, 3, 4, 8}) {
    const auto x = random_tensor(37, 129, 11 + bw, 1.0, 0.01);
    const auto a = qft::quantize_state(x, bw, qft::QuantMode::affine);
    const auto b = qft_b200::quantize_state(x, bw, qft::QuantMode::affine);
    expect(same_qt(a, b), "quantize_state affine b" + std::to_string(bw));
    expect(same_tensor(qft::dequantize(a), qft_b200::dequantize(b)),
           "dequantize b" + std::to_string(bw));
  }
  {
    const auto x = random_tensor(5, 7, 3, 1.0, 0.0);
    const auto a = qft::quantize_state(x, 8, qft::QuantMode::passthrough);
    const auto b = qft_b200::quantize_state(x, 8, qft::QuantMode::passthrough);
    expect(same_qt(a, b), "quantize_state passthrough");
    expect(same_tensor(qft::dequantize(a), qft_b200::dequantize(b)), "dequantize passthrough");
  }
  for (auto kind : {qft::ThresholdKind::percentile, qft::ThresholdKind::range_fraction}) {
    for (int bw : {3, 8}) {
      const std::string tag = std::string(kind == qft::ThresholdKind::percentile ? "pct" : "rf") +
                              " b" + std::to_string(bw);
      const auto w = random_tensor(48, 300, 21 + bw, 0.02, 0.005);
      const auto ta = qft::compute_outlier_thresholds(w, 0.01, kind);
      const auto tb = qft_b200::compute_outlier_thresholds(w, 0.01, kind);
      expect(same_bytes(ta.first, tb.first) && same_bytes(ta.second, tb.second),
             "compute_outlier_thresholds " + tag);
      auto da = qft::decompose_weight(w, 0.01, bw, qft::QuantMode::affine, kind);
      auto db = qft_b200::decompose_weight(w, 0.01, bw, qft::QuantMode::affine, kind);
      expect(same_dsw(da, db), "decompose_weight " + tag);
      expect(same_tensor(qft::reconstruct(da), qft_b200::reconstruct(db)), "reconstruct " + tag);
      auto w2 = qft::reconstruct(da);
      for (size_t i = 0; i < w2.size(); i += 7) w2.data()[i] *= 1.01f;
      qft::requantize_weight(da, w2, bw);
      qft_b200::requantize_weight(db, w2, bw);
      expect(same_dsw(da, db), "requantize_weight " + tag);
    }
  }
  {
    const auto w = random_tensor(6, 9, 5, 1.0, 0.0);
    const auto da = qft::decompose_weight(w, 0.01, 8, qft::QuantMode::passthrough);
    const auto db = qft_b200::decompose_weight(w, 0.01, 8, qft::QuantMode::passthrough);
    expect(same_dsw(da, db), "decompose_weight passthrough");
  }
  // error types
  auto throws_inv = [](auto&& f) {
    try {
      f();
    } catch (const std::invalid_argument&) {
      return true;
    } catch (...) {
      return false;
    }
    return false;
  };
  const auto x = random_tensor(3, 4, 1, 1.0, 0.0);
  expect(throws_inv([&] { qft::quantize_state(x, 9, qft::QuantMode::affine); }) &&
             throws_inv([&] { qft_b200::quantize_state(x, 9, qft::QuantMode::affine); }),
         "bit width 9 -> invalid_argument");
  expect(throws_inv([&] { qft::compute_outlier_thresholds(x, 0.5); }) &&
             throws_inv([&] { qft_b200::compute_outlier_thresholds(x, 0.5); }),
         "fraction 0.5 -> invalid_argument");
}

qft::ModelConfig config(int bw, qft::QuantMode mode, uint64_t seed) {
  qft::ModelConfig cfg;
  cfg.layer_dims = {96, 256, 200, 64};
  cfg.seed = seed;
  cfg.outlier_fraction = 0.01;
  cfg.bit_width = bw;
  cfg.quant_mode = mode;
  cfg.init_outlier_fraction = 0.005;
  return cfg;
}

void lion_steps(int bw, float lr, float wd, bool with_trace) {
  const std::string tag = "b" + std::to_string(bw) + " lr " + std::to_string(lr) + " wd " +
                          std::to_string(wd) + (with_trace ? " trace" : "");
  auto a = qft::Model<float>::build(config(bw, qft::QuantMode::affine, 7 + bw));
  auto b = a;
  auto sa = qft::LionState<float>::init(a);
  auto sb = qft::LionState<float>::init(b);
  qft::LionHyper<float> h;
  h.lr = lr;
  h.weight_decay = wd;
  for (int step = 0; step < 6; ++step) {
    auto ka = make_stack(a, 1000 + 10 * step, 1e-2);
    auto kb = ka;
    if (with_trace) {
      qft::LionStepTrace<float> ta, tb;
      qft::lion_step_quantized(a, sa, ka, h, &ta);
      qft_b200::lion_step_quantized(b, sb, kb, h, &tb);
      expect(same_trace(ta, tb), tag + " step " + std::to_string(step) + " trace");
    } else {
      qft::lion_step_quantized(a, sa, ka, h);
      qft_b200::lion_step_quantized(b, sb, kb, h);
    }
    expect(ka.size() == 0 && kb.size() == 0, tag + " stacks drained");
    expect(same_model(a, b), tag + " step " + std::to_string(step) + " weights");
    expect(same_state(sa, sb), tag + " step " + std::to_string(step) + " momentum");
  }
}

void passthrough_steps() {
  auto a = qft::Model<float>::build(config(8, qft::QuantMode::passthrough, 5));
  auto b = a;
  auto sa = qft::LionState<float>::init(a);
  auto sb = qft::LionState<float>::init(b);
  qft::LionHyper<float> h;
  h.lr = 3e-3f;
  h.weight_decay = 0.01f;
  for (int step = 0; step < 5; ++step) {
    auto ka = make_stack(a, 50 + step, 1.0);
    auto kb = ka;
    qft::LionStepTrace<float> ta, tb;
    qft::lion_step_quantized(a, sa, ka, h, &ta);
    qft_b200::lion_step_quantized(b, sb, kb, h, &tb);
    expect(same_model(a, b) && same_state(sa, sb), "passthrough step " + std::to_string(step));
    expect(same_trace(ta, tb), "passthrough trace " + std::to_string(step));
  }
}

// test_optimizer.cpp:296-328, run through both implementations
void stack_validation() {
  qft::ModelConfig cfg;
  cfg.layer_dims = {4, 6, 2};
  cfg.seed = 10;
  const auto model0 = qft::Model<float>::build(cfg);
  const auto st0 = qft::LionState<float>::init(model0);
  qft::LionHyper<float> h;
  h.lr = 1e-2f;
  auto q = [](int r, int c, uint64_t s) {
    return qft::quantize_state(random_tensor(r, c, s, 1.0, 0.0), 8, qft::QuantMode::affine);
  };
  struct Case {
    const char* name;
    std::vector<std::pair<int, std::pair<int, int>>> pushes;  // (layer, (rows, cols))
    bool drop_momentum;
  };
  const std::vector<Case> cases = {
      {"wrong depth", {{1, {6, 4}}}, false},
      {"wrong order", {{1, {6, 4}}, {2, {2, 6}}}, false},
      {"wrong shape", {{2, {2, 6}}, {1, {5, 5}}}, false},
      {"momentum count mismatch", {{2, {2, 6}}, {1, {6, 4}}}, true},
      {"bad shape below a good layer", {{2, {3, 3}}, {1, {6, 4}}}, false},
  };
  for (const auto& c : cases) {
    auto ma = model0, mb = model0;
    auto sa = st0, sb = st0;
    if (c.drop_momentum) {
      sa.momentum.pop_back();
      sb.momentum.pop_back();
    }
    qft::GradientStack<float> ka, kb;
    uint64_t s = 77;
    for (const auto& p : c.pushes) {
      auto g = q(p.second.first, p.second.second, s++);
      ka.push(p.first, g);
      kb.push(p.first, g);
    }
    bool ta = false, tb = false;
    try {
      qft::lion_step_quantized(ma, sa, ka, h);
    } catch (const std::invalid_argument&) {
      ta = true;
    }
    try {
      qft_b200::lion_step_quantized(mb, sb, kb, h);
    } catch (const std::invalid_argument&) {
      tb = true;
    }
    expect(ta && tb, std::string(c.name) + ": both throw std::invalid_argument");
    expect(ka.size() == kb.size(), std::string(c.name) + ": same stack depth after the throw");
    expect(same_model(ma, mb) && same_state(sa, sb),
           std::string(c.name) + ": same (partially updated) state after the throw");
  }
}

}  // namespace

int main() {
  try {
    quantizer_surface();
    for (bool tr : {false, true}) {
      lion_steps(8, 2e-3f, 0.0f, tr);
      lion_steps(8, 2e-5f, 0.01f, tr);
      lion_steps(4, 1e-3f, 0.01f, tr);
    }
    passthrough_steps();
    stack_validation();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "FAIL: unexpected exception: %s\n", e.what());
    return 2;
  }
  std::printf("dropin %s: %d checks, %d failed\n", g_fail ? "FAILED" : "ok", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
