// ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shell around the UNMODIFIED reference headers
// (/root/reference/proj/include/qft/*.hpp, included in place, never copied).
// oracle/Makefile compiles it with the reference's own flags
// (-O3 -ffp-contract=off, CMakeLists.txt:8-14) into oracle/_ref/libqft_ref.so.
//
// Uses:
//   * pin the C restatement (qft_oracle.c) against the real reference,
//   * generate the committed golden fixtures (tests/golden/make_golden.py),
//   * bench.py --impl reference / cpu_baseline: time qft::lion_step_quantized
//     on the host cores.
// The signatures are the qo_* ones from qft_oracle.c with a qr_ prefix.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <optional>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "qft/gradflow.hpp"
#include "qft/network.hpp"
#include "qft/optimizer.hpp"
#include "qft/quantize.hpp"

extern "C" void qo_synth(float* out, int64_t n, uint64_t seed, double sigma, double spike_p);

namespace {

thread_local std::string g_err;

constexpr int kEinval = -1;
constexpr int kErange = -2;

template <typename F>
int64_t guarded(F&& f) {
  try {
    return f();
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kEinval;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return kErange;
  }
}

qft::Tensor<float> to_tensor(const float* x, int rows, int cols) {
  qft::Tensor<float> t(rows, cols);
  std::memcpy(t.data(), x, sizeof(float) * t.size());
  return t;
}

qft::QuantizedTensor<float> to_qt(const uint8_t* codes, int rows, int cols, const float* scale,
                                  const int32_t* zp, int channels, int bit_width) {
  qft::QuantizedTensor<float> q;
  q.rows = rows;
  q.cols = cols;
  q.mode = qft::QuantMode::affine;
  q.data.assign(codes, codes + static_cast<size_t>(rows) * cols);
  q.params.scale.assign(scale, scale + channels);
  q.params.zero_point.assign(zp, zp + channels);
  q.params.bit_width = bit_width;
  return q;
}

qft::DenseSparseWeight<float> to_dsw(int rows, int cols, int bit_width, const uint8_t* codes,
                                     const float* scale, const int32_t* zp, const float* t_min,
                                     const float* t_max, const int32_t* row_ptr,
                                     const int32_t* col_idx, const float* values) {
  qft::DenseSparseWeight<float> d;
  d.dense = to_qt(codes, rows, cols, scale, zp, rows, bit_width);
  d.sparse.row_ptr.assign(row_ptr, row_ptr + rows + 1);
  const int nnz = row_ptr[rows];
  d.sparse.col_idx.assign(col_idx, col_idx + nnz);
  d.sparse.values.assign(values, values + nnz);
  d.t_min.assign(t_min, t_min + rows);
  d.t_max.assign(t_max, t_max + rows);
  return d;
}

int64_t store_dsw(const qft::DenseSparseWeight<float>& d, uint8_t* codes, float* scale,
                  int32_t* zp, int32_t* row_ptr, int32_t* col_idx, float* values,
                  int64_t capacity) {
  std::memcpy(codes, d.dense.data.data(), d.dense.data.size());
  std::memcpy(scale, d.dense.params.scale.data(), sizeof(float) * d.dense.params.scale.size());
  std::memcpy(zp, d.dense.params.zero_point.data(),
              sizeof(int32_t) * d.dense.params.zero_point.size());
  std::memcpy(row_ptr, d.sparse.row_ptr.data(), sizeof(int32_t) * d.sparse.row_ptr.size());
  const int64_t nnz = static_cast<int64_t>(d.sparse.nnz());
  const int64_t keep = std::min(nnz, capacity);
  if (keep > 0) {
    std::memcpy(col_idx, d.sparse.col_idx.data(), sizeof(int32_t) * keep);
    std::memcpy(values, d.sparse.values.data(), sizeof(float) * keep);
  }
  return nnz;
}

}  // namespace

extern "C" {

const char* qr_last_error(void) { return g_err.c_str(); }

int qr_channel_minmax(const float* x, int rows, int cols, float* mins, float* maxs) {
  return static_cast<int>(guarded([&] {
    auto [lo, hi] = qft::channel_minmax(to_tensor(x, rows, cols));
    std::copy(lo.begin(), lo.end(), mins);
    std::copy(hi.begin(), hi.end(), maxs);
    return int64_t{0};
  }));
}

int qr_affine_params_from_bounds(const float* mins, const float* maxs, int64_t n, int bit_width,
                                 float* scale, int32_t* zp) {
  return static_cast<int>(guarded([&] {
    std::vector<float> lo(mins, mins + n), hi(maxs, maxs + n);
    auto p = qft::affine_params_from_bounds(lo, hi, bit_width);
    std::copy(p.scale.begin(), p.scale.end(), scale);
    std::copy(p.zero_point.begin(), p.zero_point.end(), zp);
    return int64_t{0};
  }));
}

int qr_compute_affine_params(const float* x, int rows, int cols, int bit_width, float* scale,
                             int32_t* zp) {
  return static_cast<int>(guarded([&] {
    auto p = qft::compute_affine_params(to_tensor(x, rows, cols), bit_width, true);
    std::copy(p.scale.begin(), p.scale.end(), scale);
    std::copy(p.zero_point.begin(), p.zero_point.end(), zp);
    return int64_t{0};
  }));
}

int qr_quantize(const float* x, int rows, int cols, const float* scale, const int32_t* zp,
                int channels, int bit_width, uint8_t* codes) {
  return static_cast<int>(guarded([&] {
    qft::AffineParams<float> p;
    p.scale.assign(scale, scale + channels);
    p.zero_point.assign(zp, zp + channels);
    p.bit_width = bit_width;
    auto q = qft::quantize(to_tensor(x, rows, cols), p);
    std::memcpy(codes, q.data.data(), q.data.size());
    return int64_t{0};
  }));
}

int qr_quantize_state(const float* x, int rows, int cols, int bit_width, uint8_t* codes,
                      float* scale, int32_t* zp) {
  return static_cast<int>(guarded([&] {
    auto q = qft::quantize_state(to_tensor(x, rows, cols), bit_width, qft::QuantMode::affine);
    std::memcpy(codes, q.data.data(), q.data.size());
    std::copy(q.params.scale.begin(), q.params.scale.end(), scale);
    std::copy(q.params.zero_point.begin(), q.params.zero_point.end(), zp);
    return int64_t{0};
  }));
}

int qr_accumulate(const uint8_t* codes, const float* scale, const int32_t* zp, int rows,
                  int cols, int bit_width, const float* g, uint8_t* codes_out,
                  float* scale_out, int32_t* zp_out) {
  return static_cast<int>(guarded([&] {
    qft::QuantizedTensor<float> acc;
    acc.rows = rows;
    acc.cols = cols;
    acc.mode = qft::QuantMode::affine;
    acc.params.bit_width = bit_width;
    acc.params.scale.assign(scale, scale + rows);
    acc.params.zero_point.assign(zp, zp + rows);
    acc.data.assign(codes, codes + (size_t)rows * cols);
    auto q = qft::accumulate(acc, to_tensor(g, rows, cols));
    std::memcpy(codes_out, q.data.data(), q.data.size());
    std::copy(q.params.scale.begin(), q.params.scale.end(), scale_out);
    std::copy(q.params.zero_point.begin(), q.params.zero_point.end(), zp_out);
    return int64_t{0};
  }));
}

int qr_dequantize(const uint8_t* codes, int rows, int cols, const float* scale, const int32_t* zp,
                  int channels, float* out) {
  return static_cast<int>(guarded([&] {
    auto t = qft::dequantize(to_qt(codes, rows, cols, scale, zp, channels, 8));
    std::memcpy(out, t.data(), sizeof(float) * t.size());
    return int64_t{0};
  }));
}

int qr_outlier_thresholds(const float* w, int rows, int cols, double fraction, int kind,
                          float* t_min, float* t_max) {
  return static_cast<int>(guarded([&] {
    auto [lo, hi] = qft::compute_outlier_thresholds(to_tensor(w, rows, cols), fraction,
                                                    static_cast<qft::ThresholdKind>(kind));
    std::copy(lo.begin(), lo.end(), t_min);
    std::copy(hi.begin(), hi.end(), t_max);
    return int64_t{0};
  }));
}

int64_t qr_decompose_dense_sparse(const float* w, int rows, int cols, const float* t_min,
                                  const float* t_max, int bit_width, uint8_t* codes, float* scale,
                                  int32_t* zp, int32_t* row_ptr, int32_t* col_idx, float* values,
                                  int64_t capacity) {
  return guarded([&] {
    std::vector<float> lo(t_min, t_min + rows), hi(t_max, t_max + rows);
    auto d = qft::decompose_dense_sparse(to_tensor(w, rows, cols), lo, hi, bit_width);
    return store_dsw(d, codes, scale, zp, row_ptr, col_idx, values, capacity);
  });
}

int64_t qr_decompose_weight(const float* w, int rows, int cols, double fraction, int bit_width,
                            int kind, float* t_min, float* t_max, uint8_t* codes, float* scale,
                            int32_t* zp, int32_t* row_ptr, int32_t* col_idx, float* values,
                            int64_t capacity) {
  return guarded([&] {
    auto d = qft::decompose_weight(to_tensor(w, rows, cols), fraction, bit_width,
                                   qft::QuantMode::affine, static_cast<qft::ThresholdKind>(kind));
    std::copy(d.t_min.begin(), d.t_min.end(), t_min);
    std::copy(d.t_max.begin(), d.t_max.end(), t_max);
    return store_dsw(d, codes, scale, zp, row_ptr, col_idx, values, capacity);
  });
}

int qr_reconstruct(const uint8_t* codes, int rows, int cols, const float* scale,
                   const int32_t* zp, const int32_t* row_ptr, const int32_t* col_idx,
                   const float* values, float* out) {
  return static_cast<int>(guarded([&] {
    std::vector<float> dummy(rows, 0.0f);
    auto d = to_dsw(rows, cols, 8, codes, scale, zp, dummy.data(), dummy.data(), row_ptr, col_idx,
                    values);
    auto t = qft::reconstruct(d);
    std::memcpy(out, t.data(), sizeof(float) * t.size());
    return int64_t{0};
  }));
}

void qr_lion_apply(float* w, float* m, const float* g, int64_t n, float lr, float beta1,
                   float beta2, float wd) {
  qft::Tensor<float> tw(1, static_cast<int>(n)), tm(1, static_cast<int>(n)),
      tg(1, static_cast<int>(n));
  std::memcpy(tw.data(), w, sizeof(float) * n);
  std::memcpy(tm.data(), m, sizeof(float) * n);
  std::memcpy(tg.data(), g, sizeof(float) * n);
  qft::LionHyper<float> h{lr, beta1, beta2, wd};
  qft::detail::lion_apply(tw, tm, tg, h);
  std::memcpy(w, tw.data(), sizeof(float) * n);
  std::memcpy(m, tm.data(), sizeof(float) * n);
}

namespace {
// Wrap one layer into a 1-layer Model so the real lion_step_quantized runs.
qft::Model<float> one_layer_model(qft::DenseSparseWeight<float> w, int bit_width) {
  qft::ModelConfig cfg;
  cfg.layer_dims = {w.cols(), w.rows()};
  cfg.bit_width = bit_width;
  cfg.quant_mode = qft::QuantMode::affine;
  qft::QuantizedLinearLayer<float> layer;
  layer.index = 1;
  layer.weight = std::move(w);
  std::vector<qft::QuantizedLinearLayer<float>> layers;
  layers.push_back(std::move(layer));
  return qft::Model<float>::from_parts(cfg, std::move(layers));
}
}  // namespace

int64_t qr_lion_step_layer(int rows, int cols, int bit_width,
                           const uint8_t* g_codes, const float* g_scale, const int32_t* g_zp,
                           const uint8_t* m_codes, const float* m_scale, const int32_t* m_zp,
                           const uint8_t* w_codes, const float* w_scale, const int32_t* w_zp,
                           const float* t_min, const float* t_max, const int32_t* row_ptr,
                           const int32_t* col_idx, const float* values,
                           uint8_t* m_codes_out, float* m_scale_out, int32_t* m_zp_out,
                           uint8_t* w_codes_out, float* w_scale_out, int32_t* w_zp_out,
                           int32_t* row_ptr_out, int32_t* col_idx_out, float* values_out,
                           int64_t capacity, float lr, float beta1, float beta2, float wd,
                           float* trace_w_in, float* trace_g, float* trace_m_in,
                           float* trace_w_upd, float* trace_m_upd) {
  return guarded([&] {
    auto model = one_layer_model(to_dsw(rows, cols, bit_width, w_codes, w_scale, w_zp, t_min,
                                        t_max, row_ptr, col_idx, values),
                                 bit_width);
    qft::LionState<float> st;
    st.momentum.push_back(to_qt(m_codes, rows, cols, m_scale, m_zp, rows, bit_width));
    qft::GradientStack<float> stack;
    stack.push(1, to_qt(g_codes, rows, cols, g_scale, g_zp, rows, bit_width));
    qft::LionHyper<float> h{lr, beta1, beta2, wd};
    qft::LionStepTrace<float> trace;
    qft::lion_step_quantized(model, st, stack, h, &trace);
    const size_t n = static_cast<size_t>(rows) * cols;
    auto cp = [n](float* dst, const qft::Tensor<float>& t) {
      if (dst) std::memcpy(dst, t.data(), sizeof(float) * n);
    };
    cp(trace_w_in, trace.weights_in[0]);
    cp(trace_g, trace.gradients[0]);
    cp(trace_m_in, trace.momentum_in[0]);
    cp(trace_w_upd, trace.weights_updated[0]);
    cp(trace_m_upd, trace.momentum_updated[0]);
    const auto& m = st.momentum[0];
    std::memcpy(m_codes_out, m.data.data(), m.data.size());
    std::copy(m.params.scale.begin(), m.params.scale.end(), m_scale_out);
    std::copy(m.params.zero_point.begin(), m.params.zero_point.end(), m_zp_out);
    return store_dsw(model.layers()[0].weight, w_codes_out, w_scale_out, w_zp_out, row_ptr_out,
                     col_idx_out, values_out, capacity);
  });
}

// ---------------------------------------------------------------------------
// CPU timing harness (bench.py --impl reference, cpu_baseline).
// Holds reference-typed state for a list of layers and times
// qft::lion_step_quantized on them, one 1-layer model per tensor, the tensors
// spread over `threads` host threads (the reference itself is single-threaded;
// SPEC.md:431 allows the per-layer step to run in parallel).
// ---------------------------------------------------------------------------
struct QrBench {
  std::vector<qft::Model<float>> models;
  std::vector<qft::LionState<float>> states;
  std::vector<qft::QuantizedTensor<float>> grads;
  int bit_width = 8;
  qft::LionHyper<float> h;
};

void* qr_bench_create(int n_layers, const int* rows, const int* cols, uint64_t seed,
                      int bit_width, double fraction, float lr, float beta1, float beta2,
                      float wd, int threads) {
  auto* b = new QrBench;
  b->bit_width = bit_width;
  b->h = qft::LionHyper<float>{lr, beta1, beta2, wd};
  std::vector<std::optional<qft::Model<float>>> models(n_layers);
  std::vector<qft::QuantizedTensor<float>> grads(n_layers);
  threads = std::max(1, std::min(threads, n_layers));
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (int l = t; l < n_layers; l += threads) {
        qft::Tensor<float> w(rows[l], cols[l]);
        qo_synth(w.data(), static_cast<int64_t>(w.size()), seed + 2 * l, 0.02, 0.005);
        auto dsw = qft::decompose_weight(w, fraction, bit_width, qft::QuantMode::affine,
                                         qft::ThresholdKind::percentile);
        models[l].emplace(one_layer_model(std::move(dsw), bit_width));
        qft::Tensor<float> g(rows[l], cols[l]);
        qo_synth(g.data(), static_cast<int64_t>(g.size()), seed + 2 * l + 1, 1e-3, 0.0);
        grads[l] = qft::quantize_state(g, bit_width, qft::QuantMode::affine);
      }
    });
  }
  for (auto& th : pool) th.join();
  for (int l = 0; l < n_layers; ++l) {
    b->models.push_back(std::move(*models[l]));
    b->states.push_back(qft::LionState<float>::init(b->models.back()));
    b->grads.push_back(std::move(grads[l]));
  }
  return b;
}

// Runs one quantized Lion step over every layer; returns wall seconds.  The layers are
// handed out longest-first from a shared counter (dynamic scheduling), so `threads` host
// threads stay busy until the last few layers; the sample should hold several times
// more layers than threads.
double qr_bench_step(void* handle, int threads) {
  auto* b = static_cast<QrBench*>(handle);
  const int L = static_cast<int>(b->models.size());
  threads = std::max(1, std::min(threads, L));
  std::vector<int> order(L);
  for (int l = 0; l < L; ++l) order[l] = l;
  std::stable_sort(order.begin(), order.end(), [b](int x, int y) {
    return b->grads[x].size() > b->grads[y].size();
  });
  std::atomic<int> next{0};
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([b, &next, &order, L] {
      for (int k = next.fetch_add(1); k < L; k = next.fetch_add(1)) {
        const int l = order[k];
        qft::GradientStack<float> stack;
        stack.push(1, b->grads[l]);  // the stack entry the backward sink would hand over
        qft::lion_step_quantized(b->models[l], b->states[l], stack, b->h);
      }
    });
  }
  for (auto& th : pool) th.join();
  const auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

int64_t qr_bench_params(void* handle) {
  auto* b = static_cast<QrBench*>(handle);
  int64_t n = 0;
  for (auto& m : b->models) n += static_cast<int64_t>(m.layers()[0].weight.dense.data.size());
  return n;
}

void qr_bench_destroy(void* handle) { delete static_cast<QrBench*>(handle); }

}  // extern "C"
