// qft_b200/qft.hpp -- C++ drop-in shim over the C-ABI (include/qft_b200.h).
//
// Reproduces the reference's quantizer/optimizer entry points for T = float
// (/root/reference/proj/include/qft/{quantize,optimizer}.hpp) with the SAME signatures
// over the reference's own types, so a caller swaps the namespace and nothing else:
//
//   auto q  = qft_b200::quantize_state(x, 8, qft::QuantMode::affine);   // quantize.hpp:189
//   auto x2 = qft_b200::dequantize(q);                                   // quantize.hpp:195
//   auto w  = qft_b200::decompose_weight(t, 0.01, 8, qft::QuantMode::affine);  // :301
//   qft_b200::requantize_weight(w, t2, 8);                               // quantize.hpp:318
//   qft_b200::lion_step_quantized(model, state, stack, hyper, &trace);   // optimizer.hpp:85
//
// The reference's types are only forward-declared here; their definitions come from the
// caller's own `#include "qft/..."` (the functions are templates, instantiated where the
// types are complete).  Each call moves its host arrays to the device, runs the sm_100a
// kernels and copies the results back -- the reference API is host-resident.  The
// whole-model device-resident step is qftc_plan_* (C) / QftModelState (Python).
//
// qft_b200::generic holds the same operations over any host types with the reference's
// public field names (used by the pybind drop-in, which has no reference headers).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "qft_b200.h"

// the reference's types (definitions: qft/tensor.hpp, quantize.hpp, network.hpp, gradflow.hpp,
// optimizer.hpp)
namespace qft {
template <typename T> class Tensor;
template <typename T> struct QuantizedTensor;
template <typename T> struct DenseSparseWeight;
enum class QuantMode : std::uint8_t;
enum class ThresholdKind : std::uint8_t;
template <typename T> class Model;
template <typename T> struct LionState;
template <typename T> class GradientStack;
template <typename T> struct LionHyper;
template <typename T> struct LionStepTrace;
}  // namespace qft

namespace qft_b200 {

inline void check(int rc) {
  switch (rc) {
    case QFTC_OK: return;
    case QFTC_EINVAL: throw std::invalid_argument(qftc_last_error());
    case QFTC_ERANGE: throw std::out_of_range(qftc_last_error());
    case QFTC_EOVERFLOW: throw std::length_error(qftc_last_error());
    default: throw std::runtime_error(qftc_last_error());
  }
}

// RAII device buffer (stream 0)
template <class T>
class dbuf {
 public:
  dbuf() = default;
  explicit dbuf(size_t n) : n_(n) { check(qftc_device_alloc(reinterpret_cast<void**>(&p_), bytes())); }
  dbuf(const T* host, size_t n) : dbuf(n) { up(host, n); }
  explicit dbuf(const std::vector<T>& v) : dbuf(v.data(), v.size()) {}
  ~dbuf() { if (p_) qftc_device_free(p_); }
  dbuf(const dbuf&) = delete;
  dbuf& operator=(const dbuf&) = delete;
  dbuf(dbuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return (n_ ? n_ : 1) * sizeof(T); }
  void up(const T* h, size_t n) {
    if (n) check(qftc_copy_to_device(p_, h, n * sizeof(T), nullptr));
  }
  void down(T* h, size_t n) const {
    if (n) check(qftc_copy_to_host(h, p_, n * sizeof(T), nullptr));
    check(qftc_stream_synchronize(nullptr));
  }
  std::vector<T> vec(size_t n) const {
    std::vector<T> v(n);
    if (n) down(v.data(), n);
    return v;
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

namespace detail {
constexpr int kAffine = 0;       // QuantMode::affine (quantize.hpp:17)
constexpr int kPassthrough = 1;  // QuantMode::passthrough

template <class QT>
void fill_qt(QT& q, int rows, int cols, std::vector<uint8_t> data, std::vector<float> s,
             std::vector<int32_t> z, int bw) {
  q.rows = rows;
  q.cols = cols;
  q.mode = static_cast<decltype(q.mode)>(kAffine);
  q.data = std::move(data);
  q.params.scale = std::move(s);
  q.params.zero_point = std::move(z);
  q.params.bit_width = bw;
}

template <class TensorOut>
TensorOut tensor_from_device(const dbuf<float>& d, int r, int c) {
  TensorOut out(r, c);
  d.down(out.data(), static_cast<size_t>(r) * c);
  return out;
}

template <class TensorOut>
TensorOut tensor_from_host(const std::vector<float>& v, int r, int c) {
  TensorOut out(r, c);
  for (size_t i = 0; i < v.size(); ++i) out.data()[i] = v[i];
  return out;
}

struct NoTrace {  // lion_step_quantized without a trace
  template <class Tn> void push(Tn&&) {}
};
}  // namespace detail

// ============================================================================ generic
// The operations over any host types with the reference's public field names
// (Tensor::rows()/cols()/data(); QuantizedTensor::{rows,cols,mode,data,raw,params};
// AffineParams::{scale,zero_point,bit_width}; SparseOutliers::{row_ptr,col_idx,values};
// DenseSparseWeight::{dense,sparse,t_min,t_max,outlier_fraction}).  Affine mode.
namespace generic {

// quantize.hpp:189-193 (affine)
template <class QT, class TensorT>
QT quantize_state(const TensorT& x, int bit_width) {
  const int r = x.rows(), c = x.cols();
  if (r <= 0 || c <= 0) throw std::invalid_argument("compute_affine_params: empty tensor");
  const size_t n = static_cast<size_t>(r) * c;
  dbuf<float> dx(x.data(), n);
  dbuf<uint8_t> dq(n);
  dbuf<float> ds(r);
  dbuf<int32_t> dz(r);
  check(qftc_quantize_state(dx.get(), r, c, bit_width, dq.get(), ds.get(), dz.get(), 1, nullptr));
  QT q;
  detail::fill_qt(q, r, c, dq.vec(n), ds.vec(r), dz.vec(r), bit_width);
  return q;
}

// quantize.hpp:195-212
template <class TensorOut, class QT>
TensorOut dequantize(const QT& q) {
  if (q.rows <= 0 || q.cols <= 0) throw std::invalid_argument("dequantize: empty tensor");
  TensorOut out(q.rows, q.cols);
  const size_t n = static_cast<size_t>(q.rows) * q.cols;
  if (static_cast<int>(q.mode) == detail::kPassthrough) {
    for (size_t i = 0; i < q.raw.size(); ++i) out.data()[i] = q.raw[i];
    return out;
  }
  dbuf<uint8_t> dq(q.data);
  dbuf<float> ds(q.params.scale);
  dbuf<int32_t> dz(q.params.zero_point);
  dbuf<float> dout(n);
  check(qftc_dequantize(dq.get(), q.rows, q.cols, ds.get(), dz.get(),
                        static_cast<int>(q.params.scale.size()), dout.get(), nullptr));
  dout.down(out.data(), n);
  return out;
}

// quantize.hpp:216-247
template <class TensorT>
std::pair<std::vector<float>, std::vector<float>> compute_outlier_thresholds(
    const TensorT& w, double fraction, int kind = QFTC_PERCENTILE) {
  const int r = w.rows(), c = w.cols();
  if (r <= 0 || c <= 0) throw std::invalid_argument("compute_outlier_thresholds: empty tensor");
  dbuf<float> dw(w.data(), static_cast<size_t>(r) * c);
  dbuf<float> lo(r), hi(r);
  check(qftc_outlier_thresholds(dw.get(), r, c, fraction, kind, lo.get(), hi.get(), nullptr));
  return {lo.vec(r), hi.vec(r)};
}

// quantize.hpp:253-290
template <class DSW, class TensorT>
DSW decompose_dense_sparse(const TensorT& w, const std::vector<float>& t_min,
                           const std::vector<float>& t_max, int bit_width = 8) {
  const int r = w.rows(), c = w.cols();
  if (static_cast<int>(t_min.size()) != r || static_cast<int>(t_max.size()) != r)
    throw std::invalid_argument("decompose_dense_sparse: threshold count must equal rows");
  const size_t n = static_cast<size_t>(r) * c;
  dbuf<float> dw(w.data(), n), dlo(t_min), dhi(t_max);
  dbuf<uint8_t> dq(n);
  dbuf<float> ds(r);
  dbuf<int32_t> dz(r), drp(r + 1);
  int64_t cap = static_cast<int64_t>(n / 32 + 64), nnz = 0;
  for (;;) {
    dbuf<int32_t> dcol(cap);
    dbuf<float> dval(cap);
    const int rc = qftc_decompose_dense_sparse(dw.get(), r, c, dlo.get(), dhi.get(), bit_width,
                                               dq.get(), ds.get(), dz.get(), drp.get(),
                                               dcol.get(), dval.get(), cap, &nnz, nullptr);
    if (rc == QFTC_EOVERFLOW) {
      cap = nnz;
      continue;
    }
    check(rc);
    DSW out;
    detail::fill_qt(out.dense, r, c, dq.vec(n), ds.vec(r), dz.vec(r), bit_width);
    out.sparse.row_ptr = drp.vec(r + 1);
    out.sparse.col_idx = dcol.vec(static_cast<size_t>(nnz));
    out.sparse.values = dval.vec(static_cast<size_t>(nnz));
    out.t_min = t_min;
    out.t_max = t_max;
    return out;
  }
}

// quantize.hpp:301-314 (affine)
template <class DSW, class TensorT>
DSW decompose_weight(const TensorT& w, double fraction, int bit_width,
                     int kind = QFTC_PERCENTILE) {
  auto th = compute_outlier_thresholds(w, fraction, kind);
  DSW out = decompose_dense_sparse<DSW>(w, th.first, th.second, bit_width);
  out.outlier_fraction = fraction;
  return out;
}

// quantize.hpp:331-338
template <class TensorOut, class DSW>
TensorOut reconstruct(const DSW& d) {
  const int r = d.dense.rows, c = d.dense.cols;
  const size_t n = static_cast<size_t>(r) * c;
  if (static_cast<int>(d.dense.mode) == detail::kPassthrough) {
    TensorOut out(r, c);
    for (size_t i = 0; i < d.dense.raw.size(); ++i) out.data()[i] = d.dense.raw[i];
    return out;
  }
  TensorOut out(r, c);
  dbuf<uint8_t> dq(d.dense.data);
  dbuf<float> ds(d.dense.params.scale);
  dbuf<int32_t> dz(d.dense.params.zero_point), drp(d.sparse.row_ptr), dcol(d.sparse.col_idx);
  dbuf<float> dval(d.sparse.values), dout(n);
  check(qftc_reconstruct(dq.get(), r, c, ds.get(), dz.get(), drp.get(), dcol.get(), dval.get(),
                         dout.get(), nullptr));
  dout.down(out.data(), n);
  return out;
}

}  // namespace generic

// ============================================================================ reference
// signatures (T = float; the reference's double instantiation stays on its CPU code)

// quantize.hpp:189-193: fresh channel-wise params + quantize (affine), identity
// (pass-through)
template <typename T>
qft::QuantizedTensor<T> quantize_state(const qft::Tensor<T>& x, int bit_width,
                                       qft::QuantMode mode) {
  static_assert(std::is_same<T, float>::value, "the B200 path is fp32 (T = float)");
  if (static_cast<int>(mode) == detail::kPassthrough) {
    qft::QuantizedTensor<T> out;  // quantize_passthrough, quantize.hpp:177-185
    out.rows = x.rows();
    out.cols = x.cols();
    out.mode = mode;
    out.raw.assign(x.data(), x.data() + x.size());
    return out;
  }
  if (bit_width < 2 || bit_width > 8)  // require_bit_width precedes the empty check
    throw std::invalid_argument("bit width must be in [2, 8], got " + std::to_string(bit_width));
  return generic::quantize_state<qft::QuantizedTensor<T>>(x, bit_width);
}

// quantize.hpp:195-212
template <typename T>
qft::Tensor<T> dequantize(const qft::QuantizedTensor<T>& q) {
  static_assert(std::is_same<T, float>::value, "the B200 path is fp32 (T = float)");
  return generic::dequantize<qft::Tensor<T>>(q);
}

// quantize.hpp:216-247
template <typename T, typename KindT = qft::ThresholdKind>
std::pair<std::vector<T>, std::vector<T>> compute_outlier_thresholds(
    const qft::Tensor<T>& w, double fraction, KindT kind = static_cast<KindT>(0)) {
  static_assert(std::is_same<T, float>::value, "the B200 path is fp32 (T = float)");
  return generic::compute_outlier_thresholds(w, fraction, static_cast<int>(kind));
}

// quantize.hpp:253-290
template <typename T>
qft::DenseSparseWeight<T> decompose_dense_sparse(const qft::Tensor<T>& w,
                                                 const std::vector<T>& t_min,
                                                 const std::vector<T>& t_max, int bit_width = 8) {
  static_assert(std::is_same<T, float>::value, "the B200 path is fp32 (T = float)");
  return generic::decompose_dense_sparse<qft::DenseSparseWeight<T>>(w, t_min, t_max, bit_width);
}

// quantize.hpp:292-299 (make_passthrough_weight)
template <typename T>
qft::DenseSparseWeight<T> make_passthrough_weight(const qft::Tensor<T>& w) {
  qft::DenseSparseWeight<T> out;
  out.dense = qft_b200::quantize_state(w, 8, static_cast<qft::QuantMode>(detail::kPassthrough));
  out.sparse.row_ptr.assign(static_cast<size_t>(w.rows()) + 1, 0);
  return out;
}

// quantize.hpp:301-314
template <typename T, typename KindT = qft::ThresholdKind>
qft::DenseSparseWeight<T> decompose_weight(const qft::Tensor<T>& w, double fraction,
                                           int bit_width, qft::QuantMode mode,
                                           KindT kind = static_cast<KindT>(0)) {
  static_assert(std::is_same<T, float>::value, "the B200 path is fp32 (T = float)");
  if (static_cast<int>(mode) == detail::kPassthrough) {
    auto out = qft_b200::make_passthrough_weight(w);
    out.outlier_fraction = fraction;
    return out;
  }
  return generic::decompose_weight<qft::DenseSparseWeight<T>>(w, fraction, bit_width,
                                                              static_cast<int>(kind));
}

// quantize.hpp:318-329: against the cached thresholds (dense params stay fixed)
template <typename T>
void requantize_weight(qft::DenseSparseWeight<T>& dsw, const qft::Tensor<T>& w_fp, int bit_width) {
  if (static_cast<int>(dsw.dense.mode) == detail::kPassthrough) {
    const double fraction = dsw.outlier_fraction;
    dsw = qft_b200::make_passthrough_weight(w_fp);
    dsw.outlier_fraction = fraction;
    return;
  }
  auto next = qft_b200::decompose_dense_sparse(w_fp, dsw.t_min, dsw.t_max, bit_width);
  next.outlier_fraction = dsw.outlier_fraction;
  dsw = std::move(next);
}

// quantize.hpp:331-338
template <typename T>
qft::Tensor<T> reconstruct(const qft::DenseSparseWeight<T>& d) {
  static_assert(std::is_same<T, float>::value, "the B200 path is fp32 (T = float)");
  return generic::reconstruct<qft::Tensor<T>>(d);
}

// optimizer.hpp:85-120.  Same validation, same order, same exception types and the same
// partial state on a throw: layer li is popped, validated and updated before layer li+1
// is popped (a malformed entry at li leaves layers 1..li-1 updated, as the reference
// does).  Each layer's update is ONE fused kernel (qftc_lion_step: dequant g, m,
// reconstruct w -> Lion -> quantize_state(m') -> requantize_weight(w') in registers).
// With a trace, the layer's fp tensors are produced on the device too: dequantize /
// reconstruct, then lion_apply (bitwise equal to the fused step's arithmetic).
template <class ModelT, class StateT, class StackT, class HyperT, class TraceT = detail::NoTrace>
void lion_step_quantized(ModelT& model, StateT& state, StackT& stack, const HyperT& h,
                         TraceT* trace = nullptr) {
  const int L = model.config().num_layers();
  if (static_cast<int>(stack.size()) != L)
    throw std::invalid_argument("lion step: stack holds " + std::to_string(stack.size()) +
                                " gradients for " + std::to_string(L) + " layers");
  if (static_cast<int>(state.momentum.size()) != L)
    throw std::invalid_argument("lion step: momentum count does not match layers");
  const qftc_lion_hyper hc{static_cast<float>(h.lr), static_cast<float>(h.beta1),
                           static_cast<float>(h.beta2), static_cast<float>(h.weight_decay)};
  const int bw = model.config().bit_width;
  const bool model_pt = static_cast<int>(model.config().quant_mode) == detail::kPassthrough;
  for (int li = 1; li <= L; ++li) {
    auto e = stack.pop();
    if (e.layer_index != li)
      throw std::invalid_argument("lion step: popped layer " + std::to_string(e.layer_index) +
                                  ", expected " + std::to_string(li));
    auto& layer = model.layers()[li - 1];
    if (e.grad.rows != layer.weight.rows() || e.grad.cols != layer.weight.cols())
      throw std::invalid_argument("lion step: gradient shape mismatch at layer " +
                                  std::to_string(li));
    auto& d = layer.weight;
    auto& m = state.momentum[li - 1];
    const auto& g = e.grad;
    const int r = d.dense.rows, c = d.dense.cols;
    const size_t n = static_cast<size_t>(r) * c;
    const bool g_pt = static_cast<int>(g.mode) == detail::kPassthrough;
    const bool m_pt = static_cast<int>(m.mode) == detail::kPassthrough;
    const bool w_pt = static_cast<int>(d.dense.mode) == detail::kPassthrough;
    if (model_pt || (g_pt && m_pt && w_pt)) {
      // pass-through: lion_apply on the raw fp32 state (optimizer.hpp:103-118 with the
      // identity quantizers), then the reference's re-wrapping
      if (!(g_pt && m_pt && w_pt))
        throw std::invalid_argument("lion step: mixed quantization modes are not supported");
      dbuf<float> dw(d.dense.raw), dm(m.raw), dg(g.raw);
      if constexpr (!std::is_same<TraceT, detail::NoTrace>::value) {
        if (trace) {
          using TensorT = typename std::decay_t<decltype(trace->weights_in)>::value_type;
          trace->weights_in.push_back(detail::tensor_from_host<TensorT>(d.dense.raw, r, c));
          trace->gradients.push_back(detail::tensor_from_host<TensorT>(g.raw, r, c));
          trace->momentum_in.push_back(detail::tensor_from_host<TensorT>(m.raw, r, c));
        }
      }
      check(qftc_lion_apply(dw.get(), dm.get(), dg.get(), static_cast<int64_t>(n), hc, nullptr));
      std::vector<float> w2 = dw.vec(n), m2 = dm.vec(n);
      if constexpr (!std::is_same<TraceT, detail::NoTrace>::value) {
        if (trace) {
          using TensorT = typename std::decay_t<decltype(trace->weights_in)>::value_type;
          trace->weights_updated.push_back(detail::tensor_from_host<TensorT>(w2, r, c));
          trace->momentum_updated.push_back(detail::tensor_from_host<TensorT>(m2, r, c));
        }
      }
      m.rows = r;  // quantize_state(m, bw, passthrough)
      m.cols = c;
      m.raw = std::move(m2);
      const double fraction = d.outlier_fraction;  // requantize_weight, pass-through branch
      d.dense.rows = r;
      d.dense.cols = c;
      d.dense.raw = std::move(w2);
      d.sparse.row_ptr.assign(static_cast<size_t>(r) + 1, 0);
      d.sparse.col_idx.clear();
      d.sparse.values.clear();
      d.t_min.clear();
      d.t_max.clear();
      d.outlier_fraction = fraction;
      continue;
    }
    if (g_pt || m_pt || w_pt)
      throw std::invalid_argument("lion step: mixed quantization modes are not supported");
    dbuf<uint8_t> gq(g.data), mq(m.data), wq(d.dense.data), mq2(n), wq2(n);
    dbuf<float> gs(g.params.scale), ms(m.params.scale), ws(d.dense.params.scale), ms2(r);
    dbuf<int32_t> gz(g.params.zero_point), mz(m.params.zero_point), wz(d.dense.params.zero_point),
        mz2(r), rp(d.sparse.row_ptr), rp2(r + 1), col(d.sparse.col_idx);
    dbuf<float> lo(d.t_min), hi(d.t_max), val(d.sparse.values);
    if constexpr (!std::is_same<TraceT, detail::NoTrace>::value) {
      if (trace) {
        // the fp tensors the reference's step works on: dequantize(g), dequantize(m),
        // reconstruct(w), then lion_apply -- on the device
        using TensorT = typename std::decay_t<decltype(trace->weights_in)>::value_type;
        dbuf<float> tw(n), tm(n), tg(n);
        check(qftc_reconstruct(wq.get(), r, c, ws.get(), wz.get(), rp.get(), col.get(), val.get(),
                               tw.get(), nullptr));
        check(qftc_dequantize(gq.get(), r, c, gs.get(), gz.get(),
                              static_cast<int>(g.params.scale.size()), tg.get(), nullptr));
        check(qftc_dequantize(mq.get(), r, c, ms.get(), mz.get(),
                              static_cast<int>(m.params.scale.size()), tm.get(), nullptr));
        trace->weights_in.push_back(detail::tensor_from_device<TensorT>(tw, r, c));
        trace->gradients.push_back(detail::tensor_from_device<TensorT>(tg, r, c));
        trace->momentum_in.push_back(detail::tensor_from_device<TensorT>(tm, r, c));
        check(qftc_lion_apply(tw.get(), tm.get(), tg.get(), static_cast<int64_t>(n), hc, nullptr));
        trace->weights_updated.push_back(detail::tensor_from_device<TensorT>(tw, r, c));
        trace->momentum_updated.push_back(detail::tensor_from_device<TensorT>(tm, r, c));
      }
    }
    int64_t cap = static_cast<int64_t>(d.sparse.values.size() * 5 / 4) + r + 64, nnz = 0;
    for (;;) {
      dbuf<int32_t> col2(cap);
      dbuf<float> val2(cap);
      const int rc = qftc_lion_step(r, c, bw, gq.get(), gs.get(), gz.get(), mq.get(), ms.get(),
                                    mz.get(), wq.get(), ws.get(), wz.get(), lo.get(), hi.get(),
                                    rp.get(), col.get(), val.get(), mq2.get(), ms2.get(),
                                    mz2.get(), wq2.get(), rp2.get(), col2.get(), val2.get(), cap,
                                    hc, &nnz, nullptr);
      if (rc == QFTC_EOVERFLOW) {
        cap = nnz;
        continue;
      }
      check(rc);
      // state.momentum[li-1] = quantize_state(m', bw, affine)
      detail::fill_qt(m, r, c, mq2.vec(n), ms2.vec(r), mz2.vec(r), bw);
      m.raw.clear();
      // requantize_weight(layer.weight, w', bw): thresholds, params, fraction kept
      d.dense.data = wq2.vec(n);
      d.sparse.row_ptr = rp2.vec(r + 1);
      d.sparse.col_idx = col2.vec(static_cast<size_t>(nnz));
      d.sparse.values = val2.vec(static_cast<size_t>(nnz));
      break;
    }
  }
}

}  // namespace qft_b200
