// qft_b200/qft.hpp -- C++ drop-in shim over the C-ABI (include/qft_b200.h).
//
// Mirrors the reference's quantizer/optimizer entry points for T = float
// (/root/reference/proj/include/qft/{quantize,optimizer}.hpp) with the same
// argument order, value semantics and exception types.  The functions are
// templates over the caller's host types, so they accept the reference's own
// structs unchanged (they only touch the public fields the reference exposes:
// Tensor::rows()/cols()/data(); QuantizedTensor::{rows,cols,mode,data,raw,params};
// AffineParams::{scale,zero_point,bit_width}; SparseOutliers::{row_ptr,col_idx,
// values}; DenseSparseWeight::{dense,sparse,t_min,t_max,outlier_fraction};
// Model::config()/layers(); LionState::momentum; GradientStack::size()/pop()).
//
//   auto q  = qft_b200::quantize_state<qft::QuantizedTensor<float>>(x, 8);
//   auto x2 = qft_b200::dequantize<qft::Tensor<float>>(q);
//   auto w  = qft_b200::decompose_weight<qft::DenseSparseWeight<float>>(t, 0.01, 8);
//   qft_b200::requantize_weight(w, t2, 8);
//   qft_b200::lion_step_quantized(model, state, stack, hyper);   // same call as qft::
//
// Each call moves its host arrays to the device, runs the sm_100a kernels and
// copies the results back (the reference API is host-resident).  Whole-model
// device-resident stepping is QftModelState (Python) / qftc_plan_* (C).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "qft_b200.h"

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
  void up(const T* h, size_t n) { check(qftc_copy_to_device(p_, h, n * sizeof(T), nullptr)); }
  void down(T* h, size_t n) const {
    check(qftc_copy_to_host(h, p_, n * sizeof(T), nullptr));
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
constexpr int kPassthrough = 1;  // QuantMode::passthrough (quantize.hpp:17)

template <class QT>
void fill_qt(QT& q, int rows, int cols, std::vector<uint8_t> data, std::vector<float> s,
             std::vector<int32_t> z, int bw) {
  q.rows = rows;
  q.cols = cols;
  q.mode = static_cast<decltype(q.mode)>(0);
  q.data = std::move(data);
  q.params.scale = std::move(s);
  q.params.zero_point = std::move(z);
  q.params.bit_width = bw;
}
}  // namespace detail

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
    for (size_t i = 0; i < n; ++i) out.data()[i] = q.raw[i];
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

// quantize.hpp:318-329
template <class DSW, class TensorT>
void requantize_weight(DSW& dsw, const TensorT& w_fp, int bit_width) {
  DSW next = decompose_dense_sparse<DSW>(w_fp, dsw.t_min, dsw.t_max, bit_width);
  next.outlier_fraction = dsw.outlier_fraction;
  dsw = std::move(next);
}

// quantize.hpp:331-338
template <class TensorOut, class DSW>
TensorOut reconstruct(const DSW& d) {
  const int r = d.dense.rows, c = d.dense.cols;
  const size_t n = static_cast<size_t>(r) * c;
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

// optimizer.hpp:85-120.  Same validation order and exception types; each layer is
// then updated by one fused kernel launch (qftc_lion_step).
template <class ModelT, class StateT, class StackT, class HyperT>
void lion_step_quantized(ModelT& model, StateT& state, StackT& stack, const HyperT& h) {
  const int L = model.config().num_layers();
  if (static_cast<int>(stack.size()) != L)
    throw std::invalid_argument("lion step: stack holds " + std::to_string(stack.size()) +
                                " gradients for " + std::to_string(L) + " layers");
  if (static_cast<int>(state.momentum.size()) != L)
    throw std::invalid_argument("lion step: momentum count does not match layers");
  using QT = std::decay_t<decltype(state.momentum[0])>;
  std::vector<QT> grads;
  grads.reserve(L);
  for (int li = 1; li <= L; ++li) {
    auto e = stack.pop();
    if (e.layer_index != li)
      throw std::invalid_argument("lion step: popped layer " + std::to_string(e.layer_index) +
                                  ", expected " + std::to_string(li));
    auto& layer = model.layers()[li - 1];
    if (e.grad.rows != layer.weight.rows() || e.grad.cols != layer.weight.cols())
      throw std::invalid_argument("lion step: gradient shape mismatch at layer " +
                                  std::to_string(li));
    grads.push_back(std::move(e.grad));
  }
  const qftc_lion_hyper hc{static_cast<float>(h.lr), static_cast<float>(h.beta1),
                           static_cast<float>(h.beta2), static_cast<float>(h.weight_decay)};
  const int bw = model.config().bit_width;
  if (static_cast<int>(model.config().quant_mode) == detail::kPassthrough) {
    for (int l = 0; l < L; ++l) {  // pass-through: lion_apply on raw fp32 state
      auto& w = model.layers()[l].weight.dense.raw;
      auto& m = state.momentum[l].raw;
      const auto& g = grads[l].raw;
      dbuf<float> dw(w), dm(m), dg(g);
      check(qftc_lion_apply(dw.get(), dm.get(), dg.get(), static_cast<int64_t>(w.size()), hc,
                            nullptr));
      dw.down(w.data(), w.size());
      dm.down(m.data(), m.size());
    }
    return;
  }
  for (int l = 0; l < L; ++l) {
    auto& d = model.layers()[l].weight;
    auto& m = state.momentum[l];
    const auto& g = grads[l];
    const int r = d.dense.rows, c = d.dense.cols;
    const size_t n = static_cast<size_t>(r) * c;
    dbuf<uint8_t> gq(g.data), mq(m.data), wq(d.dense.data), mq2(n), wq2(n);
    dbuf<float> gs(g.params.scale), ms(m.params.scale), ws(d.dense.params.scale), ms2(r);
    dbuf<int32_t> gz(g.params.zero_point), mz(m.params.zero_point), wz(d.dense.params.zero_point),
        mz2(r), rp(d.sparse.row_ptr), rp2(r + 1), col(d.sparse.col_idx);
    dbuf<float> lo(d.t_min), hi(d.t_max), val(d.sparse.values);
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
      m.data = mq2.vec(n);
      m.params.scale = ms2.vec(r);
      m.params.zero_point = mz2.vec(r);
      d.dense.data = wq2.vec(n);
      d.sparse.row_ptr = rp2.vec(r + 1);
      d.sparse.col_idx = col2.vec(static_cast<size_t>(nnz));
      d.sparse.values = val2.vec(static_cast<size_t>(nnz));
      break;
    }
  }
}

}  // namespace qft_b200
