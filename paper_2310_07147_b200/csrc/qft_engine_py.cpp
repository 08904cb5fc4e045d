// qft_engine_py.cpp -- pybind11 drop-in for the reference's `qft_engine` quantizer
// surface (bindings/qft_bindings.cpp:85-150): same function names, argument names,
// defaults, return dicts and error mapping (std::invalid_argument -> ValueError).
// The work runs on the GPU through the C-ABI via the C++ shim (qft_b200/qft.hpp).
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "qft_b200/qft.hpp"

namespace py = pybind11;

namespace {

// Minimal host containers with the reference's public field names.
struct Tensor {
  int r = 0, c = 0;
  std::vector<float> v;
  Tensor() = default;
  Tensor(int rows, int cols) : r(rows), c(cols), v(static_cast<size_t>(rows) * cols) {}
  int rows() const { return r; }
  int cols() const { return c; }
  float* data() { return v.data(); }
  const float* data() const { return v.data(); }
  size_t size() const { return v.size(); }
};
struct Params {
  std::vector<float> scale;
  std::vector<int32_t> zero_point;
  int bit_width = 8;
};
struct QT {
  int rows = 0, cols = 0;
  int mode = 0;
  std::vector<uint8_t> data;
  std::vector<float> raw;
  Params params;
};
struct Sparse {
  std::vector<int32_t> row_ptr, col_idx;
  std::vector<float> values;
  size_t nnz() const { return values.size(); }
};
struct DSW {
  QT dense;
  Sparse sparse;
  std::vector<float> t_min, t_max;
  double outlier_fraction = 0.0;
};

using FloatArray = py::array_t<float, py::array::c_style | py::array::forcecast>;

Tensor to_tensor(const FloatArray& a) {
  if (a.ndim() != 2) throw std::invalid_argument("expected a 2-d array");
  const auto rows = static_cast<int>(a.shape(0));
  const auto cols = static_cast<int>(a.shape(1));
  if (rows <= 0 || cols <= 0) throw std::invalid_argument("expected a non-empty 2-d array");
  Tensor t(rows, cols);
  std::memcpy(t.data(), a.data(), sizeof(float) * t.size());
  return t;
}

py::array_t<float> to_array(const Tensor& t) {
  py::array_t<float> a({t.rows(), t.cols()});
  std::memcpy(a.mutable_data(), t.data(), sizeof(float) * t.size());
  return a;
}

int kind_from_name(const std::string& name) {
  if (name == "percentile") return QFTC_PERCENTILE;
  if (name == "range-fraction") return QFTC_RANGE_FRACTION;
  throw std::invalid_argument("threshold kind must be percentile or range-fraction, got '" +
                              name + "'");
}

size_t byte_size(const DSW& d) {  // quantize.hpp:353-376
  const size_t r = static_cast<size_t>(d.dense.rows);
  return d.dense.data.size() + 8 * r + 4 * (r + 1) + 8 * d.sparse.nnz() + 8 * r;
}

double l2(const Tensor& a, const Tensor& b) {
  double sq = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double d = double(a.data()[i]) - double(b.data()[i]);
    sq += d * d;
  }
  return std::sqrt(sq);
}

}  // namespace

PYBIND11_MODULE(qft_engine, m) {
  m.doc() = "QFT quantizer surface on B200 (sm_100a kernels behind the qftc C-ABI)";

  m.def(
      "quantize_roundtrip",
      [](const FloatArray& x, int bit_width) {
        const auto t = to_tensor(x);
        const auto q = qft_b200::generic::quantize_state<QT>(t, bit_width);
        return to_array(qft_b200::generic::dequantize<Tensor>(q));
      },
      py::arg("x"), py::arg("bit_width") = 8,
      "Channel-wise affine quantize + dequantize; rows are channels.");

  m.def(
      "quantize_params",
      [](const FloatArray& x, int bit_width) {
        const auto q = qft_b200::generic::quantize_state<QT>(to_tensor(x), bit_width);
        py::dict d;
        d["scale"] = py::cast(q.params.scale);
        d["zero_point"] = py::cast(q.params.zero_point);
        d["bit_width"] = q.params.bit_width;
        return d;
      },
      py::arg("x"), py::arg("bit_width") = 8, "Per-row scale and zero point the quantizer would use.");

  m.def(
      "decompose",
      [](const FloatArray& x, double outlier_fraction, int bit_width,
         const std::string& threshold_kind) {
        const auto t = to_tensor(x);
        const auto dsw = qft_b200::generic::decompose_weight<DSW>(t, outlier_fraction, bit_width,
                                                         kind_from_name(threshold_kind));
        const auto back = qft_b200::generic::reconstruct<Tensor>(dsw);
        py::dict d;
        d["reconstructed"] = to_array(back);
        d["nnz"] = dsw.sparse.nnz();
        d["bytes"] = byte_size(dsw);
        d["l2_error"] = l2(t, back);
        return d;
      },
      py::arg("x"), py::arg("outlier_fraction") = 0.01, py::arg("bit_width") = 8,
      py::arg("threshold_kind") = "percentile",
      "Dense-and-sparse split: quantized core plus exact outliers.");

  m.def(
      "threshold_sweep",
      [](const FloatArray& x, const std::vector<double>& fractions, int bit_width,
         const std::string& threshold_kind) {
        if (fractions.empty()) throw std::invalid_argument("threshold_sweep: no fractions");
        const auto t = to_tensor(x);
        const int kind = kind_from_name(threshold_kind);
        py::list out;
        for (double f : fractions) {  // profiler.cpp:187-201
          const auto dsw = qft_b200::generic::decompose_weight<DSW>(t, f, bit_width, kind);
          py::dict d;
          d["fraction"] = f;
          d["bytes"] = byte_size(dsw);
          d["l2_error"] = l2(qft_b200::generic::reconstruct<Tensor>(dsw), t);
          out.append(d);
        }
        return out;
      },
      py::arg("x"), py::arg("fractions"), py::arg("bit_width") = 8,
      py::arg("threshold_kind") = "percentile",
      "Storage vs reconstruction error across outlier fractions.");
}
