/*
 * qft_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference's quantized model-state update path
 * (QFT, arXiv 2310.07147; reference tree /root/reference/proj).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this
 * library.  The CUDA product path never links or calls it.
 *
 * Pinning: tests/test_oracle.py checks every function here against
 *   (a) the reference's own known-answer tests (test_quantize.cpp,
 *       test_optimizer.cpp) restated as golden vectors, and
 *   (b) oracle/_ref/libqft_ref.so -- the reference headers compiled unmodified
 *       from /root/reference by oracle/Makefile -- on seeded random inputs,
 *       with committed fixtures under tests/golden/ for the GPU box.
 *
 * Build contract mirrored from the reference (CMakeLists.txt:12-14):
 *   -O3 -ffp-contract=off (no FMA contraction; every product/sum rounds).
 *
 * Error convention: functions return 0 (or a non-negative count) on success,
 * QO_EINVAL for what the reference throws as std::invalid_argument,
 * QO_ERANGE for std::out_of_range.  qo_last_error() has the message.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define QO_EINVAL (-1)
#define QO_ERANGE (-2)

static _Thread_local char g_err[256];

const char* qo_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* ------------------------------------------------------------------------ */
/* L0: channel_minmax                       tensor.hpp:133-148               */
/* ------------------------------------------------------------------------ */
int qo_channel_minmax(const float* x, int rows, int cols, float* mins, float* maxs) {
  if (rows <= 0 || cols <= 0) return fail(QO_EINVAL, "channel_minmax: empty tensor");
  for (int r = 0; r < rows; ++r) {
    const float* row = x + (size_t)r * cols;
    float lo = row[0], hi = row[0];
    for (int c = 1; c < cols; ++c) {
      const float v = row[c];
      if (v < lo) lo = v;  /* NaN never replaces; a NaN at col 0 sticks */
      if (v > hi) hi = v;
    }
    mins[r] = lo;
    maxs[r] = hi;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* L1: affine params                         quantize.hpp:89-92, 105-131     */
/* ------------------------------------------------------------------------ */
static int require_bit_width(int b) {
  if (b < 2 || b > 8) {
    snprintf(g_err, sizeof g_err, "bit width must be in [2, 8], got %d", b);
    return QO_EINVAL;
  }
  return 0;
}

int qo_affine_params_from_bounds(const float* mins, const float* maxs, int64_t n, int bit_width,
                                 float* scale, int32_t* zp) {
  if (require_bit_width(bit_width)) return QO_EINVAL;
  if (n <= 0) return fail(QO_EINVAL, "affine_params_from_bounds: bad channel count");
  const double qmax = (double)((1 << bit_width) - 1);
  for (int64_t ch = 0; ch < n; ++ch) {
    const double lo = (double)mins[ch];
    const double hi = (double)maxs[ch];
    if (!(lo <= hi)) {
      snprintf(g_err, sizeof g_err, "affine_params_from_bounds: min > max in channel %lld",
               (long long)ch);
      return QO_EINVAL;
    }
    /* degenerate channel: max(|lo|, 1) * 2^-20  (std::max(a,b) == a<b ? b : a) */
    const double a = fabs(lo);
    const double s = (lo == hi) ? ((a < 1.0 ? 1.0 : a) * ldexp(1.0, -20)) : (hi - lo) / qmax;
    double z = round(-lo / s);
    /* std::clamp(z, INT32_MIN, INT32_MAX) */
    if (z < -2147483648.0) z = -2147483648.0;
    else if (2147483647.0 < z) z = 2147483647.0;
    scale[ch] = (float)s;
    zp[ch] = (int32_t)z;
  }
  return 0;
}

/* compute_affine_params, channel-wise           quantize.hpp:133-147 */
int qo_compute_affine_params(const float* x, int rows, int cols, int bit_width, float* scale,
                             int32_t* zp) {
  if (rows <= 0 || cols <= 0) return fail(QO_EINVAL, "compute_affine_params: empty tensor");
  float* mins = (float*)malloc(sizeof(float) * (size_t)rows);
  float* maxs = (float*)malloc(sizeof(float) * (size_t)rows);
  qo_channel_minmax(x, rows, cols, mins, maxs);
  const int rc = qo_affine_params_from_bounds(mins, maxs, rows, bit_width, scale, zp);
  free(mins);
  free(maxs);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* L1: quantize / quantize_state / dequantize  quantize.hpp:149-212         */
/* ------------------------------------------------------------------------ */
static uint8_t quantize_one(float x, double s, double z, double qmax) {
  /* round half away from zero of the double quotient, + z, clip */
  double q = round((double)x / s) + z;
  if (!(q > 0.0)) q = 0.0; /* also catches NaN */
  if (q > qmax) q = qmax;
  return (uint8_t)q;
}

int qo_quantize(const float* x, int rows, int cols, const float* scale, const int32_t* zp,
                int channels, int bit_width, uint8_t* codes) {
  if (channels != 1 && channels != rows) {
    snprintf(g_err, sizeof g_err, "quantize: channel count %d does not match rows %d", channels,
             rows);
    return QO_EINVAL;
  }
  const double qmax = (double)((1 << bit_width) - 1);
  size_t i = 0;
  for (int r = 0; r < rows; ++r) {
    const int ch = channels == 1 ? 0 : r;
    const double s = (double)scale[ch];
    const double z = (double)zp[ch];
    for (int c = 0; c < cols; ++c, ++i) codes[i] = quantize_one(x[i], s, z, qmax);
  }
  return 0;
}

int qo_quantize_state(const float* x, int rows, int cols, int bit_width, uint8_t* codes,
                      float* scale, int32_t* zp) {
  int rc = qo_compute_affine_params(x, rows, cols, bit_width, scale, zp);
  if (rc) return rc;
  return qo_quantize(x, rows, cols, scale, zp, rows, bit_width, codes);
}

int qo_dequantize(const uint8_t* codes, int rows, int cols, const float* scale,
                  const int32_t* zp, int channels, float* out) {
  if (rows <= 0 || cols <= 0) return fail(QO_EINVAL, "dequantize: empty tensor");
  size_t i = 0;
  for (int r = 0; r < rows; ++r) {
    const int ch = channels == 1 ? 0 : r;
    const float s = scale[ch];
    const int32_t z = zp[ch];
    for (int c = 0; c < cols; ++c, ++i) out[i] = s * (float)((int32_t)codes[i] - z);
  }
  return 0;
}

/* accumulate (gradflow.hpp:52-58): quantize_state(dequantize(acc) + g_new) with the
 * accumulator's bit width; the sum is fp32 (tensor add, one rounding per element). */
int qo_accumulate(const uint8_t* codes, const float* scale, const int32_t* zp, int rows,
                  int cols, int bit_width, const float* g, uint8_t* codes_out,
                  float* scale_out, int32_t* zp_out) {
  if (rows <= 0 || cols <= 0) return fail(QO_EINVAL, "accumulate: empty tensor");
  const size_t n = (size_t)rows * (size_t)cols;
  float* sum = (float*)malloc(n * sizeof(float));
  if (!sum) return fail(QO_EINVAL, "accumulate: out of memory");
  int rc = qo_dequantize(codes, rows, cols, scale, zp, rows, sum);
  if (!rc) {
    for (size_t i = 0; i < n; ++i) sum[i] = sum[i] + g[i];
    rc = qo_quantize_state(sum, rows, cols, bit_width, codes_out, scale_out, zp_out);
  }
  free(sum);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* L1: outlier thresholds                    quantize.hpp:76-87, 216-247     */
/* ------------------------------------------------------------------------ */
static int cmp_float(const void* a, const void* b) {
  const float x = *(const float*)a, y = *(const float*)b;
  return (x < y) ? -1 : (y < x) ? 1 : 0;
}

static double sorted_quantile(const float* s, size_t n, double q) {
  if (n == 1) return (double)s[0];
  const double h = q * (double)(n - 1);
  const size_t i0 = (size_t)h;
  if (i0 >= n - 1) return (double)s[n - 1];
  const double frac = h - (double)i0;
  return (double)s[i0] + frac * ((double)s[i0 + 1] - (double)s[i0]);
}

/* kind: 0 = percentile, 1 = range_fraction (ThresholdKind, quantize.hpp:20) */
int qo_outlier_thresholds(const float* w, int rows, int cols, double fraction, int kind,
                          float* t_min, float* t_max) {
  if (rows <= 0 || cols <= 0) return fail(QO_EINVAL, "compute_outlier_thresholds: empty tensor");
  if (!(fraction >= 0.0) || fraction >= 0.5)
    return fail(QO_EINVAL, "outlier fraction must be in [0, 0.5)");
  float* row = (float*)malloc(sizeof(float) * (size_t)cols);
  for (int r = 0; r < rows; ++r) {
    const float* src = w + (size_t)r * cols;
    if (fraction == 0.0 || kind == 1) {
      float lo = src[0], hi = src[0];
      for (int c = 1; c < cols; ++c) {
        if (src[c] < lo) lo = src[c];
        if (src[c] > hi) hi = src[c];
      }
      if (fraction == 0.0) {
        t_min[r] = lo;
        t_max[r] = hi;
      } else {
        const double span = (double)hi - (double)lo;
        t_min[r] = (float)((double)lo + (fraction / 2) * span);
        t_max[r] = (float)((double)hi - (fraction / 2) * span);
      }
    } else {
      memcpy(row, src, sizeof(float) * (size_t)cols);
      qsort(row, (size_t)cols, sizeof(float), cmp_float);
      t_min[r] = (float)sorted_quantile(row, (size_t)cols, fraction / 2);
      t_max[r] = (float)sorted_quantile(row, (size_t)cols, 1.0 - fraction / 2);
    }
  }
  free(row);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* L1: dense-and-sparse split                quantize.hpp:253-290            */
/* Returns nnz (>= 0).  Sparse entries beyond `capacity` are counted but not */
/* stored, so a caller can size its buffers with a first call.               */
/* ------------------------------------------------------------------------ */
int64_t qo_decompose_dense_sparse(const float* w, int rows, int cols, const float* t_min,
                                  const float* t_max, int bit_width, uint8_t* codes, float* scale,
                                  int32_t* zp, int32_t* row_ptr, int32_t* col_idx, float* values,
                                  int64_t capacity) {
  int rc = qo_affine_params_from_bounds(t_min, t_max, rows, bit_width, scale, zp);
  if (rc) return rc;
  const int32_t qmax_i = (1 << bit_width) - 1;
  const double qmax = (double)qmax_i;
  int64_t nnz = 0;
  size_t i = 0;
  row_ptr[0] = 0;
  for (int r = 0; r < rows; ++r) {
    const double s = (double)scale[r];
    const int32_t z = zp[r];
    const uint8_t z_payload = (uint8_t)(z < 0 ? 0 : (qmax_i < z ? qmax_i : z));
    for (int c = 0; c < cols; ++c, ++i) {
      const float v = w[i];
      if (v < t_min[r] || v > t_max[r]) {
        if (nnz < capacity) {
          col_idx[nnz] = c;
          values[nnz] = v;
        }
        ++nnz;
        codes[i] = z_payload;
      } else {
        codes[i] = quantize_one(v, s, (double)z, qmax);
      }
    }
    row_ptr[r + 1] = (int32_t)nnz;
  }
  return nnz;
}

/* decompose_weight = thresholds + split         quantize.hpp:301-314 */
int64_t qo_decompose_weight(const float* w, int rows, int cols, double fraction, int bit_width,
                            int kind, float* t_min, float* t_max, uint8_t* codes, float* scale,
                            int32_t* zp, int32_t* row_ptr, int32_t* col_idx, float* values,
                            int64_t capacity) {
  int rc = qo_outlier_thresholds(w, rows, cols, fraction, kind, t_min, t_max);
  if (rc) return rc;
  return qo_decompose_dense_sparse(w, rows, cols, t_min, t_max, bit_width, codes, scale, zp,
                                   row_ptr, col_idx, values, capacity);
}

/* reconstruct = dequantize, then overwrite CSR positions  quantize.hpp:331-338 */
int qo_reconstruct(const uint8_t* codes, int rows, int cols, const float* scale,
                   const int32_t* zp, const int32_t* row_ptr, const int32_t* col_idx,
                   const float* values, float* out) {
  int rc = qo_dequantize(codes, rows, cols, scale, zp, rows, out);
  if (rc) return rc;
  for (int r = 0; r < rows; ++r)
    for (int32_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k)
      out[(size_t)r * cols + col_idx[k]] = values[k];
  return 0;
}

/* ------------------------------------------------------------------------ */
/* L4: Lion                                   optimizer.hpp:15-42            */
/* ------------------------------------------------------------------------ */
static float sign_of(float v) { return v > 0.0f ? 1.0f : (v < 0.0f ? -1.0f : 0.0f); }

void qo_lion_apply(float* w, float* m, const float* g, int64_t n, float lr, float beta1,
                   float beta2, float wd) {
  for (int64_t i = 0; i < n; ++i) {
    const float d = beta1 * m[i] + (1.0f - beta1) * g[i];
    w[i] = w[i] - lr * (sign_of(d) + wd * w[i]);
    m[i] = beta2 * m[i] + (1.0f - beta2) * g[i];
  }
}

/* One layer of lion_step_quantized (optimizer.hpp:103-118):
 *   g = dequantize(grad); m = dequantize(momentum); w = reconstruct(weight);
 *   lion_apply(w, m, g); momentum = quantize_state(m); requantize_weight(w).
 * Weight dense params are re-derived from the cached thresholds
 * (requantize_weight, quantize.hpp:318-329 -> decompose_dense_sparse).
 * The five optional trace_* buffers mirror LionStepTrace (optimizer.hpp:71-78).
 * Returns the new nnz (entries beyond `capacity` counted, not stored). */
int64_t qo_lion_step_layer(int rows, int cols, int bit_width,
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
  const size_t n = (size_t)rows * (size_t)cols;
  float* g = (float*)malloc(sizeof(float) * n);
  float* m = (float*)malloc(sizeof(float) * n);
  float* w = (float*)malloc(sizeof(float) * n);
  int64_t rc = qo_dequantize(g_codes, rows, cols, g_scale, g_zp, rows, g);
  if (!rc) rc = qo_dequantize(m_codes, rows, cols, m_scale, m_zp, rows, m);
  if (!rc) rc = qo_reconstruct(w_codes, rows, cols, w_scale, w_zp, row_ptr, col_idx, values, w);
  if (!rc) {
    if (trace_w_in) memcpy(trace_w_in, w, sizeof(float) * n);
    if (trace_g) memcpy(trace_g, g, sizeof(float) * n);
    if (trace_m_in) memcpy(trace_m_in, m, sizeof(float) * n);
    qo_lion_apply(w, m, g, (int64_t)n, lr, beta1, beta2, wd);
    if (trace_w_upd) memcpy(trace_w_upd, w, sizeof(float) * n);
    if (trace_m_upd) memcpy(trace_m_upd, m, sizeof(float) * n);
    rc = qo_quantize_state(m, rows, cols, bit_width, m_codes_out, m_scale_out, m_zp_out);
  }
  if (!rc)
    rc = qo_decompose_dense_sparse(w, rows, cols, t_min, t_max, bit_width, w_codes_out,
                                   w_scale_out, w_zp_out, row_ptr_out, col_idx_out, values_out,
                                   capacity);
  free(g);
  free(m);
  free(w);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* byte accounting                            quantize.hpp:353-376           */
/* ------------------------------------------------------------------------ */
int64_t qo_byte_size_dense_sparse(int rows, int cols, int64_t nnz) {
  const int64_t dense = (int64_t)rows * cols + 4ll * rows + 4ll * rows;
  const int64_t sparse = 4ll * (rows + 1) + 8ll * nnz;
  return dense + sparse + 8ll * rows;
}
