// capi.cu -- extern "C" boundary (include/qft_b200.h) over the sm_100a kernels.
//
// Validation order and messages follow the reference so the C++ shim can map
// QFTC_EINVAL/QFTC_ERANGE back onto std::invalid_argument/std::out_of_range.
// There is no host fallback: without a CUDA device every compute entry point
// fails with QFTC_ECUDA.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "qft_b200.h"
#include <cuda.h>
#include <cstring>

#include "qft_internal.h"

namespace qftk {
cudaError_t launch_channel_minmax(const float*, int, int, float*, float*, cudaStream_t);
cudaError_t launch_affine_params(const float*, const float*, int64_t, int, float*, int32_t*,
                                 uint32_t*, cudaStream_t);
cudaError_t launch_accumulate_state(const uint8_t*, const float*, const int32_t*, int, int, int,
                                    const float*, uint8_t*, float*, int32_t*, uint32_t*,
                                    cudaStream_t);
cudaError_t launch_quantize_state(const float*, int, int, int, uint8_t*, float*, int32_t*,
                                  uint32_t*, cudaStream_t);
cudaError_t launch_quantize(const float*, int, int, const float*, const int32_t*, int, int,
                            uint8_t*, cudaStream_t);
cudaError_t launch_dequantize(const uint8_t*, int, int, const float*, const int32_t*, int, void*,
                              bool, cudaStream_t);
cudaError_t launch_thresholds(const float*, int, int, double, int, float*, float*, cudaStream_t);
cudaError_t launch_lion_apply(float*, float*, const float*, int64_t, float, float, float, float,
                              cudaStream_t);
cudaError_t launch_synth(float*, int64_t, uint64_t, double, double, cudaStream_t);
cudaError_t csr_plan_slots(const int32_t*, const int32_t*, int, int, int32_t*, cudaStream_t);
cudaError_t csr_copy_rows(int, const int32_t*, const int32_t*, const int32_t*, const float*,
                          const int32_t*, int32_t*, float*, int64_t, cudaStream_t);
}  // namespace qftk

using namespace qftk;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(QFTC_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define QFTC_CUDA(expr, where)                           \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return cuda_fail(_e, where);  \
  } while (0)

int require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(QFTC_ECUDA, "no CUDA device: the QFT B200 path has no CPU fallback");
  return QFTC_OK;
}

int require_bit_width(int b) {
  if (b < 2 || b > 8)
    return fail(QFTC_EINVAL, "bit width must be in [2, 8], got " + std::to_string(b));
  return QFTC_OK;
}

int require_shape(int rows, int cols, const char* what) {
  if (rows <= 0 || cols <= 0) return fail(QFTC_EINVAL, std::string(what) + ": empty tensor");
  return QFTC_OK;
}

inline bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

constexpr int kSlack = 8;  // extra slot entries per row beyond count + count/4

// Device workspace: header | tensors | blocks | status words
struct Scratch {
  void* base = nullptr;
  Header* hdr = nullptr;
  DevTensor* tensors = nullptr;
  RowBlock* blocks = nullptr;
  unsigned long long* status = nullptr;
  int n_blocks = 0;
};

std::vector<RowBlock> make_blocks(const std::vector<DevTensor>& ts) {
  std::vector<RowBlock> b;
  for (int t = 0; t < (int)ts.size(); ++t)
    for (int r0 = 0; r0 < ts[t].rows; r0 += kBlockRows)
      b.push_back(RowBlock{t, r0, std::min(kBlockRows, ts[t].rows - r0), 0});
  return b;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// allocate + upload descriptors and the block table (stream-ordered)
int scratch_alloc(Scratch& s, const std::vector<DevTensor>& ts, int64_t status_rows,
                  cudaStream_t st) {
  const std::vector<RowBlock> blocks = make_blocks(ts);
  const size_t hb = 256;
  const size_t tb = align256(sizeof(DevTensor) * ts.size());
  const size_t bb = align256(sizeof(RowBlock) * (blocks.size() ? blocks.size() : 1));
  const size_t sb = sizeof(unsigned long long) * (size_t)(status_rows > 0 ? status_rows : 1);
  const size_t total = hb + tb + bb + sb;
  QFTC_CUDA(cudaMallocAsync(&s.base, total, st), "cudaMallocAsync");
  QFTC_CUDA(cudaMemsetAsync(s.base, 0, hb, st), "cudaMemsetAsync");
  if (status_rows > 0)
    QFTC_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(s.base) + hb + tb + bb, 0, sb, st),
              "cudaMemsetAsync");
  char* p = reinterpret_cast<char*>(s.base);
  s.hdr = reinterpret_cast<Header*>(p);
  s.tensors = reinterpret_cast<DevTensor*>(p + hb);
  s.blocks = reinterpret_cast<RowBlock*>(p + hb + tb);
  s.status = reinterpret_cast<unsigned long long*>(p + hb + tb + bb);
  s.n_blocks = (int)blocks.size();
  static const uint32_t one = 1;  // epoch starts at 1: zeroed status words read "not ready"
  QFTC_CUDA(cudaMemcpyAsync(&s.hdr->epoch, &one, 4, cudaMemcpyHostToDevice, st), "init epoch");
  QFTC_CUDA(cudaMemcpyAsync(s.tensors, ts.data(), sizeof(DevTensor) * ts.size(),
                            cudaMemcpyHostToDevice, st),
            "upload descriptors");
  if (!blocks.empty())
    QFTC_CUDA(cudaMemcpyAsync(s.blocks, blocks.data(), sizeof(RowBlock) * blocks.size(),
                              cudaMemcpyHostToDevice, st),
              "upload blocks");
  // the pageable host vectors must outlive the copies
  QFTC_CUDA(cudaStreamSynchronize(st), "sync");
  return QFTC_OK;
}

// step kernel shape (warp-per-row kernel): the old-outlier table per warp, sized for
// the width class (rows with more old outliers take the general path).
// QFT_STEP_CFG="oldcap" overrides it (tuning).
struct StepCfg {
  int oldcap;
};
StepCfg pick_step_config(int gk, int cols_p) {
  StepCfg c{cols_p <= 4096 ? 128 : 256};
  if (const char* env = getenv("QFT_STEP_CFG")) {
    int oc = 0;
    if (sscanf(env, "%d", &oc) == 1 && oc >= 32 && oc <= 4096 &&
        step_kernel_smem(gk, cols_p, oc) <= 227 * 1024)
      c.oldcap = oc;
  }
  return c;
}

int read_header(const Header* d_hdr, Header* h, cudaStream_t st) {
  QFTC_CUDA(cudaMemcpyAsync(h, d_hdr, sizeof(Header), cudaMemcpyDeviceToHost, st), "read header");
  QFTC_CUDA(cudaStreamSynchronize(st), "cudaStreamSynchronize");
  return QFTC_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

const char* qftc_last_error(void) { return g_err.c_str(); }
int qftc_version(void) { return 2; }
int qftc_max_cols(void) { return step_kernel_max_cols(); }

int qftc_channel_minmax(const float* x, int rows, int cols, float* mins, float* maxs,
                        qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, "channel_minmax")) return rc;
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_channel_minmax(x, rows, cols, mins, maxs, (cudaStream_t)stream),
            "channel_minmax");
  return QFTC_OK;
}

int qftc_affine_params_from_bounds(const float* mins, const float* maxs, int64_t n,
                                   int bit_width, float* scale, int32_t* zp,
                                   qftc_stream_t stream) {
  if (int rc = require_bit_width(bit_width)) return rc;
  if (n <= 0) return fail(QFTC_EINVAL, "affine_params_from_bounds: bad channel count");
  if (int rc = require_device()) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* err = nullptr;
  QFTC_CUDA(cudaMallocAsync((void**)&err, 4, st), "cudaMallocAsync");
  QFTC_CUDA(cudaMemsetAsync(err, 0, 4, st), "memset");
  QFTC_CUDA(launch_affine_params(mins, maxs, n, bit_width, scale, zp, err, st), "affine_params");
  uint32_t h = 0;
  QFTC_CUDA(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, st), "copy");
  QFTC_CUDA(cudaFreeAsync(err, st), "free");
  QFTC_CUDA(cudaStreamSynchronize(st), "sync");
  if (h) return fail(QFTC_EINVAL, "affine_params_from_bounds: min > max in a channel");
  return QFTC_OK;
}

int qftc_quantize(const float* x, int rows, int cols, const float* scale, const int32_t* zp,
                  int channels, int bit_width, uint8_t* codes, qftc_stream_t stream) {
  if (channels != 1 && channels != rows)
    return fail(QFTC_EINVAL, "quantize: channel count " + std::to_string(channels) +
                                 " does not match rows " + std::to_string(rows));
  if (int rc = require_shape(rows, cols, "quantize")) return rc;
  if (int rc = require_bit_width(bit_width)) return rc;
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_quantize(x, rows, cols, scale, zp, channels, bit_width, codes,
                            (cudaStream_t)stream),
            "quantize");
  return QFTC_OK;
}

int qftc_quantize_state(const float* x, int rows, int cols, int bit_width, uint8_t* codes,
                        float* scale, int32_t* zp, int check, qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, "compute_affine_params")) return rc;
  if (int rc = require_bit_width(bit_width)) return rc;
  if (int rc = require_device()) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* err = nullptr;
  QFTC_CUDA(cudaMallocAsync((void**)&err, 4, st), "cudaMallocAsync");
  QFTC_CUDA(cudaMemsetAsync(err, 0, 4, st), "memset");
  QFTC_CUDA(launch_quantize_state(x, rows, cols, bit_width, codes, scale, zp, err, st),
            "quantize_state");
  uint32_t h = 0;
  if (check) QFTC_CUDA(cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, st), "copy");
  QFTC_CUDA(cudaFreeAsync(err, st), "free");
  if (check) {
    QFTC_CUDA(cudaStreamSynchronize(st), "sync");
    if (h) return fail(QFTC_EINVAL, "affine_params_from_bounds: min > max in a channel");
  }
  return QFTC_OK;
}

int qftc_accumulate_state(const uint8_t* codes, const float* scale, const int32_t* zero_point,
                          int rows, int cols, int bit_width, const float* g_new,
                          uint8_t* codes_out, float* scale_out, int32_t* zero_point_out,
                          qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, "accumulate")) return rc;
  if (int rc = require_bit_width(bit_width)) return rc;
  if (!codes || !scale || !zero_point || !g_new || !codes_out || !scale_out || !zero_point_out)
    return fail(QFTC_EINVAL, "accumulate: null pointer");
  if (int rc = require_device()) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  // the error flag lives in pinned host memory the kernel writes directly (no device
  // allocation, memset or copy per call; the call is one launch + one synchronisation)
  static thread_local uint32_t* flag = nullptr;
  if (!flag) QFTC_CUDA(cudaHostAlloc((void**)&flag, 4, cudaHostAllocMapped), "cudaHostAlloc");
  *flag = 0;
  uint32_t* dflag = nullptr;
  QFTC_CUDA(cudaHostGetDevicePointer((void**)&dflag, flag, 0), "cudaHostGetDevicePointer");
  QFTC_CUDA(launch_accumulate_state(codes, scale, zero_point, rows, cols, bit_width, g_new,
                                    codes_out, scale_out, zero_point_out, dflag, st),
            "accumulate");
  QFTC_CUDA(cudaStreamSynchronize(st), "sync");
  if (*(volatile uint32_t*)flag)
    return fail(QFTC_EINVAL, "affine_params_from_bounds: min > max in a channel");
  return QFTC_OK;
}

int qftc_dequantize(const uint8_t* codes, int rows, int cols, const float* scale,
                    const int32_t* zp, int channels, float* out, qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, "dequantize")) return rc;
  if (channels != 1 && channels != rows)
    return fail(QFTC_EINVAL, "dequantize: channel count does not match rows");
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_dequantize(codes, rows, cols, scale, zp, channels, out, false,
                              (cudaStream_t)stream),
            "dequantize");
  return QFTC_OK;
}

int qftc_dequantize_bf16(const uint8_t* codes, int rows, int cols, const float* scale,
                         const int32_t* zp, int channels, uint16_t* out,
                         qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, "dequantize")) return rc;
  if (channels != 1 && channels != rows)
    return fail(QFTC_EINVAL, "dequantize: channel count does not match rows");
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_dequantize(codes, rows, cols, scale, zp, channels, out, true,
                              (cudaStream_t)stream),
            "dequantize_bf16");
  return QFTC_OK;
}

int qftc_outlier_thresholds(const float* w, int rows, int cols, double fraction, int kind,
                            float* t_min, float* t_max, qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, "compute_outlier_thresholds")) return rc;
  if (!(fraction >= 0.0) || fraction >= 0.5)
    return fail(QFTC_EINVAL, "outlier fraction must be in [0, 0.5)");
  if (kind != QFTC_PERCENTILE && kind != QFTC_RANGE_FRACTION)
    return fail(QFTC_EINVAL, "threshold kind must be percentile or range-fraction");
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_thresholds(w, rows, cols, fraction, kind, t_min, t_max, (cudaStream_t)stream),
            "outlier_thresholds");
  return QFTC_OK;
}

int qftc_decompose_dense_sparse(const float* w, int rows, int cols, const float* t_min,
                                const float* t_max, int bit_width, uint8_t* codes, float* scale,
                                int32_t* zp, int32_t* row_ptr, int32_t* col_idx, float* values,
                                int64_t capacity, int64_t* nnz_host, qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, "decompose_dense_sparse")) return rc;
  if (int rc = require_bit_width(bit_width)) return rc;
  if (!w || !codes || !row_ptr) return fail(QFTC_EINVAL, "decompose: null pointer");
  if (int rc = require_device()) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  // params from thresholds (quantize.hpp:264) -- validates t_min <= t_max
  int rc = qftc_affine_params_from_bounds(t_min, t_max, rows, bit_width, scale, zp, stream);
  if (rc) return rc;
  int32_t* counts = nullptr;
  QFTC_CUDA(cudaMallocAsync((void**)&counts, (size_t)rows * 4, st), "alloc");
  cudaError_t e = decompose_codes(w, rows, cols, scale, zp, t_min, t_max, bit_width, codes,
                                  counts, st);
  if (e == cudaSuccess) e = csr_row_ptr(counts, rows, row_ptr, st, nullptr);
  int32_t nnz = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&nnz, row_ptr + rows, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(counts, st);
  QFTC_CUDA(e, "decompose codes");
  if (nnz_host) *nnz_host = nnz;
  if (nnz < 0) return fail(QFTC_ENOTSUP, "decompose: nnz above 2^31");
  if ((int64_t)nnz > capacity)
    return fail(QFTC_EOVERFLOW, "decompose: nnz " + std::to_string(nnz) + " exceeds capacity " +
                                    std::to_string(capacity));
  if (nnz > 0) {
    if (!col_idx || !values) return fail(QFTC_EINVAL, "decompose: null CSR arrays");
    QFTC_CUDA(decompose_csr(w, rows, cols, t_min, t_max, row_ptr, col_idx, values, st),
              "decompose csr");
  }
  return QFTC_OK;
}

static int reconstruct_impl(const uint8_t* codes, int rows, int cols, const float* scale,
                            const int32_t* zp, const int32_t* row_start,
                            const int32_t* row_count, const int32_t* col_idx,
                            const float* values, void* out, bool bf16, qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, "reconstruct")) return rc;
  if (!codes || !scale || !zp || !row_start || !out)
    return fail(QFTC_EINVAL, "reconstruct: null pointer");
  if (int rc = require_device()) return rc;
  qftc_expand_tensor t{};
  t.rows = rows;
  t.cols = cols;
  t.codes = codes;
  t.scale = scale;
  t.zero_point = zp;
  t.row_start = row_start;
  t.row_count = row_count;
  t.col_idx = col_idx;
  t.values = values;
  t.out = out;
  QFTC_CUDA(launch_expand(&t, 1, bf16, (cudaStream_t)stream), "reconstruct kernel");
  return QFTC_OK;
}

int qftc_expand(const qftc_expand_tensor* tensors, int n_tensors, int bf16,
                qftc_stream_t stream) {
  if (n_tensors < 0 || (n_tensors > 0 && !tensors))
    return fail(QFTC_EINVAL, "expand: bad tensor list");
  for (int i = 0; i < n_tensors; ++i) {
    const qftc_expand_tensor& t = tensors[i];
    if (int rc = require_shape(t.rows, t.cols, "expand")) return rc;
    if (!t.codes || !t.scale || !t.zero_point || !t.row_start || !t.out)
      return fail(QFTC_EINVAL, "expand: null pointer in tensor " + std::to_string(i));
  }
  if (n_tensors == 0) return QFTC_OK;
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_expand(tensors, n_tensors, bf16 != 0, (cudaStream_t)stream), "expand kernel");
  return QFTC_OK;
}

int qftc_expand_plan_create(qftc_expand_plan** plan, const qftc_expand_tensor* tensors,
                            int n_tensors, int bf16, qftc_stream_t stream) {
  if (!plan || n_tensors < 0 || (n_tensors > 0 && !tensors))
    return fail(QFTC_EINVAL, "expand_plan_create: bad tensor list");
  for (int i = 0; i < n_tensors; ++i) {
    const qftc_expand_tensor& t = tensors[i];
    if (int rc = require_shape(t.rows, t.cols, "expand")) return rc;
    if (!t.codes || !t.scale || !t.zero_point || !t.row_start || !t.out)
      return fail(QFTC_EINVAL, "expand: null pointer in tensor " + std::to_string(i));
  }
  if (int rc = require_device()) return rc;
  void* p = nullptr;
  QFTC_CUDA(expand_plan_create(tensors, n_tensors, bf16 != 0, (cudaStream_t)stream, &p),
            "expand_plan_create");
  *plan = reinterpret_cast<qftc_expand_plan*>(p);
  return QFTC_OK;
}

int qftc_expand_plan_run(qftc_expand_plan* plan, qftc_stream_t stream) {
  if (!plan) return fail(QFTC_EINVAL, "expand_plan_run: null plan");
  QFTC_CUDA(expand_plan_run(plan, (cudaStream_t)stream), "expand kernel");
  return QFTC_OK;
}

int qftc_expand_plan_destroy(qftc_expand_plan* plan) {
  expand_plan_destroy(plan);
  return QFTC_OK;
}

int64_t qftc_dequant_gemm_workspace_bytes(int n, int k) {
  return n > 0 && k > 0 ? (int64_t)dq_gemm_workspace_bytes(n, k) : 0;
}

int qftc_dequant_gemm(const void* x_bf16, int m, int k, const uint8_t* codes, int n,
                      const float* scale, const int32_t* zero_point, const int32_t* row_start,
                      const int32_t* row_count, const int32_t* col_idx, const float* values,
                      void* y_bf16, void* workspace, qftc_stream_t stream) {
  if (m <= 0 || n <= 0 || k <= 0) return fail(QFTC_EINVAL, "dequant_gemm: empty shape");
  if (k % 64 != 0) return fail(QFTC_ENOTSUP, "dequant_gemm: K must be a multiple of 64");
  if (!x_bf16 || !codes || !scale || !zero_point || !row_start || !col_idx || !values ||
      !y_bf16 || !workspace)
    return fail(QFTC_EINVAL, "dequant_gemm: null pointer");
  if (!al16(x_bf16) || !al16(codes) || !al16(y_bf16))
    return fail(QFTC_EINVAL, "dequant_gemm: x, codes and y must be 16-byte aligned");
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_dq_gemm(x_bf16, m, k, codes, n, scale, zero_point, row_start, row_count,
                           col_idx, values, y_bf16, workspace, (cudaStream_t)stream),
            "dequant_gemm kernel");
  return QFTC_OK;
}

int64_t qftc_dequant_gemm_t_workspace_bytes(int out_features, int in_features) {
  return out_features > 0 && in_features > 0
             ? (int64_t)dq_gemm_t_workspace_bytes(out_features, in_features)
             : 0;
}

int qftc_dequant_gemm_t(const void* dy_bf16, int tokens, int out_features, const uint8_t* codes,
                        int in_features, const float* scale, const int32_t* zero_point,
                        const int32_t* row_start, const int32_t* row_count,
                        const int32_t* col_idx, const float* values, void* dx_bf16,
                        void* workspace, qftc_stream_t stream) {
  if (tokens <= 0 || out_features <= 0 || in_features <= 0)
    return fail(QFTC_EINVAL, "dequant_gemm_t: empty shape");
  if (out_features % 64 != 0 || in_features % 64 != 0)
    return fail(QFTC_ENOTSUP, "dequant_gemm_t: out_features and in_features must be multiples of 64");
  if (!dy_bf16 || !codes || !scale || !zero_point || !row_start || !col_idx || !values ||
      !dx_bf16 || !workspace)
    return fail(QFTC_EINVAL, "dequant_gemm_t: null pointer");
  if (!al16(dy_bf16) || !al16(codes) || !al16(dx_bf16))
    return fail(QFTC_EINVAL, "dequant_gemm_t: dy, codes and dx must be 16-byte aligned");
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_dq_gemm_t(dy_bf16, tokens, out_features, codes, in_features, scale, zero_point,
                             row_start, row_count, col_idx, values, dx_bf16, workspace,
                             (cudaStream_t)stream),
            "dequant_gemm_t kernel");
  return QFTC_OK;
}

int qftc_dequant_gemm_index(const int32_t* row_start, const int32_t* row_count,
                            const int32_t* col_idx, int rows, int cols, void* index,
                            qftc_stream_t stream) {
  if (rows <= 0 || cols <= 0 || cols % 64 != 0)
    return fail(QFTC_EINVAL, "dequant_gemm_index: bad shape (cols must be a multiple of 64)");
  if (!row_start || !col_idx || !index) return fail(QFTC_EINVAL, "dequant_gemm_index: null pointer");
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_csr_tile_index(row_start, row_count, col_idx, rows, cols / 32, 32,
                                  reinterpret_cast<int32_t*>(index), (cudaStream_t)stream),
            "dequant_gemm_index kernel");
  return QFTC_OK;
}

int qftc_dequant_gemm_prebuilt(const void* x_bf16, int m, int k, const uint8_t* codes, int n,
                               const float* scale, const int32_t* zero_point,
                               const int32_t* col_idx, const float* values, const void* index,
                               void* y_bf16, qftc_stream_t stream) {
  if (m <= 0 || n <= 0 || k <= 0) return fail(QFTC_EINVAL, "dequant_gemm: empty shape");
  if (k % 64 != 0) return fail(QFTC_ENOTSUP, "dequant_gemm: K must be a multiple of 64");
  if (!x_bf16 || !codes || !scale || !zero_point || !col_idx || !values || !index || !y_bf16)
    return fail(QFTC_EINVAL, "dequant_gemm: null pointer");
  if (!al16(x_bf16) || !al16(codes) || !al16(y_bf16))
    return fail(QFTC_EINVAL, "dequant_gemm: x, codes and y must be 16-byte aligned");
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_dq_gemm(x_bf16, m, k, codes, n, scale, zero_point, nullptr, nullptr, col_idx,
                           values, y_bf16, const_cast<void*>(index), (cudaStream_t)stream, false),
            "dequant_gemm kernel");
  return QFTC_OK;
}

int qftc_dequant_gemm_t_prebuilt(const void* dy_bf16, int tokens, int out_features,
                                 const uint8_t* codes, int in_features, const float* scale,
                                 const int32_t* zero_point, const int32_t* col_idx,
                                 const float* values, const void* index, void* dx_bf16,
                                 qftc_stream_t stream) {
  if (tokens <= 0 || out_features <= 0 || in_features <= 0)
    return fail(QFTC_EINVAL, "dequant_gemm_t: empty shape");
  if (out_features % 64 != 0 || in_features % 64 != 0)
    return fail(QFTC_ENOTSUP, "dequant_gemm_t: out_features and in_features must be multiples of 64");
  if (!dy_bf16 || !codes || !scale || !zero_point || !col_idx || !values || !index || !dx_bf16)
    return fail(QFTC_EINVAL, "dequant_gemm_t: null pointer");
  if (!al16(dy_bf16) || !al16(codes) || !al16(dx_bf16))
    return fail(QFTC_EINVAL, "dequant_gemm_t: dy, codes and dx must be 16-byte aligned");
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_dq_gemm_t(dy_bf16, tokens, out_features, codes, in_features, scale, zero_point,
                             nullptr, nullptr, col_idx, values, dx_bf16, const_cast<void*>(index),
                             (cudaStream_t)stream, false),
            "dequant_gemm_t kernel");
  return QFTC_OK;
}

int64_t qftc_wgrad_workspace_bytes(int out_features) {
  return out_features > 0 ? (int64_t)wgrad_workspace_bytes(out_features) : 0;
}

int qftc_wgrad_quant(const void* dy_bf16, const void* x_bf16, int tokens, int out_features,
                     int in_features, int bit_width, int accumulate, uint8_t* codes, float* scale,
                     int32_t* zero_point, float* g_out, double* norm_sq, void* workspace,
                     int check, qftc_stream_t stream) {
  if (tokens <= 0 || out_features <= 0 || in_features <= 0)
    return fail(QFTC_EINVAL, "wgrad_quant: empty shape");
  if (int rc = require_bit_width(bit_width)) return rc;
  if (in_features % 64 != 0 || out_features % 8 != 0)
    return fail(QFTC_ENOTSUP, "wgrad_quant: in_features % 64 and out_features % 8 must be 0");
  if (!dy_bf16 || !x_bf16 || !codes || !scale || !zero_point || !workspace)
    return fail(QFTC_EINVAL, "wgrad_quant: null pointer");
  if (!al16(dy_bf16) || !al16(x_bf16) || !al16(codes) || (g_out && !al16(g_out)))
    return fail(QFTC_EINVAL, "wgrad_quant: dy, x, codes and g_out must be 16-byte aligned");
  if (int rc = require_device()) return rc;
  static const uint32_t lbo = (uint32_t)(getenv("QFT_WG_LBO") ? atoi(getenv("QFT_WG_LBO")) : 0);
  static const uint32_t sbo = (uint32_t)(getenv("QFT_WG_SBO") ? atoi(getenv("QFT_WG_SBO")) : 0);
  cudaStream_t st = (cudaStream_t)stream;
  const cudaError_t e = launch_wgrad_quant(dy_bf16, x_bf16, tokens, out_features, in_features,
                                           bit_width, accumulate, codes, scale, zero_point, g_out,
                                           norm_sq, workspace, lbo, sbo, st);
  if (e == cudaErrorInvalidConfiguration)
    return fail(QFTC_ENOTSUP, "wgrad_quant: a gradient row spans more tiles than SMs");
  QFTC_CUDA(e, "wgrad_quant kernel");
  if (check) {
    const int64_t wb = (int64_t)wgrad_workspace_bytes(out_features);
    uint32_t h = 0;
    QFTC_CUDA(cudaMemcpyAsync(&h, reinterpret_cast<char*>(workspace) + wb - 4, 4,
                              cudaMemcpyDeviceToHost, st), "copy");
    QFTC_CUDA(cudaStreamSynchronize(st), "sync");
    if (h) return fail(QFTC_EINVAL, "affine_params_from_bounds: min > max in a channel");
  }
  return QFTC_OK;
}

static int pack_impl(const uint8_t* src, int rows, int cols, int bits, uint8_t* dst,
                     bool unpack, qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, unpack ? "unpack_codes" : "pack_codes")) return rc;
  if (bits < 2 || bits > 8) return fail(QFTC_EINVAL, "pack_codes: bits must be in [2, 8]");
  if (!src || !dst) return fail(QFTC_EINVAL, "pack_codes: null pointer");
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_pack_codes(src, rows, cols, bits, dst, unpack, (cudaStream_t)stream),
            "pack_codes kernel");
  return QFTC_OK;
}

int qftc_pack_codes(const uint8_t* codes, int rows, int cols, int bits, uint8_t* packed,
                    qftc_stream_t stream) {
  return pack_impl(codes, rows, cols, bits, packed, false, stream);
}

int qftc_unpack_codes(const uint8_t* packed, int rows, int cols, int bits, uint8_t* codes,
                      qftc_stream_t stream) {
  return pack_impl(packed, rows, cols, bits, codes, true, stream);
}

static int mom_impl(const uint8_t* codes, const float* scale, const int32_t* zp, int rows,
                    int cols, int bits, int block, uint8_t* out, float* oscale, int32_t* ozp,
                    bool from_blocks, qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, "momentum_blocks")) return rc;
  if (int rc = require_bit_width(bits)) return rc;
  if (block <= 0) return fail(QFTC_EINVAL, "momentum_blocks: block must be positive");
  if (!codes || !scale || !zp || !out || !oscale || !ozp)
    return fail(QFTC_EINVAL, "momentum_blocks: null pointer");
  if (int rc = require_device()) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* err = nullptr;
  QFTC_CUDA(cudaMallocAsync((void**)&err, 4, st), "momentum_blocks: alloc");
  QFTC_CUDA(cudaMemsetAsync(err, 0, 4, st), "momentum_blocks: memset");
  cudaError_t e = launch_mom_blocks(codes, scale, zp, rows, cols, bits, block, out, oscale, ozp,
                                    from_blocks, err, st);
  uint32_t h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, err, 4, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(err, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  QFTC_CUDA(e, "momentum_blocks kernel");
  if (h) return fail(QFTC_EINVAL, "affine_params_from_bounds: min > max in momentum channel");
  return QFTC_OK;
}

int qftc_momentum_to_blocks(const uint8_t* codes, const float* scale, const int32_t* zero_point,
                            int rows, int cols, int bit_width, int block, uint8_t* block_codes,
                            float* block_scale, int32_t* block_zero_point,
                            qftc_stream_t stream) {
  return mom_impl(codes, scale, zero_point, rows, cols, bit_width, block, block_codes,
                  block_scale, block_zero_point, false, stream);
}

int qftc_momentum_from_blocks(const uint8_t* block_codes, const float* block_scale,
                              const int32_t* block_zero_point, int rows, int cols, int bit_width,
                              int block, uint8_t* codes, float* scale, int32_t* zero_point,
                              qftc_stream_t stream) {
  return mom_impl(block_codes, block_scale, block_zero_point, rows, cols, bit_width, block, codes,
                  scale, zero_point, true, stream);
}

int qftc_reconstruct(const uint8_t* codes, int rows, int cols, const float* scale,
                     const int32_t* zp, const int32_t* row_ptr, const int32_t* col_idx,
                     const float* values, float* out, qftc_stream_t stream) {
  return reconstruct_impl(codes, rows, cols, scale, zp, row_ptr, nullptr, col_idx, values, out,
                          false, stream);
}

int qftc_reconstruct_bf16(const uint8_t* codes, int rows, int cols, const float* scale,
                          const int32_t* zp, const int32_t* row_ptr, const int32_t* col_idx,
                          const float* values, uint16_t* out, qftc_stream_t stream) {
  return reconstruct_impl(codes, rows, cols, scale, zp, row_ptr, nullptr, col_idx, values, out,
                          true, stream);
}

int qftc_reconstruct_slots(const uint8_t* codes, int rows, int cols, const float* scale,
                           const int32_t* zp, const int32_t* row_start,
                           const int32_t* row_count, const int32_t* col_idx,
                           const float* values, void* out, int bf16, qftc_stream_t stream) {
  if (!row_count) return fail(QFTC_EINVAL, "reconstruct_slots: row_count is required");
  return reconstruct_impl(codes, rows, cols, scale, zp, row_start, row_count, col_idx, values,
                          out, bf16 != 0, stream);
}

// ------------------------------------------------------------------ slotted CSR
int qftc_csr_replan_caps(const uint8_t* codes, int rows, int cols, int bit_width,
                         const int32_t* count_out, const int32_t* count_in, int level,
                         int growth_mult, int64_t* caps, qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, "csr_replan_caps")) return rc;
  if (int rc = require_bit_width(bit_width)) return rc;
  if (!codes || !count_out || !count_in || !caps)
    return fail(QFTC_EINVAL, "csr_replan_caps: null pointer");
  if (level < 0 || growth_mult < 0) return fail(QFTC_EINVAL, "csr_replan_caps: negative level");
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_replan_caps(codes, rows, cols, bit_width, count_out, count_in, level,
                               growth_mult, caps, (cudaStream_t)stream),
            "csr_replan_caps");
  return QFTC_OK;
}

int qftc_csr_plan_slots(const int32_t* counts, const int32_t* row_ptr, int rows, int slack,
                        int32_t* row_start, int64_t* total_host, qftc_stream_t stream) {
  if (rows <= 0) return fail(QFTC_EINVAL, "csr_plan_slots: no rows");
  if (!counts && !row_ptr) return fail(QFTC_EINVAL, "csr_plan_slots: need counts or row_ptr");
  if (int rc = require_device()) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  QFTC_CUDA(csr_plan_slots(counts, row_ptr, rows, slack < 0 ? 0 : slack, row_start, st),
            "csr_plan_slots");
  if (total_host) {
    int32_t t = 0;
    QFTC_CUDA(cudaMemcpyAsync(&t, row_start + rows, 4, cudaMemcpyDeviceToHost, st), "copy");
    QFTC_CUDA(cudaStreamSynchronize(st), "sync");
    *total_host = t;
  }
  return QFTC_OK;
}

int qftc_csr_copy_rows(int rows, const int32_t* src_start, const int32_t* src_count,
                       const int32_t* src_col, const float* src_val, const int32_t* dst_start,
                       int32_t* dst_col, float* dst_val, int64_t dst_capacity,
                       qftc_stream_t stream) {
  if (rows <= 0) return QFTC_OK;
  if (int rc = require_device()) return rc;
  QFTC_CUDA(csr_copy_rows(rows, src_start, src_count, src_col, src_val, dst_start, dst_col,
                          dst_val, dst_capacity, (cudaStream_t)stream),
            "csr_copy_rows");
  return QFTC_OK;
}

int qftc_csr_compact(int rows, const int32_t* row_start, const int32_t* row_count,
                     const int32_t* col_idx, const float* values, int32_t* row_ptr,
                     int32_t* col_out, float* val_out, int64_t capacity, int64_t* nnz_host,
                     qftc_stream_t stream) {
  if (rows <= 0) return fail(QFTC_EINVAL, "csr_compact: no rows");
  if (!row_count) return fail(QFTC_EINVAL, "csr_compact: row_count is required");
  if (int rc = require_device()) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  QFTC_CUDA(csr_row_ptr(row_count, rows, row_ptr, st, row_start), "csr_row_ptr");
  QFTC_CUDA(csr_copy_rows(rows, row_start, row_count, col_idx, values, row_ptr, col_out, val_out,
                          capacity, st),
            "csr_copy_rows");
  int32_t n = 0;
  QFTC_CUDA(cudaMemcpyAsync(&n, row_ptr + rows, 4, cudaMemcpyDeviceToHost, st), "copy");
  QFTC_CUDA(cudaStreamSynchronize(st), "sync");
  if (nnz_host) *nnz_host = n;
  if (n > capacity)
    return fail(QFTC_EOVERFLOW, "csr_compact: nnz " + std::to_string(n) + " exceeds capacity " +
                                    std::to_string(capacity));
  return QFTC_OK;
}

int qftc_csr_pack_plan_create(qftc_csr_pack_plan** plan, const qftc_pack_segment* segs,
                              int nseg, int nwidth, qftc_stream_t stream) {
  if (!plan || nseg < 0 || (nseg > 0 && !segs) || nwidth <= 0 || nwidth > QFT_PACK_MAXW)
    return fail(QFTC_EINVAL, "csr_pack_plan_create: need a segment table and 1..8 classes");
  for (int i = 0; i < nseg; ++i)
    if (segs[i].rows < 0 || segs[i].width < 0 || segs[i].width >= nwidth || segs[i].rs_off < 0 ||
        segs[i].cnt_off < 0 || segs[i].rs_off + segs[i].rows >= (int64_t)INT32_MAX ||
        segs[i].cnt_off + segs[i].rows > (int64_t)INT32_MAX)
      return fail(QFTC_EINVAL, "csr_pack_plan_create: bad segment " + std::to_string(i));
  if (int rc = require_device()) return rc;
  void* p = nullptr;
  QFTC_CUDA(csr_pack_plan_create(segs, nseg, nwidth, (cudaStream_t)stream, &p),
            "csr_pack_plan_create");
  *plan = reinterpret_cast<qftc_csr_pack_plan*>(p);
  return QFTC_OK;
}

int qftc_csr_pack_run(qftc_csr_pack_plan* plan, const int32_t* row_start,
                      const int32_t* row_count, const int32_t* const* col_in,
                      const float* const* val_in, int32_t* const* col_out,
                      float* const* val_out, const int64_t* base, int32_t* row_start_out,
                      qftc_stream_t stream) {
  if (!plan || !row_start || !row_count || !row_start_out || !col_in || !val_in || !col_out ||
      !val_out || !base)
    return fail(QFTC_EINVAL, "csr_pack_run: null argument");
  PackWidths P{};
  const int nwidth = csr_pack_nwidth(plan);
  for (int w = 0; w < nwidth; ++w) {
    P.col_in[w] = col_in[w];
    P.val_in[w] = val_in[w];
    P.col_out[w] = col_out[w];
    P.val_out[w] = val_out[w];
    P.base[w] = base[w];
  }
  QFTC_CUDA(csr_pack_run(plan, row_start, row_count, P, row_start_out, (cudaStream_t)stream),
            "csr_pack");
  return QFTC_OK;
}

int qftc_csr_pack_plan_destroy(qftc_csr_pack_plan* plan) {
  csr_pack_plan_destroy(plan);
  return QFTC_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ plans
struct qftc_plan {
  Scratch sc;
  int n = 0;
  int total_rows = 0;
  int bit_width = 8;
  int grad_kind = 0;
  int cols_p = 16;
  int oldcap = 128;
  int use_bulk = 1;
  int uniform_cols = 0;       // every tensor's row length (0: mixed)
  bool rows_path = false;     // v6 rows kernel (prep + stable rows + general rows)
  RowPrep* prep = nullptr;    // per-row records
  RowBlock* xlist = nullptr;  // general-tier rows
  RowsCache rc;               // resolved launches of the rows path (+ its row-list counters)
  // raw (f32/bf16) gradient on the rows path: k_grad_quant writes quantize_state(g) into
  // this u8 scratch (the GradientStack entry) and the rows kernel steps from it
  bool gq = false;
  void* gq_base = nullptr;
  KLaunch gql;
  // the fused ZeRO-1 reduce-scatter: the raw gradient summed from npeer peer buffers
  int npeer = 0;
  int64_t* peer_deltas = nullptr;  // device [16]
  KLaunch rsl;
  KLaunch gen[2];             // general path (no rows kernel): by weight decay == 0
  cudaStream_t side = nullptr;     // qftc_plans_step: this plan's stream ...
  cudaEvent_t ev_fork = nullptr;   // ... forked from the caller's stream
  cudaEvent_t ev_done = nullptr;   // ... and joined back
  const char* last_kernel = "";  // the main kernel instance of the last step
  volatile uint32_t* oflag_host = nullptr;  // mapped pinned copy of the overflow flag
  uint32_t* oflag_dev = nullptr;
  int slotted[2] = {0, 0};
  int32_t* col[2] = {nullptr, nullptr};
  float* val[2] = {nullptr, nullptr};
  int64_t cap[2] = {0, 0};
};

extern "C" {

int qftc_plan_create(qftc_plan** out, const qftc_lion_tensor* ts, int n, int bit_width,
                     int grad_kind, int32_t* col_idx[2], float* values[2],
                     const int64_t capacity[2], qftc_stream_t stream) {
  if (!out || !ts || n <= 0) return fail(QFTC_EINVAL, "plan_create: no tensors");
  if (int rc = require_bit_width(bit_width)) return rc;
  if (grad_kind < QFTC_GRAD_U8 || grad_kind > QFTC_GRAD_BF16)
    return fail(QFTC_EINVAL, "plan_create: bad gradient kind");
  if (int rc = require_device()) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<DevTensor> dts((size_t)n);
  int64_t rows = 0;
  int maxc = 1;
  int ucols = ts[0].cols;
  bool bulk = true;
  bool slotted[2] = {true, true};
  for (int i = 0; i < n; ++i) {
    const qftc_lion_tensor& t = ts[i];
    if (t.rows <= 0 || t.cols <= 0)
      return fail(QFTC_EINVAL, "lion step: empty tensor " + std::to_string(i));
    if (t.cols > step_kernel_max_cols())
      return fail(QFTC_ENOTSUP, "lion step: cols above " + std::to_string(step_kernel_max_cols()));
    DevTensor& d = dts[(size_t)i];
    d = DevTensor{};
    d.rows = t.rows;
    d.cols = t.cols;
    d.row_base = (int32_t)rows;
    for (int k = 0; k < 2; ++k) {
      d.w_codes[k] = t.w_codes[k];
      d.rs[k] = t.row_start[k];
      d.cnt[k] = t.row_count[k];
      d.m_codes[k] = t.m_codes[k];
      d.m_scale[k] = t.m_scale[k];
      d.m_zp[k] = t.m_zero_point[k];
      bulk = bulk && al16(t.w_codes[k]) && al16(t.m_codes[k]);
      slotted[k] = slotted[k] && t.row_count[k] != nullptr;
    }
    d.w_scale = t.w_scale;
    d.w_zp = t.w_zero_point;
    d.t_min = t.t_min;
    d.t_max = t.t_max;
    d.g_codes = t.g_codes;
    d.g_scale = t.g_scale;
    d.g_zp = t.g_zero_point;
    d.g_raw = t.g_raw;
    if (grad_kind == QFTC_GRAD_U8) {
      if (!t.g_codes || !t.g_scale || !t.g_zero_point)
        return fail(QFTC_EINVAL, "lion step: gradient codes/params missing");
      bulk = bulk && al16(t.g_codes);
    } else {
      if (!t.g_raw) return fail(QFTC_EINVAL, "lion step: raw gradient missing");
      bulk = bulk && al16(t.g_raw);
    }
    bulk = bulk && (t.cols % 16 == 0);
    rows += t.rows;
    if (t.cols > maxc) maxc = t.cols;
    if (t.cols != ucols) ucols = 0;
  }
  if (rows > 0x7fffffff) return fail(QFTC_ENOTSUP, "plan: more than 2^31 rows");
  const char* no_rows = getenv("QFT_NO_ROWS_KERNEL");
  const char* no_gq = getenv("QFT_NO_GRAD_QUANT");
  const bool rows_ok = rows_kernel_eligible(QFTC_GRAD_U8, bulk ? 1 : 0, ucols) &&
                       !(no_rows && no_rows[0] == '1');
  // raw gradients on the rows path: quantize_state(g) into a plan-owned u8 entry first
  const bool gq = rows_ok && grad_kind != QFTC_GRAD_U8 && !(no_gq && no_gq[0] == '1');
  void* gq_base = nullptr;
  if (gq) {
    size_t code_bytes = 0;
    for (int i = 0; i < n; ++i) code_bytes += ((size_t)ts[i].rows * ts[i].cols + 15) & ~(size_t)15;
    const size_t row_bytes = ((size_t)rows * 4 + 255) & ~(size_t)255;
    cudaError_t e = cudaMallocAsync(&gq_base, code_bytes + 2 * row_bytes, st);
    if (e != cudaSuccess)
      return fail(QFTC_ECUDA, std::string("plan_create: gradient scratch: ") + cudaGetErrorString(e));
    uint8_t* c = reinterpret_cast<uint8_t*>(gq_base);
    float* sc = reinterpret_cast<float*>(c + code_bytes);
    int32_t* zp = reinterpret_cast<int32_t*>(c + code_bytes + row_bytes);
    int64_t r0 = 0;
    for (int i = 0; i < n; ++i) {
      dts[(size_t)i].g_codes = c;
      dts[(size_t)i].g_scale = sc + r0;
      dts[(size_t)i].g_zp = zp + r0;
      c += ((size_t)ts[i].rows * ts[i].cols + 15) & ~(size_t)15;
      r0 += ts[i].rows;
    }
  }
  auto* p = new qftc_plan;
  p->gq = gq;
  p->gq_base = gq_base;
  int rc = scratch_alloc(p->sc, dts, 0, st);
  if (rc) {
    if (gq_base) cudaFree(gq_base);
    delete p;
    return rc;
  }
  p->n = n;
  p->total_rows = (int)rows;
  p->bit_width = bit_width;
  p->grad_kind = grad_kind;
  p->cols_p = (maxc + 15) & ~15;
  p->use_bulk = bulk ? 1 : 0;
  {
    const StepCfg cfg = pick_step_config(grad_kind, p->cols_p);
    p->oldcap = cfg.oldcap;
  }
  p->uniform_cols = ucols;
  p->rows_path = rows_ok && (grad_kind == QFTC_GRAD_U8 || gq);
  if (gq) {
    cudaError_t e = resolve_grad_quant(grad_kind, ucols, (int)rows, &p->gql);
    if (e != cudaSuccess) {
      qftc_plan_destroy(p);
      return fail(QFTC_ECUDA, std::string("plan_create: gradient quantizer: ") + cudaGetErrorString(e));
    }
  }
  if (p->rows_path) {
    cudaError_t e = cudaMallocAsync((void**)&p->prep, sizeof(RowPrep) * (size_t)rows, st);
    if (e == cudaSuccess)
      e = cudaMallocAsync((void**)&p->xlist, sizeof(RowBlock) * (size_t)rows, st);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&p->rc.xcount, 64, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->rc.xcount, 0, 64, st);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&p->rc.slist, sizeof(int32_t) * (size_t)rows, st);
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&p->rc.glist, sizeof(int32_t) * (size_t)rows, st);
    const size_t nb = ((size_t)rows + 255) / 256;
    if (e == cudaSuccess) e = cudaMallocAsync((void**)&p->rc.pstatus, 8 * nb, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->rc.pstatus, 0, 8 * nb, st);
    const char* no_gen = getenv("QFT_NO_GEN");
    p->rc.gen_on = (no_gen && no_gen[0] == '1') ? 0 : 1;
    const char* allrows = getenv("QFT_STABLE_ALLROWS");
    p->rc.stable_allrows = (allrows && allrows[0] == '1') ? 1 : 0;
    const char* no_route = getenv("QFT_NO_ROUTE");
    p->rc.route_on = (no_route && no_route[0] == '1') ? 0 : 1;
    if (e == cudaSuccess) {
      void* hp = nullptr;
      if (cudaHostAlloc(&hp, 64, cudaHostAllocMapped) == cudaSuccess) {
        p->rc.seen_host = reinterpret_cast<volatile int32_t*>(hp);
        p->rc.seen_host[0] = p->rc.seen_host[1] = (int32_t)rows;  // unknown: full grids
        p->rc.seen_host[2] = (int32_t)rows;                         // ... and no routing
        void* dp = nullptr;
        if (cudaHostGetDevicePointer(&dp, hp, 0) == cudaSuccess) p->rc.seen_dev = (int32_t*)dp;
      }
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&p->rc.sms, cudaDevAttrMultiProcessorCount, dev);
    }
    if (e != cudaSuccess) {
      qftc_plan_destroy(p);
      return fail(QFTC_ECUDA, std::string("plan_create: ") + cudaGetErrorString(e));
    }
  }
  {
    // the overflow flag, also written to mapped pinned memory so the host sees it at the
    // next step without a synchronisation (qftc_plan_pending_overflow)
    void* hp = nullptr;
    if (cudaHostAlloc(&hp, 64, cudaHostAllocMapped) == cudaSuccess) {
      p->oflag_host = reinterpret_cast<volatile uint32_t*>(hp);
      *p->oflag_host = 0u;
      void* dp = nullptr;
      if (cudaHostGetDevicePointer(&dp, hp, 0) == cudaSuccess) p->oflag_dev = (uint32_t*)dp;
    }
  }
  for (int k = 0; k < 2; ++k) {
    p->col[k] = col_idx ? col_idx[k] : nullptr;
    p->val[k] = values ? values[k] : nullptr;
    p->cap[k] = capacity ? capacity[k] : 0;
    p->slotted[k] = slotted[k] && al16(p->col[k]) && al16(p->val[k]) ? 1 : 0;
  }
  *out = p;
  return QFTC_OK;
}

int qftc_plan_set_arena(qftc_plan* p, int32_t* col_idx[2], float* values[2],
                        const int64_t capacity[2]) {
  if (!p) return fail(QFTC_EINVAL, "plan: null");
  for (int k = 0; k < 2; ++k) {
    p->col[k] = col_idx[k];
    p->val[k] = values[k];
    p->cap[k] = capacity[k];
    p->slotted[k] = p->slotted[k] && al16(col_idx[k]) && al16(values[k]);
  }
  return QFTC_OK;
}

int qftc_plan_step(qftc_plan* p, int flip, qftc_lion_hyper h, qftc_stream_t stream) {
  if (!p) return fail(QFTC_EINVAL, "plan: null");
  if (flip != 0 && flip != 1) return fail(QFTC_EINVAL, "plan_step: flip must be 0 or 1");
  LaunchArgs a{};
  a.tensors = p->sc.tensors;
  a.blocks = p->sc.blocks;
  a.n_tensors = p->n;
  a.n_blocks = p->sc.n_blocks;
  a.total_rows = p->total_rows;
  a.flip = flip;
  a.bit_width = p->bit_width;
  a.lr = h.lr;
  a.b1 = h.beta1;
  a.b2 = h.beta2;
  a.wd = h.weight_decay;
  a.col_in = p->col[flip];
  a.val_in = p->val[flip];
  a.col_out = p->col[1 - flip];
  a.val_out = p->val[1 - flip];
  a.cap_out = p->cap[1 - flip];
  a.hdr = p->sc.hdr;
  a.status = p->sc.status;
  a.cols_p = p->cols_p;
  a.oldcap = p->oldcap;
  a.use_bulk = p->use_bulk;
  a.slotted_in = p->slotted[flip];
  a.oflag = p->oflag_dev;
  if (p->rows_path) {
    a.cols_p = p->uniform_cols;
    a.oldcap6 = rows_kernel_oldcap(p->uniform_cols);
    a.prep = p->prep;
    a.xlist = p->xlist;
    if (p->gq && p->npeer > 0)
      QFTC_CUDA(launch_rs_grad_quant(p->rsl, a, p->peer_deltas, p->npeer, (cudaStream_t)stream),
                "fused reduce-scatter + quantize_state");
    else if (p->gq)
      QFTC_CUDA(launch_k2(p->gql, a, (cudaStream_t)stream), "gradient quantize_state");
    QFTC_CUDA(launch_rows_step(a, p->rc, (cudaStream_t)stream), "lion step (rows kernel)");
    p->last_kernel = (p->rc.routed ? p->rc.genrows : p->rc.rows)[a.slotted_in ? 1 : 0].name;
    return QFTC_OK;
  }
  KLaunch& k = p->gen[a.wd == 0.0f ? 1 : 0];
  if (!k.fn) QFTC_CUDA(resolve_step_kernel(p->grad_kind, a, &k), "lion step kernel (resolve)");
  QFTC_CUDA(launch_k(k, a, (cudaStream_t)stream), "lion step kernel");
  p->last_kernel = k.name;
  return QFTC_OK;
}

int qftc_plan_set_peer_gradients(qftc_plan* p, const int64_t* byte_deltas, int npeer) {
  if (!p || npeer < 0 || npeer > 16 || (npeer > 0 && !byte_deltas))
    return fail(QFTC_EINVAL, "plan_set_peer_gradients: bad arguments");
  if (npeer > 0 && !(p->gq && p->grad_kind == QFTC_GRAD_BF16))
    return fail(QFTC_ENOTSUP, "plan_set_peer_gradients: needs a bf16 raw-gradient rows-path plan");
  if (!p->peer_deltas)
    QFTC_CUDA(cudaMalloc((void**)&p->peer_deltas, 16 * sizeof(int64_t)), "peer deltas");
  if (npeer > 0) {
    QFTC_CUDA(cudaMemcpy(p->peer_deltas, byte_deltas, (size_t)npeer * sizeof(int64_t),
                         cudaMemcpyHostToDevice), "peer deltas");
    if (!p->rsl.fn) QFTC_CUDA(resolve_rs_grad_quant(p->uniform_cols, p->total_rows, &p->rsl),
                              "fused reduce-scatter kernel (resolve)");
  }
  p->npeer = npeer;
  return QFTC_OK;
}

int qftc_ipc_handle(const void* ptr, unsigned char handle[64], int64_t* offset) {
  if (!ptr || !handle || !offset) return fail(QFTC_EINVAL, "ipc_handle: null argument");
  if (int rc = require_device()) return rc;
  using PFN_range = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static PFN_range range = nullptr;
  if (!range) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return fail(QFTC_ENOTSUP, "ipc_handle: cuMemGetAddressRange unavailable");
    range = reinterpret_cast<PFN_range>(fp);
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range(&base, &size, (CUdeviceptr)(uintptr_t)ptr) != CUDA_SUCCESS)
    return fail(QFTC_EINVAL, "ipc_handle: not a device allocation");
  cudaIpcMemHandle_t h;
  QFTC_CUDA(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base), "cudaIpcGetMemHandle");
  memcpy(handle, &h, 64);
  *offset = (int64_t)((uintptr_t)ptr - (uintptr_t)base);
  return QFTC_OK;
}

int qftc_ipc_open(const unsigned char handle[64], void** base) {
  if (!handle || !base) return fail(QFTC_EINVAL, "ipc_open: null argument");
  if (int rc = require_device()) return rc;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, 64);
  QFTC_CUDA(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  return QFTC_OK;
}

int qftc_ipc_close(void* base) {
  if (!base) return QFTC_OK;
  QFTC_CUDA(cudaIpcCloseMemHandle(base), "cudaIpcCloseMemHandle");
  return QFTC_OK;
}

int qftc_plan_set_ctas_per_sm(qftc_plan* p, int ctas_per_sm) {
  if (!p || ctas_per_sm < 0) return fail(QFTC_EINVAL, "plan_set_ctas_per_sm: bad arguments");
  if (p->rc.cap_per_sm != ctas_per_sm) {
    p->rc.cap_per_sm = ctas_per_sm;
    p->rc.rows[0] = KLaunch{};  // re-resolved at the next step
    p->rc.rows[1] = KLaunch{};
  }
  return QFTC_OK;
}

int qftc_plans_step(qftc_plan* const* plans, int n, int flip, qftc_lion_hyper h,
                    qftc_stream_t stream) {
  if (!plans || n <= 0) return fail(QFTC_EINVAL, "plans_step: no plans");
  for (int i = 0; i < n; ++i)
    if (!plans[i]) return fail(QFTC_EINVAL, "plans_step: null plan");
  if (n == 1) return qftc_plan_step(plans[0], flip, h, stream);
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < n; ++i) {
    qftc_plan* p = plans[i];
    if (!p->side) {
      QFTC_CUDA(cudaStreamCreateWithFlags(&p->side, cudaStreamNonBlocking), "plans_step: stream");
      QFTC_CUDA(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming), "plans_step: event");
      QFTC_CUDA(cudaEventCreateWithFlags(&p->ev_done, cudaEventDisableTiming), "plans_step: event");
    }
  }
  QFTC_CUDA(cudaEventRecord(plans[0]->ev_fork, st), "plans_step: fork");
  for (int i = 0; i < n; ++i) {
    qftc_plan* p = plans[i];
    QFTC_CUDA(cudaStreamWaitEvent(p->side, plans[0]->ev_fork, 0), "plans_step: fork wait");
    if (int rc = qftc_plan_step(p, flip, h, (qftc_stream_t)p->side)) return rc;
    QFTC_CUDA(cudaEventRecord(p->ev_done, p->side), "plans_step: join");
  }
  for (int i = 0; i < n; ++i)
    QFTC_CUDA(cudaStreamWaitEvent(st, plans[i]->ev_done, 0), "plans_step: join wait");
  return QFTC_OK;
}

int qftc_plan_result(qftc_plan* p, int64_t* nnz_total, qftc_stream_t stream) {
  if (!p) return fail(QFTC_EINVAL, "plan: null");
  cudaStream_t st = (cudaStream_t)stream;
  Header h{};
  if (int rc = read_header(p->sc.hdr, &h, st)) return rc;
  if (nnz_total) *nnz_total = h.total_nnz;
  // clear the sticky flags for the next check
  QFTC_CUDA(cudaMemsetAsync(&p->sc.hdr->overflow, 0, 8, st), "clear flags");
  QFTC_CUDA(cudaStreamSynchronize(st), "sync");
  if (p->oflag_host) *p->oflag_host = 0u;
  if (h.err & ERR_MPARAMS)
    return fail(QFTC_EINVAL, "affine_params_from_bounds: min > max in momentum channel");
  if (h.err & ERR_GPARAMS)
    return fail(QFTC_EINVAL, "affine_params_from_bounds: min > max in gradient channel");
  if (h.overflow)
    return fail(QFTC_EOVERFLOW, "lion step: a row's new outlier count exceeds its CSR slot");
  return QFTC_OK;
}

int qftc_plan_launches(const qftc_plan* p) {
  return p ? (p->rows_path ? 3 + (p->rc.gen_on ? 1 : 0) + (p->gq ? 1 : 0) : 1) : 0;
}

const char* qftc_plan_kernel_name(const qftc_plan* p) { return p ? p->last_kernel : ""; }

int qftc_plan_pending_overflow(const qftc_plan* p) {
  return (p && p->oflag_host && *p->oflag_host) ? 1 : 0;
}

int qftc_plan_tier_rows(qftc_plan* p, int64_t* stable_rows, int64_t* general_rows,
                        qftc_stream_t stream) {
  if (!p) return fail(QFTC_EINVAL, "plan: null");
  int64_t t3[3];
  if (int rc = qftc_plan_tiers(p, t3, stream)) return rc;
  if (stable_rows) *stable_rows = t3[0];
  if (general_rows) *general_rows = t3[1] + t3[2];
  return QFTC_OK;
}

int qftc_plan_tiers(qftc_plan* p, int64_t rows_out[3], qftc_stream_t stream) {
  if (!p || !rows_out) return fail(QFTC_EINVAL, "plan_tiers: bad arguments");
  rows_out[0] = 0;
  rows_out[1] = 0;
  rows_out[2] = p->total_rows;  // without the rows kernel every row runs the general kernel
  if (p->rows_path && p->rc.last_flip >= 0) {
    int32_t x[4] = {0, 0, 0, 0};
    QFTC_CUDA(cudaMemcpyAsync(x, p->rc.xcount + 4 * p->rc.last_flip, 12, cudaMemcpyDeviceToHost,
                              (cudaStream_t)stream), "read row lists");
    QFTC_CUDA(cudaStreamSynchronize((cudaStream_t)stream), "sync");
    rows_out[1] = x[2];
    rows_out[2] = x[0];
    rows_out[0] = p->total_rows - x[0] - x[2];  // the stable rows kernel walks every row
  }
  return QFTC_OK;
}

int qftc_plan_destroy(qftc_plan* p) {
  if (!p) return QFTC_OK;
  cudaFree(p->sc.base);
  if (p->prep) cudaFree(p->prep);
  if (p->xlist) cudaFree(p->xlist);
  if (p->rc.xcount) cudaFree(p->rc.xcount);
  if (p->rc.slist) cudaFree(p->rc.slist);
  if (p->rc.glist) cudaFree(p->rc.glist);
  if (p->rc.pstatus) cudaFree(p->rc.pstatus);
  if (p->gq_base) cudaFree(p->gq_base);
  if (p->peer_deltas) cudaFree(p->peer_deltas);
  if (p->rc.seen_host) cudaFreeHost(const_cast<int32_t*>(p->rc.seen_host));
  if (p->side) {
    cudaStreamSynchronize(p->side);
    cudaStreamDestroy(p->side);
    cudaEventDestroy(p->ev_fork);
    cudaEventDestroy(p->ev_done);
  }
  if (p->oflag_host) cudaFreeHost(const_cast<uint32_t*>(p->oflag_host));
  delete p;
  return QFTC_OK;
}

int qftc_lion_step(int rows, int cols, int bit_width, const uint8_t* g_codes,
                   const float* g_scale, const int32_t* g_zp, const uint8_t* m_codes,
                   const float* m_scale, const int32_t* m_zp, const uint8_t* w_codes,
                   const float* w_scale, const int32_t* w_zp, const float* t_min,
                   const float* t_max, const int32_t* row_ptr, const int32_t* col_idx,
                   const float* values, uint8_t* m_codes_out, float* m_scale_out,
                   int32_t* m_zp_out, uint8_t* w_codes_out, int32_t* row_ptr_out,
                   int32_t* col_idx_out, float* values_out, int64_t capacity,
                   qftc_lion_hyper hyper, int64_t* nnz_host, qftc_stream_t stream) {
  if (int rc = require_shape(rows, cols, "lion step")) return rc;
  if (int rc = require_device()) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  // output slots planned from the input counts; strict CSR via compaction
  int32_t* rs_out = nullptr;
  int32_t* cnt_out = nullptr;
  QFTC_CUDA(cudaMallocAsync((void**)&rs_out, sizeof(int32_t) * (rows + 1), st), "alloc");
  QFTC_CUDA(cudaMallocAsync((void**)&cnt_out, sizeof(int32_t) * rows, st), "alloc");
  int64_t slots = 0;
  int rc = qftc_csr_plan_slots(nullptr, row_ptr, rows, kSlack, rs_out, &slots, stream);
  int32_t* col_tmp = nullptr;
  float* val_tmp = nullptr;
  for (int attempt = 0; attempt < 3 && rc == QFTC_OK; ++attempt) {
    QFTC_CUDA(cudaMallocAsync((void**)&col_tmp, sizeof(int32_t) * (slots + 4), st), "alloc");
    QFTC_CUDA(cudaMallocAsync((void**)&val_tmp, sizeof(float) * (slots + 4), st), "alloc");
    qftc_lion_tensor t{};
    t.rows = rows;
    t.cols = cols;
    t.w_codes[0] = const_cast<uint8_t*>(w_codes);
    t.w_codes[1] = w_codes_out;
    t.row_start[0] = const_cast<int32_t*>(row_ptr);
    t.row_count[0] = nullptr;  // strict input
    t.row_start[1] = rs_out;
    t.row_count[1] = cnt_out;
    t.w_scale = w_scale;
    t.w_zero_point = w_zp;
    t.t_min = t_min;
    t.t_max = t_max;
    t.m_codes[0] = const_cast<uint8_t*>(m_codes);
    t.m_codes[1] = m_codes_out;
    t.m_scale[0] = const_cast<float*>(m_scale);
    t.m_scale[1] = m_scale_out;
    t.m_zero_point[0] = const_cast<int32_t*>(m_zp);
    t.m_zero_point[1] = m_zp_out;
    t.g_codes = g_codes;
    t.g_scale = g_scale;
    t.g_zero_point = g_zp;
    int32_t* cols_arr[2] = {const_cast<int32_t*>(col_idx), col_tmp};
    float* vals_arr[2] = {const_cast<float*>(values), val_tmp};
    const int64_t caps[2] = {0, slots};
    qftc_plan* p = nullptr;
    rc = qftc_plan_create(&p, &t, 1, bit_width, QFTC_GRAD_U8, cols_arr, vals_arr, caps, stream);
    if (rc) break;
    rc = qftc_plan_step(p, 0, hyper, stream);
    if (!rc) rc = qftc_plan_result(p, nullptr, stream);
    qftc_plan_destroy(p);
    if (rc == QFTC_EOVERFLOW && attempt < 2) {
      // re-plan the slots from the true counts and re-run (inputs are intact)
      cudaFreeAsync(col_tmp, st);
      cudaFreeAsync(val_tmp, st);
      col_tmp = nullptr;
      val_tmp = nullptr;
      rc = qftc_csr_plan_slots(cnt_out, nullptr, rows, kSlack, rs_out, &slots, stream);
      continue;  // rc == QFTC_OK -> next attempt
    }
    break;
  }
  if (rc == QFTC_OK)
    rc = qftc_csr_compact(rows, rs_out, cnt_out, col_tmp, val_tmp, row_ptr_out, col_idx_out,
                          values_out, capacity, nnz_host, stream);
  if (col_tmp) cudaFreeAsync(col_tmp, st);
  if (val_tmp) cudaFreeAsync(val_tmp, st);
  cudaFreeAsync(rs_out, st);
  cudaFreeAsync(cnt_out, st);
  cudaStreamSynchronize(st);
  return rc;
}

int qftc_lion_apply(float* w, float* m, const float* g, int64_t n, qftc_lion_hyper h,
                    qftc_stream_t stream) {
  if (n < 0) return fail(QFTC_EINVAL, "lion_apply: negative size");
  if (n == 0) return QFTC_OK;
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_lion_apply(w, m, g, n, h.lr, h.beta1, h.beta2, h.weight_decay,
                              (cudaStream_t)stream),
            "lion_apply");
  return QFTC_OK;
}

int qftc_crc32(const void* const* segments, const int64_t* lengths, int n, uint32_t* crc_out,
               qftc_stream_t stream) {
  if (!crc_out || n < 0 || (n > 0 && (!segments || !lengths)))
    return fail(QFTC_EINVAL, "crc32: bad arguments");
  for (int i = 0; i < n; ++i)
    if (lengths[i] < 0 || (lengths[i] > 0 && !segments[i]))
      return fail(QFTC_EINVAL, "crc32: bad segment " + std::to_string(i));
  if (int rc = require_device()) return rc;
  QFTC_CUDA(crc32_device(segments, lengths, n, crc_out, (cudaStream_t)stream), "crc32");
  return QFTC_OK;
}

int qftc_device_alloc(void** ptr, size_t bytes) {
  if (!ptr) return fail(QFTC_EINVAL, "device_alloc: null out pointer");
  if (int rc = require_device()) return rc;
  QFTC_CUDA(cudaMalloc(ptr, bytes ? bytes : 1), "cudaMalloc");
  return QFTC_OK;
}

int qftc_device_free(void* ptr) {
  if (!ptr) return QFTC_OK;
  QFTC_CUDA(cudaFree(ptr), "cudaFree");
  return QFTC_OK;
}

int qftc_copy_to_device(void* dst, const void* src, size_t bytes, qftc_stream_t stream) {
  if (!bytes) return QFTC_OK;
  QFTC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream),
            "copy_to_device");
  return QFTC_OK;
}

int qftc_copy_peer(void* dst, const void* src, size_t bytes, qftc_stream_t stream) {
  if (!bytes) return QFTC_OK;
  QFTC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream),
            "copy_peer");
  return QFTC_OK;
}

int qftc_copy_to_host(void* dst, const void* src, size_t bytes, qftc_stream_t stream) {
  if (!bytes) return QFTC_OK;
  QFTC_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, (cudaStream_t)stream),
            "copy_to_host");
  return QFTC_OK;
}

int qftc_memset(void* dst, int value, size_t bytes, qftc_stream_t stream) {
  if (!bytes) return QFTC_OK;
  QFTC_CUDA(cudaMemsetAsync(dst, value, bytes, (cudaStream_t)stream), "memset");
  return QFTC_OK;
}

int qftc_stream_synchronize(qftc_stream_t stream) {
  QFTC_CUDA(cudaStreamSynchronize((cudaStream_t)stream), "stream synchronize");
  return QFTC_OK;
}

int qftc_synth(float* out, int64_t n, uint64_t seed, double sigma, double spike_p,
               qftc_stream_t stream) {
  if (n <= 0) return QFTC_OK;
  if (int rc = require_device()) return rc;
  QFTC_CUDA(launch_synth(out, n, seed, sigma, spike_p, (cudaStream_t)stream), "synth");
  return QFTC_OK;
}

}  // extern "C"
