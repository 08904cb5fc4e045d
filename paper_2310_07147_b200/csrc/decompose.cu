// Dense-and-sparse decomposition with given thresholds (decompose_dense_sparse,
// quantize.hpp:253-290): per row, params from (t_min, t_max) (computed by the caller
// with affine_params_from_bounds, quantize.hpp:264); per element, outlier iff
// v < t_min || v > t_max -> CSR (col, v) and dense code clamp(z, 0, qmax); otherwise the
// channel quantizer (quantize.hpp:149-175, fp32 scale, half-away rounding, NaN -> 0).
//
// Init / threshold-refresh path (not the per-step hot path), built as two warp-per-row
// passes around a device scan so the CSR comes out strict (row_ptr) with no cross-row
// dependency inside a kernel:
//   A  codes + per-row outlier counts   (one read of the f32 row, codes written)
//   -  row_ptr = exclusive_scan(counts) (CUB, csr.cu)
//   B  ordered outlier extraction       (second read; warp ballot + popc ranks)
#include "qft_internal.h"
#include "qft_device.cuh"

using namespace qftd;
using namespace qftk;

namespace {

constexpr int DC_WARPS = 8;

__device__ __forceinline__ bool is_outlier(float v, float lo, float hi) {
  return (v < lo) || (v > hi);
}

// pass A: warp per row, 4 consecutive elements per lane per step
template <bool VEC>
__global__ void __launch_bounds__(DC_WARPS * 32)
k_decompose_codes(const float* __restrict__ w, int rows, int cols, const float* __restrict__ scale,
                  const int32_t* __restrict__ zp, const float* __restrict__ t_min,
                  const float* __restrict__ t_max, int bit_width, uint8_t* __restrict__ codes,
                  int32_t* __restrict__ counts) {
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * DC_WARPS;
  for (int r = blockIdx.x * DC_WARPS + (threadIdx.x >> 5); r < rows; r += nw) {
    const QuantRow q = make_quant_row(scale[r], zp[r], bit_width);
    const float lo = t_min[r], hi = t_max[r];
    const uint32_t zpay = (uint32_t)min(max(q.z, 0), q.qmax);
    const float* src = w + (size_t)r * cols;
    uint8_t* dst = codes + (size_t)r * cols;
    int n = 0;
    if (VEC) {
      for (int c = lane * 4; c < cols; c += 128) {
        const float4 v4 = __ldcs(reinterpret_cast<const float4*>(src + c));
        const float x[4] = {v4.x, v4.y, v4.z, v4.w};
        float em = 0.0f;
        uint32_t code = quant4_fast(x, q, em);
        if (!q.fast || !(em < q.thr)) code = quant4_exact(x, q);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (is_outlier(x[i], lo, hi)) {
            code = (code & ~(0xFFu << (8 * i))) | (zpay << (8 * i));
            ++n;
          }
        }
        *reinterpret_cast<uint32_t*>(dst + c) = code;
      }
    } else {
      for (int c = lane; c < cols; c += 32) {
        const float x = src[c];
        uint32_t code;
        if (is_outlier(x, lo, hi)) {
          code = zpay;
          ++n;
        } else {
          code = quant_exact(x, q.s, q.z, q.qmax);
        }
        dst[c] = (uint8_t)code;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if (lane == 0) counts[r] = n;
  }
}

// pass B: warp per row, 32 consecutive columns per step; ballot keeps column order
__global__ void __launch_bounds__(DC_WARPS * 32)
k_decompose_csr(const float* __restrict__ w, int rows, int cols, const float* __restrict__ t_min,
                const float* __restrict__ t_max, const int32_t* __restrict__ row_ptr,
                int32_t* __restrict__ col_idx, float* __restrict__ values) {
  const int lane = threadIdx.x & 31;
  const int nw = gridDim.x * DC_WARPS;
  const uint32_t below = (1u << lane) - 1u;
  for (int r = blockIdx.x * DC_WARPS + (threadIdx.x >> 5); r < rows; r += nw) {
    int pos = row_ptr[r];
    const int end = row_ptr[r + 1];
    if (pos == end) continue;
    const float lo = t_min[r], hi = t_max[r];
    const float* src = w + (size_t)r * cols;
    for (int c0 = 0; c0 < cols && pos < end; c0 += 32) {
      const int c = c0 + lane;
      const float x = c < cols ? __ldcs(src + c) : 0.0f;
      const bool o = c < cols && is_outlier(x, lo, hi);
      const uint32_t b = __ballot_sync(0xffffffffu, o);
      if (o) {
        const int p = pos + __popc(b & below);
        col_idx[p] = c;
        values[p] = x;
      }
      pos += __popc(b);
    }
  }
}

int dc_grid(int rows) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int need = (rows + DC_WARPS - 1) / DC_WARPS;
  const int cap = sms * 8;
  return need < cap ? need : cap;
}

}  // namespace

namespace qftk {

cudaError_t decompose_codes(const float* w, int rows, int cols, const float* scale,
                            const int32_t* zp, const float* t_min, const float* t_max,
                            int bit_width, uint8_t* codes, int32_t* counts, cudaStream_t st) {
  const bool vec = (cols % 4 == 0) && (((uintptr_t)w & 15u) == 0) && (((uintptr_t)codes & 3u) == 0);
  if (vec)
    k_decompose_codes<true><<<dc_grid(rows), DC_WARPS * 32, 0, st>>>(
        w, rows, cols, scale, zp, t_min, t_max, bit_width, codes, counts);
  else
    k_decompose_codes<false><<<dc_grid(rows), DC_WARPS * 32, 0, st>>>(
        w, rows, cols, scale, zp, t_min, t_max, bit_width, codes, counts);
  return cudaGetLastError();
}

cudaError_t decompose_csr(const float* w, int rows, int cols, const float* t_min,
                          const float* t_max, const int32_t* row_ptr, int32_t* col_idx,
                          float* values, cudaStream_t st) {
  k_decompose_csr<<<dc_grid(rows), DC_WARPS * 32, 0, st>>>(w, rows, cols, t_min, t_max, row_ptr,
                                                          col_idx, values);
  return cudaGetLastError();
}

}  // namespace qftk
