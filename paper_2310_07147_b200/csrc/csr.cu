// csr.cu -- CSR layout utilities (not on the step's hot path).
//
// The fused step keeps outliers in a SLOTTED CSR: row r owns arena entries
// [row_start[r], row_start[r+1]) of which row_count[r] are used (columns
// ascending, quantize.hpp:48-49).  Slots are 16-byte aligned (capacity a multiple
// of 4 entries) so the step's producer can TMA-stage them.  These kernels
//   * plan slots from counts (capacity = count + count/4 + slack, rounded to 4),
//   * copy rows between a strict reference CSR (row_ptr) and a slotted arena,
//   * compact a slotted arena into the strict reference CSR (row_ptr = exclusive
//     scan of the counts; what the reference's SparseOutliers holds).
#include <cub/device/device_scan.cuh>

#include "qft_internal.h"

namespace qftk {

__global__ void k_slot_caps(const int32_t* counts, const int32_t* row_ptr, int rows, int slack,
                            int32_t* caps) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= rows; r += gridDim.x * blockDim.x) {
    if (r == rows) {
      caps[r] = 0;
      continue;
    }
    const int c = counts ? counts[r] : row_ptr[r + 1] - row_ptr[r];
    caps[r] = ((c + c / 4 + slack) + 3) & ~3;
  }
}

// per-row entry counts: from a strict row_ptr, or from slot counts clamped to their slot
// (slot_start != nullptr: a count above its slot -- an overflowed step that was not re-run
// -- never reaches into the next row's entries)
__global__ void k_counts(const int32_t* counts, const int32_t* row_ptr, int rows, int32_t* out,
                         const int32_t* slot_start) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r <= rows; r += gridDim.x * blockDim.x) {
    int n = 0;
    if (r < rows) {
      n = counts ? counts[r] : row_ptr[r + 1] - row_ptr[r];
      if (counts && slot_start) n = min(n, slot_start[r + 1] - slot_start[r]);
    }
    out[r] = n;
  }
}

// copy each row's entries from src (slotted: start+count, or strict: row_ptr) to
// dst (start array); one warp per row
__global__ void k_copy_rows(int rows, const int32_t* src_start, const int32_t* src_count,
                            const int32_t* src_col, const float* src_val, const int32_t* dst_start,
                            int32_t* dst_col, float* dst_val, int64_t dst_cap) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
    const int s = src_start[r];
    // slotted source: the used entries, never past the slot end (see k_counts)
    const int n = src_count ? min(src_count[r], src_start[r + 1] - s) : src_start[r + 1] - s;
    const int64_t d = dst_start[r];
    for (int i = lane; i < n; i += 32) {
      if (d + i < dst_cap) {
        dst_col[d + i] = src_col[s + i];
        dst_val[d + i] = src_val[s + i];
      }
    }
  }
}

static cudaError_t exclusive_scan(const int32_t* in, int32_t* out, int n, cudaStream_t st) {
  size_t tmp = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, st);
  if (e != cudaSuccess) return e;
  void* buf = nullptr;
  e = cudaMallocAsync(&buf, tmp ? tmp : 1, st);
  if (e != cudaSuccess) return e;
  e = cub::DeviceScan::ExclusiveSum(buf, tmp, in, out, n, st);
  cudaFreeAsync(buf, st);
  return e;
}

static int grid_for(int64_t n, int per_block) {
  int64_t g = (n + per_block - 1) / per_block;
  if (g > 148 * 32) g = 148 * 32;
  return g < 1 ? 1 : (int)g;
}

// row_start[0..rows] of slots sized from counts (or from a strict row_ptr)
cudaError_t csr_plan_slots(const int32_t* counts, const int32_t* row_ptr, int rows, int slack,
                           int32_t* row_start, cudaStream_t st) {
  int32_t* caps = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&caps, sizeof(int32_t) * (rows + 1), st);
  if (e != cudaSuccess) return e;
  k_slot_caps<<<grid_for(rows + 1, 256), 256, 0, st>>>(counts, row_ptr, rows, slack, caps);
  e = exclusive_scan(caps, row_start, rows + 1, st);
  cudaFreeAsync(caps, st);
  return e;
}

cudaError_t csr_copy_rows(int rows, const int32_t* src_start, const int32_t* src_count,
                          const int32_t* src_col, const float* src_val, const int32_t* dst_start,
                          int32_t* dst_col, float* dst_val, int64_t dst_cap, cudaStream_t st) {
  k_copy_rows<<<grid_for((int64_t)rows * 32, 256), 256, 0, st>>>(
      rows, src_start, src_count, src_col, src_val, dst_start, dst_col, dst_val, dst_cap);
  return cudaGetLastError();
}

// strict row_ptr (rows+1) from counts (clamped to their slots when slot_start is given)
cudaError_t csr_row_ptr(const int32_t* counts, int rows, int32_t* row_ptr, cudaStream_t st,
                        const int32_t* slot_start) {
  int32_t* tmp = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&tmp, sizeof(int32_t) * (rows + 1), st);
  if (e != cudaSuccess) return e;
  k_counts<<<grid_for(rows + 1, 256), 256, 0, st>>>(counts, nullptr, rows, tmp, slot_start);
  e = exclusive_scan(tmp, row_ptr, rows + 1, st);
  cudaFreeAsync(tmp, st);
  return e;
}

}  // namespace qftk
