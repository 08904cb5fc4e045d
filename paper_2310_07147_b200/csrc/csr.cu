// csr.cu -- CSR layout utilities (not on the step's hot path).
//
// The fused step keeps outliers in a SLOTTED CSR: row r owns arena entries
// [row_start[r], row_start[r+1]) of which row_count[r] are used (columns
// ascending, quantize.hpp:48-49).  Slots are 16-byte aligned (capacity a multiple
// of 4 entries) so the step's producer can TMA-stage them.  These kernels
//   * plan slots from counts (capacity = count + count/4 + slack, rounded to 4),
//   * copy rows between a strict reference CSR (row_ptr) and a slotted arena,
//   * compact a slotted arena into the strict reference CSR (row_ptr = exclusive
//     scan of the counts; what the reference's SparseOutliers holds),
//   * pack the used entries of many slotted segments per width class for the ZeRO-1
//     all-gather (only used entries travel; the row starts are re-based to the rank's
//     offset inside the gathered arena).
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <vector>

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

// Slot capacities for a re-plan (engine._replan): per row, the used count of the step's
// output plus its dense codes at 0 / qmax (the only elements a stable-tier step can turn
// into new outliers: the placement's no-overflow padding), plus growth headroom.  One warp
// per row, 16 codes per lane load (__vcmpeq4 on 4 words), no temporaries.
//   want = cnt_out + edge;  grow = max(cnt_out - cnt_in, 0)
//   cap  = want + want/4 + gmul*grow + want*lvl/4 + min(8 << 2 lvl, 64), rounded up to 4
__global__ void k_replan_caps(const uint8_t* codes, int rows, int cols, int qmax,
                              const int32_t* cnt_out, const int32_t* cnt_in, int lvl, int gmul,
                              int64_t* caps) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const uint32_t qm4 = 0x01010101u * (uint32_t)qmax;
  const bool vec = (cols % 16) == 0 && (reinterpret_cast<uintptr_t>(codes) & 15) == 0;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < rows; r += warps) {
    const uint8_t* cr = codes + (size_t)r * cols;
    int edge = 0;
    if (vec) {
      const uint4* v = reinterpret_cast<const uint4*>(cr);
      for (int i = lane; i < cols / 16; i += 32) {
        const uint4 q = v[i];
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          edge += __popc(__vcmpeq4(w[k], 0u) | __vcmpeq4(w[k], qm4)) >> 3;
      }
    } else {
      for (int i = lane; i < cols; i += 32) edge += (cr[i] == 0 || cr[i] == qmax) ? 1 : 0;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) edge += __shfl_xor_sync(0xffffffffu, edge, o);
    if (lane == 0) {
      const int64_t c = cnt_out[r];
      const int64_t want = c + edge;
      const int64_t grow = c > cnt_in[r] ? c - cnt_in[r] : 0;
      const int64_t slack = (8LL << (2 * lvl)) < 64 ? (8LL << (2 * lvl)) : 64;
      const int64_t cap = want + want / 4 + gmul * grow + (want * lvl) / 4 + slack;
      caps[r] = (cap + 3) & ~3LL;
    }
  }
}

cudaError_t launch_replan_caps(const uint8_t* codes, int rows, int cols, int bit_width,
                               const int32_t* cnt_out, const int32_t* cnt_in, int lvl, int gmul,
                               int64_t* caps, cudaStream_t st) {
  const int blocks = std::min(4096, (rows + 7) / 8);
  k_replan_caps<<<blocks, 256, 0, st>>>(codes, rows, cols, (1 << bit_width) - 1, cnt_out, cnt_in,
                                        lvl, gmul, caps);
  return cudaGetLastError();
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

// ------------------------------------------------------------------ ZeRO-1 packed gather
// The rows of every segment (one tensor's row range: rows+1 slot starts at rs_off, rows
// counts at cnt_off) are cut into chunks of <= PACK_T rows, ordered by width class, then
// segment.  Per run: the used entries of every chunk (one CTA per chunk), an exclusive scan
// of the chunk totals (cub), and the pack (one CTA per chunk: a block scan of its rows'
// used counts -> row starts + base; the chunk's entries are one contiguous output range,
// copied with consecutive threads on consecutive entries).
constexpr int PACK_T = 256;

struct PackChunk {
  int32_t rs_off;   // first row's slot start (the segment's rs_off + r0)
  int32_t cnt_off;  // first row's count
  int32_t rows;     // rows in the chunk (0: an empty segment's terminator only)
  int32_t flags;    // width class | 0x100: last chunk of its segment
};

__device__ __forceinline__ int used_entries(const int32_t* rs, const int32_t* cnt, int r) {
  const int s = rs[r];
  return max(0, min(cnt[r], rs[r + 1] - s));  // clamped to the slot (an unrepaired overflow)
}

__global__ void __launch_bounds__(PACK_T) k_chunk_totals(const PackChunk* __restrict__ ch,
                                                          const int32_t* __restrict__ rs,
                                                          const int32_t* __restrict__ cnt,
                                                          int32_t* __restrict__ tot) {
  __shared__ int red[PACK_T / 32];
  const PackChunk c = ch[blockIdx.x];
  int n = threadIdx.x < c.rows ? used_entries(rs + c.rs_off, cnt + c.cnt_off, threadIdx.x) : 0;
  for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < PACK_T / 32; ++w) n += red[w];
    tot[blockIdx.x] = n;
  }
}

__global__ void __launch_bounds__(PACK_T) k_pack_chunks(const PackChunk* __restrict__ ch,
                                                         const int32_t* __restrict__ scan,
                                                         const int32_t* __restrict__ rs_all,
                                                         const int32_t* __restrict__ cnt_all,
                                                         PackWidths P,
                                                         int32_t* __restrict__ rs_out_all) {
  __shared__ int wsum[PACK_T / 32];
  __shared__ int r_src[PACK_T], r_dst[PACK_T], s_total;
  const PackChunk c = ch[blockIdx.x];
  const int w = c.flags & 0xFF;
  const int32_t* rs = rs_all + c.rs_off;
  const int32_t* cnt = cnt_all + c.cnt_off;
  int32_t* rs_out = rs_out_all + c.rs_off;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int off = scan[blockIdx.x] - scan[P.first_chunk[w]];  // within the class
  const int64_t base = P.base[w];
  int n = 0, src = 0;
  if (tid < c.rows) {
    src = rs[tid];
    n = used_entries(rs, cnt, tid);
  }
  int x = n;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  int before = 0;
  for (int k = 0; k < wid; ++k) before += wsum[k];
  const int excl = off + before + x - n;
  if (tid < c.rows) rs_out[tid] = (int32_t)(base + excl);
  if ((c.flags & 0x100) && tid == PACK_T - 1) rs_out[c.rows] = (int32_t)(base + excl + n);
  r_src[tid] = src;
  r_dst[tid] = excl - off;  // the row's first entry within the chunk's output range
  if (tid == PACK_T - 1) s_total = excl + n - off;
  __syncthreads();
  const int32_t* col_in = P.col_in[w];
  const float* val_in = P.val_in[w];
  int32_t* col_out = P.col_out[w] + off;
  float* val_out = P.val_out[w] + off;
  // the chunk's output is one contiguous range: thread tid writes entries tid, tid+256, ...
  // (coalesced), finding each entry's row with a cursor that only moves forward
  const int total = s_total;
  int row = 0;
  for (int e = tid; e < total; e += PACK_T) {
    while (row + 1 < c.rows && r_dst[row + 1] <= e) ++row;
    const int src_e = r_src[row] + (e - r_dst[row]);
    col_out[e] = __ldcs(col_in + src_e);
    val_out[e] = __ldcs(val_in + src_e);
  }
}

struct PackPlan {
  PackChunk* chunks = nullptr;
  int32_t* tot = nullptr;
  int32_t* scan = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int nchunks = 0, nwidth = 0;
  int first_chunk[QFT_PACK_MAXW] = {};
};

cudaError_t csr_pack_plan_create(const qftc_pack_segment* segs, int nseg, int nwidth,
                                 cudaStream_t st, void** out) {
  std::vector<PackChunk> v;
  PackPlan* p = new PackPlan;
  p->nwidth = nwidth;
  for (int w = 0; w < nwidth; ++w) {
    p->first_chunk[w] = (int)v.size();
    for (int i = 0; i < nseg; ++i) {
      const qftc_pack_segment& s = segs[i];
      if (s.width != w) continue;
      for (int r0 = 0; r0 < s.rows || (r0 == 0 && s.rows == 0); r0 += PACK_T) {
        const int n = std::min(PACK_T, s.rows - r0);
        const bool last = r0 + PACK_T >= s.rows;
        v.push_back(PackChunk{(int32_t)(s.rs_off + r0), (int32_t)(s.cnt_off + r0), n,
                              w | (last ? 0x100 : 0)});
      }
    }
  }
  p->nchunks = (int)v.size();
  const int nc = std::max(1, p->nchunks);
  cudaError_t e = cudaMalloc((void**)&p->chunks, sizeof(PackChunk) * nc);
  if (e == cudaSuccess) e = cudaMalloc((void**)&p->tot, sizeof(int32_t) * nc);
  if (e == cudaSuccess) e = cudaMalloc((void**)&p->scan, sizeof(int32_t) * nc);
  if (e == cudaSuccess && p->nchunks)
    e = cudaMemcpyAsync(p->chunks, v.data(), sizeof(PackChunk) * v.size(),
                        cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(nullptr, p->tmp_bytes, p->tot, p->scan, nc, st);
  if (e == cudaSuccess) e = cudaMalloc(&p->tmp, p->tmp_bytes ? p->tmp_bytes : 1);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    csr_pack_plan_destroy(p);
    return e;
  }
  *out = p;
  return cudaSuccess;
}

cudaError_t csr_pack_run(void* plan, const int32_t* row_start, const int32_t* row_count,
                         PackWidths P, int32_t* row_start_out, cudaStream_t st) {
  PackPlan* p = static_cast<PackPlan*>(plan);
  if (!p->nchunks) return cudaSuccess;
  for (int w = 0; w < p->nwidth; ++w) P.first_chunk[w] = std::min(p->first_chunk[w], p->nchunks - 1);
  k_chunk_totals<<<p->nchunks, PACK_T, 0, st>>>(p->chunks, row_start, row_count, p->tot);
  cudaError_t e = cub::DeviceScan::ExclusiveSum(p->tmp, p->tmp_bytes, p->tot, p->scan,
                                                p->nchunks, st);
  if (e != cudaSuccess) return e;
  k_pack_chunks<<<p->nchunks, PACK_T, 0, st>>>(p->chunks, p->scan, row_start, row_count, P,
                                               row_start_out);
  return cudaGetLastError();
}

int csr_pack_nwidth(const void* plan) { return static_cast<const PackPlan*>(plan)->nwidth; }

void csr_pack_plan_destroy(void* plan) {
  PackPlan* p = static_cast<PackPlan*>(plan);
  if (!p) return;
  cudaFree(p->chunks);
  cudaFree(p->tot);
  cudaFree(p->scan);
  cudaFree(p->tmp);
  delete p;
}

}  // namespace qftk
