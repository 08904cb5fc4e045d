// Weight expansion for the next forward: dense codes + CSR outliers -> f32 or bf16.
//
// reconstruct (quantize.hpp:331-338): dequantize every code with the row's (scale, zp)
// (quantize.hpp:195-212, fp32, no FMA), then overwrite each CSR position with its exact
// f32 value.  The bf16 output is the RNE rounding of that f32 tensor (the consumer
// format of the forward, network.hpp:199-212 with bf16 in place of f32).
//
// HBM-bound elementwise kernel (1 B read + 2 or 4 B written per parameter + 8 B per CSR
// entry): a warp owns a row, lanes stream 16-code vectors with 128-bit loads/stores,
// several in flight per lane; then, after __syncwarp (which orders the warp's global
// stores), the lanes scatter the row's outliers.  A whole model goes in one launch: the
// tensor table travels in the kernel parameter space (no device allocation, no host
// sync), and a warp finds its tensor by a warp-uniform binary search over the row
// prefix.
#include "qft_internal.h"

#include <vector>
#include "qft_device.cuh"

using namespace qftd;
using namespace qftk;

namespace {

#ifndef QFT_EXP_WARPS
#define QFT_EXP_WARPS 2
#endif
#ifndef QFT_EXP_UNROLL
#define QFT_EXP_UNROLL 10
#endif
constexpr int EXP_MAXT = 224;      // tensors per launch (param space: <= 32 KB)
constexpr int EXP_WARPS = QFT_EXP_WARPS;    // warps per CTA
constexpr int EXP_UNROLL = QFT_EXP_UNROLL;  // 16-code vectors in flight per lane

struct ExpT {
  const uint8_t* codes;
  const float* scale;
  const int32_t* zp;
  const int32_t* rs;
  const int32_t* cnt;   // null: strict CSR (row_ptr = rs)
  const int32_t* col;
  const float* val;
  void* out;
  int32_t rows, cols;
  int32_t aligned;      // 16-byte vector path usable for every row
  int32_t pad_;
};

struct ExpArgs {
  int n;
  int bf16;
  long long total_rows;
  long long prefix[EXP_MAXT + 1];
  ExpT t[EXP_MAXT];
};

__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

__device__ __forceinline__ uint16_t to_bf16(float a) {
  return (uint16_t)(pack_bf16x2(a, 0.0f) & 0xFFFFu);
}

template <bool BF16>
__device__ __forceinline__ void store16(void* out, size_t idx, const float* f) {
  if (BF16) {
    uint4 a, b;
    a.x = pack_bf16x2(f[0], f[1]);   a.y = pack_bf16x2(f[2], f[3]);
    a.z = pack_bf16x2(f[4], f[5]);   a.w = pack_bf16x2(f[6], f[7]);
    b.x = pack_bf16x2(f[8], f[9]);   b.y = pack_bf16x2(f[10], f[11]);
    b.z = pack_bf16x2(f[12], f[13]); b.w = pack_bf16x2(f[14], f[15]);
    uint4* o = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(out) + idx);
    o[0] = a;
    o[1] = b;
  } else {
    float4* o = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + idx);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      o[q] = make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
  }
}

template <bool BF16>
__device__ __forceinline__ void store1(void* out, size_t idx, float v) {
  if (BF16) reinterpret_cast<uint16_t*>(out)[idx] = to_bf16(v);
  else reinterpret_cast<float*>(out)[idx] = v;
}

struct RowMeta {
  int ti, r;
  float s;
  int32_t z;
  int b, n;
};

__device__ __forceinline__ RowMeta row_meta(const ExpT* tab, const long long* prefix, int n,
                                            long long grow) {
  // warp-uniform binary search: tensor ti with prefix[ti] <= grow < prefix[ti+1]
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= grow) lo = mid; else hi = mid - 1;
  }
  const ExpT& T = tab[lo];
  RowMeta m;
  m.ti = lo;
  m.r = (int)(grow - prefix[lo]);
  m.s = T.scale[m.r];
  m.z = T.zp[m.r];
  m.b = T.rs[m.r];
  // a slotted row uses at most its slot: a count above it (an overflowed step that was
  // not re-run) must not read the next row's entries
  m.n = T.cnt ? min(T.cnt[m.r], T.rs[m.r + 1] - m.b) : (T.rs[m.r + 1] - m.b);
  return m;
}

// A warp expands one row at a time.  Latency hiding: the next row's metadata is
// loaded while the current row streams, the row's first 64 CSR entries are loaded
// before its dense loads, and each lane keeps EXP_UNROLL 16-byte loads in flight.
template <bool BF16>
__device__ __forceinline__ void expand_rows(const ExpT* tab, const long long* prefix, int n,
                                            long long total_rows) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * EXP_WARPS;
  long long grow = (long long)blockIdx.x * EXP_WARPS + (threadIdx.x >> 5);
  if (grow >= total_rows) return;
  RowMeta nxt = row_meta(tab, prefix, n, grow);
  for (; grow < total_rows; grow += nwarps) {
    const RowMeta m = nxt;
    if (grow + nwarps < total_rows) nxt = row_meta(tab, prefix, n, grow + nwarps);
    const ExpT& T = tab[m.ti];
    const int cols = T.cols;
    const size_t base = (size_t)m.r * (size_t)cols;
    // the row's first 64 outliers, loaded early
    int c0 = -1, c1 = -1;
    float v0 = 0.0f, v1 = 0.0f;
    if (lane < m.n) { c0 = T.col[m.b + lane]; v0 = T.val[m.b + lane]; }
    if (lane + 32 < m.n) { c1 = T.col[m.b + lane + 32]; v1 = T.val[m.b + lane + 32]; }
    const DequantRow d = make_dequant_row(m.s, m.z);
    const uint8_t* src = T.codes + base;
    if (T.aligned) {
      const int nvec = cols >> 4;
      for (int vb = 0; vb < nvec; vb += 32 * EXP_UNROLL) {
        uint4 q[EXP_UNROLL];
#pragma unroll
        for (int u = 0; u < EXP_UNROLL; ++u) {
          const int v = vb + u * 32 + lane;
          if (v < nvec) q[u] = __ldcs(reinterpret_cast<const uint4*>(src) + v);
        }
#pragma unroll
        for (int u = 0; u < EXP_UNROLL; ++u) {
          const int v = vb + u * 32 + lane;
          if (v < nvec) {
            float f[16];
            dequant4(q[u].x, d, f);     dequant4(q[u].y, d, f + 4);
            dequant4(q[u].z, d, f + 8); dequant4(q[u].w, d, f + 12);
            store16<BF16>(T.out, base + (size_t)v * 16, f);
          }
        }
      }
    } else {
      for (int c = lane; c < cols; c += 32) {
        const uint32_t q = src[c];
        const float f = d.fast ? __fmul_rn(__fadd_rn(magic_byte(q, 0), d.negc), d.s)
                               : dequant_exact(q, d.s, d.z);
        store1<BF16>(T.out, base + c, f);
      }
    }
    __syncwarp();
    // outliers: exact f32 values over the dense payload (quantize.hpp:335-337)
    if (c0 >= 0) store1<BF16>(T.out, base + c0, v0);
    if (c1 >= 0) store1<BF16>(T.out, base + c1, v1);
    for (int j = 64 + lane; j < m.n; j += 32) store1<BF16>(T.out, base + T.col[m.b + j], T.val[m.b + j]);
  }
}

// the table in the kernel parameter space (up to EXP_MAXT tensors, nothing to upload) ...
template <bool BF16>
__global__ void __launch_bounds__(EXP_WARPS * 32) expand_kernel(const __grid_constant__ ExpArgs a) {
  expand_rows<BF16>(a.t, a.prefix, a.n, a.total_rows);
}
// ... or in device memory (an expand plan: any number of tensors, one launch)
template <bool BF16>
__global__ void __launch_bounds__(EXP_WARPS * 32) expand_kernel_dev(const ExpT* tab,
                                                                  const long long* prefix, int n,
                                                                  long long total_rows) {
  expand_rows<BF16>(tab, prefix, n, total_rows);
}

}  // namespace

static bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

namespace qftk {
int expand_max_tensors() { return EXP_MAXT; }

cudaError_t launch_expand(const qftc_expand_tensor* ts, int n, bool bf16, cudaStream_t st) {
  static int sms = 0, per_sm[2] = {0, 0};
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[0], expand_kernel<false>, EXP_WARPS * 32, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[1], expand_kernel<true>, EXP_WARPS * 32, 0);
    if (per_sm[0] < 1) per_sm[0] = 1;
    if (per_sm[1] < 1) per_sm[1] = 1;
  }
  for (int off = 0; off < n; off += EXP_MAXT) {
    const int m = (n - off < EXP_MAXT) ? n - off : EXP_MAXT;
    ExpArgs a;
    a.n = m;
    a.bf16 = bf16 ? 1 : 0;
    long long acc = 0;
    int k = 0;
    for (int i = 0; i < m; ++i) {
      const qftc_expand_tensor& s = ts[off + i];
      if (s.rows <= 0 || s.cols <= 0) continue;
      ExpT& t = a.t[k];
      t.codes = s.codes; t.scale = s.scale; t.zp = s.zero_point; t.rs = s.row_start;
      t.cnt = s.row_count; t.col = s.col_idx; t.val = s.values; t.out = s.out;
      t.rows = s.rows; t.cols = s.cols;
      const int esz = bf16 ? 2 : 4;
      t.aligned = (s.cols % 16 == 0) && al16(s.codes) && al16(s.out) &&
                  ((size_t)s.cols * esz % 16 == 0);
      t.pad_ = 0;
      a.prefix[k] = acc;
      acc += s.rows;
      ++k;
    }
    if (k == 0) continue;
    a.n = k;
    a.prefix[k] = acc;
    a.total_rows = acc;
    long long warps_needed = acc;
    long long grid = (warps_needed + EXP_WARPS - 1) / EXP_WARPS;
    const long long cap = (long long)sms * per_sm[bf16 ? 1 : 0];  // one resident wave
    if (grid > cap) grid = cap;
    if (bf16) expand_kernel<true><<<(unsigned)grid, EXP_WARPS * 32, 0, st>>>(a);
    else expand_kernel<false><<<(unsigned)grid, EXP_WARPS * 32, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ------------------------------------------------------------------ expand plans
struct ExpandPlan {
  ExpT* tab = nullptr;          // device table
  long long* prefix = nullptr;  // device row prefix (n + 1)
  int n = 0;
  long long total = 0;
  bool bf16 = false;
  int grid = 0;
};

cudaError_t expand_plan_create(const qftc_expand_tensor* ts, int n, bool bf16, cudaStream_t st,
                               void** out) {
  std::vector<ExpT> tab;
  std::vector<long long> pre;
  long long acc = 0;
  for (int i = 0; i < n; ++i) {
    const qftc_expand_tensor& s = ts[i];
    if (s.rows <= 0 || s.cols <= 0) continue;
    ExpT t{};
    t.codes = s.codes; t.scale = s.scale; t.zp = s.zero_point; t.rs = s.row_start;
    t.cnt = s.row_count; t.col = s.col_idx; t.val = s.values; t.out = s.out;
    t.rows = s.rows; t.cols = s.cols;
    const int esz = bf16 ? 2 : 4;
    t.aligned = (s.cols % 16 == 0) && al16(s.codes) && al16(s.out) && ((size_t)s.cols * esz % 16 == 0);
    pre.push_back(acc);
    acc += s.rows;
    tab.push_back(t);
  }
  pre.push_back(acc);
  auto* p = new ExpandPlan;
  p->n = (int)tab.size();
  p->total = acc;
  p->bf16 = bf16;
  cudaError_t e = cudaSuccess;
  if (p->n > 0) {
    e = cudaMalloc(&p->tab, sizeof(ExpT) * tab.size());
    if (e == cudaSuccess) e = cudaMalloc(&p->prefix, sizeof(long long) * pre.size());
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->tab, tab.data(), sizeof(ExpT) * tab.size(), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(p->prefix, pre.data(), sizeof(long long) * pre.size(), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the host vectors die here
  }
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &per_sm, bf16 ? (const void*)expand_kernel_dev<true> : (const void*)expand_kernel_dev<false>,
        EXP_WARPS * 32, 0);
  long long grid = (acc + EXP_WARPS - 1) / EXP_WARPS;
  const long long cap = (long long)sms * (per_sm > 0 ? per_sm : 1);
  p->grid = (int)(grid < cap ? (grid < 1 ? 1 : grid) : cap);
  if (e != cudaSuccess) {
    expand_plan_destroy(p);
    return e;
  }
  *out = p;
  return cudaSuccess;
}

cudaError_t expand_plan_run(void* plan, cudaStream_t st) {
  auto* p = static_cast<ExpandPlan*>(plan);
  if (p->n == 0) return cudaSuccess;
  if (p->bf16) expand_kernel_dev<true><<<p->grid, EXP_WARPS * 32, 0, st>>>(p->tab, p->prefix, p->n, p->total);
  else expand_kernel_dev<false><<<p->grid, EXP_WARPS * 32, 0, st>>>(p->tab, p->prefix, p->n, p->total);
  return cudaGetLastError();
}

void expand_plan_destroy(void* plan) {
  auto* p = static_cast<ExpandPlan*>(plan);
  if (!p) return;
  if (p->tab) cudaFree(p->tab);
  if (p->prefix) cudaFree(p->prefix);
  delete p;
}

}  // namespace qftk
