// gradquant.cu -- quantize_state of a plan's RAW (f32 / bf16) gradient into the plan's
// u8 gradient scratch, so the rows kernel can run the step (the GradientStack entry the
// reference's sink would have pushed: gradflow.hpp:77 -> quantize_state,
// quantize.hpp:189-193 -> compute_affine_params (:133-137) -> quantize (:143-175)).
//
// A warp (or a CTA of 4 / 8 warps for wide rows) per row, persistent over a static row
// stride, the tensor found by binary search over the row bases: every lane loads its
// 16-byte vectors of the row into registers (all loads in flight at once), the team
// reduces the row's min/max with the reference's NaN semantics (tensor.hpp:133-148: NaN
// never replaces a bound, a NaN in column 0 sticks), derives the affine params, and writes
// the codes from the registers -- the row is read from HBM once.  Traffic per element: 4 / 2 B
// read, 1 B written; per row 8 B of params.
#include <cuda_bf16.h>

#include <cstdio>

#include "qft_device.cuh"
#include "qft_internal.h"

namespace qftk {
using namespace qftd;

namespace gq {
__device__ __forceinline__ void minmax2(float& lo, float& hi, float a, float b) {
  float t;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(lo), "f"(a), "f"(b));
  lo = t;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(hi), "f"(a), "f"(b));
  hi = t;
}

// the 8 (bf16) or 4 (f32) values of a 16-byte vector as floats
template <bool BF16>
__device__ __forceinline__ void unpack(const uint4& q, float* x) {
  if (BF16) {
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[2 * i] = __uint_as_float(w[i] << 16);
      x[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  } else {
    x[0] = __uint_as_float(q.x);
    x[1] = __uint_as_float(q.y);
    x[2] = __uint_as_float(q.z);
    x[3] = __uint_as_float(q.w);
  }
}
}  // namespace gq

// One CTA of NT threads per row (persistent, static row stride); every thread holds VPL
// 16-byte vectors of the row in registers, so a row is read from HBM once and the CTA's
// loads are all in flight together.  The min/max partials of the warps go through shared
// memory (double-buffered by row parity, so ONE barrier per row suffices) and every thread
// derives the row's affine params itself (FMA-proven fast divide, exact fp64 fallback).
// Quantization is range-proven (every value lies in [lo, hi], whose codes are 0 and
// qmax, so no clip is needed): per element one multiply, the magic-number rint and its
// tie distance; a thread whose values come within the error bound of a tie redoes its
// vectors with the reference's fp64 formula.
// register budget: the row in flight twice (current + prefetched next row, 8 regs per
// vector) plus ~24; a budget below that would spill the prefetch to local memory
template <int NT, int VPL>
constexpr int gq_minb() { return VPL <= 2 ? 65536 / (NT * 64) : 65536 / (NT * 128); }
template <bool BF16, int NT, int VPL>
__global__ void __launch_bounds__(NT, gq_minb<NT, VPL>()) k_grad_quant(const LaunchArgs a) {
  using namespace gq;
  constexpr int EPV = BF16 ? 8 : 4;  // elements per 16-byte vector
  constexpr int NW = NT / 32;
  __shared__ float red[2][2][NW];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int bw = a.bit_width;
  const int qmax = (1 << bw) - 1;
  const double rq = __drcp_rn((double)qmax);
  int par = 0;
  // the row's tensor (binary search over the row bases) and its first 16-byte vector
  auto locate = [&](int row, int& ti) -> const uint4* {
    int lo_t = 0, hi_t = a.n_tensors - 1;
    while (lo_t < hi_t) {
      const int mid = (lo_t + hi_t + 1) >> 1;
      if (a.tensors[mid].row_base <= row) lo_t = mid;
      else hi_t = mid - 1;
    }
    ti = lo_t;
    const DevTensor& T = a.tensors[lo_t];
    return reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(T.g_raw) +
                                          (size_t)(row - T.row_base) * T.cols * (BF16 ? 2 : 4));
  };
  // loads of a row into registers; vectors past the row end repeat vector 0 (same range)
  auto load = [&](const uint4* src, int nv, uint4* v) {
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int i = t + j * NT;
      v[j] = __ldcs(src + (i < nv ? i : 0));
    }
  };
  int gr = blockIdx.x;
  if (gr >= a.total_rows) return;
  int ti;
  const uint4* src = locate(gr, ti);
  uint4 v[VPL], vn[VPL];
  load(src, a.tensors[ti].cols / EPV, v);
  for (;; gr += gridDim.x, par ^= 1) {
    const DevTensor& T = a.tensors[ti];
    const int r = gr - T.row_base;
    const int cols = T.cols;
    const int nv = cols / EPV;  // cols % 16 == 0 on this path
    // the CTA's next row streams in while this one is reduced and quantized
    const int gn = gr + (int)gridDim.x;
    int tin = ti;
    const uint4* srcn = nullptr;
    if (gn < a.total_rows) {
      srcn = locate(gn, tin);
      load(srcn, a.tensors[tin].cols / EPV, vn);
    }
    float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      float x[EPV];
      unpack<BF16>(v[j], x);
#pragma unroll
      for (int e = 0; e < EPV; e += 2) minmax2(lo, hi, x[e], x[e + 1]);
    }
    asm("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(lo) : "f"(lo));
    asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(hi) : "f"(hi));
    if (lane == 0) {
      red[par][0][wid] = lo;
      red[par][1][wid] = hi;
    }
    __syncthreads();
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      lo = fminf(lo, red[par][0][w]);
      hi = fmaxf(hi, red[par][1][w]);
    }
    // column 0: a NaN there is the initial bound and sticks (tensor.hpp:133-148)
    if (t == 0) {
      const float c0 = BF16 ? __uint_as_float(v[0].x << 16) : __uint_as_float(v[0].x);
      if (c0 != c0) atomicOr(&a.hdr->err, ERR_GPARAMS);
    }
    const float c0 = BF16 ? __uint_as_float(__ldg(reinterpret_cast<const uint32_t*>(src)) << 16)
                          : __ldg(reinterpret_cast<const float*>(src));
    if (c0 != c0) lo = hi = c0;
    float s;
    int32_t z;
    bool ok = affine_fast(lo, hi, (double)qmax, rq, s, z);
    if (!ok) {
      ok = affine_from_bounds(lo, hi, bw, s, z);
      if (!ok) {
        s = 1.0f;
        z = 0;
      }
    }
    if (t == 0) {
      if (!ok) atomicOr(&a.hdr->err, ERR_GPARAMS);
      const_cast<float*>(T.g_scale)[r] = s;
      const_cast<int32_t*>(T.g_zp)[r] = z;
    }
    const QuantRow q = make_quant_row(s, z, bw);
    // range proof: lo and hi quantize (fast form, unclamped) to codes inside [0, qmax]
    float el = 0.0f;
    const float lh[4] = {lo, hi, lo, hi};
    (void)quant4_e(lh, q, el);
    const float ylo = __fmul_rn(lo, q.inv_s), yhi = __fmul_rn(hi, q.inv_s);
    const bool fast = ok && q.fast && el < q.thr && ylo > q.ylo - 0.5f && yhi < q.yhi + 0.5f;
    uint32_t c[VPL][EPV / 4];
    float em = 0.0f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      float x[EPV];
      unpack<BF16>(v[j], x);
#pragma unroll
      for (int k = 0; k < EPV / 4; ++k) c[j][k] = quant4_e(x + 4 * k, q, em);
    }
    if (!(fast && em < q.thr)) {  // near a tie (or no range proof): the reference formula
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        float x[EPV];
        unpack<BF16>(v[j], x);
#pragma unroll
        for (int k = 0; k < EPV / 4; ++k) c[j][k] = quant4_exact(x + 4 * k, q);
      }
    }
    uint8_t* dst = const_cast<uint8_t*>(T.g_codes) + (size_t)r * cols;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int i = t + j * NT;
      if (i < nv) {
        if constexpr (BF16)
          __stcs(reinterpret_cast<uint2*>(dst) + i, make_uint2(c[j][0], c[j][1]));
        else
          __stcs(reinterpret_cast<uint32_t*>(dst) + i, c[j][0]);
      }
    }
    if (gn >= a.total_rows) break;
    ti = tin;
    src = srcn;
#pragma unroll
    for (int j = 0; j < VPL; ++j) v[j] = vn[j];
  }
}

template <bool BF16, int NT, int VPL>
static cudaError_t gq_resolve_t(int total_rows, const char* name, KLaunch* out) {
  const void* fn = reinterpret_cast<const void*>(k_grad_quant<BF16, NT, VPL>);
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT, 0);
  if (e != cudaSuccess) return e;
  long grid = (long)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > total_rows) grid = total_rows;
  out->fn = fn;
  out->grid = (int)(grid < 1 ? 1 : grid);
  out->block = NT;
  out->smem = 0;
  snprintf(out->name, sizeof(out->name), "%s", name);
  return cudaSuccess;
}

// the launch for a plan of raw-gradient kind gk over rows of <= max_cols columns
cudaError_t resolve_grad_quant(int gk, int max_cols, int total_rows, KLaunch* out) {
  if (gk == G_BF16) {  // 8 elements per vector
    if (max_cols <= 8 * 256 * 2) return gq_resolve_t<true, 256, 2>(total_rows, "k_grad_quant<bf16,256,2>", out);
    if (max_cols <= 8 * 1024 * 2) return gq_resolve_t<true, 1024, 2>(total_rows, "k_grad_quant<bf16,1024,2>", out);
  } else if (gk == G_F32) {  // 4 elements per vector
    if (max_cols <= 4 * 512 * 2) return gq_resolve_t<false, 512, 2>(total_rows, "k_grad_quant<f32,512,2>", out);
    if (max_cols <= 4 * 1024 * 2) return gq_resolve_t<false, 1024, 2>(total_rows, "k_grad_quant<f32,1024,2>", out);
    if (max_cols <= 4 * 512 * 8) return gq_resolve_t<false, 512, 8>(total_rows, "k_grad_quant<f32,512,8>", out);
  }
  return cudaErrorInvalidValue;
}

}  // namespace qftk
