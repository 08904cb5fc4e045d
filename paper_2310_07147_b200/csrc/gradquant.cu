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

// One CTA of NT threads per row (persistent, static row stride).  Rows stream into a
// 4-stage shared-memory ring by TMA bulk copies (thread 0, two rows ahead, one mbarrier
// per stage), and the rows are SOFTWARE-PIPELINED: while row r's min/max is reduced
// (every thread its VPL 16-byte vectors, from the stage), row r-1 -- whose quantizer
// thread 0 derived during the previous iteration -- is quantized from its stage and
// stored.  The row's serial part (thread 0: the fp64 affine params, FMA-proven fast divide
// or the reference formula) overlaps the other threads' quantization; a row costs ONE
// barrier, and the row is read from HBM once.
// Quantization: the fast quantizer (range-proven, no clamp: gq_quant4) with its tie proof
// per group of 4 elements, the reference's fp64 formula for a group near a tie
// (quantize.hpp:160-166).
constexpr int GQ_NS = 4;  // ring stages
#ifndef QFT_GQ_NOCLAMP
#define QFT_GQ_NOCLAMP 1
#endif

// The fast quantizer of a value of the row's own [lo, hi] range.  The clamp to the code
// range is provably unnecessary (QFT_GQ_NOCLAMP): with s = the fp32 scale and z the zero
// point of affine_params_from_bounds(lo, hi), every x in [lo, hi] has x/s in
// [-z - 0.5 - d, qmax - z + 0.5 + d], d <= (qmax + |z| + 1) * 2^-23.9 (the fp32 rounding of
// s and the +-0.5 of z's rounding), so a value whose nearest integer lies outside the code
// range sits within d + (the product's error) of a half-integer: its tie check
// (|y - rint(y)| < 0.5 - (qmax + |z| + 2) * 2^-21) fails and it takes the exact formula,
// which clips.  NaN propagates into the check (max.NaN) and takes the exact path too.
__device__ __forceinline__ uint32_t gq_quant4(const float* x, const QuantRow& q, float& em) {
#if QFT_GQ_NOCLAMP
  return quant4_e(x, q, em);
#else
  return quant4_fast(x, q, em);
#endif
}

#ifndef QFT_GQ_BRANCHFREE
#define QFT_GQ_BRANCHFREE 1
#endif
// the codes of four values of a row whose quantizer is q (bf: the branch-free form applies)
__device__ __forceinline__ uint32_t gq_codes4(const float* x, const QuantRow& q, bool bf) {
  if (QFT_GQ_BRANCHFREE && bf) return quant4_bf(x, q);
  float em = 0.0f;
  uint32_t c = q.fast ? gq_quant4(x, q, em) : 0u;
  if (!q.fast || !(em < q.thr)) c = quant4_exact_fast(x, q);
  return c;
}

template <bool BF16, int NT, int VPL>
__global__ void __launch_bounds__(NT + 32) k_grad_quant(const LaunchArgs a, int stage_bytes) {
  using namespace gq;
  constexpr int EPV = BF16 ? 8 : 4;  // elements per 16-byte vector
  constexpr int NW = NT / 32;        // worker warps; warp NW is the control warp
  extern __shared__ __align__(128) uint8_t gsm[];
  __shared__ float red[2][2][NW];
  __shared__ float prm[2][4];  // per row parity: s, z, RN(1/s), fast
  __shared__ __align__(8) uint64_t bars[GQ_NS];
  // the tensor of the row each stage holds: written by the issuing thread before the
  // stage's TMA (read after the stage's barrier), so the workers never walk the table
  __shared__ int s_ti[GQ_NS];
  // the tensors' first rows (the issuing thread's walk reads them per row): in shared
  // memory when the table is small, so the control warp's serial section per row has no
  // global load
  constexpr int RBMAX = 512;
  __shared__ int s_rb[RBMAX];
  const bool rb_smem = a.n_tensors <= RBMAX;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const bool ctrl = wid == NW;  // the control warp: TMA issue + the row's quantizer
  const int tc = NT;            // its lane 0
  const int bw = a.bit_width;
  const int qmax = (1 << bw) - 1;
  const double rq = __drcp_rn((double)qmax);
  const int G = (int)gridDim.x;
  const int TR = a.total_rows;
  // rows come in increasing order per CTA: the tensor index only moves forward
  int ti_issue = 0;
  auto tensor_of = [&](int row, int& ti) -> const DevTensor& {
    if (rb_smem)
      while (ti + 1 < a.n_tensors && s_rb[ti + 1] <= row) ++ti;
    else
      while (ti + 1 < a.n_tensors && a.tensors[ti + 1].row_base <= row) ++ti;
    return a.tensors[ti];
  };
  // the control thread: row `row` into stage st (one bulk copy of the row)
  auto issue = [&](int row, int st) {
    const DevTensor& T = tensor_of(row, ti_issue);
    s_ti[st] = ti_issue;
    const uint32_t nb = (uint32_t)T.cols * (BF16 ? 2u : 4u);
    mbar_arrive_expect_tx(&bars[st], nb);
    bulk_g2s(gsm + (size_t)st * stage_bytes,
             reinterpret_cast<const uint8_t*>(T.g_raw) + (size_t)(row - T.row_base) * nb, nb,
             &bars[st]);
  };
  auto vec = [&](int st, int i) {
    return reinterpret_cast<const uint4*>(gsm + (size_t)st * stage_bytes)[i];
  };
  // quantize row `row` (stage st, quantizer of parity p) and store its codes
  auto quantize_store = [&](int row, int st, int p) {
    if (ctrl) return;
    const DevTensor& T = a.tensors[s_ti[st]];
    const int nv = T.cols / EPV;
    uint8_t* dst = const_cast<uint8_t*>(T.g_codes) + (size_t)(row - T.row_base) * T.cols;
    QuantRow q;
    q.s = prm[p][0];
    q.z = __float_as_int(prm[p][1]);
    q.inv_s = prm[p][2];
    q.qmax = qmax;
    q.ylo = (float)(-q.z);
    q.yhi = (float)(qmax - q.z);
    q.magic = __fadd_rn(kMagicRound, (float)q.z);
    q.thr = 0.5f - (float)((q.z < 0 ? -(int64_t)q.z : (int64_t)q.z) + qmax + 2) * 0x1.0p-21f;
    q.fast = prm[p][3] != 0.0f;
    const bool bf = q.fast && q.s >= 0x1.0p-100f;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int i = t + j * NT;
      if (i < nv) {
        float x[EPV];
        unpack<BF16>(vec(st, i), x);
        uint32_t c[EPV / 4];
#pragma unroll
        for (int k = 0; k < EPV / 4; ++k) c[k] = gq_codes4(x + 4 * k, q, bf);
        if constexpr (BF16)
          __stcs(reinterpret_cast<uint2*>(dst) + i, make_uint2(c[0], c[1]));
        else
          __stcs(reinterpret_cast<uint32_t*>(dst) + i, c[0]);
      }
    }
  };

  int gr = blockIdx.x;
  if (gr >= TR) return;
  if (t == tc) {
    for (int i = 0; i < GQ_NS; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  if (rb_smem)
    for (int i = t; i < a.n_tensors; i += NT + 32) s_rb[i] = a.tensors[i].row_base;
  __syncthreads();
  if (t == tc) {  // this CTA's first two rows in flight
    for (int k = 0; k < GQ_NS - 2; ++k)
      if (gr + k * G < TR) issue(gr + k * G, k);
  }
  int it = 0, par = 0;
  for (;; ++it, par ^= 1) {
    const int st = it % GQ_NS;
    float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
    if (!ctrl) {
      mbar_wait(&bars[st], (uint32_t)((it / GQ_NS) & 1));
      const int nv = a.tensors[s_ti[st]].cols / EPV;
      // row gr: min/max partials (vectors past the row end repeat vector 0: same range)
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int i = t + j * NT;
        float x[EPV];
        unpack<BF16>(vec(st, i < nv ? i : 0), x);
#pragma unroll
        for (int e = 0; e < EPV; e += 2) minmax2(lo, hi, x[e], x[e + 1]);
      }
      asm("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(lo) : "f"(lo));
      asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(hi) : "f"(hi));
      if (lane == 0) {
        red[par][0][wid] = lo;
        red[par][1][wid] = hi;
      }
    }
    __syncthreads();  // red[par] complete; the previous row's quantizer published; the
                      // stage of row gr - 2G is free (its quantization ended before this)
    if (t == tc) {
      // two rows ahead: row gr + 2G into the stage row gr - 2G vacated (the stages hold
      // gr - G (quantized now), gr, gr + G and this one)
      const int gi = gr + (GQ_NS - 2) * G;
      if (gi < TR) issue(gi, (it + GQ_NS - 2) % GQ_NS);
      // row gr's quantizer (quantize_state: channel_minmax -> affine_params_from_bounds)
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        lo = fminf(lo, red[par][0][w]);
        hi = fmaxf(hi, red[par][1][w]);
      }
      // column 0: a NaN there is the initial bound and sticks (tensor.hpp:133-148)
      float x0[EPV];
      mbar_wait(&bars[st], (uint32_t)((it / GQ_NS) & 1));  // (complete: the workers saw it)
      const DevTensor& T = a.tensors[s_ti[st]];
      unpack<BF16>(vec(st, 0), x0);
      if (x0[0] != x0[0]) lo = hi = x0[0];
      float s;
      int32_t z;
      bool ok = affine_fast(lo, hi, (double)qmax, rq, s, z);
      if (!ok) {
        ok = affine_from_bounds(lo, hi, bw, s, z);
        if (!ok) {
          atomicOr(&a.hdr->err, ERR_GPARAMS);
          s = 1.0f;
          z = 0;
        }
      }
      const_cast<float*>(T.g_scale)[gr - T.row_base] = s;
      const_cast<int32_t*>(T.g_zp)[gr - T.row_base] = z;
      const QuantRow q0 = make_quant_row(s, z, bw);
      prm[par][0] = s;
      prm[par][1] = __int_as_float(z);
      prm[par][2] = q0.inv_s;
      prm[par][3] = q0.fast ? 1.0f : 0.0f;
    }
    if (it > 0) quantize_store(gr - G, (it + GQ_NS - 1) % GQ_NS, par ^ 1);
    if (gr + G >= TR) break;
    gr += G;
  }
  __syncthreads();  // the last row's quantizer
  quantize_store(gr, it % GQ_NS, par);
}

template <bool BF16, int NT, int VPL>
static cudaError_t gq_resolve_t(int total_rows, int max_cols, const char* name, KLaunch* out) {
  const void* fn = reinterpret_cast<const void*>(k_grad_quant<BF16, NT, VPL>);
  const int stage = ((max_cols * (BF16 ? 2 : 4)) + 127) & ~127;
  const size_t smem = (size_t)GQ_NS * stage;
  int dev = 0, sms = 0, per_sm = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa{};
  cudaError_t e = cudaFuncGetAttributes(&fa, fn);
  if (e != cudaSuccess) return e;
  const int maxdyn = optin - (int)fa.sharedSizeBytes;  // the static part counts against it
  if ((size_t)maxdyn < smem) return cudaErrorInvalidValue;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, maxdyn);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, NT + 32, smem);
  if (e != cudaSuccess) return e;
  long grid = (long)sms * (per_sm > 0 ? per_sm : 1);
  if (grid > total_rows) grid = total_rows;
  out->fn = fn;
  out->grid = (int)(grid < 1 ? 1 : grid);
  out->block = NT + 32;
  out->smem = smem;
  out->arg1 = stage;
  snprintf(out->name, sizeof(out->name), "%s", name);
  return cudaSuccess;
}

// the launch for a plan of raw-gradient kind gk over rows of <= max_cols columns
cudaError_t resolve_grad_quant(int gk, int max_cols, int total_rows, KLaunch* out) {
  if (gk == G_BF16) {  // 8 elements per vector
    if (max_cols <= 8 * 128 * 4) return gq_resolve_t<true, 128, 4>(total_rows, max_cols, "k_grad_quant<bf16,128,4>", out);
    if (max_cols <= 8 * 256 * 8) return gq_resolve_t<true, 256, 8>(total_rows, max_cols, "k_grad_quant<bf16,256,8>", out);
  } else if (gk == G_F32) {  // 4 elements per vector
    if (max_cols <= 4 * 128 * 8) return gq_resolve_t<false, 128, 8>(total_rows, max_cols, "k_grad_quant<f32,128,8>", out);
    if (max_cols <= 4 * 256 * 16) return gq_resolve_t<false, 256, 16>(total_rows, max_cols, "k_grad_quant<f32,256,16>", out);
  }
  return cudaErrorInvalidValue;
}

}  // namespace qftk

// ---------------------------------------------------------------------------------------
// The ZeRO-1 reduce-scatter fused with the sink's quantize_state:
// rank k's shard rows of the summed gradient are read straight from every peer's full
// (shard-major) bf16 gradient buffer over NVLink peer memory -- the source of a row for
// peer j is its local address + deltas[j] bytes -- summed in fp32 in rank order
// (deterministic), reduced for the row's min/max and quantized into the plan's u8 entry.
// No reduced gradient is ever written: the collective and the quantization are one pass.
// One CTA per row; every thread keeps its VPL vectors' fp32 sums in registers.
namespace qftk {
using namespace qftd;

template <int NT, int VPL>
__global__ void __launch_bounds__(NT) k_rs_grad_quant(const LaunchArgs a, const int64_t* deltas,
                                                       int npeer) {
  using namespace gq;
  constexpr int NW = NT / 32;
  __shared__ float red[2][NW];
  __shared__ float prm[4];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int bw = a.bit_width;
  const int qmax = (1 << bw) - 1;
  const double rq = __drcp_rn((double)qmax);
  int ti = 0;
  for (int gr = blockIdx.x; gr < a.total_rows; gr += gridDim.x) {
    while (ti + 1 < a.n_tensors && a.tensors[ti + 1].row_base <= gr) ++ti;
    const DevTensor& T = a.tensors[ti];
    const int r = gr - T.row_base;
    const int nv = T.cols / 8;  // bf16 vectors
    const uint8_t* local = reinterpret_cast<const uint8_t*>(T.g_raw) + (size_t)r * T.cols * 2;
    float sum[VPL][8];
#pragma unroll
    for (int j = 0; j < VPL; ++j)
#pragma unroll
      for (int e = 0; e < 8; ++e) sum[j][e] = 0.0f;
    for (int p = 0; p < npeer; ++p) {
      const uint4* src = reinterpret_cast<const uint4*>(local + deltas[p]);
      uint4 v[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const int i = t + j * NT;
        v[j] = __ldcv(src + (i < nv ? i : 0));  // peers' buffers: never cached stale
      }
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        float x[8];
        unpack<true>(v[j], x);
#pragma unroll
        for (int e = 0; e < 8; ++e) sum[j][e] = p == 0 ? x[e] : __fadd_rn(sum[j][e], x[e]);
      }
    }
    float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
#pragma unroll
    for (int j = 0; j < VPL; ++j)
#pragma unroll
      for (int e = 0; e < 8; e += 2) minmax2(lo, hi, sum[j][e], sum[j][e + 1]);
    asm("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(lo) : "f"(lo));
    asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(hi) : "f"(hi));
    if (lane == 0) {
      red[0][wid] = lo;
      red[1][wid] = hi;
    }
    __syncthreads();
    if (t == 0) {
#pragma unroll
      for (int w = 1; w < NW; ++w) {
        lo = fminf(lo, red[0][w]);
        hi = fmaxf(hi, red[1][w]);
      }
      if (sum[0][0] != sum[0][0]) lo = hi = sum[0][0];  // column 0's NaN sticks
      float s;
      int32_t z;
      bool ok = affine_fast(lo, hi, (double)qmax, rq, s, z);
      if (!ok) {
        ok = affine_from_bounds(lo, hi, bw, s, z);
        if (!ok) {
          atomicOr(&a.hdr->err, ERR_GPARAMS);
          s = 1.0f;
          z = 0;
        }
      }
      const_cast<float*>(T.g_scale)[r] = s;
      const_cast<int32_t*>(T.g_zp)[r] = z;
      prm[0] = s;
      prm[1] = __int_as_float(z);
    }
    __syncthreads();
    const QuantRow q = make_quant_row(prm[0], __float_as_int(prm[1]), bw);
    const bool bf = q.fast && q.s >= 0x1.0p-100f;
    uint8_t* dst = const_cast<uint8_t*>(T.g_codes) + (size_t)r * T.cols;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int i = t + j * NT;
      if (i < nv) {
        uint32_t c[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) c[k] = gq_codes4(sum[j] + 4 * k, q, bf);
        __stcs(reinterpret_cast<uint2*>(dst) + i, make_uint2(c[0], c[1]));
      }
    }
    __syncthreads();  // red / prm are rewritten by the next row
  }
}

template <int NT, int VPL>
static cudaError_t rs_resolve_t(int total_rows, const char* name, KLaunch* out) {
  const void* fn = reinterpret_cast<const void*>(k_rs_grad_quant<NT, VPL>);
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

cudaError_t resolve_rs_grad_quant(int max_cols, int total_rows, KLaunch* out) {
  if (max_cols <= 8 * 256 * 2) return rs_resolve_t<256, 2>(total_rows, "k_rs_grad_quant<256,2>", out);
  if (max_cols <= 8 * 512 * 4) return rs_resolve_t<512, 4>(total_rows, "k_rs_grad_quant<512,4>", out);
  return cudaErrorInvalidValue;
}

cudaError_t launch_rs_grad_quant(const KLaunch& k, const LaunchArgs& a, const int64_t* deltas,
                                 int npeer, cudaStream_t st) {
  LaunchArgs aa = a;
  const int64_t* d = deltas;
  int np = npeer;
  void* args[] = {&aa, &d, &np};
  return cudaLaunchKernel(k.fn, dim3((unsigned)k.grid), dim3((unsigned)k.block), args, k.smem, st);
}

}  // namespace qftk
