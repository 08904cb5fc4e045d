// wgrad.cu -- the backward's weight gradient with the gradient quantization fused into the
// GEMM epilogue: G[O,I] = dY[T,O]^T . X[T,I] (network.hpp:139,
// backward_core: wgrad = matmul(transpose(out_grad), in)) and, in the same kernel, the
// backward sink (gradflow.hpp:70-84): the first micro-batch pushes quantize_state(G)
// (:77 -> quantize.hpp:189-193: per-row min/max, affine_params_from_bounds, quantize); later
// ones fold in integer form, quantize_state(dequantize(acc) + G) (accumulate, :52-58).  The
// fp32 gradient never reaches HBM: what leaves the chip is the u8 codes + per-row params, the
// GradientStack entry lion_step_quantized pops.  dY, X are bf16 activations; the products
// accumulate in fp32 in TMEM.
//
// The quantizer needs each row's min/max over ALL of its I columns, which span I/256 CTAs.
// The grid is persistent and co-resident (cooperative launch, one CTA per SM), tiles are
// assigned round-robin in row-block-major order, and the CTAs of a row block meet through
// global memory: each epilogue thread (one per row and column half) reduces its values,
// merges them into the row's global bounds (order-preserving integer atomics), and the row
// block's counter releases them once every tile of the block has contributed; then every
// CTA derives the same params (fp64, the reference's formula) and quantizes its values
// straight from TMEM.  Deadlock-free when a row block has at most gridDim tiles (checked by
// the launcher): a CTA waiting in round k waits only for tiles of rounds k-1..k+1, and the
// round-(k+1) tiles of a straddling block belong to CTAs whose round-k tile completes
// without waiting on round k+1.  TMEM holds two 256-column accumulators, so the next tile's
// MMAs run while this tile's epilogue waits.
//
// sm_100a, one 128 x 256 output tile (O rows x I columns) per CTA iteration, K (= tokens)
// in blocks of 64:
//   warp 0 (lane 0)  TMA: dY^T and X tiles, both MN-major (the activations' natural
//                    layout: no transpose pass) -- dY box {64 O, 64 T} x 2, X box {64 I,
//                    64 T} x 4, SWIZZLE_128B -- into a 4-stage ring (mbarrier tx)
//   warp 1 (lane 0)  tcgen05.mma.cta_group::1.kind::f16, M=128, N=256, K=16 x 4 per block,
//                    A and B MN-major, into TMEM accumulator (tile & 1); commits
//   warp 2           TMEM allocation (512 columns) and release
//   warps 4-11       the epilogue: warp 4 + 4h + q reads TMEM lanes 32q.. (rows), columns
//                    [128h, 128h + 128) of the tile, 32 at a time (tcgen05.ld 32x32b.x32)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cstdio>

#include "qft_device.cuh"
#include "qft_internal.h"
#include "umma.cuh"

namespace qftk {
using namespace qftd;

namespace wg {
using namespace um;
constexpr int BM = 128;  // gradient rows (O) per tile: UMMA M
constexpr int BN = 256;  // gradient columns (I) per tile: UMMA N
constexpr int BK = 64;   // tokens per K block
#ifndef WG_STAGES
#define WG_STAGES 4
#endif
constexpr int STAGES = WG_STAGES;
constexpr int A_BYTES = BM * BK * 2;  // 2 MN chunks of 64 x 64 bf16 (8 KB each)
constexpr int B_BYTES = BN * BK * 2;  // 4 MN chunks
constexpr int CHUNK = 64 * BK * 2;    // one TMA box: 64 MN elements x 64 K rows = 8 KB
constexpr int SMEM_BYTES = STAGES * (A_BYTES + B_BYTES) + 1024;
constexpr int NT = 128 + 256;  // TMA, MMA, TMEM, idle warps + 8 epilogue warps
constexpr int NEPI = 8;
// instruction descriptor: D f32, A/B bf16, A and B MN-major (bits 15, 16), N = 256, M = 128
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | (1u << 16) |
                           ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
constexpr int TMEM_COLS = 2 * BN;

// order-preserving float -> u32 (u32 compare == float compare for non-NaN values)
__device__ __forceinline__ uint32_t ord(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float unord(uint32_t u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}
__device__ __forceinline__ void epi_bar() {  // the 256 epilogue threads
  asm volatile("bar.sync 1, 256;" ::: "memory");
}
}  // namespace wg

struct WgArgs {
  int T, O, I, bw;
  int accumulate;        // 0: push quantize_state(G); 1: quantize_state(dequantize(acc) + G)
  uint8_t* codes;        // [O, I] stack entry codes (read first when accumulating; in place)
  float* scale;          // [O]
  int32_t* zp;           // [O]
  float* g_out;          // optional [O, I] fp32 G (tests: the materialised gradient)
  double* norm_sq;       // optional: += sum of G^2 (backward_core's norm, network.hpp:140)
  uint32_t* rmin;        // [O] workspace: row bounds (ord), NaN-in-column-0 flags, counters
  uint32_t* rmax;        // [O]
  uint32_t* nan0;        // [O]
  uint32_t* cnt;         // [tiles_m]
  uint32_t* err;         // NaN in column 0 (the reference's min > max)
  int tiles_m, tiles_n;
  uint32_t lbo, sbo;     // MN-major descriptor strides
};

__global__ void __launch_bounds__(wg::NT, 1)
    k_wgrad_quant(const __grid_constant__ CUtensorMap tm_dy, const __grid_constant__ CUtensorMap tm_x,
                  const WgArgs a) {
  using namespace wg;
  extern __shared__ uint8_t dsm_raw[];
  uint8_t* dsm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntiles = a.tiles_m * a.tiles_n;
  const int nkb = (a.T + BK - 1) / BK;
  auto a_tile = [&](int s) { return dsm + s * (A_BYTES + B_BYTES); };
  auto b_tile = [&](int s) { return dsm + s * (A_BYTES + B_BYTES) + A_BYTES; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], NEPI);
    }
    mbar_fence_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_base)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before_sync();
  __syncthreads();
  tc_after_sync();
  const uint32_t tmem_d = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int o0 = (t / a.tiles_n) * BM, i0 = (t % a.tiles_n) * BN;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], (uint32_t)(((it / STAGES) & 1) ^ 1));
          mbar_arrive_expect_tx(&full[s], (uint32_t)(A_BYTES + B_BYTES));
#pragma unroll
          for (int h = 0; h < BM / 64; ++h)
            tma_load_2d(a_tile(s) + h * CHUNK, &tm_dy, o0 + 64 * h, kb * BK, &full[s]);
#pragma unroll
          for (int h = 0; h < BN / 64; ++h)
            tma_load_2d(b_tile(s) + h * CHUNK, &tm_x, i0 + 64 * h, kb * BK, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      int it = 0, lt = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
        const int buf = lt & 1;
        mbar_wait(&acc_empty[buf], (uint32_t)(((lt >> 1) & 1) ^ 1));
        tc_after_sync();
        const uint32_t acc_addr = tmem_d + (uint32_t)(buf * BN);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % STAGES;
          mbar_wait(&full[s], (uint32_t)((it / STAGES) & 1));
          tc_after_sync();
          const uint32_t sa = smem_u32(a_tile(s)), sb = smem_u32(b_tile(s));
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)  // 16 K rows = two 8-row swizzle atoms
            mma_bf16(acc_addr, sw128_desc_mn(sa + kk * 2048, a.lbo, a.sbo),
                     sw128_desc_mn(sb + kk * 2048, a.lbo, a.sbo), IDESC,
                     (kb > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[buf]);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue
    const int q = (warp - 4) & 3, h = (warp - 4) >> 2;
    const uint32_t lane_base = (uint32_t)(32 * q) << 16;
    const int bw = a.bw;
    double nsq = 0.0;
    int lt = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++lt) {
      const int tm = t / a.tiles_n;
      const int o0 = tm * BM, i0 = (t % a.tiles_n) * BN;
      const int buf = lt & 1;
      const int row = o0 + 32 * q + lane;
      const bool live = row < a.O;
      const int cbase = i0 + 128 * h;  // this thread's 128 columns of the row
      const uint32_t tbase = tmem_d + lane_base + (uint32_t)(buf * BN + 128 * h);
      mbar_wait(&acc_full[buf], (uint32_t)((lt >> 1) & 1));
      tc_after_sync();
      // old entry (accumulating): its params, read before this block's counter completes
      DequantRow d{};
      if (a.accumulate && live) d = make_dequant_row(a.scale[row], a.zp[row]);
      const uint8_t* crow = a.codes + (size_t)row * a.I;
      // the value of column c of the chunk: G, or dequantize(acc) + G (gradflow.hpp:57, the
      // reference's add(dequantize(acc), g_new): one fp32 rounding each)
      auto values = [&](int c, uint32_t* r, float* v) {
        tmem_ld32(tbase + (uint32_t)(32 * c), r);
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]);
        if (a.accumulate && live && cbase + 32 * c < a.I) {
          const uint4* cp = reinterpret_cast<const uint4*>(crow + cbase + 32 * c);
          const uint4 c0 = cp[0], c1 = cp[1];
          const uint32_t w[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            float dq[4];
            if (d.fast) {
              dequant4(w[k], d, dq);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) dq[e] = dequant_exact((w[k] >> (8 * e)) & 0xFFu, d.s, d.z);
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) v[4 * k + e] = __fadd_rn(dq[e], v[4 * k + e]);
          }
        }
      };
      // ---- phase A: the row's bounds over this thread's columns
      float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
      bool nan_c0 = false;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        if (cbase + 32 * c >= a.I) break;
        uint32_t r[32];
        float v[32];
        values(c, r, v);
        if (a.norm_sq) {
          float ss = 0.0f;
#pragma unroll
          for (int e = 0; e < 32; ++e) ss = __fadd_rn(ss, __fmul_rn(__uint_as_float(r[e]), __uint_as_float(r[e])));
          nsq += (double)ss;
        }
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          float m;
          asm("min.f32 %0, %1, %2, %3;" : "=f"(m) : "f"(lo), "f"(v[e]), "f"(v[e + 1]));
          lo = m;
          asm("max.f32 %0, %1, %2, %3;" : "=f"(m) : "f"(hi), "f"(v[e]), "f"(v[e + 1]));
          hi = m;
        }
        if (cbase + 32 * c == 0) nan_c0 = v[0] != v[0];
        if (a.g_out && live) {
          float4* gp = reinterpret_cast<float4*>(a.g_out + (size_t)row * a.I + cbase + 32 * c);
#pragma unroll
          for (int k = 0; k < 8; ++k) gp[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        }
      }
      if (live) {
        if (lo == lo) atomicMin(a.rmin + row, ord(lo));  // all-NaN span: nothing to merge
        if (hi == hi) atomicMax(a.rmax + row, ord(hi));
        if (nan_c0) atomicOr(a.nan0 + row, 1u);
      }
      __threadfence();
      epi_bar();
      if (threadIdx.x == 128) {
        atomicAdd(a.cnt + tm, 1u);
        const uint32_t target = (uint32_t)a.tiles_n;  // one arrival per tile
        uint32_t ns = 64;
        while (*(volatile uint32_t*)(a.cnt + tm) < target) {
          __nanosleep(ns);
          ns = ns < 1024 ? ns * 2 : 1024;
        }
        __threadfence();
      }
      epi_bar();
      // ---- phase B: the row's params (every CTA of the block derives the same ones) and
      // its codes straight from TMEM
      float s = 1.0f;
      int32_t z = 0;
      if (live) {
        float rlo = unord(__ldcg(a.rmin + row)), rhi = unord(__ldcg(a.rmax + row));
        if (__ldcg(a.nan0 + row)) rlo = rhi = __int_as_float(0x7fffffff);
        if (!affine_from_bounds(rlo, rhi, bw, s, z)) {
          if (i0 == 0 && h == 0) *(volatile uint32_t*)a.err = 1u;
          s = 1.0f;
          z = 0;
        }
      }
      const QuantRow qr = make_quant_row(s, z, bw);
      // (every lane runs the tcgen05.ld calls -- they are warp-collective -- dead rows only
      // skip the stores)
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        if (cbase + 32 * c >= a.I) break;
        uint32_t r[32];
        float v[32];
        values(c, r, v);
        uint32_t pk[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          float em = 0.0f;
          uint32_t cc = qr.fast ? quant4_e(v + 4 * k, qr, em) : 0u;
          if (!qr.fast || !(em < qr.thr)) {
            cc = 0u;
#pragma unroll
            for (int e = 0; e < 4; ++e)
              cc |= quant_exact(v[4 * k + e], qr.s, qr.z, qr.qmax) << (8 * e);
          }
          pk[k] = cc;
        }
        if (live) {
          uint4* dst = reinterpret_cast<uint4*>(a.codes + (size_t)row * a.I + cbase + 32 * c);
          dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
          dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
        }
      }
      if (live && i0 == 0 && h == 0) {  // one writer per row (every reader holds the old params)
        a.scale[row] = s;
        a.zp[row] = z;
      }
      tc_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
    if (a.norm_sq) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
      if (lane == 0 && nsq != 0.0) atomicAdd(a.norm_sq, nsq);
    }
  }
  tc_before_sync();
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d),
                 "n"(TMEM_COLS));
}

// ------------------------------------------------------------------ host side
size_t wgrad_workspace_bytes(int O) {
  const int tiles_m = (O + wg::BM - 1) / wg::BM;
  return (size_t)(3 * O + tiles_m + 1) * sizeof(uint32_t);
}

cudaError_t launch_wgrad_quant(const void* dy, const void* x, int T, int O, int I, int bw,
                               int accumulate, uint8_t* codes, float* scale, int32_t* zp,
                               float* g_out, double* norm_sq, void* workspace, uint32_t lbo,
                               uint32_t sbo, cudaStream_t st) {
  using namespace wg;
  auto enc = um::encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tdy{}, tx{};
  {
    const cuuint64_t dims[2] = {(cuuint64_t)O, (cuuint64_t)T};
    const cuuint64_t strides[1] = {(cuuint64_t)O * 2};
    const cuuint32_t box[2] = {64, BK};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&tdy, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(dy), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)I, (cuuint64_t)T};
    const cuuint64_t strides[1] = {(cuuint64_t)I * 2};
    const cuuint32_t box[2] = {64, BK};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  static int sms = 0;
  if (!sms) {
    cudaError_t e = cudaFuncSetAttribute(k_wgrad_quant, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         SMEM_BYTES);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
  }
  WgArgs A{};
  A.T = T;
  A.O = O;
  A.I = I;
  A.bw = bw;
  A.accumulate = accumulate;
  A.codes = codes;
  A.scale = scale;
  A.zp = zp;
  A.g_out = g_out;
  A.norm_sq = norm_sq;
  A.tiles_m = (O + BM - 1) / BM;
  A.tiles_n = (I + BN - 1) / BN;
  uint32_t* ws = reinterpret_cast<uint32_t*>(workspace);
  A.rmin = ws;
  A.rmax = ws + O;
  A.nan0 = ws + 2 * O;
  A.cnt = ws + 3 * O;
  A.err = ws + 3 * O + A.tiles_m;  // the workspace's last word
  A.lbo = lbo ? lbo : (uint32_t)CHUNK;
  A.sbo = sbo ? sbo : 1024u;
  const int ntiles = A.tiles_m * A.tiles_n;
  const int grid = ntiles < sms ? ntiles : sms;
  if (A.tiles_n > grid) return cudaErrorInvalidConfiguration;  // see the header
  cudaError_t e = cudaMemsetAsync(ws, 0xFF, (size_t)O * sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(ws + O, 0, (size_t)(2 * O + A.tiles_m + 1) * sizeof(uint32_t), st);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = SMEM_BYTES;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // the row blocks' CTAs must be co-resident
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_wgrad_quant, tdy, tx, A);
}

}  // namespace qftk
