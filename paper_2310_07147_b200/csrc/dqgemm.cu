// dqgemm.cu -- the forward consumer's GEMM with the weight dequantization fused into its
// operand producer: Y[M,N] = X[M,K] . W^T, where W is a QFT
// dense-and-sparse weight -- u8 codes [N,K] (rows = output channels, tensor.hpp:13-16),
// per-row (scale, zero point) and the CSR outliers -- and X, Y are bf16.  The reference
// consumer reconstructs W (quantize.hpp:331-338: dequantize every code, then overwrite the
// CSR positions with their fp32 values) and multiplies (network.hpp:113-129,
// forward_core: matmul(cur, transpose(weight_at(l)))); here the bf16 operand the tensor
// cores read is exactly RNE(reconstruct(W)) -- the bytes qftc_expand(bf16) would write --
// but it never exists in HBM: W streams as 1 byte per element instead of 2.
//
// sm_100a, one 512 x 128 output tile per CTA (DQ_BN=128: 4 accumulators; DQ_BN=256 gives
// 256 x 256 with 2), K in blocks of 64:
//   warp 0 (lane 0)  TMA: the X tile (512 x 64 bf16, two 256-row boxes, SWIZZLE_128B) of a
//                    K block into a stage of the X ring (2 stages, mbarrier tx); the
//                    dequantized W operand has its own 4-stage ring, so the producers run
//                    up to three blocks ahead of the MMAs
//   warp 3 (lane 0)  TMA: the W code tile (128 x 64 u8) into its own 4-stage ring
//   warps 4-11       the dequant producers: a thread pair owns W row n0 + j, each thread
//                    32 columns of a block: its codes of
//                    the stage -> s*(q-z) (fp32, one rounding, quantize.hpp:209) -> its
//                    CSR outliers in [k0, k0+64) overwrite their positions -> bf16 (RNE)
//                    -> the K-major SWIZZLE_128B layout tcgen05 reads; fence.proxy.async;
//                    one arrive per warp.  Each keeps a cursor into its row's CSR slot
//                    (columns ascending), so the outliers cost O(nnz) per row in total.
//   warp 1 (lane 0)  tcgen05.mma.cta_group::1.kind::f16, M=128, N=128, K=16 x 4 per block
//                    for each of the four 128-row blocks of X (all read the same
//                    dequantized W operand: each dequantized element feeds 4 x 128 rows of
//                    MMA), into four TMEM accumulators (fp32); tcgen05.commit frees the stage
//   warps 4-11       the epilogue after the last block: tcgen05.ld 32x32b -> bf16 -> HBM
//   warp 2           TMEM allocation (512 columns: the accumulators) and release
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cstdio>

#include "qft_device.cuh"
#include "qft_internal.h"
#include "umma.cuh"

namespace qftk {
using namespace qftd;

#ifndef DQ_NOPROD
#define DQ_NOPROD 0
#endif
#ifndef DQ_NOFENCE
#define DQ_NOFENCE 0
#endif
namespace dq {
using namespace um;
#ifndef DQ_BN
#define DQ_BN 128
#endif
constexpr int BN = DQ_BN;          // output columns (W rows) per CTA: UMMA N
constexpr int NACC = 512 / BN;     // M=128 accumulators: all 512 TMEM columns
constexpr int BM = 128 * NACC;     // output rows (X rows) per CTA
constexpr int BK = 64;      // K per block: 128 bytes of bf16 = one SWIZZLE_128B row
#ifndef DQ_STAGES
#define DQ_STAGES 2
#endif
#ifndef DQ_CSTAGES
#define DQ_CSTAGES 4
#endif
#ifndef DQ_WSTAGES
#define DQ_WSTAGES 4
#endif
constexpr int STAGES = DQ_STAGES;    // X ring
constexpr int WSTAGES = DQ_WSTAGES;  // dequantized W-operand ring (producers run ahead)
constexpr int CSTAGES = DQ_CSTAGES;  // W-code ring
constexpr int A_BYTES = BM * BK * 2;  // NACC 128-row blocks of 16 KB
constexpr int B_BYTES = BN * BK * 2;
constexpr int C_BYTES = BN * BK;      // codes
constexpr int SMEM_BYTES = STAGES * A_BYTES + WSTAGES * B_BYTES + CSTAGES * C_BYTES + 1024;
#ifndef DQ_HALVES
#define DQ_HALVES 2
#endif
constexpr int HALVES = DQ_HALVES;     // producer threads per W row
constexpr int CPT = BK / HALVES;      // columns of a K block per producer thread
constexpr int NQ = CPT / 16;          // 16-code vectors per producer thread and block
constexpr int NPW = BN * HALVES / 32; // producer warps
constexpr int NT = 128 + BN * HALVES; // TMA (X), MMA, TMEM, TMA (codes) warps + producers

// instruction descriptor: D f32, A/B bf16, both K-major, N = BN, M = 128 (per accumulator)
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(128 >> 4) << 24);
constexpr int TMEM_COLS = NACC * BN;  // NACC fp32 accumulators of BN columns (512)
constexpr int XBOX = BM < 256 ? BM : 256;  // TMA box rows (<= 256): BM / XBOX loads per X tile

}  // namespace dq

struct DqArgs {
  const float* scale;        // [N]
  const int32_t* zp;         // [N]
  const int32_t* row_start;  // [N] CSR slot starts (arena offsets)
  const int32_t* row_count;  // [N] used entries (null: strict CSR, count = rs[n+1]-rs[n])
  const int32_t* col;        // arena
  const float* val;
  __nv_bfloat16* y;          // [M, N]
  int M, N, K;
};

__global__ void __launch_bounds__(dq::NT, 1)
    k_dq_gemm(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
              const DqArgs a) {
  using namespace dq;
  extern __shared__ uint8_t dsm_raw[];
  // 1024-byte aligned (SWIZZLE_128B atoms); pointer arithmetic on the shared array keeps
  // the address space visible to the compiler (LDS/STS, not generic loads and stores)
  uint8_t* dsm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full_a[STAGES], empty_a[STAGES], full_b[WSTAGES], empty_b[WSTAGES];
  __shared__ __align__(8) uint64_t full_c[CSTAGES], empty_c[CSTAGES], acc_full;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nkb = a.K / BK;
  auto a_tile = [&](int s) { return dsm + s * A_BYTES; };
  auto b_tile = [&](int w) { return dsm + STAGES * A_BYTES + w * B_BYTES; };
  auto c_tile = [&](int c) { return dsm + STAGES * A_BYTES + WSTAGES * B_BYTES + c * C_BYTES; };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_a[s], 1);
      mbar_init(&empty_a[s], 1);
    }
    for (int w = 0; w < WSTAGES; ++w) {
      mbar_init(&full_b[w], NPW);
      mbar_init(&empty_b[w], 1);
    }
    for (int c = 0; c < CSTAGES; ++c) {
      mbar_init(&full_c[c], 1);
      mbar_init(&empty_c[c], NPW);
    }
    mbar_init(&acc_full, 1);
    mbar_fence_init();
  }
  if (warp == 2) {  // TMEM: two accumulators of BN fp32 columns x 128 lanes
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
    if (lane == 0) {  // ---------------- TMA: X tiles
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&empty_a[s], (uint32_t)(((kb / STAGES) & 1) ^ 1));
        mbar_arrive_expect_tx(&full_a[s], (uint32_t)A_BYTES);
#pragma unroll
        for (int xb = 0; xb < BM / XBOX; ++xb)
          tma_load_2d(a_tile(s) + xb * XBOX * 128, &tm_x, kb * BK, m0 + xb * XBOX, &full_a[s]);
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {  // ---------------- TMA: W code tiles (their own, deeper ring)
      for (int kb = 0; kb < nkb; ++kb) {
        const int c = kb % CSTAGES;
        mbar_wait(&empty_c[c], (uint32_t)(((kb / CSTAGES) & 1) ^ 1));
        mbar_arrive_expect_tx(&full_c[c], (uint32_t)C_BYTES);
        tma_load_2d(c_tile(c), &tm_w, kb * BK, n0, &full_c[c]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES, w = kb % WSTAGES;
        mbar_wait(&full_a[s], (uint32_t)((kb / STAGES) & 1));
        mbar_wait(&full_b[w], (uint32_t)((kb / WSTAGES) & 1));
        tc_after_sync();
        const uint32_t sa = smem_u32(a_tile(s)), sb = smem_u32(b_tile(w));
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {  // every 128-row block shares the W operand
          const uint64_t bd = sw128_desc(sb + 32 * kk);
          const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
#pragma unroll
          for (int ab = 0; ab < NACC; ++ab)
            mma_bf16(tmem_d + ab * BN, sw128_desc(sa + ab * 128 * 128 + 32 * kk), bd, IDESC, acc);
        }
        mma_commit(&empty_a[s]);  // the X and W-operand slots are free once these MMAs read them
        mma_commit(&empty_b[w]);
      }
      mma_commit(&acc_full);
    }
  } else if (warp >= 4) {
    // ---------------- dequant producers (then the epilogue)
    const int pt = threadIdx.x - 128;
    const int j = pt % BN;            // W row n0 + j of the tile ...
    const int hf = pt / BN;           // ... columns [32 hf, 32 hf + 32) of each block
    const int n = n0 + j;
    const bool live = n < a.N;
    float s_n = 0.0f, negc = 0.0f;
    int32_t z_n = 0;
    int cur = 0, end = 0;
    if (live) {
      s_n = a.scale[n];
      z_n = a.zp[n];
      negc = make_dequant_row(s_n, z_n).negc;
      cur = a.row_start[n];
      end = cur + (a.row_count ? min(a.row_count[n], a.row_start[n + 1] - cur)
                               : a.row_start[n + 1] - cur);
    }
    const bool fast = make_dequant_row(s_n, z_n).fast;
    // a 4-entry register window over the row's CSR slot (columns ascending): the per-block
    // test is a register compare, and an entry's load is issued 4 outliers before it is used
    constexpr int NONE = 0x7fffffff;
    int oc0 = NONE, oc1 = NONE, oc2 = NONE, oc3 = NONE;
    float ov0 = 0.0f, ov1 = 0.0f, ov2 = 0.0f, ov3 = 0.0f;
    int nxt = cur;  // next CSR entry to load into the window
    auto fetch = [&](int& c, float& v) {
      if (nxt < end) {
        c = __ldg(a.col + nxt);
        v = __ldg(a.val + nxt);
        ++nxt;
      } else {
        c = NONE;
      }
    };
    fetch(oc0, ov0);
    fetch(oc1, ov1);
    fetch(oc2, ov2);
    fetch(oc3, ov3);
    for (int kb = 0; kb < nkb; ++kb) {
      const int w = kb % WSTAGES, c = kb % CSTAGES;
      mbar_wait(&full_c[c], (uint32_t)((kb / CSTAGES) & 1));
#if DQ_NOPROD  // A/B: the pipeline without the dequantization work (wrong results)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_c[c]);
      mbar_wait(&empty_b[w], (uint32_t)(((kb / WSTAGES) & 1) ^ 1));
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_b[w]);
      continue;
#endif
      // the code tile is TMA-swizzled (SWIZZLE_64B: 16-byte chunk k of the 64-byte row j at
      // k ^ ((j >> 1) & 3)), so a warp's 32 rows spread over all banks
      const uint4* cr = reinterpret_cast<const uint4*>(c_tile(c) + j * BK);
      uint4 q4[NQ];
#pragma unroll
      for (int c4 = 0; c4 < NQ; ++c4)
        q4[c4] = live ? cr[(c4 + NQ * hf) ^ ((j >> 1) & 3)] : make_uint4(0, 0, 0, 0);
      // generic-proxy reads of the slot, then the TMA (async proxy) refills it: order them
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_c[c]);  // the code slot is consumed
      // the W-operand slot w is free once the MMAs of its previous use completed
      mbar_wait(&empty_b[w], (uint32_t)(((kb / WSTAGES) & 1) ^ 1));
      uint8_t* bt = b_tile(w) + j * 128;
      // 32 codes -> 4 swizzled 16-byte chunks of bf16: the row's branch (fast magic-number
      // dequant, or the exact form for |z| >= 2^22) is taken once per block
      uint32_t pk[NQ][8];
      if (fast) {
#pragma unroll
        for (int c4 = 0; c4 < NQ; ++c4) {
          const uint32_t w4[4] = {q4[c4].x, q4[c4].y, q4[c4].z, q4[c4].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float2 u = make_float2(magic_byte(w4[i], 0), magic_byte(w4[i], 1));
            float2 v = make_float2(magic_byte(w4[i], 2), magic_byte(w4[i], 3));
            u = mul2(add2(u, f2(negc)), f2(s_n));
            v = mul2(add2(v, f2(negc)), f2(s_n));
            pk[c4][2 * i] = pack_bf16(u.x, u.y);
            pk[c4][2 * i + 1] = pack_bf16(v.x, v.y);
          }
        }
      } else {
#pragma unroll
        for (int c4 = 0; c4 < NQ; ++c4) {
          const uint32_t w4[4] = {q4[c4].x, q4[c4].y, q4[c4].z, q4[c4].w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float f[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) f[e] = dequant_exact((w4[i] >> (8 * e)) & 0xFFu, s_n, z_n);
            pk[c4][2 * i] = pack_bf16(f[0], f[1]);
            pk[c4][2 * i + 1] = pack_bf16(f[2], f[3]);
          }
        }
      }
#pragma unroll
      for (int c4 = 0; c4 < NQ; ++c4) {
        const int c0 = (CPT / 8) * hf + 2 * c4, c1 = c0 + 1;  // 8 bf16 per 16-byte chunk
        *reinterpret_cast<uint4*>(bt + ((c0 ^ (j & 7)) << 4)) =
            make_uint4(pk[c4][0], pk[c4][1], pk[c4][2], pk[c4][3]);
        *reinterpret_cast<uint4*>(bt + ((c1 ^ (j & 7)) << 4)) =
            make_uint4(pk[c4][4], pk[c4][5], pk[c4][6], pk[c4][7]);
      }
      // the row's outliers in this K block overwrite their positions with their exact
      // fp32 values (RNE to bf16)
      const int k0 = kb * BK + CPT * hf;  // this thread's part of the block
      // (the other half's entries below it are skipped: they belong to the other thread)
      while (oc0 < k0) {
        oc0 = oc1; ov0 = ov1;
        oc1 = oc2; ov1 = ov2;
        oc2 = oc3; ov2 = ov3;
        fetch(oc3, ov3);
      }
      while (oc0 < k0 + CPT) {
        const int k = oc0 - kb * BK;
        const uint32_t h = pack_bf16(ov0, 0.0f) & 0xFFFFu;
        *reinterpret_cast<uint16_t*>(bt + ((((k >> 3) ^ (j & 7)) << 4) | ((k & 7) << 1))) = (uint16_t)h;
        oc0 = oc1; ov0 = ov1;
        oc1 = oc2; ov1 = ov2;
        oc2 = oc3; ov2 = ov3;
        fetch(oc3, ov3);
      }
#if !DQ_NOFENCE
      fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor cores
#endif
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_b[w]);
    }
    // ---------------- epilogue: TMEM -> bf16 -> HBM
    mbar_wait(&acc_full, 0u);
    tc_after_sync();
    epilogue_bf16<BN, NACC, NPW>(tmem_d, warp, lane, m0, n0, a.M, a.N, a.y);
  }
  tc_before_sync();
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d),
                 "n"(TMEM_COLS));
}

// ------------------------------------------------------------------ host side
cudaError_t launch_dq_gemm(const void* x, int M, int K, const uint8_t* codes, int N,
                           const float* scale, const int32_t* zp, const int32_t* row_start,
                           const int32_t* row_count, const int32_t* col, const float* val,
                           void* y, cudaStream_t st) {
  using namespace dq;
  auto enc = um::encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tx{}, tw{};
  {
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
    const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    const cuuint32_t box[2] = {BK, XBOX};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
    const cuuint64_t strides[1] = {(cuuint64_t)K};
    const cuuint32_t box[2] = {BK, BN};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(codes), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(k_dq_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  DqArgs a{scale, zp, row_start, row_count, col, val, reinterpret_cast<__nv_bfloat16*>(y), M, N, K};
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM));
  k_dq_gemm<<<grid, NT, SMEM_BYTES, st>>>(tx, tw, a);
  return cudaGetLastError();
}

}  // namespace qftk
