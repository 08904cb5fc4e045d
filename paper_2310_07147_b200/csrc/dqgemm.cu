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
// sm_100a, K in blocks of 64; two shapes (dq::Shape): a CTA pair (cta_group::2, M > 256)
// with a 512 x 256 output tile per pair, or one CTA with a 512 x 128 tile.  Per CTA:
//   warp 0 (lane 0)  TMA: the CTA's X rows of a K block (SWIZZLE_128B, 256-row boxes) into
//                    the X ring (pair: 4 stages of 256 rows, both CTAs' bytes completing
//                    on the leader's barrier; single: 2 stages of 512 rows)
//   warp 3 (lane 0)  TMA: the CTA's 128 x 64 W code tile into its own 4-stage ring
//   warps 4-11       the dequant producers: a thread pair owns one of the CTA's 128 W rows,
//                    each thread 32 columns of a block: codes -> s*(q-z) (fp32, one
//                    rounding, quantize.hpp:209) -> its CSR outliers of the block (from the
//                    per-(row, 32-column) slot index, loaded a block ahead) overwrite their
//                    positions -> bf16 (RNE) -> the K-major SWIZZLE_128B operand ring (4
//                    stages); one fence.proxy.async, then the code slot and the operand
//                    slot are released / published (pair: on the leader's barrier)
//   warp 1 (lane 0)  the MMA issuer (pair: the leader only): tcgen05.mma kind::f16 --
//                    pair M=256 x N=256 (cta_group::2, each SM supplies its A and B halves)
//                    into two TMEM accumulators, single M=128 x N=128 into four; all read
//                    the same dequantized W operand; tcgen05.commit (multicast to both
//                    CTAs of a pair) frees the slots and finally signals the accumulators
//   warps 4-11       the epilogue: tcgen05.ld 32x32b (double-buffered) -> bf16 -> HBM
//   warp 2           TMEM allocation (512 columns) and release
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
#ifndef DQ_PUNROLL
#define DQ_PUNROLL 2  // producer loop unrolled by 2 (measured +4%; 4: no better)
#endif
#ifndef DQ_ONEFENCE
#define DQ_ONEFENCE 1  // one proxy fence per block (measured +0.5-1%)
#endif
namespace dq {
using namespace um;
constexpr int kProdUnroll = DQ_PUNROLL;
constexpr int BK = 64;      // K per block: 128 bytes of bf16 = one SWIZZLE_128B row
constexpr int WROWS = 128;  // W rows dequantized per CTA (output columns of a CTA's operand)
#ifndef DQ_CSTAGES
#define DQ_CSTAGES 4
#endif
#ifndef DQ_WSTAGES
#define DQ_WSTAGES 4
#endif
constexpr int WSTAGES = DQ_WSTAGES;  // dequantized W-operand ring (producers run ahead)
constexpr int CSTAGES = DQ_CSTAGES;  // W-code ring
constexpr int B_BYTES = WROWS * BK * 2;
constexpr int C_BYTES = WROWS * BK;  // codes
#ifndef DQ_HALVES
#define DQ_HALVES 2
#endif
constexpr int HALVES = DQ_HALVES;        // producer threads per W row
constexpr int CPT = BK / HALVES;         // columns of a K block per producer thread
constexpr int NQ = CPT / 16;             // 16-code vectors per producer thread and block
constexpr int NPW = WROWS * HALVES / 32; // producer warps
constexpr int NT = 128 + WROWS * HALVES; // TMA (X), MMA, TMEM, TMA (codes) warps + producers

// The two tile shapes.  Single CTA: 512 x 128 output tile, four M=128 x N=128 accumulators
// (cta_group::1), a 2-stage 64 KB X ring.  CTA pair (cta_group::2, cluster of 2): a
// 512 x 256 output tile per pair -- each CTA holds 256 X rows (two M=256 halves) and
// dequantizes 128 of the 256 W rows; the leader's M=256 x N=256 MMAs read both CTAs'
// halves, so each SM's tensor core streams half the operand bytes per flop (the
// single-CTA shape is shared-memory-bandwidth bound), and a 4-stage 32 KB X ring fits.
template <bool PAIR>
struct Shape {
  static constexpr int BN = PAIR ? 256 : 128;          // UMMA N (output columns per tile)
  static constexpr int NACC = PAIR ? 2 : 4;            // accumulators (512 TMEM columns)
  static constexpr int BM = PAIR ? 256 : 512;          // X rows per CTA
#ifndef DQ_PSTAGES
#define DQ_PSTAGES 4
#endif
  static constexpr int STAGES = PAIR ? DQ_PSTAGES : 2;  // X ring
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int SMEM_BYTES = STAGES * A_BYTES + WSTAGES * B_BYTES + CSTAGES * C_BYTES + 1024;
  // instruction descriptor: D f32, A/B bf16, both K-major, N = BN, M = 128 or 256 (pair)
  static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) |
                                    ((uint32_t)(BN >> 3) << 17) |
                                    ((uint32_t)((PAIR ? 256 : 128) >> 4) << 24);
  static constexpr int TMEM_COLS = NACC * BN;  // 512
  static constexpr int XBOX = 256;             // TMA box rows: BM / XBOX loads per X tile
};

}  // namespace dq

struct DqArgs {
  const uint8_t* codes;      // [N, K] u8 W codes
  const float* scale;        // [N]
  const int32_t* zp;         // [N]
  const int32_t* row_start;  // [N] CSR slot starts (arena offsets)
  const int32_t* row_count;  // [N] used entries (null: strict CSR, count = rs[n+1]-rs[n])
  const int32_t* col;        // arena
  const float* val;
  const int32_t* tix;        // [N][K/32 + 1] per-(row, 32-column) slot index (k_csr_tile_index)
  __nv_bfloat16* y;          // [M, N]
  int M, N, K;
};

template <bool PAIR>
__device__ __forceinline__ void dq_gemm_body(const CUtensorMap* tm_x, const CUtensorMap* tm_w,
                                             const DqArgs& a) {
  using namespace dq;
  using S = Shape<PAIR>;
  constexpr int STAGES = S::STAGES, A_BYTES = S::A_BYTES, BM = S::BM, BN = S::BN;
  constexpr int NACC = S::NACC, XBOX = S::XBOX;
  extern __shared__ uint8_t dsm_raw[];
  // 1024-byte aligned (SWIZZLE_128B atoms); pointer arithmetic on the shared array keeps
  // the address space visible to the compiler (LDS/STS, not generic loads and stores).
  // Both CTAs of a pair compute the same offsets (the leader's descriptors address both).
  uint8_t* dsm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full_a[STAGES], empty_a[STAGES], full_b[WSTAGES], empty_b[WSTAGES];
  __shared__ __align__(8) uint64_t full_c[CSTAGES], empty_c[CSTAGES], acc_full;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  // pair: blockIdx.x = 2 * (256-column tile) + rank; CTA `rank` holds X rows
  // m0 = 512 * blockIdx.y + 256 * rank and dequantizes W rows wn0 = n0 + 128 * rank
  const int n0 = PAIR ? (int)(blockIdx.x >> 1) * BN : (int)blockIdx.x * BN;
  const int m0 = PAIR ? (int)blockIdx.y * 2 * BM + (int)rank * BM : (int)blockIdx.y * BM;
  const int wn0 = n0 + (int)rank * WROWS;
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
      mbar_init(&full_b[w], PAIR ? 2 * NPW : NPW);  // pair: both CTAs' producers (leader's)
      mbar_init(&empty_b[w], 1);
    }
    for (int c = 0; c < CSTAGES; ++c) {
      mbar_init(&full_c[c], 1);
      mbar_init(&empty_c[c], NPW);
    }
    mbar_init(&acc_full, 1);
    mbar_fence_init();
  }
  if (warp == 2) {  // TMEM: the accumulators (pair: the same columns on both SMs)
    if (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base)),
                   "n"(S::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base)),
                   "n"(S::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_before_sync();
  if (PAIR)
    cluster_sync_all();  // barrier inits and the allocation visible to the peer
  else
    __syncthreads();
  tc_after_sync();
  const uint32_t tmem_d = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA: X tiles
      const uint32_t fa0 = PAIR ? mapa_cl(&full_a[0], 0) : 0u;
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&empty_a[s], (uint32_t)(((kb / STAGES) & 1) ^ 1));
        if (PAIR) {
          // both CTAs' bytes complete on the leader's barrier; the leader expects them all
          if (rank == 0) mbar_arrive_expect_tx(&full_a[s], (uint32_t)(2 * A_BYTES));
          const uint32_t bar = fa0 + (uint32_t)(s * sizeof(uint64_t));
#pragma unroll
          for (int xb = 0; xb < BM / XBOX; ++xb)
            tma_load_2d_pair(a_tile(s) + xb * XBOX * 128, tm_x, kb * BK, m0 + xb * XBOX, bar);
        } else {
          mbar_arrive_expect_tx(&full_a[s], (uint32_t)A_BYTES);
#pragma unroll
          for (int xb = 0; xb < BM / XBOX; ++xb)
            tma_load_2d(a_tile(s) + xb * XBOX * 128, tm_x, kb * BK, m0 + xb * XBOX, &full_a[s]);
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {  // ---------------- TMA: W code tiles (their own, deeper ring)
      for (int kb = 0; kb < nkb; ++kb) {
        const int c = kb % CSTAGES;
        mbar_wait(&empty_c[c], (uint32_t)(((kb / CSTAGES) & 1) ^ 1));
        mbar_arrive_expect_tx(&full_c[c], (uint32_t)C_BYTES);
        tma_load_2d(c_tile(c), tm_w, kb * BK, wn0, &full_c[c]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // ---------------- MMA issuer (the pair's leader)
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES, w = kb % WSTAGES;
        if (PAIR) {
          mbar_wait_cl(&full_a[s], (uint32_t)((kb / STAGES) & 1));
          mbar_wait_cl(&full_b[w], (uint32_t)((kb / WSTAGES) & 1));
        } else {
          mbar_wait(&full_a[s], (uint32_t)((kb / STAGES) & 1));
          mbar_wait(&full_b[w], (uint32_t)((kb / WSTAGES) & 1));
        }
        tc_after_sync();
        const uint32_t sa = smem_u32(a_tile(s)), sb = smem_u32(b_tile(w));
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {  // every 128-row block shares the W operand
          const uint64_t bd = sw128_desc(sb + 32 * kk);
          const uint32_t acc = (kb > 0 || kk > 0) ? 1u : 0u;
#pragma unroll
          for (int ab = 0; ab < NACC; ++ab) {
            const uint64_t ad = sw128_desc(sa + ab * 128 * 128 + 32 * kk);
            if (PAIR)
              mma_bf16_pair(tmem_d + ab * BN, ad, bd, S::IDESC, acc);
            else
              mma_bf16(tmem_d + ab * BN, ad, bd, S::IDESC, acc);
          }
        }
        // the X and W-operand slots (of both CTAs) are free once these MMAs read them
        if (PAIR) {
          mma_commit_pair(&empty_a[s], 3);
          mma_commit_pair(&empty_b[w], 3);
        } else {
          mma_commit(&empty_a[s]);
          mma_commit(&empty_b[w]);
        }
      }
      if (PAIR)
        mma_commit_pair(&acc_full, 3);
      else
        mma_commit(&acc_full);
    }
  } else if (warp >= 4) {
    // ---------------- dequant producers (then the epilogue)
    const int pt = threadIdx.x - 128;
    const int j = pt % WROWS;         // W row wn0 + j of the tile ...
    const int hf = pt / WROWS;        // ... columns [32 hf, 32 hf + 32) of each block
    const int n = wn0 + j;
    const bool live = n < a.N;
    float s_n = 0.0f, negc = 0.0f;
    int32_t z_n = 0;
    if (live) {
      s_n = a.scale[n];
      z_n = a.zp[n];
      negc = make_dequant_row(s_n, z_n).negc;
    }
    const bool fast = make_dequant_row(s_n, z_n).fast;
    const uint32_t fb0 = PAIR ? mapa_cl(&full_b[0], 0) : 0u;
    // The thread's outliers of block kb are slot entries [tix[H kb + hf], tix[H kb + hf + 1])
    // of its row (H = HALVES; columns ascending, CPT-column granularity = exactly its part
    // of the block).
    // Pipelined without dependent chains: block kb+2's index pair is loaded during block
    // kb, and block kb+1's first two entries during block kb -- each load is consumed one
    // block (~1 us) after issue.  More than two entries in a half block (rare at p <= 1%)
    // are loaded where they are written.
    const int32_t* tr = a.tix + (size_t)(live ? n : 0) * (size_t)(HALVES * nkb + 1) + hf;
    auto tload = [&](int kb, int& s0, int& e0) {
      if (live && kb < nkb) {
        s0 = __ldg(tr + HALVES * kb);
        e0 = __ldg(tr + HALVES * kb + 1);
      } else {
        s0 = e0 = 0;
      }
    };
    int s1, e1, s2, e2;  // index pairs of the next block and the one after
    tload(0, s1, e1);
    tload(1, s2, e2);
    int nS = s1, nN = e1 - s1, nc0 = 0, nc1 = 0;  // the next block's first two entries
    float nv0 = 0.0f, nv1 = 0.0f;
    auto eload = [&](int s0, int e0) {
      nS = s0;
      nN = e0 - s0;
      if (nN > 0) {
        nc0 = __ldg(a.col + s0);
        nv0 = __ldg(a.val + s0);
      }
      if (nN > 1) {
        nc1 = __ldg(a.col + s0 + 1);
        nv1 = __ldg(a.val + s0 + 1);
      }
    };
    eload(s1, e1);
#pragma unroll kProdUnroll
    for (int kb = 0; kb < nkb; ++kb) {
      const int w = kb % WSTAGES, c = kb % CSTAGES;
      // this block's outliers (loaded during the previous block); issue the next block's
      // entries and the index pair of the block after it
      const int cS = nS, cN = nN, cc0 = nc0, cc1 = nc1;
      const float cv0 = nv0, cv1 = nv1;
      eload(s2, e2);
      tload(kb + 2, s2, e2);
      mbar_wait(&full_c[c], (uint32_t)((kb / CSTAGES) & 1));
#if DQ_NOPROD  // A/B: the pipeline without the dequantization work (wrong results)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_c[c]);
      mbar_wait(&empty_b[w], (uint32_t)(((kb / WSTAGES) & 1) ^ 1));
      __syncwarp();
      if (lane == 0) {
        if (PAIR)
          mbar_arrive_cl(fb0 + (uint32_t)(w * sizeof(uint64_t)));
        else
          mbar_arrive(&full_b[w]);
      }
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
      // (DQ_ONEFENCE: the slot is released after the block's operand writes, behind the
      // one fence that also publishes them)
      if (!DQ_ONEFENCE) {
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_c[c]);  // the code slot is consumed
      }
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
      // the row's outliers in this half block overwrite their positions with their exact
      // fp32 values (RNE to bf16)
      auto put = [&](int col, float v) {
        const int k = col - kb * BK;
        const uint32_t h = pack_bf16(v, 0.0f) & 0xFFFFu;
        *reinterpret_cast<uint16_t*>(bt + ((((k >> 3) ^ (j & 7)) << 4) | ((k & 7) << 1))) = (uint16_t)h;
      };
      if (cN > 0) {
        put(cc0, cv0);
        if (cN > 1) put(cc1, cv1);
        for (int e = 2; e < cN; ++e) put(__ldg(a.col + cS + e), __ldg(a.val + cS + e));
      }
#if !DQ_NOFENCE
      fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor cores
#endif
      __syncwarp();
      if (lane == 0) {
        if (DQ_ONEFENCE) mbar_arrive(&empty_c[c]);  // the code slot is consumed
        if (PAIR)  // the leader's MMA reads this CTA's half: arrive on the leader's barrier
          mbar_arrive_cl(fb0 + (uint32_t)(w * sizeof(uint64_t)));
        else
          mbar_arrive(&full_b[w]);
      }
    }
    // ---------------- epilogue: TMEM -> bf16 -> HBM (each CTA its own X rows x all BN)
    mbar_wait(&acc_full, 0u);
    tc_after_sync();
    epilogue_bf16<BN, NACC, NPW>(tmem_d, warp, lane, m0, n0, a.M, a.N, a.y);
  }
  tc_before_sync();
  if (PAIR) {
    cluster_sync_all();  // both CTAs done with the pair's TMEM and barriers
    if (warp == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_d),
                   "n"(S::TMEM_COLS));
  } else {
    __syncthreads();
    if (warp == 2)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d),
                   "n"(S::TMEM_COLS));
  }
}

__global__ void __launch_bounds__(dq::NT, 1)
    k_dq_gemm(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
              const DqArgs a) {
  dq_gemm_body<false>(&tm_x, &tm_w, a);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(dq::NT, 1)
    k_dq_gemm_pair(const __grid_constant__ CUtensorMap tm_x,
                   const __grid_constant__ CUtensorMap tm_w, const DqArgs a) {
  dq_gemm_body<true>(&tm_x, &tm_w, a);
}

// ------------------------------------------------------------------ host side
// The pair kernel for M > 256 (its 512-row tile would idle half of a pair below that),
// the single-CTA one otherwise; QFT_DQ_PAIR=0/1 forces either (A/B).
static int dq_pair_mode() {
  static int mode = -2;
  if (mode == -2) {
    const char* e = getenv("QFT_DQ_PAIR");
    mode = e ? atoi(e) : -1;
  }
  return mode;
}

size_t dq_gemm_workspace_bytes(int N, int K) {
  return (size_t)N * (size_t)(K / dq::CPT + 1) * sizeof(int32_t);
}

cudaError_t launch_dq_gemm(const void* x, int M, int K, const uint8_t* codes, int N,
                           const float* scale, const int32_t* zp, const int32_t* row_start,
                           const int32_t* row_count, const int32_t* col, const float* val,
                           void* y, void* workspace, cudaStream_t st, bool build_index) {
  using namespace dq;
  auto enc = um::encode_fn();
  if (!enc) return cudaErrorNotSupported;
  const int pm = dq_pair_mode();
  const bool pair = pm >= 0 ? pm != 0 : M > 256;
  const int XB = 256;
  CUtensorMap tx{}, tw{};
  {
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
    const cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    const cuuint32_t box[2] = {BK, (cuuint32_t)XB};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&tx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(x), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N};
    const cuuint64_t strides[1] = {(cuuint64_t)K};
    const cuuint32_t box[2] = {BK, WROWS};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(codes), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  int32_t* tix = reinterpret_cast<int32_t*>(workspace);
  if (build_index) {  // (else: the caller's workspace already holds this CSR's index)
    cudaError_t e = launch_csr_tile_index(row_start, row_count, col, N, K / CPT, CPT, tix, st);
    if (e != cudaSuccess) return e;
  }
  DqArgs a{codes, scale, zp, row_start, row_count, col, val, tix,
           reinterpret_cast<__nv_bfloat16*>(y), M, N, K};
  if (pair) {
    using S = Shape<true>;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(k_dq_gemm_pair,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM_BYTES);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    dim3 grid((unsigned)(2 * ((N + S::BN - 1) / S::BN)), (unsigned)((M + 2 * S::BM - 1) / (2 * S::BM)));
    k_dq_gemm_pair<<<grid, NT, S::SMEM_BYTES, st>>>(tx, tw, a);
  } else {
    using S = Shape<false>;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(k_dq_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           S::SMEM_BYTES);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    dim3 grid((unsigned)((N + S::BN - 1) / S::BN), (unsigned)((M + S::BM - 1) / S::BM));
    k_dq_gemm<<<grid, NT, S::SMEM_BYTES, st>>>(tx, tw, a);
  }
  return cudaGetLastError();
}

}  // namespace qftk
