// dqgemm_t.cu -- the backward's input gradient with the weight dequantization fused into
// the GEMM's operand producer (the backward weight operand):
// dX[T,I] = dY[T,O] . W, W a QFT dense-and-sparse weight [O,I] (u8 codes, per-row params,
// CSR outliers).  The reference reconstructs W for the backward too (gradflow.hpp:78,
// weight_at = reconstruct, quantize.hpp:331-338) and multiplies (network.hpp:145,
// backward_core: in_grad = matmul(out_grad, w)); here the tensor cores read
// RNE(reconstruct(W)) -- the bytes qftc_expand(bf16) writes -- built in shared memory from the
// codes: W streams as 1 byte per element and never exists in HBM as bf16.
//
// The forward kernel (dqgemm.cu) reads W K-major (rows of W = output channels = N); here W's
// rows are the REDUCTION dimension, so the operand is MN-major: a K block is 64 rows of W,
// each contributing BN contiguous columns -- one 128-byte SWIZZLE_128B row per 64 columns.
// A W row's CSR outliers inside a producer's 32 columns are located through a per-(row, 32-column
// tile) index built by a small pre-pass (k_csr_tile_index: the first slot entry at or past
// each tile's first column), so a producer scans only the ~1-2 entries of its own window.
//
// sm_100a, K in blocks of 64 W rows; a CTA pair (cta_group::2, more than 256 tokens: a
// 512 x 256 tile per pair, each CTA 256 dY rows and 128 of the W columns, two M=256
// accumulators) or one CTA (512 x 128, four M=128 accumulators), per CTA:
//   warp 0 (lane 0)  TMA: the dY tile (512 x 64 bf16, K-major, SWIZZLE_128B) -> X/W ring
//   warp 3 (lane 0)  TMA: the W code tile (64 rows x 128 columns u8, SWIZZLE_128B) -> its
//                    own 4-stage ring; the W operand has a 4-stage ring of its own
//   warps 4-11       producers: thread (r, j, h) dequantizes W row k0 + r, columns
//                    [64j + 32h, +32) of the tile -> 4 swizzled 16-byte chunks of row r of
//                    the operand's MN chunk j; then its outliers; fence.proxy.async; arrive
//   warp 1 (lane 0)  tcgen05.mma kind::f16, A K-major, B MN-major (pair: the leader only)
//   warps 4-11       the bf16 epilogue (umma.cuh)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>

#include "qft_device.cuh"
#include "qft_internal.h"
#include "umma.cuh"

namespace qftk {
using namespace qftd;

#ifndef DQT_PUNROLL
#define DQT_PUNROLL 2  // producer loop unroll (A/B)
#endif
namespace dqt {
using namespace um;
constexpr int kProdUnrollT = DQT_PUNROLL;
constexpr int WC = 128;          // W columns dequantized per CTA (= UMMA N of one CTA)
constexpr int BK = 64;           // W rows per K block
constexpr int WSTAGES = 4;       // dequantized W-operand ring (producers run ahead)
constexpr int CSTAGES = 4;       // W-code ring
constexpr int B_BYTES = WC * BK * 2;  // WC/64 MN chunks of 64 x 64 bf16 (8 KB each)
constexpr int C_BYTES = WC * BK;
constexpr int NPW = 8;                // producer warps
constexpr int NT = 128 + 32 * NPW;
constexpr int XBOX = 256;
constexpr uint32_t B_LBO = 64 * BK * 2;  // bytes between the operand's 64-column MN chunks
// single CTA: 512 x 128 output tile, four M=128 x N=128 accumulators, 2-stage dY ring;
// CTA pair (cta_group::2): 512 x 256 tile per pair, each CTA 256 dY rows (two M=256
// halves) and 128 of the 256 W columns, 4-stage dY ring (dqgemm.cu has the plumbing notes)
template <bool PAIR>
struct ShapeT {
  static constexpr int BN = PAIR ? 256 : 128;  // UMMA N: output columns per tile
  static constexpr int NACC = PAIR ? 2 : 4;
  static constexpr int BM = PAIR ? 256 : 512;  // dY rows per CTA
  static constexpr int STAGES = PAIR ? 4 : 2;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int SMEM_BYTES = STAGES * A_BYTES + WSTAGES * B_BYTES + CSTAGES * C_BYTES + 1024;
  // D f32, A/B bf16, A K-major, B MN-major (bit 16), N = BN, M = 128 or 256 (pair)
  static constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                                    ((uint32_t)(BN >> 3) << 17) |
                                    ((uint32_t)((PAIR ? 256 : 128) >> 4) << 24);
  static constexpr int TMEM_COLS = NACC * BN;  // 512
};
constexpr int TC = 32;                   // columns per tile of the CSR index (a producer's)
}  // namespace dqt

struct DqtArgs {
  const float* scale;     // [O]
  const int32_t* zp;      // [O]
  const int32_t* tix;     // [O, tiles_n + 1] arena positions: first entry of each 32-column tile
  const int32_t* col;     // arena
  const float* val;
  __nv_bfloat16* y;       // [M, N] = dX [T, I]
  int M, N, K;            // T, I, O
  int tiles_n;
};

// tix[o][t] = the first entry of row o's slot whose column is >= t * tile_cols (t < tiles_n), and
// tix[o][tiles_n] = the slot's used end; slot entries are column-ascending.  A warp per row,
// linear in the row's entries: entry i is the answer for the tiles (tile(i-1), tile(i)], the
// used end for the tiles past the last entry's.
__global__ void k_csr_tile_index(const int32_t* row_start, const int32_t* row_count,
                                 const int32_t* col, int O, int tiles_n, int tile_cols,
                                 int32_t* tix) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int o = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; o < O; o += warps) {
    const int b = row_start[o];
    const int e = b + (row_count ? min(row_count[o], row_start[o + 1] - b) : row_start[o + 1] - b);
    int32_t* out = tix + (size_t)o * (tiles_n + 1);
    for (int i = b + lane; i < e; i += 32) {
      const int t = col[i] / tile_cols;
      const int tp = i > b ? col[i - 1] / tile_cols : -1;
      for (int u = tp + 1; u <= t; ++u) out[u] = i;
    }
    const int tl = e > b ? col[e - 1] / tile_cols : -1;
    for (int u = tl + 1 + lane; u <= tiles_n; u += 32) out[u] = e;
  }
}

template <bool PAIR>
__device__ __forceinline__ void dq_gemm_t_body(const CUtensorMap* tm_dy, const CUtensorMap* tm_w,
                                               const DqtArgs& a) {
  using namespace dqt;
  using S = ShapeT<PAIR>;
  constexpr int BN = S::BN, NACC = S::NACC, BM = S::BM, STAGES = S::STAGES, A_BYTES = S::A_BYTES;
  extern __shared__ uint8_t dsm_raw[];
  uint8_t* dsm = dsm_raw + ((1024u - (smem_u32(dsm_raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full_a[STAGES], empty_a[STAGES], full_b[WSTAGES], empty_b[WSTAGES];
  __shared__ __align__(8) uint64_t full_c[CSTAGES], empty_c[CSTAGES], acc_full;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  // pair: blockIdx.x = 2 * (256-column tile) + rank; CTA `rank` holds dY rows
  // m0 = 512 * blockIdx.y + 256 * rank and dequantizes W columns wn0 = n0 + 128 * rank
  const int n0 = PAIR ? (int)(blockIdx.x >> 1) * BN : (int)blockIdx.x * BN;
  const int m0 = PAIR ? (int)blockIdx.y * 2 * BM + (int)rank * BM : (int)blockIdx.y * BM;
  const int wn0 = n0 + (int)rank * WC;
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
  if (warp == 2) {
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
    cluster_sync_all();
  else
    __syncthreads();
  tc_after_sync();
  const uint32_t tmem_d = tmem_base;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA: dY tiles
      for (int kb = 0; kb < nkb; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&empty_a[s], (uint32_t)(((kb / STAGES) & 1) ^ 1));
        if (PAIR) {  // both CTAs' bytes complete on the leader's barrier
          if (rank == 0) mbar_arrive_expect_tx(&full_a[s], (uint32_t)(2 * A_BYTES));
          const uint32_t bar = mapa_cl(&full_a[s], 0);
#pragma unroll
          for (int xb = 0; xb < BM / XBOX; ++xb)
            tma_load_2d_pair(a_tile(s) + xb * XBOX * 128, tm_dy, kb * BK, m0 + xb * XBOX, bar);
        } else {
          mbar_arrive_expect_tx(&full_a[s], (uint32_t)A_BYTES);
#pragma unroll
          for (int xb = 0; xb < BM / XBOX; ++xb)
            tma_load_2d(a_tile(s) + xb * XBOX * 128, tm_dy, kb * BK, m0 + xb * XBOX, &full_a[s]);
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {  // ---------------- TMA: W code tiles (64 W rows x BN columns)
      for (int kb = 0; kb < nkb; ++kb) {
        const int c = kb % CSTAGES;
        mbar_wait(&empty_c[c], (uint32_t)(((kb / CSTAGES) & 1) ^ 1));
        mbar_arrive_expect_tx(&full_c[c], (uint32_t)C_BYTES);
        tma_load_2d(c_tile(c), tm_w, wn0, kb * BK, &full_c[c]);
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
        for (int kk = 0; kk < BK / 16; ++kk) {
          // B MN-major: 16 K rows = two 8-row swizzle atoms (2048 B) per K=16 step
          const uint64_t bd = sw128_desc_mn(sb + 2048 * kk, B_LBO, 1024u);
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
    // ---------------- dequant producers: thread (r, j, h) of the 64 x 2 x 2 units
    const int pt = threadIdx.x - 128;
    const int r = pt >> 2, j = (pt >> 1) & 1, h = pt & 1;
    const int cbeg = wn0 + 64 * j + 32 * h;  // this thread's 32 columns of the W rows
    const uint32_t fb0 = PAIR ? mapa_cl(&full_b[0], 0) : 0u;
    const int tq = cbeg / TC;                // ... = column tile tq of the index
    // The block's row parameters are loaded one block ahead; the row's slot range of the
    // thread's 32 columns (the index) two blocks ahead, and its first two entries one block
    // ahead -- no load is consumed within a block of its issue (a scan that loaded each
    // entry where it was written stalled every producer on that load)
    auto load_row = [&](int kb, float& s, int32_t& z) {
      const int o = kb * BK + r;
      s = __ldg(a.scale + o);
      z = __ldg(a.zp + o);
    };
    auto load_ix = [&](int kb, int& eb, int& ee) {
      if (kb < nkb && cbeg < a.N) {  // (columns past I: no entries, no index tile)
        const int32_t* t = a.tix + (size_t)(kb * BK + r) * (a.tiles_n + 1) + tq;
        eb = __ldg(t);
        ee = __ldg(t + 1);
      } else {
        eb = ee = 0;
      }
    };
    int nS = 0, nN = 0, nc0 = 0, nc1 = 0;  // the next block's range and first two entries
    float nv0 = 0.0f, nv1 = 0.0f;
    auto eload = [&](int e0, int e1) {
      nS = e0;
      nN = e1 - e0;
      if (nN > 0) {
        nc0 = __ldg(a.col + e0);
        nv0 = __ldg(a.val + e0);
      }
      if (nN > 1) {
        nc1 = __ldg(a.col + e0 + 1);
        nv1 = __ldg(a.val + e0 + 1);
      }
    };
    float s_n, s_nx = 0.0f;
    int32_t z_n, z_nx = 0;
    int ebA, eeA;
    load_row(0, s_n, z_n);
    load_ix(0, ebA, eeA);
    eload(ebA, eeA);
    load_ix(1, ebA, eeA);
#pragma unroll kProdUnrollT
    for (int kb = 0; kb < nkb; ++kb) {
      const int w = kb % WSTAGES, c = kb % CSTAGES;
      const int cS = nS, cN = nN, cc0 = nc0, cc1 = nc1;
      const float cv0 = nv0, cv1 = nv1;
      eload(ebA, eeA);
      load_ix(kb + 2, ebA, eeA);
      if (kb + 1 < nkb) load_row(kb + 1, s_nx, z_nx);
      mbar_wait(&full_c[c], (uint32_t)((kb / CSTAGES) & 1));
      // the code tile is TMA-swizzled (SWIZZLE_128B: 16-byte chunk k of row r at k ^ (r & 7)),
      // so the 8 rows a warp reads hit distinct banks
      const uint4* cr = reinterpret_cast<const uint4*>(c_tile(c) + r * WC);
      const int k0 = 4 * j + 2 * h;
      const uint4 q0 = cr[k0 ^ (r & 7)], q1 = cr[(k0 + 1) ^ (r & 7)];
      // (the code slot is released after the block's operand writes, behind the one fence
      // that also publishes them: one proxy fence per block)
      mbar_wait(&empty_b[w], (uint32_t)(((kb / WSTAGES) & 1) ^ 1));
      // row r of MN chunk j: 64 bf16 = 128 bytes, 16-byte chunk k at (k ^ (r & 7)) << 4
      uint8_t* bt = b_tile(w) + j * B_LBO + r * 128;
      const DequantRow d = make_dequant_row(s_n, z_n);
      const uint32_t w8[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
      uint32_t pk[16];
      if (d.fast) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float2 u = make_float2(magic_byte(w8[i], 0), magic_byte(w8[i], 1));
          float2 v = make_float2(magic_byte(w8[i], 2), magic_byte(w8[i], 3));
          u = mul2(add2(u, f2(d.negc)), f2(s_n));
          v = mul2(add2(v, f2(d.negc)), f2(s_n));
          pk[2 * i] = pack_bf16(u.x, u.y);
          pk[2 * i + 1] = pack_bf16(v.x, v.y);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float f[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) f[e] = dequant_exact((w8[i] >> (8 * e)) & 0xFFu, s_n, z_n);
          pk[2 * i] = pack_bf16(f[0], f[1]);
          pk[2 * i + 1] = pack_bf16(f[2], f[3]);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int ch = 4 * h + k;  // 16-byte chunk of the 128-byte row (8 bf16)
        *reinterpret_cast<uint4*>(bt + ((ch ^ (r & 7)) << 4)) =
            make_uint4(pk[4 * k], pk[4 * k + 1], pk[4 * k + 2], pk[4 * k + 3]);
      }
      // the row's outliers in [cbeg, cbeg + 32): exact fp32 values, RNE to bf16
      auto put = [&](int cc, float v) {
        const int k = cc - wn0 - 64 * j;  // 0..63 within the MN chunk row
        const uint32_t hv = pack_bf16(v, 0.0f) & 0xFFFFu;
        *reinterpret_cast<uint16_t*>(bt + ((((k >> 3) ^ (r & 7)) << 4) | ((k & 7) << 1))) =
            (uint16_t)hv;
      };
      if (cN > 0) {
        put(cc0, cv0);
        if (cN > 1) put(cc1, cv1);
        for (int e = 2; e < cN; ++e) put(__ldg(a.col + cS + e), __ldg(a.val + cS + e));
      }
      fence_proxy_async();  // smem reads and writes of the block -> ordered with the async proxy
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty_c[c]);  // the code slot is consumed
        if (PAIR)  // the leader's MMA reads this CTA's half: arrive on the leader's barrier
          mbar_arrive_cl(fb0 + (uint32_t)(w * sizeof(uint64_t)));
        else
          mbar_arrive(&full_b[w]);
      }
      s_n = s_nx;
      z_n = z_nx;
    }
    mbar_wait(&acc_full, 0u);
    tc_after_sync();
    epilogue_bf16<BN, NACC, NPW>(tmem_d, warp, lane, m0, n0, a.M, a.N, a.y);
  }
  tc_before_sync();
  if (PAIR) {
    cluster_sync_all();
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

__global__ void __launch_bounds__(dqt::NT, 1)
    k_dq_gemm_t(const __grid_constant__ CUtensorMap tm_dy, const __grid_constant__ CUtensorMap tm_w,
                const DqtArgs a) {
  dq_gemm_t_body<false>(&tm_dy, &tm_w, a);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(dqt::NT, 1)
    k_dq_gemm_t_pair(const __grid_constant__ CUtensorMap tm_dy,
                     const __grid_constant__ CUtensorMap tm_w, const DqtArgs a) {
  dq_gemm_t_body<true>(&tm_dy, &tm_w, a);
}

// ------------------------------------------------------------------ host side
cudaError_t launch_csr_tile_index(const int32_t* row_start, const int32_t* row_count,
                                  const int32_t* col, int rows, int tiles, int tile_cols,
                                  int32_t* tix, cudaStream_t st) {
  const int blocks = (rows + 7) / 8 < 4096 ? (rows + 7) / 8 : 4096;  // a warp per row
  k_csr_tile_index<<<blocks, 256, 0, st>>>(row_start, row_count, col, rows, tiles, tile_cols, tix);
  return cudaGetLastError();
}

size_t dq_gemm_t_workspace_bytes(int O, int I) {
  return (size_t)O * ((I + dqt::TC - 1) / dqt::TC + 1) * sizeof(int32_t);
}

cudaError_t launch_dq_gemm_t(const void* dy, int T, int O, const uint8_t* codes, int I,
                             const float* scale, const int32_t* zp, const int32_t* row_start,
                             const int32_t* row_count, const int32_t* col, const float* val,
                             void* dx, void* workspace, cudaStream_t st, bool build_index) {
  using namespace dqt;
  auto enc = um::encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tdy{}, tw{};
  {
    const cuuint64_t dims[2] = {(cuuint64_t)O, (cuuint64_t)T};
    const cuuint64_t strides[1] = {(cuuint64_t)O * 2};
    const cuuint32_t box[2] = {BK, XBOX};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&tdy, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(dy), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    const cuuint64_t dims[2] = {(cuuint64_t)I, (cuuint64_t)O};
    const cuuint64_t strides[1] = {(cuuint64_t)I};
    const cuuint32_t box[2] = {WC, BK};
    const cuuint32_t es[2] = {1, 1};
    if (enc(&tw, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<uint8_t*>(codes), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  const int ix_tiles = (I + TC - 1) / TC;  // index tiles: one per producer thread's columns
  int32_t* tix = reinterpret_cast<int32_t*>(workspace);
  if (build_index) {  // (else: the caller's workspace already holds this CSR's index)
    cudaError_t e = launch_csr_tile_index(row_start, row_count, col, O, ix_tiles, TC, tix, st);
    if (e != cudaSuccess) return e;
  }
  DqtArgs a{scale, zp, tix, col, val, reinterpret_cast<__nv_bfloat16*>(dx), T, I, O, ix_tiles};
  // the CTA pair for T > 256 (as the forward GEMM; QFT_DQ_PAIR=0/1 forces either)
  const char* pe = getenv("QFT_DQ_PAIR");
  const bool pair = pe ? atoi(pe) != 0 : T > 256;
  if (pair) {
    using S = ShapeT<true>;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(k_dq_gemm_t_pair,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, S::SMEM_BYTES);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    dim3 grid((unsigned)(2 * ((I + S::BN - 1) / S::BN)), (unsigned)((T + 2 * S::BM - 1) / (2 * S::BM)));
    k_dq_gemm_t_pair<<<grid, NT, S::SMEM_BYTES, st>>>(tdy, tw, a);
  } else {
    using S = ShapeT<false>;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(k_dq_gemm_t, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           S::SMEM_BYTES);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    dim3 grid((unsigned)((I + S::BN - 1) / S::BN), (unsigned)((T + S::BM - 1) / S::BM));
    k_dq_gemm_t<<<grid, NT, S::SMEM_BYTES, st>>>(tdy, tw, a);
  }
  return cudaGetLastError();
}

}  // namespace qftk
