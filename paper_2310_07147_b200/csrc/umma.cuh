// umma.cuh -- the sm_100a tensor-core plumbing shared by the two GEMMs (dqgemm.cu: the
// forward consumer with the dequantizing operand producer; wgrad.cu: the weight gradient
// with the quantizing epilogue): tcgen05 shared-memory matrix descriptors (SWIZZLE_128B,
// K-major and MN-major), TMA tensor loads, tcgen05.mma / commit, the tcgen05 thread-sync
// fences, and the driver's tensor-map encoder.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdint>

#include "qft_device.cuh"

namespace qftk {
namespace um {
using qftd::smem_u32;

// K-major SWIZZLE_128B smem descriptor (tcgen05 matrix descriptor): start >> 4,
// leading byte offset 1 (unused for swizzled K-major), stride byte offset 1024 B between
// 8-row groups, version 1, layout type 2 (SWIZZLE_128B)
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1u << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
#ifndef UMMA_EPI_V8
#define UMMA_EPI_V8 1
#endif
// ---- CTA-pair (cta_group::2) plumbing: the MMA of a 2-SM pair is issued by the leader
// (cluster rank 0) and reads A and B halves from both CTAs' shared memory at the same
// offsets; barriers the leader waits on receive the peer's TMA bytes and arrivals through
// shared::cluster addresses (mapa)
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// the shared::cluster address of `p` (this CTA's shared variable) in cluster CTA `rank`
__device__ __forceinline__ uint32_t mapa_cl(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_arrive_cl(uint32_t cl_addr) {
  // default semantics (release.cta), the form CUTLASS's 2-SM pipelines use; .release.cluster
  // compiles to MEMBAR.ALL.GPU + ERRBAR per arrive and cost the pair kernel ~40%
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cl(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// wait with cluster-scope acquire: arrivals came from the peer CTA
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait_cl(bar, parity)) {
  }
}
// TMA 2-D load into this CTA's shared memory whose completion bytes are counted on a
// barrier of either CTA of the pair (`bar_cl`: shared::cluster address)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint32_t bar_cl) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar_cl)
      : "memory");
}
__device__ __forceinline__ void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// arrive (once, when the pair's prior MMAs complete) on the barrier at `bar`'s offset in
// every CTA of `mask`
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 "
      "[%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}

// tcgen05.ld 32x32b.x32: lane i of the warp gets 32 consecutive fp32 columns of TMEM lane
// (warp % 4) * 32 + i (the warp's lane quarter) starting at `addr`; waits for completion
__device__ __forceinline__ void tmem_ld32(uint32_t addr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// tcgen05.ld 32x32b.x32 without the wait (the registers are undefined until tmem_wait32)
__device__ __forceinline__ void tmem_ld32_issue(uint32_t addr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(addr));
}
// wait for the thread's outstanding tcgen05.ld; `r` as in-out operands, so no use of the
// loaded registers moves above the wait
__device__ __forceinline__ void tmem_wait32(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]),
                 "+r"(r[6]), "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]),
                 "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]),
                 "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]),
                 "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]),
                 "+r"(r[30]), "+r"(r[31])
               :
               : "memory");
}

// The bf16 epilogue of the GEMMs with NACC M=128 accumulators of BN fp32 columns: warp
// (4 + 4g + q) drains TMEM lanes 32q.. for warp group g of NPW/4 -- the (accumulator,
// 32-column chunk) units g, g + NPW/4, ... (accumulator a: rows m0 + 128a ..) -- rounds to
// bf16 (RNE) and stores y[row, n0 + c ..] of the row-major [M, N] output.
template <int BN, int NACC, int NPW>
__device__ __forceinline__ void epilogue_bf16(uint32_t tmem_d, int warp, int lane, int m0, int n0,
                                              int M, int N, __nv_bfloat16* y) {
  const int wq = (warp - 4) & 3, grp = (warp - 4) >> 2;
  const uint32_t lane_base = (uint32_t)(32 * wq) << 16;
  constexpr int CH = BN / 32, GROUPS = NPW / 4, NU = NACC * CH / GROUPS;
  static_assert(NACC * CH % GROUPS == 0, "epilogue units per warp");
  // the warp's units k = 0..NU-1 (unit u = grp + k * GROUPS: accumulator u / CH, columns
  // (u % CH) * 32 ..), double-buffered: unit k+1's TMEM load is in flight while unit k
  // is converted and stored
  auto taddr = [&](int k) {
    const int u = grp + k * GROUPS;
    return tmem_d + lane_base + (uint32_t)((u / CH) * BN + (u % CH) * 32);
  };
  uint32_t rb[2][32];
  tmem_ld32_issue(taddr(0), rb[0]);
  tmem_wait32(rb[0]);
#pragma unroll
  for (int k = 0; k < NU; ++k) {
    if (k + 1 < NU) tmem_ld32_issue(taddr(k + 1), rb[(k + 1) & 1]);
    uint32_t* r = rb[k & 1];
    const int u = grp + k * GROUPS;
    const int accn = u / CH, c0 = (u % CH) * 32;
    const int row = m0 + 128 * accn + 32 * wq + lane;
    if (row < M) {
      __nv_bfloat16* yr = y + (size_t)row * N + n0 + c0;
      if (UMMA_EPI_V8 && n0 + c0 + 32 <= N && (N % 16) == 0) {
        // two 32-byte stores (STG.256): every store fills whole L2 sectors of its row
        // (16-byte stores left each sector half-written per instruction: ncu-measured
        // the epilogue at ~1.6 TB/s, 15% of a 4096^3 GEMM)
        uint32_t o[16];
#pragma unroll
        for (int q = 0; q < 16; ++q)
          o[q] = pack_bf16(__uint_as_float(r[2 * q]), __uint_as_float(r[2 * q + 1]));
#pragma unroll
        for (int h = 0; h < 2; ++h)
          asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(yr + 16 * h),
                       "r"(o[8 * h]), "r"(o[8 * h + 1]), "r"(o[8 * h + 2]), "r"(o[8 * h + 3]),
                       "r"(o[8 * h + 4]), "r"(o[8 * h + 5]), "r"(o[8 * h + 6]), "r"(o[8 * h + 7])
                       : "memory");
      } else if (n0 + c0 + 32 <= N && (N % 8) == 0) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 o;
          o.x = pack_bf16(__uint_as_float(r[8 * q]), __uint_as_float(r[8 * q + 1]));
          o.y = pack_bf16(__uint_as_float(r[8 * q + 2]), __uint_as_float(r[8 * q + 3]));
          o.z = pack_bf16(__uint_as_float(r[8 * q + 4]), __uint_as_float(r[8 * q + 5]));
          o.w = pack_bf16(__uint_as_float(r[8 * q + 6]), __uint_as_float(r[8 * q + 7]));
          reinterpret_cast<uint4*>(yr)[q] = o;
        }
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e)  // (static indices: r stays in registers)
          if (n0 + c0 + e < N) yr[e] = __float2bfloat16_rn(__uint_as_float(r[e]));
      }
    }
    if (k + 1 < NU) tmem_wait32(rb[(k + 1) & 1]);
  }
}

// MN-major SWIZZLE_128B descriptor (canonical layout ((8,n),(8,k)) : ((1,LBO),(8,SBO)) in
// 16-byte units): 64 contiguous MN elements (128 B, one TMA box row) per K row, 8 K rows per
// 1024-byte swizzle atom; `lbo` = bytes between 64-element MN chunks, `sbo` = bytes between
// 8-row K groups
__device__ __forceinline__ uint64_t sw128_desc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | ((uint64_t)1u << 46) | ((uint64_t)2u << 61);
}

// cuTensorMapEncodeTiled from the driver (no -lcuda link)
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}
}  // namespace um
}  // namespace qftk
