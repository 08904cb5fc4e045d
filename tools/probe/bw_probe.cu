// Bandwidth probe for the step's access pattern: per row, read w|m|g (1 B/elem each),
// write w|m.  Variants: (0) LDG.128/STG.128 warp-per-row, (1) TMA loads into smem +
// STG.128 from smem, (2) plain copy of 2 arrays (read 2, write 2).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2310_07147_b200/csrc bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "qft_device.cuh"
using namespace qftd;

__global__ void k_ldg(const uint4* w, const uint4* m, const uint4* g, uint4* wo, uint4* mo,
                      long rows, int vpr) {
  const int lane = threadIdx.x & 31;
  const long tw = (long)gridDim.x * (blockDim.x >> 5);
  for (long r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += tw) {
    const long b = r * vpr;
    for (int v = lane; v < vpr; v += 32) {
      uint4 a = __ldcs(w + b + v), c = __ldcs(m + b + v), d = __ldcs(g + b + v);
      c.x ^= d.x; c.y ^= d.y; c.z ^= d.z; c.w ^= d.w;
      __stcs(wo + b + v, a);
      __stcs(mo + b + v, c);
    }
  }
}

__global__ void k_tma(const uint8_t* w, const uint8_t* m, const uint8_t* g, uint8_t* wo,
                      uint8_t* mo, long rows, int cols) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint8_t* st = sm + wid * (3 * cols + 16);
  uint64_t* bar = reinterpret_cast<uint64_t*>(st + 3 * cols);
  if (lane == 0) { mbar_init(bar, 1); mbar_fence_init(); }
  __syncwarp();
  const long tw = (long)gridDim.x * (blockDim.x >> 5);
  uint32_t ph = 0;
  for (long r = blockIdx.x * (blockDim.x >> 5) + wid; r < rows; r += tw) {
    const long b = r * cols;
    if (lane == 0) {
      mbar_arrive_expect_tx(bar, 3 * cols);
      bulk_g2s(st, w + b, cols, bar);
      bulk_g2s(st + cols, m + b, cols, bar);
      bulk_g2s(st + 2 * cols, g + b, cols, bar);
    }
    mbar_wait(bar, ph);
    ph ^= 1;
    for (int v = lane; v < cols / 16; v += 32) {
      uint4 a = reinterpret_cast<uint4*>(st)[v];
      uint4 c = reinterpret_cast<uint4*>(st + cols)[v];
      uint4 d = reinterpret_cast<uint4*>(st + 2 * cols)[v];
      c.x ^= d.x; c.y ^= d.y; c.z ^= d.z; c.w ^= d.w;
      __stcs(reinterpret_cast<uint4*>(wo + b) + v, a);
      __stcs(reinterpret_cast<uint4*>(mo + b) + v, c);
    }
    __syncwarp();
  }
}

int main() {
  const long cols = 4096, rows = 1290000;  // the 4096-column group of LLaMA-2-7B
  const size_t n = (size_t)rows * cols;
  uint8_t *w, *m, *g, *wo, *mo;
  cudaMalloc(&w, n); cudaMalloc(&m, n); cudaMalloc(&g, n); cudaMalloc(&wo, n); cudaMalloc(&mo, n);
  cudaMemset(w, 1, n); cudaMemset(m, 2, n); cudaMemset(g, 3, n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int variant = 0; variant < 3; ++variant) {
    for (int wpb : {4, 8}) {
      for (int bps : {2, 4, 8}) {
        const int smem = variant == 1 ? wpb * (3 * cols + 16) : 0;
        if (smem > 227 * 1024) continue;
        if (variant == 1) cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int grid = sms * bps;
        float best = 1e9;
        for (int it = 0; it < 4; ++it) {
          cudaEventRecord(e0);
          if (variant == 0)
            k_ldg<<<grid, wpb * 32>>>((uint4*)w, (uint4*)m, (uint4*)g, (uint4*)wo, (uint4*)mo, rows, cols / 16);
          else if (variant == 1)
            k_tma<<<grid, wpb * 32, smem>>>(w, m, g, wo, mo, rows, cols);
          else {
            cudaMemcpyAsync(wo, w, n, cudaMemcpyDeviceToDevice);
            cudaMemcpyAsync(mo, m, n, cudaMemcpyDeviceToDevice);
          }
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1);
          if (it) best = ms < best ? ms : best;
        }
        const double bytes = (variant == 2 ? 4.0 : 5.0) * n;
        printf("variant %d wpb %d ctas/sm %d: %.3f ms  %.0f GB/s  (%s)\n", variant, wpb, bps, best,
               bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
        if (variant == 2) break;
      }
      if (variant == 2) break;
    }
  }
  return 0;
}
