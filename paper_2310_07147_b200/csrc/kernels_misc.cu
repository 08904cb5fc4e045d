// kernels_misc.cu -- the non-fused kernels of the path (sm_100a):
//   channel_minmax, affine params, quantize / quantize_state, dequantize (f32,
//   bf16), outlier thresholds (exact per-row radix select), pass-through Lion,
//   and the synthetic-input generator.
// All arithmetic follows qft_device.cuh (bit-exact with the reference CPU code).
#include <cuda_bf16.h>

#include "qft_device.cuh"
#include "qft_internal.h"

namespace qftk {
using namespace qftd;

constexpr int RT = 256;  // threads per row-CTA

// block-wide min/max reduce over RT threads; returns the result in every thread
__device__ __forceinline__ void block_minmax(float& lo, float& hi, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) {
    red[w] = lo;
    red[32 + w] = hi;
  }
  __syncthreads();
  lo = red[0];
  hi = red[32];
#pragma unroll
  for (int i = 1; i < RT / 32; ++i) {
    lo = fminf(lo, red[i]);
    hi = fmaxf(hi, red[32 + i]);
  }
}

// row min/max with the reference's sequential semantics (tensor.hpp:133-148):
// NaN never replaces a bound, but a NaN in column 0 is the initial bound and sticks.
__device__ __forceinline__ void row_minmax(const float* x, int cols, bool vec4, float& lo,
                                           float& hi, float* red) {
  lo = __int_as_float(0x7f800000);
  hi = __int_as_float(0xff800000);
  if (vec4) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int i = threadIdx.x; i < cols / 4; i += RT) {
      const float4 f = x4[i];
      float t;
      asm("min.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(lo), "f"(f.x), "f"(f.y)); lo = t;
      asm("min.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(lo), "f"(f.z), "f"(f.w)); lo = t;
      asm("max.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(hi), "f"(f.x), "f"(f.y)); hi = t;
      asm("max.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(hi), "f"(f.z), "f"(f.w)); hi = t;
    }
  } else {
    for (int i = threadIdx.x; i < cols; i += RT) {
      lo = fminf(lo, x[i]);
      hi = fmaxf(hi, x[i]);
    }
  }
  block_minmax(lo, hi, red);
  if (isnan(x[0])) lo = hi = x[0];
}

// ------------------------------------------------------------- channel_minmax
__global__ void __launch_bounds__(RT) k_channel_minmax(const float* __restrict__ x, int rows,
                                                       int cols, int vec4, float* mins,
                                                       float* maxs) {
  __shared__ float red[64];
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    float lo, hi;
    row_minmax(x + (size_t)r * cols, cols, vec4, lo, hi, red);
    if (threadIdx.x == 0) {
      mins[r] = lo;
      maxs[r] = hi;
    }
  }
}

// ------------------------------------------------------------- affine params
__global__ void k_affine_params(const float* mins, const float* maxs, int64_t n, int bw,
                                float* scale, int32_t* zp, uint32_t* err) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float s;
    int32_t z;
    if (!affine_from_bounds(mins[i], maxs[i], bw, s, z)) {
      atomicOr(err, 1u);
      s = 1.0f;
      z = 0;
    }
    scale[i] = s;
    zp[i] = z;
  }
}

// ------------------------------------------------------------- quantize rows
// quantize 4 values with validation, exact fallback
__device__ __forceinline__ uint32_t quant4(const float* x, const QuantRow& q) {
  float em = 0.0f;
  uint32_t c = q.fast ? quant4_fast(x, q, em) : 0u;
  if (!q.fast || !(em < q.thr)) c = quant4_exact(x, q);
  return c;
}

__device__ __forceinline__ void quantize_row(const float* x, int cols, bool vec4,
                                             const QuantRow& q, uint8_t* out) {
  if (vec4) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    for (int i = threadIdx.x; i < cols / 4; i += RT) {
      const float4 f = x4[i];
      const float v[4] = {f.x, f.y, f.z, f.w};
      reinterpret_cast<uint32_t*>(out)[i] = quant4(v, q);
    }
  } else {
    for (int i = threadIdx.x; i < cols; i += RT)
      out[i] = (uint8_t)quant_exact(x[i], q.s, q.z, q.qmax);
  }
}

// quantize_state: fresh per-row params from the row's own min/max, then quantize
// (quantize.hpp:189-193 -> compute_affine_params -> quantize).  Fused: the row is
// read once for the bounds and once (from L2) for the codes.
__global__ void __launch_bounds__(RT) k_quantize_state(const float* __restrict__ x, int rows,
                                                       int cols, int bw, int vec4,
                                                       uint8_t* codes, float* scale,
                                                       int32_t* zp, uint32_t* err) {
  __shared__ float red[64];
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const float* xr = x + (size_t)r * cols;
    float lo, hi;
    row_minmax(xr, cols, vec4, lo, hi, red);
    float s;
    int32_t z;
    if (!affine_from_bounds(lo, hi, bw, s, z)) {
      if (threadIdx.x == 0) atomicOr(err, 1u);
      s = 1.0f;
      z = 0;
    }
    if (threadIdx.x == 0) {
      scale[r] = s;
      zp[r] = z;
    }
    quantize_row(xr, cols, vec4, make_quant_row(s, z, bw), codes + (size_t)r * cols);
  }
}

// accumulate (gradflow.hpp:52-58): the micro-batch running sum kept in integer form,
// sum = dequantize(acc) + g_new in fp32 (quantize.hpp:195-212, then tensor add), then
// quantize_state(sum) with fresh per-row params.  Fused: the sum never exists in HBM
// (pass 1: bounds; pass 2: recomputed from the L2-resident row and quantized).  The
// old params are read before the block barrier, so the update may be in place.
__device__ __forceinline__ float acc_sum(const uint8_t* c, const float* g, int i,
                                         const DequantRow& d) {
  return __fadd_rn(dequant_exact(c[i], d.s, d.z), g[i]);
}
__global__ void __launch_bounds__(RT) k_accumulate_state(
    const uint8_t* codes, const float* scale, const int32_t* zp, int rows, int cols, int bw,
    const float* __restrict__ g, int vec4, int staged, uint8_t* codes_out, float* scale_out,
    int32_t* zp_out, uint32_t* err) {
  __shared__ float red[64];
  extern __shared__ float4 sums[];  // staged: the row's fp32 sums between the passes
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const DequantRow d = make_dequant_row(scale[r], zp[r]);
    const uint8_t* cr = codes + (size_t)r * cols;
    const float* gr = g + (size_t)r * cols;
    float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
    if (vec4) {
#pragma unroll 4  // independent row loads in flight (the loop is latency-bound otherwise)
      for (int i = threadIdx.x; i < cols / 4; i += RT) {
        float v[4];
        dequant4(reinterpret_cast<const uint32_t*>(cr)[i], d, v);
        const float4 f = reinterpret_cast<const float4*>(gr)[i];
        v[0] = __fadd_rn(v[0], f.x); v[1] = __fadd_rn(v[1], f.y);
        v[2] = __fadd_rn(v[2], f.z); v[3] = __fadd_rn(v[3], f.w);
        if (staged) sums[i] = make_float4(v[0], v[1], v[2], v[3]);
        float t;
        asm("min.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(lo), "f"(v[0]), "f"(v[1])); lo = t;
        asm("min.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(lo), "f"(v[2]), "f"(v[3])); lo = t;
        asm("max.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(hi), "f"(v[0]), "f"(v[1])); hi = t;
        asm("max.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(hi), "f"(v[2]), "f"(v[3])); hi = t;
      }
    } else {
      for (int i = threadIdx.x; i < cols; i += RT) {
        const float v = acc_sum(cr, gr, i, d);
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
      }
    }
    const float v0 = acc_sum(cr, gr, 0, d);  // read before the barrier (in-place safe)
    block_minmax(lo, hi, red);  // (barrier: every thread has read the old params)
    if (isnan(v0)) lo = hi = v0;  // channel_minmax: a NaN in column 0 sticks
    float s;
    int32_t z;
    if (!affine_from_bounds(lo, hi, bw, s, z)) {
      if (threadIdx.x == 0) *(volatile uint32_t*)err = 1u;  // may be mapped host memory
      s = 1.0f;
      z = 0;
    }
    const QuantRow q = make_quant_row(s, z, bw);
    uint8_t* out = codes_out + (size_t)r * cols;
    if (vec4 && staged) {  // each thread re-reads only what it staged itself
#pragma unroll 4
      for (int i = threadIdx.x; i < cols / 4; i += RT) {
        const float4 f = sums[i];
        const float v[4] = {f.x, f.y, f.z, f.w};
        reinterpret_cast<uint32_t*>(out)[i] = quant4(v, q);
      }
    } else if (vec4) {
      for (int i = threadIdx.x; i < cols / 4; i += RT) {
        float v[4];
        dequant4(reinterpret_cast<const uint32_t*>(cr)[i], d, v);
        const float4 f = reinterpret_cast<const float4*>(gr)[i];
        v[0] = __fadd_rn(v[0], f.x); v[1] = __fadd_rn(v[1], f.y);
        v[2] = __fadd_rn(v[2], f.z); v[3] = __fadd_rn(v[3], f.w);
        reinterpret_cast<uint32_t*>(out)[i] = quant4(v, q);
      }
    } else {
      for (int i = threadIdx.x; i < cols; i += RT)
        out[i] = (uint8_t)quant_exact(acc_sum(cr, gr, i, d), q.s, q.z, q.qmax);
    }
    __syncthreads();  // the next row's barrier-free reads vs this row's param write
    if (threadIdx.x == 0) {
      scale_out[r] = s;
      zp_out[r] = z;
    }
  }
}

__global__ void __launch_bounds__(RT) k_quantize(const float* __restrict__ x, int rows, int cols,
                                                 const float* scale, const int32_t* zp,
                                                 int channels, int bw, int vec4,
                                                 uint8_t* codes) {
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const int ch = channels == 1 ? 0 : r;
    quantize_row(x + (size_t)r * cols, cols, vec4, make_quant_row(scale[ch], zp[ch], bw),
                 codes + (size_t)r * cols);
  }
}

// ------------------------------------------------------------- dequantize
template <bool BF16>
__global__ void __launch_bounds__(RT) k_dequantize(const uint8_t* __restrict__ codes, int rows,
                                                   int cols, const float* scale,
                                                   const int32_t* zp, int channels, int vec4,
                                                   void* out) {
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const int ch = channels == 1 ? 0 : r;
    const DequantRow d = make_dequant_row(scale[ch], zp[ch]);
    const uint8_t* cr = codes + (size_t)r * cols;
    if (vec4) {
      for (int i = threadIdx.x; i < cols / 4; i += RT) {
        float v[4];
        dequant4(reinterpret_cast<const uint32_t*>(cr)[i], d, v);
        if (BF16) {
          const __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]);
          const __nv_bfloat162 b = __floats2bfloat162_rn(v[2], v[3]);
          uint2 pk;
          pk.x = *reinterpret_cast<const uint32_t*>(&a);
          pk.y = *reinterpret_cast<const uint32_t*>(&b);
          reinterpret_cast<uint2*>(out)[((size_t)r * cols) / 4 + i] = pk;
        } else {
          reinterpret_cast<float4*>(out)[((size_t)r * cols) / 4 + i] =
              make_float4(v[0], v[1], v[2], v[3]);
        }
      }
    } else {
      for (int i = threadIdx.x; i < cols; i += RT) {
        const float v = dequant_exact(cr[i], d.s, d.z);
        if (BF16)
          reinterpret_cast<__nv_bfloat16*>(out)[(size_t)r * cols + i] = __float2bfloat16_rn(v);
        else
          reinterpret_cast<float*>(out)[(size_t)r * cols + i] = v;
      }
    }
  }
}

// ------------------------------------------------------------- thresholds
// Exact k-th smallest of a row (ascending order statistics, 0-based) by a 4-pass
// 8-bit radix select on order-preserving u32 keys.  Equivalent to std::sort then
// indexing (quantize.hpp:240-243): ties are equal values, so any sorted order
// gives the same key at every rank.
__device__ uint32_t row_select(const float* x, int cols, int k, uint32_t* hist,
                               int* bcast) {
  uint32_t prefix = 0, pmask = 0;
  int remaining = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += RT) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < cols; i += RT) {
      const uint32_t key = float_key(x[i]);
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int l = threadIdx.x;
      uint32_t c[8];
      uint32_t sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c[j] = hist[l * 8 + j];
        sum += c[j];
      }
      uint32_t incl = sum;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
        if (l >= d) incl += t;
      }
      const uint32_t excl = incl - sum;
      const bool mine = (excl <= (uint32_t)remaining) && ((uint32_t)remaining < incl);
      if (mine) {
        uint32_t run = excl;
        int b = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (run + c[j] > (uint32_t)remaining) { b = l * 8 + j; break; }
          run += c[j];
        }
        bcast[0] = b;
        bcast[1] = remaining - (int)run;
      }
    }
    __syncthreads();
    const uint32_t b = (uint32_t)bcast[0];
    remaining = bcast[1];
    prefix |= b << shift;
    pmask |= 255u << shift;
    __syncthreads();
  }
  return prefix;
}

struct QuantileSpec {
  int i0;       // lower index
  int exact;    // 1: value is s[i0] (n==1 or i0 >= n-1)
  double frac;
};

__device__ float quantile_value(const float* x, int cols, const QuantileSpec& q, uint32_t* hist,
                                int* bcast) {
  const float a = key_float(row_select(x, cols, q.i0, hist, bcast));
  if (q.exact) return a;
  const float b = key_float(row_select(x, cols, q.i0 + 1, hist, bcast));
  // sorted_quantile, quantize.hpp:85-86, in fp64 without contraction
  const double v =
      __dadd_rn((double)a, __dmul_rn(q.frac, __dsub_rn((double)b, (double)a)));
  return __double2float_rn(v);
}

__global__ void __launch_bounds__(RT) k_thresholds_percentile(const float* __restrict__ w,
                                                              int rows, int cols,
                                                              QuantileSpec qlo, QuantileSpec qhi,
                                                              float* t_min, float* t_max) {
  __shared__ uint32_t hist[256];
  __shared__ int bcast[2];
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const float* x = w + (size_t)r * cols;
    const float lo = quantile_value(x, cols, qlo, hist, bcast);
    const float hi = quantile_value(x, cols, qhi, hist, bcast);
    if (threadIdx.x == 0) {
      t_min[r] = lo;
      t_max[r] = hi;
    }
  }
}

// fraction == 0 (plain range) or range_fraction (quantize.hpp:225-238)
__global__ void __launch_bounds__(RT) k_thresholds_range(const float* __restrict__ w, int rows,
                                                         int cols, int vec4, double fraction,
                                                         float* t_min, float* t_max) {
  __shared__ float red[64];
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    float lo, hi;
    row_minmax(w + (size_t)r * cols, cols, vec4, lo, hi, red);
    if (threadIdx.x == 0) {
      if (fraction == 0.0) {
        t_min[r] = lo;
        t_max[r] = hi;
      } else {
        const double span = __dsub_rn((double)hi, (double)lo);
        const double f2 = fraction / 2;
        t_min[r] = __double2float_rn(__dadd_rn((double)lo, __dmul_rn(f2, span)));
        t_max[r] = __double2float_rn(__dsub_rn((double)hi, __dmul_rn(f2, span)));
      }
    }
  }
}

// ------------------------------------------------------------- pass-through Lion
template <bool VEC>
__global__ void k_lion_apply(float* __restrict__ w, float* __restrict__ m,
                             const float* __restrict__ g, int64_t n, Hyper h) {
  const int64_t n4 = VEC ? n / 4 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 W = reinterpret_cast<float4*>(w)[i];
    float4 M = reinterpret_cast<float4*>(m)[i];
    const float4 G = reinterpret_cast<const float4*>(g)[i];
    float2 w0 = make_float2(W.x, W.y), w1 = make_float2(W.z, W.w);
    float2 m0 = make_float2(M.x, M.y), m1 = make_float2(M.z, M.w);
    lion2(w0, m0, make_float2(G.x, G.y), h);
    lion2(w1, m1, make_float2(G.z, G.w), h);
    reinterpret_cast<float4*>(w)[i] = make_float4(w0.x, w0.y, w1.x, w1.y);
    reinterpret_cast<float4*>(m)[i] = make_float4(m0.x, m0.y, m1.x, m1.y);
  }
  for (int64_t i = n4 * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float wv = w[i], mv = m[i];
    lion1(wv, mv, g[i], h);
    w[i] = wv;
    m[i] = mv;
  }
}

// ------------------------------------------------------------- synthetic inputs
// Device twin of oracle/synth.c qo_synth (bit-identical: integer hashing plus
// +,-,* in fp64 with explicit rounding, no transcendental functions).
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double draw_u(uint64_t key, uint64_t i, unsigned k) {
  return __dmul_rn((double)(splitmix64(key + i * 8ull + k) >> 11), 0x1.0p-53);
}
__global__ void k_synth(float* out, int64_t n, uint64_t key, double sigma, double spike_p) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t u = (uint64_t)i;
    const double u0 = draw_u(key, u, 0), u1 = draw_u(key, u, 1);
    const double u2 = draw_u(key, u, 2), u3 = draw_u(key, u, 3);
    const double sum = __dsub_rn(__dadd_rn(__dadd_rn(__dadd_rn(u0, u1), u2), u3), 2.0);
    double v = __dmul_rn(__dmul_rn(sum, 1.7320508075688772), sigma);
    if (spike_p > 0.0 && draw_u(key, u, 4) < spike_p) {
      const double mag = __dadd_rn(100.0, __dmul_rn(900.0, draw_u(key, u, 5)));
      v = __dmul_rn(draw_u(key, u, 6) < 0.5 ? -mag : mag, sigma);
    }
    out[i] = __double2float_rn(v);
  }
}

// ============================================================================
// host launchers (called by capi.cu)
// ============================================================================
static int row_grid(int rows) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int g = sms * 8;
  return rows < g ? rows : g;
}
static inline bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
static inline int vec4_ok(const void* a, int cols) { return (cols % 4 == 0) && al16(a); }

cudaError_t launch_channel_minmax(const float* x, int rows, int cols, float* mins, float* maxs,
                                  cudaStream_t s) {
  k_channel_minmax<<<row_grid(rows), RT, 0, s>>>(x, rows, cols, vec4_ok(x, cols), mins, maxs);
  return cudaGetLastError();
}
cudaError_t launch_affine_params(const float* mins, const float* maxs, int64_t n, int bw,
                                 float* scale, int32_t* zp, uint32_t* err, cudaStream_t s) {
  const int64_t blocks = (n + 255) / 256;
  k_affine_params<<<(int)(blocks < 4096 ? blocks : 4096), 256, 0, s>>>(mins, maxs, n, bw, scale,
                                                                       zp, err);
  return cudaGetLastError();
}
cudaError_t launch_quantize_state(const float* x, int rows, int cols, int bw, uint8_t* codes,
                                  float* scale, int32_t* zp, uint32_t* err, cudaStream_t s) {
  const int v4 = vec4_ok(x, cols) && al16(codes);
  k_quantize_state<<<row_grid(rows), RT, 0, s>>>(x, rows, cols, bw, v4, codes, scale, zp, err);
  return cudaGetLastError();
}
cudaError_t launch_accumulate_state(const uint8_t* codes, const float* scale, const int32_t* zp,
                                    int rows, int cols, int bw, const float* g,
                                    uint8_t* codes_out, float* scale_out, int32_t* zp_out,
                                    uint32_t* err, cudaStream_t s) {
  const int v4 = (cols % 4 == 0) && vec4_ok(g, cols) && al16(codes) && al16(codes_out);
  // stage the sums in shared memory when the row fits 48 KB (the second pass then
  // reads no global memory); wider rows re-read the row from L2
  const size_t sm = (size_t)cols * 4;
  const int staged = v4 && sm <= 48 * 1024;
  k_accumulate_state<<<row_grid(rows), RT, staged ? sm : 0, s>>>(
      codes, scale, zp, rows, cols, bw, g, v4, staged, codes_out, scale_out, zp_out, err);
  return cudaGetLastError();
}
cudaError_t launch_quantize(const float* x, int rows, int cols, const float* scale,
                            const int32_t* zp, int channels, int bw, uint8_t* codes,
                            cudaStream_t s) {
  const int v4 = vec4_ok(x, cols) && al16(codes);
  k_quantize<<<row_grid(rows), RT, 0, s>>>(x, rows, cols, scale, zp, channels, bw, v4, codes);
  return cudaGetLastError();
}
cudaError_t launch_dequantize(const uint8_t* codes, int rows, int cols, const float* scale,
                              const int32_t* zp, int channels, void* out, bool bf16,
                              cudaStream_t s) {
  const int v4 = (cols % 4 == 0) && al16(codes) && al16(out);
  if (bf16)
    k_dequantize<true><<<row_grid(rows), RT, 0, s>>>(codes, rows, cols, scale, zp, channels, v4,
                                                     out);
  else
    k_dequantize<false><<<row_grid(rows), RT, 0, s>>>(codes, rows, cols, scale, zp, channels, v4,
                                                      out);
  return cudaGetLastError();
}
cudaError_t launch_thresholds(const float* w, int rows, int cols, double fraction, int kind,
                              float* t_min, float* t_max, cudaStream_t s) {
  if (fraction == 0.0 || kind == QFTC_RANGE_FRACTION) {
    k_thresholds_range<<<row_grid(rows), RT, 0, s>>>(w, rows, cols, vec4_ok(w, cols), fraction,
                                                     t_min, t_max);
    return cudaGetLastError();
  }
  // sorted_quantile index arithmetic (quantize.hpp:76-87), identical on host
  auto spec = [cols](double q) {
    QuantileSpec r{0, 1, 0.0};
    const size_t n = (size_t)cols;
    if (n == 1) return r;
    const double hh = q * (double)(n - 1);
    const size_t i0 = (size_t)hh;
    if (i0 >= n - 1) {
      r.i0 = (int)(n - 1);
      return r;
    }
    r.i0 = (int)i0;
    r.exact = 0;
    r.frac = hh - (double)i0;
    return r;
  };
  k_thresholds_percentile<<<row_grid(rows), RT, 0, s>>>(w, rows, cols, spec(fraction / 2),
                                                        spec(1.0 - fraction / 2), t_min, t_max);
  return cudaGetLastError();
}
cudaError_t launch_lion_apply(float* w, float* m, const float* g, int64_t n, float lr, float b1,
                              float b2, float wd, cudaStream_t s) {
  Hyper h;
  h.lr = lr; h.b1 = b1; h.b2 = b2; h.wd = wd;
  h.c1 = 1.0f - b1;
  h.c2 = 1.0f - b2;
  const bool ok = al16(w) && al16(m) && al16(g);
  int64_t blocks = ((ok ? n / 4 : n) + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (ok)
    k_lion_apply<true><<<(int)blocks, 256, 0, s>>>(w, m, g, n, h);
  else
    k_lion_apply<false><<<(int)blocks, 256, 0, s>>>(w, m, g, n, h);
  return cudaGetLastError();
}
cudaError_t launch_synth(float* out, int64_t n, uint64_t seed, double sigma, double spike_p,
                         cudaStream_t s) {
  uint64_t z = seed + 0x9E3779B97F4A7C15ull;  // splitmix64(seed) on the host
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  const uint64_t key = z ^ (z >> 31);
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  k_synth<<<(int)blocks, 256, 0, s>>>(out, n, key, sigma, spike_p);
  return cudaGetLastError();
}

}  // namespace qftk
