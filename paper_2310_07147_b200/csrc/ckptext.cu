// ckptext.cu -- the opt-in QFTC format extensions (not part of the
// reference's v1 format, non-parity by definition):
//   * packed sub-byte codes: a row's b-bit codes (b < 8) bit-packed LSB-first, the row
//     padded to a whole byte -- lossless;
//   * blockwise momentum scales: the momentum (per-row affine codes, quantize.hpp:189-193)
//     re-expressed with one affine (scale, zero point) per block of `block` elements of a
//     row (the block's own quantize_state, quantize.hpp:105-131 over the block), and back
//     to the per-row form on load (quantize_state of each row of the dequantized blocks) --
//     lossy, as any change of quantization grid is.
// The arithmetic of every (de)quantization is the reference's (qft_device.cuh).
#include "qft_device.cuh"
#include "qft_internal.h"

namespace qftk {
using namespace qftd;

namespace {
constexpr int XT = 256;

// one thread per group of 8 codes: 8 x b bits = b bytes out (b in [2, 8])
__global__ void k_pack_codes(const uint8_t* __restrict__ src, int rows, int cols, int bits,
                             uint8_t* __restrict__ dst) {
  const int groups = (cols + 7) / 8;
  const int row_bytes = (cols * bits + 7) / 8;
  const long long n = (long long)rows * groups;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(g / groups), k = (int)(g % groups);
    const uint8_t* s = src + (size_t)r * cols + 8 * k;
    uint64_t acc = 0;
    const int m = min(8, cols - 8 * k);
    for (int e = 0; e < m; ++e) acc |= (uint64_t)(s[e] & ((1u << bits) - 1u)) << (bits * e);
    uint8_t* d = dst + (size_t)r * row_bytes + (size_t)k * bits;
    const int nb = min(bits, row_bytes - k * bits);
    for (int b = 0; b < nb; ++b) d[b] = (uint8_t)(acc >> (8 * b));
  }
}

__global__ void k_unpack_codes(const uint8_t* __restrict__ src, int rows, int cols, int bits,
                               uint8_t* __restrict__ dst) {
  const int groups = (cols + 7) / 8;
  const int row_bytes = (cols * bits + 7) / 8;
  const long long n = (long long)rows * groups;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(g / groups), k = (int)(g % groups);
    const uint8_t* s = src + (size_t)r * row_bytes + (size_t)k * bits;
    const int nb = min(bits, row_bytes - k * bits);
    uint64_t acc = 0;
    for (int b = 0; b < nb; ++b) acc |= (uint64_t)s[b] << (8 * b);
    uint8_t* d = dst + (size_t)r * cols + 8 * k;
    const int m = min(8, cols - 8 * k);
    for (int e = 0; e < m; ++e) d[e] = (uint8_t)((acc >> (bits * e)) & ((1u << bits) - 1u));
  }
}

// per-row momentum -> per-block quantization: one thread per block (blocks are short)
__global__ void k_mom_to_blocks(const uint8_t* __restrict__ codes, const float* __restrict__ scale,
                                const int32_t* __restrict__ zp, int rows, int cols, int bits,
                                int block, uint8_t* __restrict__ out, float* __restrict__ bscale,
                                int32_t* __restrict__ bzp, uint32_t* err) {
  const int nblk = (cols + block - 1) / block;
  const long long n = (long long)rows * nblk;
  const int qmax = (1 << bits) - 1;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < n;
       g += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(g / nblk), b = (int)(g % nblk);
    const int c0 = b * block, c1 = min(cols, c0 + block);
    const float s = scale[r];
    const int32_t z = zp[r];
    const uint8_t* cr = codes + (size_t)r * cols;
    float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
    const float first = dequant_exact(cr[c0], s, z);
    for (int c = c0; c < c1; ++c) {
      const float v = dequant_exact(cr[c], s, z);
      lo = fminf(lo, v);
      hi = fmaxf(hi, v);
    }
    if (first != first) lo = hi = first;
    float bs;
    int32_t bz;
    if (!affine_from_bounds(lo, hi, bits, bs, bz)) {
      atomicOr(err, 1u);
      bs = 1.0f;
      bz = 0;
    }
    bscale[g] = bs;
    bzp[g] = bz;
    uint8_t* o = out + (size_t)r * cols;
    for (int c = c0; c < c1; ++c) o[c] = (uint8_t)quant_exact(dequant_exact(cr[c], s, z), bs, bz, qmax);
  }
}

// per-block momentum -> per-row quantize_state of the dequantized row (one CTA per row:
// pass 1 the row's min/max, pass 2 the codes; the values are recomputed from the codes)
__global__ void __launch_bounds__(XT) k_mom_from_blocks(const uint8_t* __restrict__ codes,
                                                         const float* __restrict__ bscale,
                                                         const int32_t* __restrict__ bzp,
                                                         int rows, int cols, int bits, int block,
                                                         uint8_t* __restrict__ out,
                                                         float* __restrict__ scale,
                                                         int32_t* __restrict__ zp, uint32_t* err) {
  __shared__ float red[2][XT / 32];
  __shared__ float prm[2];
  const int nblk = (cols + block - 1) / block;
  const int qmax = (1 << bits) - 1;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const uint8_t* cr = codes + (size_t)r * cols;
    auto val = [&](int c) {
      const size_t bi = (size_t)r * nblk + c / block;
      return dequant_exact(cr[c], bscale[bi], bzp[bi]);
    };
    float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
    for (int c = threadIdx.x; c < cols; c += XT) {
      const float v = val(c);
      lo = fminf(lo, v);
      hi = fmaxf(hi, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = lo;
      red[1][threadIdx.x >> 5] = hi;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < XT / 32; ++w) {
        lo = fminf(lo, red[0][w]);
        hi = fmaxf(hi, red[1][w]);
      }
      const float v0 = val(0);
      if (v0 != v0) lo = hi = v0;  // column 0's NaN sticks (tensor.hpp:133-148)
      float s;
      int32_t z;
      if (!affine_from_bounds(lo, hi, bits, s, z)) {
        atomicOr(err, 1u);
        s = 1.0f;
        z = 0;
      }
      scale[r] = s;
      zp[r] = z;
      prm[0] = s;
      prm[1] = __int_as_float(z);
    }
    __syncthreads();
    const float s = prm[0];
    const int32_t z = __float_as_int(prm[1]);
    for (int c = threadIdx.x; c < cols; c += XT)
      out[(size_t)r * cols + c] = (uint8_t)quant_exact(val(c), s, z, qmax);
    __syncthreads();
  }
}

int grid_for(long long n) {
  long long g = (n + XT - 1) / XT;
  return (int)(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}
}  // namespace

cudaError_t launch_pack_codes(const uint8_t* src, int rows, int cols, int bits, uint8_t* dst,
                              bool unpack, cudaStream_t st) {
  const long long n = (long long)rows * ((cols + 7) / 8);
  if (unpack) k_unpack_codes<<<grid_for(n), XT, 0, st>>>(src, rows, cols, bits, dst);
  else k_pack_codes<<<grid_for(n), XT, 0, st>>>(src, rows, cols, bits, dst);
  return cudaGetLastError();
}

cudaError_t launch_mom_blocks(const uint8_t* codes, const float* scale, const int32_t* zp,
                              int rows, int cols, int bits, int block, uint8_t* out,
                              float* oscale, int32_t* ozp, bool from_blocks, uint32_t* err,
                              cudaStream_t st) {
  if (from_blocks) {
    const int g = rows < 148 * 8 ? rows : 148 * 8;
    k_mom_from_blocks<<<g, XT, 0, st>>>(codes, scale, zp, rows, cols, bits, block, out, oscale,
                                        ozp, err);
  } else {
    const long long n = (long long)rows * ((cols + block - 1) / block);
    k_mom_to_blocks<<<grid_for(n), XT, 0, st>>>(codes, scale, zp, rows, cols, bits, block, out,
                                                oscale, ozp, err);
  }
  return cudaGetLastError();
}

}  // namespace qftk
