// crc32.cu -- the QFTC v1 checkpoint CRC (checkpoint.cpp:20-33: reflected polynomial
// 0xEDB88320, register preset 0xFFFFFFFF, final complement) over device-resident bytes.
//
// A checkpoint of the 7B state is ~14 GB, almost all of it device arrays (codes, CSR,
// per-row params), so the CRC is computed where the bytes live instead of on one host
// core.  The CRC register without preset/complement ("raw") is linear over GF(2):
//     raw(A || B) = X^(8|B|) * raw(A)  ^  raw(B)
// where X^(8n) is the 32x32 bit matrix "append n zero bytes".  Each warp takes one
// 64 KB chunk of a segment, each lane a 2 KB slice (table-driven, byte by byte; the
// table is replicated per lane in shared memory so lookups never bank-conflict); the
// 32 lane values are folded in a 5-level shuffle tree with the
// shift matrices for 2, 4, 8, 16, 32 KB.  A segment's short tail chunk leaves one
// value per 2 KB slice.  The host folds all values in order (fixed 64 KB / 2 KB
// matrices, a table of 2^k-byte shifts for the odd lengths) and applies the preset and
// complement once for the whole stream.
#include <algorithm>
#include <cstdint>
#include <vector>

#include "qft_internal.h"

namespace qftk {
namespace {

constexpr uint32_t kPoly = 0xEDB88320u;
constexpr int kLaneBytes = 2048;
constexpr int kChunk = 32 * kLaneBytes;  // 64 KB per warp

struct ShiftMats {
  uint32_t m[5][32];  // column j of "append 2 KB << k zero bytes", k = 0..4
};

struct ChunkJob {
  const uint8_t* p;
  int64_t len;   // <= kChunk; < kChunk only for a segment's last chunk
  int64_t oidx;  // first output slot: 1 for a full chunk, one per 2 KB slice for a tail
};

__device__ __forceinline__ uint32_t apply_mat(const uint32_t* m, uint32_t v) {
  uint32_t r = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j) r ^= ((v >> j) & 1u) ? m[j] : 0u;
  return r;
}

// The byte table, one copy per lane interleaved so that lane L's entry i sits at word
// 32*i + L: every lane reads its own bank, so the random table lookups are
// conflict-free (32 KB of shared memory per CTA).
constexpr int kCrcThreads = 512;
__global__ void __launch_bounds__(kCrcThreads) k_crc32_chunks(const ChunkJob* jobs, int n,
                                                              ShiftMats mats, uint32_t* out) {
  extern __shared__ uint32_t tab32[];  // [256][32]
  for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) {
    uint32_t c = (uint32_t)(i >> 5);
    for (int k = 0; k < 8; ++k) c = (c & 1u) ? kPoly ^ (c >> 1) : c >> 1;
    tab32[i] = c;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t* tab_l = tab32 + lane;
#define tab(i) tab_l[(i) << 5]
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += warps) {
    const ChunkJob J = jobs[w];
    if (J.len < kChunk) {  // a segment tail: one value per 2 KB slice, folded on the host
      const int64_t a = (int64_t)lane * kLaneBytes;
      if (a < J.len) {
        const int64_t b = std::min<int64_t>(J.len, a + kLaneBytes);
        uint32_t c = 0;
        for (int64_t i = a; i < b; ++i) c = tab((c ^ __ldg(J.p + i)) & 0xFFu) ^ (c >> 8);
        out[J.oidx + lane] = c;
      }
      continue;
    }
    const uint8_t* q = J.p + (int64_t)lane * kLaneBytes;
    uint32_t c = 0;
    if ((reinterpret_cast<uintptr_t>(q) & 15u) == 0) {
      // 16-byte loads, several in flight (the byte chain itself is short-latency LDS)
      const uint4* q16 = reinterpret_cast<const uint4*>(q);
#pragma unroll 4
      for (int i = 0; i < kLaneBytes / 16; ++i) {
        const uint4 x = __ldg(q16 + i);
        const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int b = 0; b < 4; ++b) c = tab((c ^ (w[k] >> (8 * b))) & 0xFFu) ^ (c >> 8);
      }
    } else if ((reinterpret_cast<uintptr_t>(q) & 3u) == 0) {
      const uint32_t* q4 = reinterpret_cast<const uint32_t*>(q);
#pragma unroll 8
      for (int i = 0; i < kLaneBytes / 4; ++i) {
        const uint32_t x = __ldg(q4 + i);
#pragma unroll
        for (int b = 0; b < 4; ++b) c = tab((c ^ (x >> (8 * b))) & 0xFFu) ^ (c >> 8);
      }
    } else {
      for (int i = 0; i < kLaneBytes; ++i) c = tab((c ^ __ldg(q + i)) & 0xFFu) ^ (c >> 8);
    }
    // fold: level k joins lane pairs 2^k apart; the left value shifts over the right
    // block of 2 KB << k bytes
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t right = __shfl_down_sync(0xffffffffu, c, 1 << k);
      if ((lane & ((2 << k) - 1)) == 0) c = apply_mat(mats.m[k], c) ^ right;
    }
    if (lane == 0) out[J.oidx] = c;
  }
#undef tab
}

// ---- host GF(2) helpers (zlib's crc32_combine construction)
uint32_t mat_times(const uint32_t* m, uint32_t v) {
  uint32_t r = 0;
  for (int j = 0; v; ++j, v >>= 1)
    if (v & 1u) r ^= m[j];
  return r;
}
void mat_square(uint32_t* sq, const uint32_t* m) {
  for (int j = 0; j < 32; ++j) sq[j] = mat_times(m, m[j]);
}
// matrix of "append n zero bytes" (n >= 1)
void shift_matrix(int64_t n, uint32_t* out) {
  uint32_t odd[32], even[32];
  odd[0] = kPoly;  // one zero BIT
  for (int j = 1; j < 32; ++j) odd[j] = 1u << (j - 1);
  mat_square(even, odd);  // 2 bits
  mat_square(odd, even);  // 4 bits
  // odd = 1 zero byte after the next squaring
  uint32_t res[32];
  for (int j = 0; j < 32; ++j) res[j] = 1u << j;
  bool first = true;
  uint32_t* cur = odd;
  uint32_t* nxt = even;
  mat_square(nxt, cur);  // 8 bits = 1 byte
  std::swap(cur, nxt);
  while (n) {
    if (n & 1) {
      if (first) {
        for (int j = 0; j < 32; ++j) res[j] = cur[j];
        first = false;
      } else {
        uint32_t t[32];
        for (int j = 0; j < 32; ++j) t[j] = mat_times(cur, res[j]);
        for (int j = 0; j < 32; ++j) res[j] = t[j];
      }
    }
    n >>= 1;
    if (n) {
      mat_square(nxt, cur);
      std::swap(cur, nxt);
    }
  }
  for (int j = 0; j < 32; ++j) out[j] = res[j];
}
// "append 2^k zero bytes" for k = 0..47: a shift by n costs one matrix-vector
// product per set bit of n
struct Pow2Shifts {
  uint32_t m[48][32];
  Pow2Shifts() {
    shift_matrix(1, m[0]);
    for (int k = 1; k < 48; ++k) mat_square(m[k], m[k - 1]);
  }
  uint32_t apply(uint32_t v, int64_t n) const {
    for (int k = 0; n && k < 48; ++k, n >>= 1)
      if (n & 1) v = mat_times(m[k], v);
    return v;
  }
};
const Pow2Shifts& pow2() {
  static const Pow2Shifts P;
  return P;
}
uint32_t shift_by(uint32_t v, int64_t n) { return n > 0 ? pow2().apply(v, n) : v; }
// a fixed shift as four 256-entry byte tables (the per-chunk host fold)
struct ByteMat {
  uint32_t t[4][256];
  explicit ByteMat(int64_t n) {
    uint32_t m[32];
    shift_matrix(n, m);
    for (int b = 0; b < 4; ++b)
      for (uint32_t x = 0; x < 256; ++x) t[b][x] = mat_times(m, x << (8 * b));
  }
  uint32_t operator()(uint32_t v) const {
    return t[0][v & 0xFFu] ^ t[1][(v >> 8) & 0xFFu] ^ t[2][(v >> 16) & 0xFFu] ^ t[3][v >> 24];
  }
};

}  // namespace

cudaError_t crc32_device(const void* const* segs, const int64_t* lens, int n, uint32_t* crc_out,
                         cudaStream_t st) {
  std::vector<ChunkJob> jobs;
  int64_t total = 0, nout = 0;
  for (int s = 0; s < n; ++s) {
    const uint8_t* p = static_cast<const uint8_t*>(segs[s]);
    for (int64_t o = 0; o < lens[s]; o += kChunk) {
      const int64_t len = std::min<int64_t>(kChunk, lens[s] - o);
      jobs.push_back(ChunkJob{p + o, len, nout});
      nout += len == kChunk ? 1 : (len + kLaneBytes - 1) / kLaneBytes;
    }
    total += lens[s];
  }
  uint32_t raw = 0;
  if (!jobs.empty()) {
    static const ShiftMats mats = [] {
      ShiftMats s;
      for (int k = 0; k < 5; ++k) shift_matrix((int64_t)kLaneBytes << k, s.m[k]);
      return s;
    }();
    ChunkJob* djobs = nullptr;
    uint32_t* dout = nullptr;
    cudaError_t e = cudaMallocAsync(&djobs, jobs.size() * sizeof(ChunkJob), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&dout, (size_t)nout * sizeof(uint32_t), st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(djobs, jobs.data(), jobs.size() * sizeof(ChunkJob),
                          cudaMemcpyHostToDevice, st);
    std::vector<uint32_t> vals((size_t)nout);
    if (e == cudaSuccess) {
      int dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int threads = kCrcThreads;
      const size_t smem = 256 * 32 * sizeof(uint32_t);
      const long want = ((long)jobs.size() * 32 + threads - 1) / threads;
      const int grid = (int)std::max(1L, std::min<long>(want, (long)sms * 4));
      k_crc32_chunks<<<grid, threads, smem, st>>>(djobs, (int)jobs.size(), mats, dout);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(vals.data(), dout, vals.size() * sizeof(uint32_t),
                          cudaMemcpyDeviceToHost, st);
    if (djobs) cudaFreeAsync(djobs, st);
    if (dout) cudaFreeAsync(dout, st);
    const cudaError_t es = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    if (es != cudaSuccess) return es;
    static const ByteMat full(kChunk), slice(kLaneBytes);
    for (const ChunkJob& J : jobs) {
      if (J.len == kChunk) {
        raw = full(raw) ^ vals[(size_t)J.oidx];
        continue;
      }
      for (int64_t a = 0, k = 0; a < J.len; a += kLaneBytes, ++k) {
        const int64_t l = std::min<int64_t>(kLaneBytes, J.len - a);
        raw = (l == kLaneBytes ? slice(raw) : shift_by(raw, l)) ^ vals[(size_t)(J.oidx + k)];
      }
    }
  }
  // preset 0xFFFFFFFF (its effect after `total` bytes) and the final complement
  *crc_out = raw ^ shift_by(0xFFFFFFFFu, total) ^ 0xFFFFFFFFu;
  return cudaSuccess;
}

}  // namespace qftk
