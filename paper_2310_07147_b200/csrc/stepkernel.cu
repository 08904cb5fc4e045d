// stepkernel.cu -- the fused quantized Lion step (sm_100a), v5: one WARP per row.
//
// Reference: the loop body of lion_step_quantized, optimizer.hpp:103-118 -- dequant g,
// m, reconstruct w -> lion_apply -> quantize_state(m') -> requantize_weight(w')
// against the cached thresholds (quantize.hpp:253-290).  Every quantity of the update
// is per ROW (scales, zero points, thresholds, the m' min/max, the CSR segment), so a
// warp can own a row end to end: its reductions are warp shuffles, its CSR prefix is
// a warp scan, and no CTA barrier exists anywhere in the step.  The 4 warps of a CTA
// only share the SM; each has its own slice of shared memory:
//
//   ring   R slots x (w | m | g) chunks of 32 x 16 codes (one 16-byte vector per
//          lane), filled by TMA 1-D bulk copies (cp.async.bulk -> UBLKCP) and
//          completed on a per-slot mbarrier.  Lane 0 keeps R chunks in flight ahead
//          of the consumer across row boundaries (its own cursor over the warp's
//          rows); a chunk's slot is refilled as soon as the warp has consumed it.
//   bitmaps of the row's old outliers (and of those that stay outliers), the first
//          rank per 32-column word (O(1) rank lookup), the sparse results, and a
//          per-lane parking slot for the w' values of a vector that holds outliers.
//
// Per row:
//   sparse pass   one lane per OLD outlier: its exact w' (the general Lion form),
//                 its class against the cached thresholds and its code;
//   pass 1        per chunk: dequant w/m/g (PRMT magic numbers, FMUL2) -> Lion ->
//                 outlier test -> payload select -> quantize -> STG.128 of W codes;
//                 m' min/max (FMNMX3); the chunk's outliers are appended to the row's
//                 CSR slot right away (warp scan of the per-lane counts);
//   row end       shuffle-reduce of the m' range, params in fp64 by lane 0
//                 (affine_params_from_bounds), old-outlier codes patched;
//   pass 2        per chunk (m and g re-streamed through the ring, L2-resident):
//                 m' recomputed -> quantized -> STG.128.
//
// Fast rows.  Whether the cheap arithmetic is exact is decided once per ROW: a row is
// "fast" when its zero points are small enough for the fp32 magic-number forms, its
// thresholds map to codes inside [0, qmax] (so every inlier, and the payload,
// quantizes without the clip -- only the tie distance is checked), and its old
// outliers fit the sparse table.  With weight decay 0 and bounded, not-too-small m
// and g scales the Lion sign update takes the saturating-FMA form (lion2_sat).  Other
// rows run the general code (per-vector exactness + range checks, exact fp64
// fallbacks).  Both produce the reference's bytes.
#include "qft_device.cuh"
#include "qft_internal.h"

#include <cstdio>

namespace qftk {
using namespace qftd;

namespace ws {
constexpr int NW = 4;          // warps per CTA (independent)
constexpr int R = 4;           // ring depth: chunks in flight per warp
constexpr int VB = 32 * 16;    // bytes of one u8 chunk
constexpr int F_FAST = 1;      // fast dequant of w/m/g, w codes range-proven, sparse table fits
constexpr int F_LSAT = 2;      // Lion sign update by saturating FMA (weight decay 0)

__host__ __device__ inline int r16(int x) { return (x + 15) & ~15; }

// per-row metadata of the warp's current block (loaded lane-parallel)
struct RowMeta {
  float sw, tmin, tmax, sm, sg;
  int32_t zw, zm, zg, ob, on, so, co, flags, _p[3];
};

struct WLayout {
  int cp, oldcap, gk;
  __host__ __device__ int gel() const { return gk == G_U8 ? 1 : (gk == G_F32 ? 4 : 2); }
  __host__ __device__ int slot_bytes() const { return VB * (2 + gel()); }  // w | m | g
  __host__ __device__ int words() const { return (cp + 31) / 32; }
  __host__ __device__ int o_bits() const { return R * slot_bytes(); }
  __host__ __device__ int o_bout() const { return o_bits() + r16(words() * 4); }
  __host__ __device__ int o_frank() const { return o_bout() + r16(words() * 4); }
  __host__ __device__ int o_sp() const { return o_frank() + r16(words() * 2); }   // val|cw|col
  __host__ __device__ int o_park() const { return o_sp() + r16(12 * oldcap); }
  __host__ __device__ int o_meta() const { return o_park() + 32 * 64; }
  __host__ __device__ int o_bar() const { return o_meta() + kBlockRows * (int)sizeof(RowMeta); }
  __host__ __device__ int warp_bytes() const { return o_bar() + 8 * R; }
  __host__ __device__ size_t total() const { return 128 + (size_t)NW * warp_bytes(); }
};

// the producer's position in the warp's row sequence
struct Cursor {
  int blk, j, nrows, row0, tensor;
};
}  // namespace ws

int step_kernel_max_cols() { return 65536; }

size_t step_kernel_smem(int gk, int cols_p, int oldcap) {
  ws::WLayout L{cols_p, oldcap, gk};
  return L.total();
}

namespace {

__device__ __forceinline__ uint32_t skbits16(const uint32_t* bits, int v) {
  return (bits[v >> 1] >> ((v & 1) * 16)) & 0xFFFFu;
}

__device__ __forceinline__ int sk_rank(const uint32_t* bits, const uint16_t* frank, int col) {
  const int w = col >> 5;
  return (int)frank[w] + __popc(bits[w] & ((1u << (col & 31)) - 1u));
}

template <int GK>
__device__ __forceinline__ float sk_graw(const uint8_t* gdata, int idx) {
  if (GK == G_F32) return reinterpret_cast<const float*>(gdata)[idx];
  const uint16_t b = reinterpret_cast<const uint16_t*>(gdata)[idx];
  return __uint_as_float((uint32_t)b << 16);
}

__device__ __forceinline__ float sk_deq1(uint32_t code, const DequantRow& d) {
  return d.fast ? __fmul_rn(__fadd_rn(magic_byte(code, 0), d.negc), d.s)
                : dequant_exact(code, d.s, d.z);
}

// fast-form dequant of 16 codes (the row is proven fast: no per-call branch)
__device__ __forceinline__ void sk_deq16(const uint4 q, const DequantRow& d, float* o) {
  const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 a = make_float2(magic_byte(wv[i], 0), magic_byte(wv[i], 1));
    float2 b = make_float2(magic_byte(wv[i], 2), magic_byte(wv[i], 3));
    a = mul2(add2(a, f2(d.negc)), f2(d.s));
    b = mul2(add2(b, f2(d.negc)), f2(d.s));
    o[4 * i] = a.x; o[4 * i + 1] = a.y; o[4 * i + 2] = b.x; o[4 * i + 3] = b.y;
  }
}

__device__ __forceinline__ void sk_deq16g(const uint4 q, const DequantRow& d, float* o) {
  dequant4(q.x, d, o); dequant4(q.y, d, o + 4); dequant4(q.z, d, o + 8); dequant4(q.w, d, o + 12);
}

__device__ __forceinline__ uint32_t sk_nib_mask(uint32_t nib) {
  return ((nib * 0x00204081u) & 0x01010101u) * 0xFFu;
}

__device__ __forceinline__ void sk_minmax16(const float* m, float& lo, float& hi) {
#pragma unroll
  for (int pp = 0; pp < 8; ++pp) {
    float tt;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(tt) : "f"(lo), "f"(m[2 * pp]), "f"(m[2 * pp + 1]));
    lo = tt;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(tt) : "f"(hi), "f"(m[2 * pp]), "f"(m[2 * pp + 1]));
    hi = tt;
  }
}

// quantize_state(g) -> dequantize of 16 raw gradient values (gradflow.hpp:77)
template <int GK>
__device__ __forceinline__ void sk_graw16(const uint8_t* gl, int nvalid, const QuantRow& qg,
                                          const DequantRow& dg, float* g) {
  float graw[16];
#pragma unroll
  for (int e = 0; e < 16; ++e) graw[e] = (e < nvalid) ? sk_graw<GK>(gl, e) : 0.0f;
  float em = 0.0f;
  uint32_t gc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) gc[q] = quant4_fast(graw + 4 * q, qg, em);
  if (!qg.fast || !(em < qg.thr)) {
#pragma unroll
    for (int q = 0; q < 4; ++q) gc[q] = quant4_exact(graw + 4 * q, qg);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) dequant4(gc[q], dg, g + 4 * q);
}

// The row-level proof for the fast path (see the file header); fp64 where the
// reference is fp64.  Evaluated lane-parallel once per row block.
template <int GK, bool ALIGNED, bool WD0>
__device__ __forceinline__ int sk_row_flags(float sw, int32_t zw, float tmin, float tmax,
                                            float sm, int32_t zm, float sg, int32_t zg, int on,
                                            int bit_width, int oldcap, const LaunchArgs& a) {
  if (GK != G_U8 || !ALIGNED) return 0;
  const int qmax = (1 << bit_width) - 1;
  const QuantRow qw = make_quant_row(sw, zw, bit_width);
  bool ok = qw.fast && make_dequant_row(sm, zm).fast && make_dequant_row(sg, zg).fast &&
            on <= oldcap;
  // bounded dense w (and w +- lr): no overflow in the update
  ok = ok && (__fmul_rn(fabsf(sw), (float)qmax + fabsf((float)zw)) < 0x1.0p126f) &&
       fabsf(a.lr) <= 0x1.0p100f;
  // every inlier v in [t_min, t_max] and the payload quantize inside [0, qmax]
  ok = ok && (tmin <= tmax) && code_unclamped(tmin, sw, zw) >= 0.0 &&
       code_unclamped(tmax, sw, zw) <= (double)qmax;
  int f = ok ? ws::F_FAST : 0;
  if (ok && WD0) {
    const double c1 = (double)__fsub_rn(1.0f, a.b1);
    const double bm = (double)sm * ((double)qmax + fabs((double)zm));
    const double bg = (double)sg * ((double)qmax + fabs((double)zg));
    const double pm = fabs((double)a.b1) * (double)sm;  // smallest non-zero |b1*m|
    const double pg = fabs(c1) * (double)sg;            // smallest non-zero |c1*g|
    const bool lsat = sm > 0.0f && sg > 0.0f && bm <= 0x1.0p120 && bg <= 0x1.0p120 &&
                      fabs((double)a.b1) <= 4.0 && fabs(c1) <= 4.0 &&
                      (a.b1 == 0.0f || pm >= 0x1.0p-100) && (c1 == 0.0 || pg >= 0x1.0p-100);
    if (lsat) f |= ws::F_LSAT;
  }
  return f;
}

}  // namespace

template <int GK, bool ALIGNED, bool WD0>
__global__ void __launch_bounds__(ws::NW * 32, QFT_STEP_MIN_CTAS) step_kernel(const LaunchArgs a) {
  using namespace ws;
  extern __shared__ __align__(128) uint8_t smem[];
  const WLayout L{a.cols_p, a.oldcap, GK};
  const int oldcap = L.oldcap;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const unsigned FULL = 0xffffffffu;
  uint8_t* wsm = smem + 128 + (size_t)wid * L.warp_bytes();
  uint8_t* ring = wsm;
  uint32_t* obits = reinterpret_cast<uint32_t*>(wsm + L.o_bits());
  uint32_t* obout = reinterpret_cast<uint32_t*>(wsm + L.o_bout());
  uint16_t* frank = reinterpret_cast<uint16_t*>(wsm + L.o_frank());
  float* sp_val = reinterpret_cast<float*>(wsm + L.o_sp());
  uint32_t* sp_cw = reinterpret_cast<uint32_t*>(wsm + L.o_sp() + 4 * oldcap);
  int32_t* sp_col = reinterpret_cast<int32_t*>(wsm + L.o_sp() + 8 * oldcap);
  float4* park = reinterpret_cast<float4*>(wsm + L.o_park());
  uint64_t* bars = reinterpret_cast<uint64_t*>(wsm + L.o_bar());
  RowMeta* meta = reinterpret_cast<RowMeta*>(wsm + L.o_meta());
  const int sbytes = L.slot_bytes();
  const int gel = L.gel();
  const int qmax = (1 << a.bit_width) - 1;
  const int in = a.flip, out = 1 - a.flip;
  const int gwarp = blockIdx.x * NW + wid;
  const int nwarps = gridDim.x * NW;
  constexpr int P0 = (GK == G_U8) ? 1 : 0;  // first pass (raw kinds: a g-range pass 0)
  // the row list of the rows kernel's general tier has a device-side length
  const int n_blocks = a.n_blocks_dev ? *a.n_blocks_dev : a.n_blocks;
  if (a.xseen && gwarp == 0 && lane == 0) *reinterpret_cast<volatile int32_t*>(a.xseen) = n_blocks;
  if (gwarp >= n_blocks) return;  // whole warp idle (warps are independent)

  if (lane == 0) {
    for (int s = 0; s < R; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncwarp();

  Hyper h;
  h.lr = a.lr; h.b1 = a.b1; h.b2 = a.b2; h.wd = a.wd;
  h.c1 = __fsub_rn(1.0f, a.b1);
  h.c2 = __fsub_rn(1.0f, a.b2);

  // ------------------------------------------------------------------ producer
  // (warp-uniform state; lane 0 issues the copies)
  Cursor pc{gwarp, 0, 0, 0, 0};
  int p_pass = P0, p_c = 0, p_nit = 0, p_off = 0, p_last = 0;
  const uint8_t *p_w = nullptr, *p_m = nullptr, *p_g = nullptr;
  bool p_live = false;
  int p_slot = 0;
  auto p_row = [&]() {  // enter the producer's current row (pc.j < pc.nrows)
    const DevTensor* Tt = a.tensors + pc.tensor;
    const int p_cols = Tt->cols;
    p_nit = (p_cols + VB - 1) / VB;
    p_last = p_cols - (p_nit - 1) * VB;  // bytes of the row's last chunk
    p_off = 0;
    const size_t roff = (size_t)(pc.row0 + pc.j) * (size_t)p_cols;
    p_w = Tt->w_codes[in] + roff;
    p_m = Tt->m_codes[in] + roff;
    p_g = (GK == G_U8) ? Tt->g_codes + roff
                       : reinterpret_cast<const uint8_t*>(Tt->g_raw) + (size_t)gel * roff;
    p_pass = P0;
    p_c = 0;
  };
  auto p_block = [&]() {  // enter block pc.blk (or finish)
    if (pc.blk >= n_blocks) {
      p_live = false;
      return;
    }
    const RowBlock B = a.blocks[pc.blk];
    pc.nrows = B.nrows;
    pc.row0 = B.row0;
    pc.tensor = B.tensor;
    pc.j = 0;
    p_live = true;
    p_row();
  };
  auto produce = [&]() {
    if (!p_live) return;
    const int s = p_slot;
    p_slot = (p_slot + 1) & (R - 1);
    uint8_t* sl = ring + s * sbytes;
    const bool last = (p_c + 1 == p_nit);
    const int nb = last ? p_last : VB;  // bytes of this chunk per u8 array
    const int b0 = p_off;
    const bool lw = (p_pass == 1), lm = (p_pass >= 1);
    if (ALIGNED) {
      if (lane == 0) {
        const uint32_t tx = (lw ? nb : 0) + (lm ? nb : 0) + nb * gel;
        mbar_arrive_expect_tx(&bars[s], tx);
        if (lw) bulk_g2s(sl, p_w + b0, nb, &bars[s]);
        if (lm) bulk_g2s(sl + VB, p_m + b0, nb, &bars[s]);
        bulk_g2s(sl + 2 * VB, p_g + (size_t)gel * b0, nb * gel, &bars[s]);
      }
    } else {
      for (int i = lane; i < nb; i += 32) {
        if (lw) sl[i] = p_w[b0 + i];
        if (lm) sl[VB + i] = p_m[b0 + i];
      }
      for (int i = lane; i < nb * gel; i += 32) sl[2 * VB + i] = p_g[(size_t)gel * b0 + i];
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars[s]);
    }
    // advance: chunk -> pass -> row -> block
    p_off += VB;
    ++p_c;
    if (last) {
      p_c = 0;
      p_off = 0;
      if (++p_pass > 2) {
        if (++pc.j < pc.nrows) {
          p_row();
        } else {
          pc.blk += nwarps;
          p_block();
        }
      }
    }
  };

  p_block();
  for (int i = 0; i < R; ++i) produce();

  // ------------------------------------------------------------------ consumer
  int c_slot = 0;
  uint32_t c_phase = 0;
  auto acquire = [&]() -> const uint8_t* {  // wait for the next chunk; returns its slot
    mbar_wait(&bars[c_slot], c_phase);
    return ring + c_slot * sbytes;
  };
  auto release = [&]() {  // the warp is done with the chunk: refill its slot
    __syncwarp();
    c_slot = (c_slot + 1) & (R - 1);
    c_phase ^= (c_slot == 0) ? 1u : 0u;
    produce();
  };

  for (int blk = gwarp; blk < n_blocks; blk += nwarps) {
    const RowBlock B = a.blocks[blk];
    const DevTensor* Tt = a.tensors + B.tensor;
    const int cols = Tt->cols;
    const int nvec = (cols + 15) >> 4;
    const int nit = (nvec + 31) >> 5;
    // lane-parallel row metadata of the block (lane j = row j) + the fast-path proof
    if (lane < B.nrows) {
      const int r = B.row0 + lane;
      RowMeta mt;
      mt.sw = Tt->w_scale[r];
      mt.zw = Tt->w_zp[r];
      mt.tmin = Tt->t_min[r];
      mt.tmax = Tt->t_max[r];
      mt.sm = Tt->m_scale[in][r];
      mt.zm = Tt->m_zp[in][r];
      mt.sg = (GK == G_U8) ? Tt->g_scale[r] : 0.0f;
      mt.zg = (GK == G_U8) ? Tt->g_zp[r] : 0;
      const int32_t* rs = Tt->rs[in];
      mt.ob = rs[r];
      const int cap_in = rs[r + 1] - mt.ob;
      mt.on = Tt->cnt[in] ? min(Tt->cnt[in][r], cap_in) : cap_in;
      mt.so = Tt->rs[out][r];
      mt.co = Tt->rs[out][r + 1] - mt.so;
      mt.flags = sk_row_flags<GK, ALIGNED, WD0>(mt.sw, mt.zw, mt.tmin, mt.tmax, mt.sm, mt.zm,
                                                mt.sg, mt.zg, mt.on, a.bit_width, oldcap, a);
      meta[lane] = mt;
    }
    __syncwarp();

    for (int j = 0; j < B.nrows; ++j) {
      const int lrow = B.row0 + j;
      const RowMeta& mt = meta[j];
      const float sw = mt.sw, tmin = mt.tmin, tmax = mt.tmax, smi = mt.sm, sgi = mt.sg;
      const int zw = mt.zw, zmi = mt.zm, zgi = mt.zg, ob = mt.ob, old_n = mt.on;
      const int slot_out = mt.so, cap_out = mt.co, flags = mt.flags;
      const bool fast = (GK == G_U8) && ALIGNED && (flags & F_FAST);
      const size_t roff = (size_t)lrow * (size_t)cols;
      uint8_t* w_out = Tt->w_codes[out] + roff;
      uint8_t* m_out = Tt->m_codes[out] + roff;
      const uint8_t* m_in_row = Tt->m_codes[in] + roff;
      const uint8_t* g_in_row = (GK == G_U8) ? Tt->g_codes + roff
                                             : reinterpret_cast<const uint8_t*>(Tt->g_raw) +
                                                   (size_t)gel * roff;

      const DequantRow dw = make_dequant_row(sw, zw);
      const DequantRow dm = make_dequant_row(smi, zmi);
      DequantRow dg = make_dequant_row(sgi, zgi);
      QuantRow qg{};
      const QuantRow qw = make_quant_row(sw, zw, a.bit_width);
      const int zpay = zw < 0 ? 0 : (zw > qmax ? qmax : zw);
      const uint32_t zpay4 = (uint32_t)zpay * 0x01010101u;
      const float wz = __fmul_rn(sw, (float)(zpay - zw));
      const bool w_ovf = !(__fmul_rn(fabsf(sw), (float)qmax + fabsf((float)zw)) < 3.0e38f);
      const bool sparse_ok = old_n <= oldcap;

      // ---- raw-gradient kinds: pass 0 = the row's g range -> quantize_state params
      if (GK != G_U8) {
        float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
        int nan0 = 0;
        for (int c = 0; c < nit; ++c) {
          const uint8_t* sl = acquire();
          const int v = c * 32 + lane;
          if (v < nvec) {
            const uint8_t* gl = sl + 2 * VB + lane * 16 * gel;
            const int nvalid = min(16, cols - v * 16);
            for (int e = 0; e < nvalid; ++e) {
              const float x = sk_graw<GK>(gl, e);
              lo = fminf(lo, x);
              hi = fmaxf(hi, x);
            }
            if (v == 0 && isnan(sk_graw<GK>(gl, 0))) nan0 = 1;
          }
          release();
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lo = fminf(lo, __shfl_xor_sync(FULL, lo, o));
          hi = fmaxf(hi, __shfl_xor_sync(FULL, hi, o));
          nan0 |= __shfl_xor_sync(FULL, nan0, o);
        }
        if (nan0) lo = hi = __int_as_float(0x7fc00000);
        float sgv = 1.0f;
        int32_t zgv = 0;
        if (lane == 0 && !affine_from_bounds(lo, hi, a.bit_width, sgv, zgv)) {
          atomicOr(&a.hdr->err, ERR_GPARAMS);
          sgv = 1.0f;
          zgv = 0;
        }
        sgv = __shfl_sync(FULL, sgv, 0);
        zgv = __shfl_sync(FULL, zgv, 0);
        qg = make_quant_row(sgv, zgv, a.bit_width);
        dg = make_dequant_row(sgv, zgv);
      }

      // ---- sparse pass over the OLD outliers
      for (int i = lane; i < L.words(); i += 32) {
        obits[i] = 0u;
        obout[i] = 0u;
      }
      __syncwarp();
      for (int i = lane; i < old_n; i += 32) {
        const int col = a.col_in[ob + i];
        const int wd = col >> 5;
        atomicOr(&obits[wd], 1u << (col & 31));
        const int prev = (i == 0) ? -1 : a.col_in[ob + i - 1];
        if (i == 0 || (prev >> 5) != wd) frank[wd] = (uint16_t)i;
        if (sparse_ok) {
          // exact w' (lion1, general form), class and code of this element
          // (quantize.hpp:274-285)
          float wv = a.val_in[ob + i];
          float mv = sk_deq1(m_in_row[col], dm);
          float gv;
          if (GK == G_U8) gv = sk_deq1(g_in_row[col], dg);
          else gv = sk_deq1(quant_exact(sk_graw<GK>(g_in_row, col), qg.s, qg.z, qg.qmax), dg);
          lion1(wv, mv, gv, h);
          const bool o = (wv < tmin) || (wv > tmax);
          const uint32_t code = o ? (uint32_t)zpay : quant_exact(wv, qw.s, qw.z, qw.qmax);
          sp_val[i] = wv;
          sp_cw[i] = code | (o ? 0x100u : 0u);
          sp_col[i] = col;
          if (o) atomicOr(&obout[wd], 1u << (col & 31));
        }
      }
      __syncwarp();

      // ================================ pass 1 ================================
      float mlo = __int_as_float(0x7f800000), mhi = __int_as_float(0xff800000);
      int mnan0 = 0;
      int base = 0;  // CSR entries of the row emitted so far
      const bool lsat = WD0 && (flags & F_LSAT);
      for (int c = 0; c < nit; ++c) {
        const uint8_t* sl = acquire();
        const int v = c * 32 + lane;
        uint32_t mask = 0, dense_new = 0, o16 = 0;
        float w[16];
        if (v < nvec) {
          const uint4 wq = *reinterpret_cast<const uint4*>(sl + lane * 16);
          const uint4 mq = *reinterpret_cast<const uint4*>(sl + VB + lane * 16);
          float m[16], g[16];
          o16 = skbits16(obits, v);
          if (fast) {
            // ---- fast rows: branch-free dequant, range-proven quantizer; old outliers
            // are excluded here (their codes are patched at the row end)
            const uint4 gq = *reinterpret_cast<const uint4*>(sl + 2 * VB + lane * 16);
            sk_deq16(wq, dw, w);
            sk_deq16(mq, dm, m);
            sk_deq16(gq, dg, g);
            if (lsat) {
#pragma unroll
              for (int pp = 0; pp < 8; ++pp) {
                float2 W = make_float2(w[2 * pp], w[2 * pp + 1]);
                float2 M = make_float2(m[2 * pp], m[2 * pp + 1]);
                lion2_sat(W, M, make_float2(g[2 * pp], g[2 * pp + 1]), h);
                w[2 * pp] = W.x; w[2 * pp + 1] = W.y;
                m[2 * pp] = M.x; m[2 * pp + 1] = M.y;
              }
            } else if (WD0) {
#pragma unroll
              for (int pp = 0; pp < 8; ++pp) {
                float2 W = make_float2(w[2 * pp], w[2 * pp + 1]);
                float2 M = make_float2(m[2 * pp], m[2 * pp + 1]);
                lion2_wd0(W, M, make_float2(g[2 * pp], g[2 * pp + 1]), h);
                w[2 * pp] = W.x; w[2 * pp + 1] = W.y;
                m[2 * pp] = M.x; m[2 * pp + 1] = M.y;
              }
            } else {
#pragma unroll
              for (int pp = 0; pp < 8; ++pp) {
                float2 W = make_float2(w[2 * pp], w[2 * pp + 1]);
                float2 M = make_float2(m[2 * pp], m[2 * pp + 1]);
                lion2(W, M, make_float2(g[2 * pp], g[2 * pp + 1]), h);
                w[2 * pp] = W.x; w[2 * pp + 1] = W.y;
                m[2 * pp] = M.x; m[2 * pp + 1] = M.y;
              }
            }
            sk_minmax16(m, mlo, mhi);
            float wq2[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) wq2[e] = outlier_select(w[e], tmin, tmax, wz, 1u << e, mask);
            float em = 0.0f;
            uint32_t cq[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) cq[q] = quant4_e(wq2 + 4 * q, qw, em);
            if (!(em < qw.thr)) {
#pragma unroll
              for (int q = 0; q < 4; ++q) cq[q] = quant4_exact(wq2 + 4 * q, qw);
            }
            *reinterpret_cast<uint4*>(w_out + v * 16) = make_uint4(cq[0], cq[1], cq[2], cq[3]);
            dense_new = mask & ~o16;
            mask = dense_new | skbits16(obout, v);
          } else {
            // ---- general rows: per-vector proofs with exact fallbacks
            const int nvalid = min(16, cols - v * 16);
            const uint32_t valid = nvalid >= 16 ? 0xFFFFu : ((1u << nvalid) - 1u);
            sk_deq16g(wq, dw, w);
            sk_deq16g(mq, dm, m);
            if (GK == G_U8) sk_deq16g(*reinterpret_cast<const uint4*>(sl + 2 * VB + lane * 16), dg, g);
            else sk_graw16<GK>(sl + 2 * VB + lane * 16 * gel, nvalid, qg, dg, g);
            // rows with more old outliers than the sparse table patch w before the update
            uint32_t op = sparse_ok ? 0u : o16;
            bool wspecial = w_ovf;
            while (op) {
              const int e = __ffs(op) - 1;
              op &= op - 1u;
              const float val = a.val_in[ob + sk_rank(obits, frank, v * 16 + e)];
              wspecial |= !isfinite(val);
#pragma unroll
              for (int q = 0; q < 16; ++q) w[q] = (q == e) ? val : w[q];
            }
            if (WD0 && !wspecial) {
#pragma unroll
              for (int pp = 0; pp < 8; ++pp) {
                float2 W = make_float2(w[2 * pp], w[2 * pp + 1]);
                float2 M = make_float2(m[2 * pp], m[2 * pp + 1]);
                lion2_wd0(W, M, make_float2(g[2 * pp], g[2 * pp + 1]), h);
                w[2 * pp] = W.x; w[2 * pp + 1] = W.y;
                m[2 * pp] = M.x; m[2 * pp + 1] = M.y;
              }
            } else {
#pragma unroll
              for (int pp = 0; pp < 8; ++pp) {
                float2 W = make_float2(w[2 * pp], w[2 * pp + 1]);
                float2 M = make_float2(m[2 * pp], m[2 * pp + 1]);
                lion2(W, M, make_float2(g[2 * pp], g[2 * pp + 1]), h);
                w[2 * pp] = W.x; w[2 * pp + 1] = W.y;
                m[2 * pp] = M.x; m[2 * pp + 1] = M.y;
              }
            }
            if (v == 0 && isnan(m[0])) mnan0 = 1;
            if (valid != 0xFFFFu) {
#pragma unroll
              for (int e = 1; e < 16; ++e)
                if (!(valid & (1u << e))) m[e] = m[0];
            }
            sk_minmax16(m, mlo, mhi);
            float wq2[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) wq2[e] = outlier_select(w[e], tmin, tmax, wz, 1u << e, mask);
            mask &= valid;
            QAcc qa = qacc_init();
            uint32_t cq[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) cq[q] = quant4_nc(wq2 + 4 * q, qw, qa);
            if (!quant_vec_ok(qa, qw)) {
#pragma unroll
              for (int q = 0; q < 4; ++q) cq[q] = quant4_exact(w + 4 * q, qw);
              if (mask) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const uint32_t bm = sk_nib_mask((mask >> (4 * q)) & 0xFu);
                  cq[q] = (cq[q] & ~bm) | (zpay4 & bm);
                }
              }
            }
            if (sparse_ok && o16) {
              // old-outlier elements: class and code from the sparse pass
              uint32_t obm = o16 & valid;
              while (obm) {
                const int e = __ffs(obm) - 1;
                obm &= obm - 1u;
                const uint32_t cw = sp_cw[sk_rank(obits, frank, v * 16 + e)];
                mask = (mask & ~(1u << e)) | (((cw >> 8) & 1u) << e);
                const uint32_t sh = (uint32_t)(e & 3) * 8u;
                const uint32_t keep = ~(0xFFu << sh), put = (cw & 0xFFu) << sh;
                const int q = e >> 2;
                cq[0] = (q == 0) ? ((cq[0] & keep) | put) : cq[0];
                cq[1] = (q == 1) ? ((cq[1] & keep) | put) : cq[1];
                cq[2] = (q == 2) ? ((cq[2] & keep) | put) : cq[2];
                cq[3] = (q == 3) ? ((cq[3] & keep) | put) : cq[3];
              }
            }
            uint8_t* wo = w_out + v * 16;
            if (ALIGNED) {
              *reinterpret_cast<uint4*>(wo) = make_uint4(cq[0], cq[1], cq[2], cq[3]);
            } else {
              for (int e = 0; e < nvalid; ++e) wo[e] = (uint8_t)(cq[e >> 2] >> ((e & 3) * 8));
            }
            dense_new = sparse_ok ? (mask & ~o16) : mask;
            if (!sparse_ok) o16 = 0;  // old-origin values come from w' (patched) here
          }
        }
        release();  // the chunk's codes are in registers / stored
        // ---- append this chunk's outliers to the row's CSR slot (columns ascending)
        const int cnt = __popc(mask);
        int incl = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int tt = __shfl_up_sync(FULL, incl, d);
          if (lane >= d) incl += tt;
        }
        const int total = __shfl_sync(FULL, incl, 31);
        if (mask) {
          int pos = base + incl - cnt;
          if (dense_new) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              park[q * 32 + lane] = make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
          }
          const float* pk = reinterpret_cast<const float*>(park);
          uint32_t mm = mask;
          while (mm) {
            const int e = __ffs(mm) - 1;
            mm &= mm - 1u;
            const int col = v * 16 + e;
            const float val = (o16 & (1u << e)) ? sp_val[sk_rank(obits, frank, col)]
                                                : pk[((e >> 2) * 32 + lane) * 4 + (e & 3)];
            if (pos < cap_out) {
              a.col_out[slot_out + pos] = col;
              a.val_out[slot_out + pos] = val;
            }
            ++pos;
          }
        }
        base += total;
      }

      // ---- row end: m' params (quantize_state: channel_minmax -> affine_params_from_bounds)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mlo = fminf(mlo, __shfl_xor_sync(FULL, mlo, o));
        mhi = fmaxf(mhi, __shfl_xor_sync(FULL, mhi, o));
        mnan0 |= __shfl_xor_sync(FULL, mnan0, o);
      }
      if (mnan0) mlo = mhi = __int_as_float(0x7fc00000);
      float smv = 1.0f;
      int32_t zmv = 0;
      int qmf = 0;
      if (lane == 0) {
        if (!affine_from_bounds(mlo, mhi, a.bit_width, smv, zmv)) {
          atomicOr(&a.hdr->err, ERR_MPARAMS);
          smv = 1.0f;
          zmv = 0;
        }
        // every m' lies in [lo, hi]: if those two codes need no clip, none does
        qmf = fast && make_quant_row(smv, zmv, a.bit_width).fast &&
              code_unclamped(mlo, smv, zmv) >= 0.0 && code_unclamped(mhi, smv, zmv) <= (double)qmax;
        Tt->m_scale[out][lrow] = smv;
        Tt->m_zp[out][lrow] = zmv;
        Tt->cnt[out][lrow] = base;
        if (base > cap_out) {
          atomicOr(&a.hdr->overflow, 1u);
          if (a.oflag) *reinterpret_cast<volatile uint32_t*>(a.oflag) = 1u;
        }
      }
      smv = __shfl_sync(FULL, smv, 0);
      zmv = __shfl_sync(FULL, zmv, 0);
      qmf = __shfl_sync(FULL, qmf, 0);
      const QuantRow qm = make_quant_row(smv, zmv, a.bit_width);

      // old-outlier codes of fast rows (pass 1 left payload-derived bytes there);
      // __syncwarp orders the warp's pass-1 vector stores before these byte stores
      if (fast) {
        __syncwarp();
        for (int i = lane; i < old_n; i += 32) w_out[sp_col[i]] = (uint8_t)(sp_cw[i] & 0xFFu);
      }

      // ================================ pass 2 ================================
      for (int c = 0; c < nit; ++c) {
        const uint8_t* sl = acquire();
        const int v = c * 32 + lane;
        if (v < nvec) {
          float m[16], g[16];
          const uint4 mq = *reinterpret_cast<const uint4*>(sl + VB + lane * 16);
          if (fast) {
            sk_deq16(mq, dm, m);
            sk_deq16(*reinterpret_cast<const uint4*>(sl + 2 * VB + lane * 16), dg, g);
          } else {
            sk_deq16g(mq, dm, m);
            if (GK == G_U8) sk_deq16g(*reinterpret_cast<const uint4*>(sl + 2 * VB + lane * 16), dg, g);
            else sk_graw16<GK>(sl + 2 * VB + lane * 16 * gel, min(16, cols - v * 16), qg, dg, g);
          }
#pragma unroll
          for (int pp = 0; pp < 8; ++pp) {
            const float2 M = sadd2(mul2(f2(h.b2), make_float2(m[2 * pp], m[2 * pp + 1])),
                                   mul2(f2(h.c2), make_float2(g[2 * pp], g[2 * pp + 1])));
            m[2 * pp] = M.x;
            m[2 * pp + 1] = M.y;
          }
          uint32_t cq[4];
          bool ok;
          if (qmf) {
            float em = 0.0f;
#pragma unroll
            for (int q = 0; q < 4; ++q) cq[q] = quant4_e(m + 4 * q, qm, em);
            ok = em < qm.thr;
          } else {
            QAcc qa = qacc_init();
#pragma unroll
            for (int q = 0; q < 4; ++q) cq[q] = quant4_nc(m + 4 * q, qm, qa);
            ok = quant_vec_ok(qa, qm);
          }
          if (!ok) {
#pragma unroll
            for (int q = 0; q < 4; ++q) cq[q] = quant4_exact(m + 4 * q, qm);
          }
          uint8_t* mo = m_out + v * 16;
          if (ALIGNED) {
            *reinterpret_cast<uint4*>(mo) = make_uint4(cq[0], cq[1], cq[2], cq[3]);
          } else {
            const int nvalid = min(16, cols - v * 16);
            for (int e = 0; e < nvalid; ++e) mo[e] = (uint8_t)(cq[e >> 2] >> ((e & 3) * 8));
          }
        }
        release();
      }
    }
  }
}

// ----------------------------------------------------------------------------
template <int GK, bool AL, bool WD0>
static cudaError_t step_resolve_t(const LaunchArgs& a, size_t smem, KLaunch* out) {
  auto k = step_kernel<GK, AL, WD0>;
  // the attribute is per FUNCTION, shared by every plan that launches this instance: raise
  // it to the device's opt-in maximum (never lower it to this plan's size, which would
  // invalidate another plan's cached launch); occupancy follows the launch's own smem
  int dev0 = 0, optin = 0;
  cudaGetDevice(&dev0);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev0);
  if ((size_t)optin < smem) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, ws::NW * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  long grid = (long)sms * per_sm;
  const long need = ((long)a.n_blocks + ws::NW - 1) / ws::NW;
  if (grid > need) grid = need;
  if (grid < 1) grid = 1;
  out->fn = reinterpret_cast<const void*>(k);
  out->grid = (int)grid;
  out->block = ws::NW * 32;
  out->smem = smem;
  snprintf(out->name, sizeof(out->name), "step_kernel<%d,%d,%d>", GK, AL ? 1 : 0, WD0 ? 1 : 0);
  return cudaSuccess;
}

cudaError_t resolve_step_kernel(int gk, const LaunchArgs& a, KLaunch* out) {
  const size_t smem = step_kernel_smem(gk, a.cols_p, a.oldcap);
  const bool al = a.use_bulk != 0;
  const bool wd0 = (a.wd == 0.0f);
#define SK_R(G)                                                                   \
  do {                                                                            \
    if (al) return wd0 ? step_resolve_t<G, true, true>(a, smem, out)              \
                       : step_resolve_t<G, true, false>(a, smem, out);            \
    return wd0 ? step_resolve_t<G, false, true>(a, smem, out)                     \
               : step_resolve_t<G, false, false>(a, smem, out);                   \
  } while (0)
  if (gk == G_U8) SK_R(G_U8);
  if (gk == G_F32) SK_R(G_F32);
  SK_R(G_BF16);
#undef SK_R
}

cudaError_t launch_step_kernel(int gk, const LaunchArgs& a, cudaStream_t st) {
  KLaunch k;
  cudaError_t e = resolve_step_kernel(gk, a, &k);
  if (e != cudaSuccess) return e;
  return launch_k(k, a, st);
}

}  // namespace qftk
