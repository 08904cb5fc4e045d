// stepkernel.cu -- the fused quantized Lion step (sm_100a), v4.
//
// One row (= one output channel) at a time per CTA of 4 warps; the whole row's
// per-channel work is row-local (scales, zero points, thresholds, the m' min/max,
// its CSR slot), so rows never wait on each other.  Reference: the loop body of
// lion_step_quantized, optimizer.hpp:103-118 (dequant g, m, reconstruct w ->
// lion_apply -> quantize_state(m') -> requantize_weight(w') against the cached
// thresholds, quantize.hpp:253-290).
//
// Pipeline (no producer warp): a ring of S >= 3 smem stages, each holding one row's
// context, w/m/g code rows and old CSR slot, filled by TMA 1-D bulk copies
// (cp.async.bulk -> UBLKCP) and completed on a per-stage mbarrier.  Row t-1's
// pass 2 still reads its stage after the row-t barrier, so warp 0 refills the
// stage of row t-2 there (with row t-2+S): S-2 rows of prefetch, no polling warp.  Rows come
// from a static round-robin list of 32-row blocks whose per-row metadata warp 0
// loads lane-parallel into smem once per block -- together with the row's
// FAST-PATH PROOF (below).
//
// Per row (128 threads, 16 elements = one 16-byte vector per thread-step):
//   sparse pass: one thread per OLD outlier computes its exact w' (the general
//     Lion form), its class against the cached thresholds and its code; bitmap +
//     first-rank table of the old outliers, bitmap of those that stay outliers;
//   barrier B0;
//   pass 1 over the dense vectors: dequant w/m/g (PRMT magic numbers, FMUL2) ->
//     Lion -> outlier test -> payload select -> quantize -> STG.128 of W codes;
//     m' row min/max (FMNMX3); vectors holding a new dense-origin outlier park
//     their 16 w' values in a per-thread smem slot;
//   barrier C; one thread derives the m' params in fp64 (affine_params_from_bounds)
//     while the others patch the old-outlier codes and write the row's CSR slot;
//   pass 2 runs ONE ROW LATE, after the next row's barrier B0 (which publishes the
//     params): m' (per-thread smem buffer, or recomputed from the still-resident
//     staged codes) -> quantize -> STG.  The fp64 param latency thus overlaps the
//     CSR phase and the next row's sparse pass instead of stalling a barrier.
//
// Fast rows.  Whether the cheap arithmetic is exact is decided once per ROW, not per
// element: a row is "fast" when its zero points are small enough for the fp32
// magic-number forms, its thresholds map to codes inside [0, qmax] (so every
// inlier, and the payload, quantizes without the clip -- only the tie distance is
// checked), and its old outliers fit the sparse table.  With weight decay 0 and
// bounded, not-too-small m and g scales the Lion sign update also takes the
// saturating-FMA form (lion2_sat, 3 FP ops/element).  Other rows run the general
// code (per-vector exactness + range checks, exact fp64 fallbacks).  Both produce
// the reference's bytes.
#include "qft_device.cuh"
#include "qft_internal.h"

namespace qftk {
using namespace qftd;

namespace sk {
constexpr int NW = 4;
constexpr int T = NW * 32;
constexpr int NCH_MAX = 32;
constexpr int MAX_STAGES = 8;
constexpr int CTX = 128;
constexpr int PW = NW - 1;  // the warp whose lane 0 derives the m' params

// per-row fast-path proof bits (Meta/Ctx::flags)
constexpr int F_FAST = 1;   // fast dequant of w/m/g, w codes range-proven, sparse table fits
constexpr int F_LSAT = 2;   // Lion sign update by saturating FMA (weight decay 0)

struct Ctx {
  int32_t lrow;  // -1: no more rows
  int32_t cols;
  int32_t old_begin, old_n, old_staged;
  int32_t zw, zm, zg, zpay;
  int32_t slot_out, cap_out, flags;
  float sw, tmin, tmax, sm, sg, _pf[3];
  uint8_t* w_out;
  uint8_t* m_out;
  float* m_scale_out;
  int32_t* m_zp_out;
  int32_t* cnt_out;
};
static_assert(sizeof(Ctx) <= CTX, "ctx");

// per-row metadata of the current issue block (warp 0 loads it lane-parallel)
struct Meta {
  float sw, tmin, tmax, sm, sg;
  int32_t zw, zm, zg, ob, on, so, co, flags;
};

struct Tabs {
  float lo[NW], hi[NW];
  int32_t nan[NW];
  float glo[NW], ghi[NW];
  int32_t gnan[NW];
  int32_t cnt[NCH_MAX][NW];
  QuantRow qm;       // m' quantizer of the current row (written by the param thread)
  int32_t qm_fast;   // m' codes range-proven: pass 2 checks only the tie distance
};

__host__ __device__ inline int r16(int x) { return (x + 15) & ~15; }

struct Layout {
  int cp, oldcap, S, K;
  bool mrec;
  int gk;
  // stage: ctx | old cols | old vals | old bitmap | kept-outlier bitmap | first ranks | w m g
  __host__ __device__ int bits_bytes() const { return r16((cp + 31) / 32 * 4); }
  __host__ __device__ int frank_bytes() const { return r16((cp + 31) / 32 * 2); }
  __host__ __device__ int gbytes() const { return gk == G_U8 ? cp : (gk == G_F32 ? 4 * cp : 2 * cp); }
  __host__ __device__ int off_bits() const { return CTX + oldcap * 8; }
  __host__ __device__ int off_bout() const { return off_bits() + bits_bytes(); }
  __host__ __device__ int off_frank() const { return off_bout() + bits_bytes(); }
  __host__ __device__ int off_data() const { return off_frank() + frank_bytes(); }
  __host__ __device__ int stage_bytes() const { return off_data() + 2 * cp + gbytes(); }
  __host__ __device__ int nch() const { return (cp / 16 + T - 1) / T; }
  __host__ __device__ int mprime_bytes() const { return mrec ? 0 : 4 * nch() * T * 16; }
  __host__ __device__ int masks_bytes() const { return r16(cp / 16 * 2); }
  __host__ __device__ int slots_bytes() const { return K * 4 * T * 16; }
  __host__ __device__ int meta_bytes() const { return 32 * (int)sizeof(Meta); }
  // sparse results (w' and code|class<<8 per old outlier), double-buffered by row
  // parity: row t writes them before barrier B0(t) while row t-1's CSR phase (which
  // ends at B0(t)) may still read the other buffer
  __host__ __device__ int sparse_bytes() const { return 16 * oldcap; }
  __host__ __device__ size_t total() const {
    return 128 + (size_t)S * stage_bytes() + r16((int)sizeof(Tabs)) + mprime_bytes() +
           masks_bytes() + slots_bytes() + meta_bytes() + sparse_bytes();
  }
};
}  // namespace sk

int step_kernel_max_cols() { return sk::NCH_MAX * sk::T * 16; }

size_t step_kernel_smem(int gk, int cols_p, int stages, int oldcap, int slots, bool mrec) {
  sk::Layout L{cols_p, oldcap, stages, slots, mrec, gk};
  return L.total();
}

namespace {

__device__ __forceinline__ uint32_t skbits16(const uint32_t* bits, int v) {
  return (bits[v >> 1] >> ((v & 1) * 16)) & 0xFFFFu;
}

__device__ __forceinline__ float sk_old_value(const uint32_t* bits, const uint16_t* frank,
                                              const float* ov, int staged, int oldcap,
                                              int old_begin, int col, const float* val_in) {
  const int w = col >> 5;
  const int r = (int)frank[w] + __popc(bits[w] & ((1u << (col & 31)) - 1u));
  return (staged && r < oldcap) ? ov[r] : val_in[old_begin + r];
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

// The row-level proof for the fast path (see the file header).  Lane-parallel, once
// per row, off the element loop; fp64 where the reference is fp64.
template <int GK, bool ALIGNED, bool WD0>
__device__ __forceinline__ int sk_row_flags(const sk::Meta& m, int bit_width, int oldcap,
                                            const LaunchArgs& a) {
  if (GK != G_U8 || !ALIGNED) return 0;
  const int qmax = (1 << bit_width) - 1;
  const QuantRow qw = make_quant_row(m.sw, m.zw, bit_width);
  bool ok = qw.fast && make_dequant_row(m.sm, m.zm).fast && make_dequant_row(m.sg, m.zg).fast &&
            m.on <= oldcap;
  // bounded dense w (and w +- lr) -- no overflow in the update
  ok = ok && (__fmul_rn(fabsf(m.sw), (float)qmax + fabsf((float)m.zw)) < 0x1.0p126f) &&
       fabsf(a.lr) <= 0x1.0p100f;
  // every inlier v in [t_min, t_max] and the payload code quantize inside [0, qmax]
  ok = ok && (m.tmin <= m.tmax) && code_unclamped(m.tmin, m.sw, m.zw) >= 0.0 &&
       code_unclamped(m.tmax, m.sw, m.zw) <= (double)qmax;
  int f = ok ? sk::F_FAST : 0;
  if (ok && WD0) {
    const double c1 = (double)__fsub_rn(1.0f, a.b1);
    const double bm = (double)m.sm * ((double)qmax + fabs((double)m.zm));
    const double bg = (double)m.sg * ((double)qmax + fabs((double)m.zg));
    const double pm = fabs((double)a.b1) * (double)m.sm;  // smallest non-zero |b1*m|
    const double pg = fabs(c1) * (double)m.sg;            // smallest non-zero |c1*g|
    const bool lsat = m.sm > 0.0f && m.sg > 0.0f && bm <= 0x1.0p120 && bg <= 0x1.0p120 &&
                      fabs((double)a.b1) <= 4.0 && fabs(c1) <= 4.0 &&
                      (a.b1 == 0.0f || pm >= 0x1.0p-100) && (c1 == 0.0 || pg >= 0x1.0p-100);
    if (lsat) f |= sk::F_LSAT;
  }
  return f;
}

}  // namespace

template <int GK, bool ALIGNED, bool WD0, bool MREC_>
__global__ void __launch_bounds__(sk::T, QFT_STEP_MIN_CTAS) step_kernel(const LaunchArgs a) {
  using namespace sk;
  constexpr bool MREC = MREC_ && GK == G_U8;  // recompute needs the staged g codes
  extern __shared__ __align__(128) uint8_t smem[];
  const Layout L{a.cols_p, a.oldcap, a.stages, a.slots, MREC, GK};
  const int cp = L.cp, S = L.S, K = L.K, oldcap = L.oldcap;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  const int sbytes = L.stage_bytes();
  uint8_t* stage0 = smem + 128;
  uint8_t* p = stage0 + (size_t)S * sbytes;
  Tabs* tabs = reinterpret_cast<Tabs*>(p);
  p += r16((int)sizeof(Tabs));
  float4* mprime = reinterpret_cast<float4*>(p);
  p += L.mprime_bytes();
  uint16_t* masks = reinterpret_cast<uint16_t*>(p);
  p += L.masks_bytes();
  float4* slots = reinterpret_cast<float4*>(p);
  p += L.slots_bytes();
  Meta* meta = reinterpret_cast<Meta*>(p);
  p += L.meta_bytes();
  float* const sp_base = reinterpret_cast<float*>(p);  // [w' | code|class<<8] x 2 (row parity)

  const int ct = threadIdx.x;
  const int warp = ct >> 5, lane = ct & 31;
  const int qmax = (1 << a.bit_width) - 1;
  const int in = a.flip, out = 1 - a.flip;

  auto stage_of = [&](int s) { return stage0 + (size_t)s * sbytes; };
  auto ctx_of = [&](int s) { return reinterpret_cast<Ctx*>(stage_of(s)); };
  auto oc_of = [&](int s) { return reinterpret_cast<int32_t*>(stage_of(s) + CTX); };
  auto ov_of = [&](int s) { return reinterpret_cast<float*>(stage_of(s) + CTX + oldcap * 4); };
  auto bits_of = [&](int s) { return reinterpret_cast<uint32_t*>(stage_of(s) + L.off_bits()); };
  auto bout_of = [&](int s) { return reinterpret_cast<uint32_t*>(stage_of(s) + L.off_bout()); };
  auto frank_of = [&](int s) { return reinterpret_cast<uint16_t*>(stage_of(s) + L.off_frank()); };
  auto data_of = [&](int s) { return stage_of(s) + L.off_data(); };

  // ------------------------------------------------------------------ issuer (warp 0)
  int i_blk = blockIdx.x, i_j = 0, i_nrows = 0, i_row0 = 0, i_tensor = 0;
  auto load_block = [&]() {  // warp 0: lane-parallel metadata of block i_blk into smem
    if (i_blk >= a.n_blocks) {
      i_nrows = 0;
      return;
    }
    const RowBlock B = a.blocks[i_blk];
    i_nrows = B.nrows;
    i_row0 = B.row0;
    i_tensor = B.tensor;
    const DevTensor* Tt = a.tensors + B.tensor;
    if (lane < B.nrows) {
      const int r = B.row0 + lane;
      Meta m;
      m.sw = Tt->w_scale[r];
      m.zw = Tt->w_zp[r];
      m.tmin = Tt->t_min[r];
      m.tmax = Tt->t_max[r];
      m.sm = Tt->m_scale[in][r];
      m.zm = Tt->m_zp[in][r];
      if (GK == G_U8) {
        m.sg = Tt->g_scale[r];
        m.zg = Tt->g_zp[r];
      } else {
        m.sg = 0.f;
        m.zg = 0;
      }
      const int32_t* rs = Tt->rs[in];
      m.ob = rs[r];
      const int cap_in = rs[r + 1] - m.ob;
      m.on = Tt->cnt[in] ? min(Tt->cnt[in][r], cap_in) : cap_in;
      m.so = Tt->rs[out][r];
      m.co = Tt->rs[out][r + 1] - m.so;
      m.flags = sk_row_flags<GK, ALIGNED, WD0>(m, a.bit_width, oldcap, a);
      meta[lane] = m;
    }
    __syncwarp();
  };
  auto issue = [&](int s) {  // warp 0: fill stage s with the next row (or the end mark)
    Ctx* cx = ctx_of(s);
    if (i_j >= i_nrows) {
      i_blk += gridDim.x;
      i_j = 0;
      load_block();
    }
    if (i_nrows == 0) {
      if (lane == 0) {
        cx->lrow = -1;
        mbar_arrive(&full[s]);
      }
      return;
    }
    const DevTensor* Tt = a.tensors + i_tensor;
    const int cols = Tt->cols;
    const int lrow = i_row0 + i_j;
    const Meta& m = meta[i_j];
    const size_t roff = (size_t)lrow * (size_t)cols;
    uint32_t* bits = bits_of(s);
    uint32_t* bout = bout_of(s);
    for (int i = lane; i < (cp + 31) / 32; i += 32) {
      bits[i] = 0u;
      bout[i] = 0u;
    }
    const bool staged = ALIGNED && a.slotted_in && m.on > 0 && ((m.ob & 3) == 0);
    const int nstage = staged ? min((m.on + 3) & ~3, oldcap) : 0;
    const int gel = (GK == G_U8) ? 1 : (GK == G_F32 ? 4 : 2);
    const uint8_t* g_base = (GK == G_U8) ? Tt->g_codes : reinterpret_cast<const uint8_t*>(Tt->g_raw);
    uint8_t* data = data_of(s);
    // context fields spread over lanes (one store each)
    switch (lane) {
      case 0: cx->lrow = lrow; break;
      case 1: cx->cols = cols; break;
      case 2: cx->old_begin = m.ob; break;
      case 3: cx->old_n = m.on; break;
      case 4: cx->old_staged = staged ? 1 : 0; break;
      case 5: cx->sw = m.sw; break;
      case 6: cx->zw = m.zw; break;
      case 7: cx->zpay = m.zw < 0 ? 0 : (m.zw > qmax ? qmax : m.zw); break;
      case 8: cx->tmin = m.tmin; break;
      case 9: cx->tmax = m.tmax; break;
      case 10: cx->sm = m.sm; break;
      case 11: cx->zm = m.zm; break;
      case 12: cx->sg = m.sg; break;
      case 13: cx->zg = m.zg; break;
      case 14: cx->slot_out = m.so; break;
      case 15: cx->cap_out = m.co; break;
      case 16: cx->w_out = Tt->w_codes[out] + roff; break;
      case 17: cx->m_out = Tt->m_codes[out] + roff; break;
      case 18: cx->m_scale_out = Tt->m_scale[out]; break;
      case 19: cx->m_zp_out = Tt->m_zp[out]; break;
      case 20: cx->cnt_out = Tt->cnt[out]; break;
      case 21: cx->flags = m.flags; break;
      default: break;
    }
    if (!ALIGNED) {
      const uint8_t* wsrc = Tt->w_codes[in] + roff;
      const uint8_t* msrc = Tt->m_codes[in] + roff;
      const uint8_t* gsrc = g_base + (size_t)gel * roff;
      for (int i = lane; i < cols; i += 32) {
        data[i] = wsrc[i];
        data[cp + i] = msrc[i];
      }
      for (int i = lane; i < gel * cols; i += 32) data[2 * cp + i] = gsrc[i];
    }
    __syncwarp();
    if (lane == 0) {
      uint32_t tx = 8u * (uint32_t)nstage;
      if (ALIGNED) tx += (uint32_t)((2 + gel) * cols);
      if (tx) mbar_expect_tx(&full[s], tx);
      if (ALIGNED) {
        bulk_g2s(data, Tt->w_codes[in] + roff, cols, &full[s]);
        bulk_g2s(data + cp, Tt->m_codes[in] + roff, cols, &full[s]);
        bulk_g2s(data + 2 * cp, g_base + (size_t)gel * roff, gel * cols, &full[s]);
      }
      if (nstage) {
        bulk_g2s(oc_of(s), a.col_in + m.ob, 4u * nstage, &full[s]);
        bulk_g2s(ov_of(s), a.val_in + m.ob, 4u * nstage, &full[s]);
      }
      mbar_arrive(&full[s]);
    }
    ++i_j;
  };

  if (ct == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (warp == 0) {
    load_block();
    for (int s = 0; s < S; ++s) issue(s);
  }

  Hyper h;
  h.lr = a.lr; h.b1 = a.b1; h.b2 = a.b2; h.wd = a.wd;
  h.c1 = __fsub_rn(1.0f, a.b1);
  h.c2 = __fsub_rn(1.0f, a.b2);

  // pass 2 of a finished row (stage ps): m' -> codes with the params the param thread
  // published; runs one row late, right after the next row's barrier B0
  auto pass2 = [&](int ps) {
    const Ctx* px = ctx_of(ps);
    const int pcols = px->cols;
    const int pnvec = (pcols + 15) >> 4;
    const int pnch = (pnvec + T - 1) / T;
    const uint8_t* pdata = data_of(ps);
    const QuantRow qm = tabs->qm;
    const bool qm_fast = tabs->qm_fast != 0;
    const DequantRow pdm = make_dequant_row(px->sm, px->zm);
    const DequantRow pdg = make_dequant_row(px->sg, px->zg);
    for (int k = 0; k < pnch; ++k) {
      const int v = k * T + ct;
      if (v >= pnvec) break;
      float m[16];
      if (MREC) {
        float g[16];
        const uint4 mq = *reinterpret_cast<const uint4*>(pdata + cp + v * 16);
        const uint4 gq = *reinterpret_cast<const uint4*>(pdata + 2 * cp + v * 16);
        dequant4(mq.x, pdm, m); dequant4(mq.y, pdm, m + 4);
        dequant4(mq.z, pdm, m + 8); dequant4(mq.w, pdm, m + 12);
        dequant4(gq.x, pdg, g); dequant4(gq.y, pdg, g + 4);
        dequant4(gq.z, pdg, g + 8); dequant4(gq.w, pdg, g + 12);
#pragma unroll
        for (int pp = 0; pp < 8; ++pp) {
          const float2 M = sadd2(mul2(f2(h.b2), make_float2(m[2 * pp], m[2 * pp + 1])),
                                 mul2(f2(h.c2), make_float2(g[2 * pp], g[2 * pp + 1])));
          m[2 * pp] = M.x;
          m[2 * pp + 1] = M.y;
        }
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 f = mprime[(k * 4 + q) * T + ct];
          m[4 * q] = f.x; m[4 * q + 1] = f.y; m[4 * q + 2] = f.z; m[4 * q + 3] = f.w;
        }
      }
      uint32_t c[4];
      bool ok;
      if (qm_fast) {
        float em = 0.0f;
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = quant4_e(m + 4 * q, qm, em);
        ok = em < qm.thr;
      } else {
        QAcc qa = qacc_init();
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = quant4_nc(m + 4 * q, qm, qa);
        ok = quant_vec_ok(qa, qm);
      }
      if (!ok) {
#pragma unroll
        for (int q = 0; q < 4; ++q) c[q] = quant4_exact(m + 4 * q, qm);
      }
      uint8_t* mo = px->m_out + v * 16;
      if (ALIGNED) {
        *reinterpret_cast<uint4*>(mo) = make_uint4(c[0], c[1], c[2], c[3]);
      } else {
        const int nvalid = min(16, pcols - v * 16);
        for (int e = 0; e < nvalid; ++e) mo[e] = (uint8_t)(c[e >> 2] >> ((e & 3) * 8));
      }
    }
  };

  for (int t = 0;; ++t) {
    const int s = t % S;
    mbar_wait(&full[s], (uint32_t)(t / S) & 1u);
    Ctx* cx = ctx_of(s);
    const int lrow = cx->lrow;
    const bool end = lrow < 0;
    const int cols = cx->cols;
    const int nvec = (cols + 15) >> 4;
    const int nch = (nvec + T - 1) / T;
    const uint8_t* data = data_of(s);
    uint32_t* obits = bits_of(s);
    uint32_t* obout = bout_of(s);
    uint16_t* frank = frank_of(s);
    const int32_t* ocols = oc_of(s);
    const float* ovals = ov_of(s);
    const int old_n = end ? 0 : cx->old_n;
    const int old_begin = cx->old_begin, staged = cx->old_staged;
    const int flags = cx->flags;
    const bool fast = (GK == G_U8) && ALIGNED && (flags & F_FAST);

    const DequantRow dw = make_dequant_row(cx->sw, cx->zw);
    const DequantRow dm = make_dequant_row(cx->sm, cx->zm);
    DequantRow dg = make_dequant_row(cx->sg, cx->zg);
    QuantRow qg{};
    const QuantRow qw = make_quant_row(cx->sw, cx->zw, a.bit_width);
    const float tmin = cx->tmin, tmax = cx->tmax;
    const int zpay = cx->zpay;
    const uint32_t zpay4 = (uint32_t)zpay * 0x01010101u;
    const uint32_t wz_bits = __float_as_uint(__fmul_rn(cx->sw, (float)(zpay - cx->zw)));
    const bool w_ovf = !(__fmul_rn(fabsf(cx->sw), (float)qmax + fabsf((float)cx->zw)) < 3.0e38f);
    // old outliers: a sparse side computation (one thread per entry) unless the row has
    // more than the per-CTA table holds
    const bool sparse_ok = old_n <= oldcap;
    float* const sp_val = sp_base + (t & 1) * 2 * oldcap;
    uint32_t* const sp_cw = reinterpret_cast<uint32_t*>(sp_val + oldcap);

    // sparse pass for one old outlier: its exact w' (lion1, the general form), its
    // class against the cached thresholds and its code -- what requantize_weight
    // gives that element (quantize.hpp:274-285)
    auto sparse_entry = [&](int i, int col) {
      const float v0 = (staged && i < oldcap) ? ovals[i] : a.val_in[old_begin + i];
      const float mv = sk_deq1(data[cp + col], dm);
      float gv;
      if (GK == G_U8) {
        gv = sk_deq1(data[2 * cp + col], dg);
      } else {
        gv = sk_deq1(quant_exact(sk_graw<GK>(data + 2 * cp, col), qg.s, qg.z, qg.qmax), dg);
      }
      float wv = v0, mm = mv;
      lion1(wv, mm, gv, h);
      const bool o = (wv < tmin) || (wv > tmax);
      const uint32_t code = o ? (uint32_t)zpay : quant_exact(wv, qw.s, qw.z, qw.qmax);
      sp_val[i] = wv;
      sp_cw[i] = code | (o ? 0x100u : 0u);
      if (o) atomicOr(&obout[col >> 5], 1u << (col & 31));
    };

    // old-outlier bitmap + first rank per 32-column word (O(1) rank/value lookup)
    for (int i = ct; i < old_n; i += T) {
      const int col = (staged && i < oldcap) ? ocols[i] : a.col_in[old_begin + i];
      const int wd = col >> 5;
      atomicOr(&obits[wd], 1u << (col & 31));
      const int prev = (i == 0) ? -1
                       : ((staged && i - 1 < oldcap) ? ocols[i - 1] : a.col_in[old_begin + i - 1]);
      if (i == 0 || (prev >> 5) != wd) frank[wd] = (uint16_t)i;
      if (GK == G_U8 && sparse_ok) sparse_entry(i, col);
    }
    __syncthreads();  // B0: bitmaps ready; row t-1's CSR phase done, its m' params published
    // refill the stage of row t-2 (row t-1's stage still feeds its pass 2)
    if (!end && warp == 0 && t >= 2) issue((t - 2) % S);
    if (t > 0) pass2((t - 1) % S);
    if (end) break;

    // ---- raw-gradient kinds: fused quantize_state(g) -> dequantize (gradflow.hpp:77)
    if (GK != G_U8) {
      float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
      int nan0 = 0;
      const uint8_t* gd = data + 2 * cp;
      for (int k = 0; k < nch; ++k) {
        const int v = k * T + ct;
        if (v < nvec) {
          const int nvalid = min(16, cols - v * 16);
          for (int e = 0; e < nvalid; ++e) {
            const float x = sk_graw<GK>(gd, v * 16 + e);
            lo = fminf(lo, x);
            hi = fmaxf(hi, x);
          }
          if (v == 0 && isnan(sk_graw<GK>(gd, 0))) nan0 = 1;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        nan0 |= __shfl_xor_sync(0xffffffffu, nan0, o);
      }
      if (lane == 0) {
        tabs->glo[warp] = lo;
        tabs->ghi[warp] = hi;
        tabs->gnan[warp] = nan0;
      }
      __syncthreads();
      lo = tabs->glo[0]; hi = tabs->ghi[0]; nan0 = tabs->gnan[0];
#pragma unroll
      for (int w2 = 1; w2 < NW; ++w2) {
        lo = fminf(lo, tabs->glo[w2]);
        hi = fmaxf(hi, tabs->ghi[w2]);
        nan0 |= tabs->gnan[w2];
      }
      if (nan0) lo = hi = __int_as_float(0x7fc00000);
      float sgv; int32_t zgv;
      if (!affine_from_bounds(lo, hi, a.bit_width, sgv, zgv)) {
        if (ct == 0) atomicOr(&a.hdr->err, ERR_GPARAMS);
        sgv = 1.0f; zgv = 0;
      }
      qg = make_quant_row(sgv, zgv, a.bit_width);
      dg = make_dequant_row(sgv, zgv);
      if (sparse_ok) {  // the sparse pass needs the gradient params: one more barrier
        for (int i = ct; i < old_n; i += T)
          sparse_entry(i, (staged && i < oldcap) ? ocols[i] : a.col_in[old_begin + i]);
        __syncthreads();
      }
    }

    float mlo = __int_as_float(0x7f800000), mhi = __int_as_float(0xff800000);
    int mnan0 = 0;
    int slots_used = 0;
    uint64_t slotmap = ~0ull;  // 2 bits per chunk: slot id, 3 = none / recompute

    // ================================ pass 1 ================================
    if (fast) {
      // ---- fast rows: branch-free dequant, range-proven quantizer, old outliers
      // excluded here (their codes are patched after barrier C from the sparse pass)
      const bool lsat = WD0 && (flags & F_LSAT);
      const float2 n2lr = f2(__fmul_rn(-2.0f, h.lr)), plr = f2(h.lr);
      for (int k = 0; k < nch; ++k) {
        const int v = k * T + ct;
        uint32_t mask = 0;
        if (v < nvec) {
          float w[16], m[16], g[16];
          sk_deq16(*reinterpret_cast<const uint4*>(data + v * 16), dw, w);
          sk_deq16(*reinterpret_cast<const uint4*>(data + cp + v * 16), dm, m);
          sk_deq16(*reinterpret_cast<const uint4*>(data + 2 * cp + v * 16), dg, g);
          if (lsat) {
#pragma unroll
            for (int pp = 0; pp < 8; ++pp) {
              float2 W = make_float2(w[2 * pp], w[2 * pp + 1]);
              float2 M = make_float2(m[2 * pp], m[2 * pp + 1]);
              lion2_sat(W, M, make_float2(g[2 * pp], g[2 * pp + 1]), h, n2lr, plr);
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
          if (!MREC) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              mprime[(k * 4 + q) * T + ct] =
                  make_float4(m[4 * q], m[4 * q + 1], m[4 * q + 2], m[4 * q + 3]);
          }
          float wq2[16];
          const float wz = __uint_as_float(wz_bits);
#pragma unroll
          for (int e = 0; e < 16; ++e) wq2[e] = outlier_select(w[e], tmin, tmax, wz, 1u << e, mask);
          float em = 0.0f;
          uint32_t c[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) c[q] = quant4_e(wq2 + 4 * q, qw, em);
          if (!(em < qw.thr)) {
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] = quant4_exact(wq2 + 4 * q, qw);
          }
          *reinterpret_cast<uint4*>(cx->w_out + v * 16) = make_uint4(c[0], c[1], c[2], c[3]);
          const uint32_t dense_new = mask & ~skbits16(obits, v);
          mask = dense_new | skbits16(obout, v);
          masks[v] = (uint16_t)mask;
          if (dense_new && slots_used < K) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              slots[(slots_used * 4 + q) * T + ct] =
                  make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
            slotmap &= ~(3ull << (2 * k));
            slotmap |= (uint64_t)slots_used << (2 * k);
            ++slots_used;
          }
        }
        const int wc = __reduce_add_sync(0xffffffffu, __popc(mask));
        if (lane == 0) tabs->cnt[k][warp] = wc;
      }
    } else {
      // ---- general rows: per-vector proofs with exact fallbacks
      for (int k = 0; k < nch; ++k) {
        const int v = k * T + ct;
        uint32_t mask = 0;
        if (v < nvec) {
          const int nvalid = min(16, cols - v * 16);
          const uint32_t valid = nvalid >= 16 ? 0xFFFFu : ((1u << nvalid) - 1u);
          float w[16], m[16], g[16];
          const uint4 wq = *reinterpret_cast<const uint4*>(data + v * 16);
          const uint4 mq = *reinterpret_cast<const uint4*>(data + cp + v * 16);
          dequant4(wq.x, dw, w); dequant4(wq.y, dw, w + 4);
          dequant4(wq.z, dw, w + 8); dequant4(wq.w, dw, w + 12);
          dequant4(mq.x, dm, m); dequant4(mq.y, dm, m + 4);
          dequant4(mq.z, dm, m + 8); dequant4(mq.w, dm, m + 12);
          if (GK == G_U8) {
            const uint4 gq = *reinterpret_cast<const uint4*>(data + 2 * cp + v * 16);
            dequant4(gq.x, dg, g); dequant4(gq.y, dg, g + 4);
            dequant4(gq.z, dg, g + 8); dequant4(gq.w, dg, g + 12);
          } else {
            float graw[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
              graw[e] = (e < nvalid) ? sk_graw<GK>(data + 2 * cp, v * 16 + e) : 0.0f;
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
          // old outliers: normally done by the sparse pass (their w here comes from the
          // payload code and is patched over below); rows with more old outliers than
          // the table holds patch w before the update instead
          const uint32_t o16_all = skbits16(obits, v);
          uint32_t o16 = sparse_ok ? 0u : o16_all;
          bool wspecial = w_ovf;
          while (o16) {
            const int e = __ffs(o16) - 1;
            o16 &= o16 - 1u;
            const float val =
                sk_old_value(obits, frank, ovals, staged, oldcap, old_begin, v * 16 + e, a.val_in);
            wspecial |= !isfinite(val);
#pragma unroll
            for (int j = 0; j < 16; ++j) w[j] = (j == e) ? val : w[j];
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
          if (!MREC) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              mprime[(k * 4 + q) * T + ct] =
                  make_float4(m[4 * q], m[4 * q + 1], m[4 * q + 2], m[4 * q + 3]);
          }
          // ---- outlier test, payload select, quantize w'
          float wq2[16];
          const float wz = __uint_as_float(wz_bits);
#pragma unroll
          for (int e = 0; e < 16; ++e) wq2[e] = outlier_select(w[e], tmin, tmax, wz, 1u << e, mask);
          mask &= valid;
          QAcc qa = qacc_init();
          uint32_t c[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) c[q] = quant4_nc(wq2 + 4 * q, qw, qa);
          if (!quant_vec_ok(qa, qw)) {
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] = quant4_exact(w + 4 * q, qw);
            if (mask) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t bm = sk_nib_mask((mask >> (4 * q)) & 0xFu);
                c[q] = (c[q] & ~bm) | (zpay4 & bm);
              }
            }
          }
          if (sparse_ok && o16_all) {
            // old-outlier elements: class and code from the sparse pass
            uint32_t ob = o16_all & valid;
            while (ob) {
              const int e = __ffs(ob) - 1;
              ob &= ob - 1u;
              const int col = v * 16 + e;
              const int wd = col >> 5;
              const int r = (int)frank[wd] + __popc(obits[wd] & ((1u << (col & 31)) - 1u));
              const uint32_t cw = sp_cw[r];
              mask = (mask & ~(1u << e)) | (((cw >> 8) & 1u) << e);
              const uint32_t sh = (uint32_t)(e & 3) * 8u;
              const uint32_t keep = ~(0xFFu << sh), put = (cw & 0xFFu) << sh;
              const int q = e >> 2;
              c[0] = (q == 0) ? ((c[0] & keep) | put) : c[0];
              c[1] = (q == 1) ? ((c[1] & keep) | put) : c[1];
              c[2] = (q == 2) ? ((c[2] & keep) | put) : c[2];
              c[3] = (q == 3) ? ((c[3] & keep) | put) : c[3];
            }
          }
          uint8_t* wo = cx->w_out + v * 16;
          if (ALIGNED) {
            *reinterpret_cast<uint4*>(wo) = make_uint4(c[0], c[1], c[2], c[3]);
          } else {
            for (int e = 0; e < nvalid; ++e) wo[e] = (uint8_t)(c[e >> 2] >> ((e & 3) * 8));
          }
          masks[v] = (uint16_t)mask;
          // park the w' values of a vector holding new dense-origin outliers (CSR values
          // later; old-origin ones come from the sparse pass)
          const uint32_t need_slot = sparse_ok ? (mask & ~o16_all) : mask;
          if (need_slot && slots_used < K) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              slots[(slots_used * 4 + q) * T + ct] =
                  make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
            slotmap &= ~(3ull << (2 * k));
            slotmap |= (uint64_t)slots_used << (2 * k);
            ++slots_used;
          }
        }
        const int wc = __reduce_add_sync(0xffffffffu, __popc(mask));
        if (lane == 0) tabs->cnt[k][warp] = wc;
      }
    }

    // ---- row reduction
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mlo = fminf(mlo, __shfl_xor_sync(0xffffffffu, mlo, o));
      mhi = fmaxf(mhi, __shfl_xor_sync(0xffffffffu, mhi, o));
      mnan0 |= __shfl_xor_sync(0xffffffffu, mnan0, o);
    }
    if (lane == 0) {
      tabs->lo[warp] = mlo;
      tabs->hi[warp] = mhi;
      tabs->nan[warp] = mnan0;
    }
    __syncthreads();  // C

    // chunk-major CSR offsets: lane l < nch holds the offset of (chunk l, this warp)
    int tot_l = 0, mine_l = 0;
    if (lane < nch) {
#pragma unroll
      for (int w2 = 0; w2 < NW; ++w2) {
        const int cv = tabs->cnt[lane][w2];
        tot_l += cv;
        if (w2 < warp) mine_l += cv;
      }
    }
    int incl_l = tot_l;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int tt = __shfl_up_sync(0xffffffffu, incl_l, d);
      if (lane >= d) incl_l += tt;
    }
    const int chunk_pref = incl_l - tot_l + mine_l;
    const int row_total = __shfl_sync(0xffffffffu, incl_l, nch - 1);
    const int slot_out = cx->slot_out, cap_out = cx->cap_out;

    if (ct == PW * 32) {
      // m' params (quantize_state: channel_minmax -> affine_params_from_bounds), once
      float lo = tabs->lo[0], hi = tabs->hi[0];
      int nan0 = tabs->nan[0];
#pragma unroll
      for (int w2 = 1; w2 < NW; ++w2) {
        lo = fminf(lo, tabs->lo[w2]);
        hi = fmaxf(hi, tabs->hi[w2]);
        nan0 |= tabs->nan[w2];
      }
      if (nan0) lo = hi = __int_as_float(0x7fc00000);
      float smv; int32_t zmv;
      if (!affine_from_bounds(lo, hi, a.bit_width, smv, zmv)) {
        atomicOr(&a.hdr->err, ERR_MPARAMS);
        smv = 1.0f; zmv = 0;
      }
      const QuantRow qm = make_quant_row(smv, zmv, a.bit_width);
      // every m' lies in [lo, hi]: if those two codes need no clip, none does
      tabs->qm = qm;
      tabs->qm_fast = fast && qm.fast && code_unclamped(lo, smv, zmv) >= 0.0 &&
                      code_unclamped(hi, smv, zmv) <= (double)qmax;
      cx->m_scale_out[lrow] = smv;
      cx->m_zp_out[lrow] = zmv;
      cx->cnt_out[lrow] = row_total;
      if (row_total > cap_out) atomicOr(&a.hdr->overflow, 1u);
    }

    // old-outlier codes of fast rows (pass 1 left payload-derived bytes there)
    if (fast) {
      for (int i = ct; i < old_n; i += T) {
        const int col = (staged && i < oldcap) ? ocols[i] : a.col_in[old_begin + i];
        cx->w_out[col] = (uint8_t)(sp_cw[i] & 0xFFu);
      }
    }

    // ============================ CSR write =================================
    for (int k = 0; k < nch; ++k) {
      const int pref_k = __shfl_sync(0xffffffffu, chunk_pref, k);
      if (tabs->cnt[k][warp] == 0) continue;  // warp-uniform
      const int v = k * T + ct;
      uint32_t mask = (v < nvec) ? (uint32_t)masks[v] : 0u;
      const int c = __popc(mask);
      int incl = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int tt = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += tt;
      }
      int pos = pref_k + incl - c;
      const int sid = (int)((slotmap >> (2 * k)) & 3ull);
      const uint32_t o16 = (sparse_ok && v < nvec) ? skbits16(obits, v) : 0u;
      while (mask) {
        const int e = __ffs(mask) - 1;
        mask &= mask - 1u;
        const int col = v * 16 + e;
        float val;
        if (o16 & (1u << e)) {  // old-origin: value from the sparse pass
          const int wd = col >> 5;
          val = sp_val[(int)frank[wd] + __popc(obits[wd] & ((1u << (col & 31)) - 1u))];
        } else if (sid < K) {
          val = reinterpret_cast<const float*>(&slots[(sid * 4 + (e >> 2)) * T + ct])[e & 3];
        } else {  // no slot left: recompute exactly as pass 1 did (scalar, exact)
          float wv = sk_deq1(data[col], dw);
          if (skbits16(obits, v) & (1u << e))
            wv = sk_old_value(obits, frank, ovals, staged, oldcap, old_begin, col, a.val_in);
          float mv = sk_deq1(data[cp + col], dm);
          float gv;
          if (GK == G_U8) {
            gv = sk_deq1(data[2 * cp + col], dg);
          } else {
            const float gr = sk_graw<GK>(data + 2 * cp, col);
            gv = sk_deq1(quant_exact(gr, qg.s, qg.z, qg.qmax), dg);
          }
          lion1(wv, mv, gv, h);
          val = wv;
        }
        if (pos < cap_out) {
          a.col_out[slot_out + pos] = col;
          a.val_out[slot_out + pos] = val;
        }
        ++pos;
      }
    }
  }
}

// ----------------------------------------------------------------------------
template <int GK, bool AL, bool WD0, bool MREC>
static cudaError_t step_launch_t(const LaunchArgs& a, size_t smem, cudaStream_t st) {
  auto k = step_kernel<GK, AL, WD0, MREC>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, sk::T, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int grid = sms * per_sm;
  if (grid > a.n_blocks) grid = a.n_blocks;
  if (grid < 1) grid = 1;
  k<<<grid, sk::T, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_step_kernel(int gk, const LaunchArgs& a, cudaStream_t st) {
  const bool mrec = a.mrec != 0 && gk == G_U8;
  const size_t smem = step_kernel_smem(gk, a.cols_p, a.stages, a.oldcap, a.slots, mrec);
  const bool al = a.use_bulk != 0;
  const bool wd0 = (a.wd == 0.0f);
#define SK_L(G)                                                                          \
  do {                                                                                   \
    if (al) {                                                                            \
      if (wd0) return mrec ? step_launch_t<G, true, true, true>(a, smem, st)             \
                           : step_launch_t<G, true, true, false>(a, smem, st);           \
      return mrec ? step_launch_t<G, true, false, true>(a, smem, st)                     \
                  : step_launch_t<G, true, false, false>(a, smem, st);                   \
    }                                                                                    \
    return wd0 ? step_launch_t<G, false, true, false>(a, smem, st)                       \
               : step_launch_t<G, false, false, false>(a, smem, st);                     \
  } while (0)
  if (gk == G_U8) SK_L(G_U8);
  if (gk == G_F32) {
    if (al) return wd0 ? step_launch_t<G_F32, true, true, false>(a, smem, st)
                       : step_launch_t<G_F32, true, false, false>(a, smem, st);
    return wd0 ? step_launch_t<G_F32, false, true, false>(a, smem, st)
               : step_launch_t<G_F32, false, false, false>(a, smem, st);
  }
  if (al) return wd0 ? step_launch_t<G_BF16, true, true, false>(a, smem, st)
                     : step_launch_t<G_BF16, true, false, false>(a, smem, st);
  return wd0 ? step_launch_t<G_BF16, false, true, false>(a, smem, st)
             : step_launch_t<G_BF16, false, false, false>(a, smem, st);
#undef SK_L
}

}  // namespace qftk
