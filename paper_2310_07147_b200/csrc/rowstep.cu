// rowstep.cu -- the fused quantized Lion step, v6: one CTA per ROW, the row's new
// momentum held in registers, and a per-row proof that lets the dense weight codes
// pass through untouched.
//
// Reference: the loop body of lion_step_quantized, optimizer.hpp:103-118 -- dequant g,
// m, reconstruct w -> lion_apply -> quantize_state(m') -> requantize_weight(w')
// against the cached thresholds (quantize.hpp:253-290, :318-329).
//
// Three launches per step (one stream, no host synchronisation):
//
//   k_step_prep   one thread per row: the row's tier, its per-row constants and CSR
//                 slot bounds (RowPrep, 64 B); rows outside the stable tier are
//                 appended to a device row list for the general kernel.
//   rows_kernel   (this file) every STABLE row, one CTA per row:
//                   phase 1  each thread owns V 16-byte vectors of the row: dequant m,
//                            g (PRMT magic numbers, FADD2/FMUL2) -> m' = b2*m + c2*g,
//                            kept in registers; m' min/max (FMNMX3, CREDUX); weight
//                            codes pass through except boundary-code candidates and
//                            old outliers; STG.128 of the weight codes.
//                   barrier  warp 0: the row's m' range -> affine_from_bounds (fp64),
//                            the CSR segment offsets; the other warps run the sparse
//                            pass of the CTA's NEXT row (one thread per old outlier).
//                   phase 2  quantize m' (range-proven fast quantizer), STG.128; CSR
//                            entries appended in column order.
//   step_kernel   (stepkernel.cu, v5) the rows of the device list: every row the
//                 stable-tier proof does not cover (large lr, weight decay that can
//                 move a code, odd zero points, NaN/Inf, over-full sparse tables).
//
// The stable tier.  Dense weight codes k (not old outliers) have w = RN(sw*(k-zw)).
// One Lion step moves w by at most D = |lr|*(1 + |wd|*Wmax)*(1+2^-20) (sign(d) is
// +-1 or 0, Wmax bounds |w|), so with K = qmax + |zw|
//       D/sw <= 0.5 - (K+2)*2^-21                                         (*)
// puts w'/sw within 0.5 - (rounding slack) of the integer k - zw: the reference's
// round((double)w'/(double)sw) + zw is k again, for EVERY value of m and g.  When
// moreover code(t_min) == 0 and code(t_max) == qmax (the thresholds define the scale,
// so this is the normal case), every code in [1, qmax-1] stays strictly inside
// (t_min, t_max): it can neither become an outlier nor change.  Only codes 0 and qmax
// ("candidates") and the old outliers need the Lion arithmetic, which they get
// exactly (fp32 reference order, fp64 quantizer).  (*) is checked per row in fp64
// (k_step_prep); at the paper's lr = 2e-5 every LLaMA row satisfies it (sw ~ 4e-4 at
// 8 bits).  The output is byte-identical to the reference either way.
#include "qft_device.cuh"
#include "qft_internal.h"

namespace qftk {
using namespace qftd;

namespace rs6 {
constexpr uint32_t I_STABLE = 1u;

struct Smem {  // per-CTA shared-memory layout (runtime sizes)
  int nvec, oldcap, nw;
  __device__ __host__ int buf_bytes() const {
    return ((nvec * 2 + 15) & ~15) + ((nvec * 2 + 15) & ~15) + oldcap * 8;
  }
  __device__ __host__ int o_bits(int b) const { return b * buf_bytes(); }
  __device__ __host__ int o_frank(int b) const { return o_bits(b) + ((nvec * 2 + 15) & ~15); }
  __device__ __host__ int o_spval(int b) const { return o_frank(b) + ((nvec * 2 + 15) & ~15); }
  __device__ __host__ int o_spcw(int b) const { return o_spval(b) + oldcap * 4; }
  __device__ __host__ int o_part() const { return 3 * buf_bytes(); }         // nw x float4
  __device__ __host__ int o_seg() const { return o_part() + nw * 16; }        // nw x int2
  __device__ __host__ int o_res() const { return o_seg() + nw * 8; }          // RowRes
  __device__ __host__ int total() const { return o_res() + 64; }
};

struct RowRes {  // the row's m' quantizer, published by warp 0
  float s, inv, magic, thr;
  float ylo, yhi;
  int32_t z, qmf;
};

// the row's identity and the pointers of the CTA's current row (uniform)
struct RowCtx {
  int gr, tensor, lrow;
  int ob, on, so, co;
  uint32_t zpay;
  DequantRow dm, dg;
  size_t roff;
};

__device__ __forceinline__ RowCtx load_ctx(const LaunchArgs& a, int gr) {
  RowCtx c;
  const RowPrep* p = a.prep + gr;
  const int4 p0 = __ldg(reinterpret_cast<const int4*>(p));
  const int4 p1 = __ldg(reinterpret_cast<const int4*>(p) + 1);
  const int4 p2 = __ldg(reinterpret_cast<const int4*>(p) + 2);
  c.gr = gr;
  c.zpay = ((uint32_t)p0.x >> 8) & 0xFFu;
  c.tensor = p0.y;
  c.lrow = p0.z;
  c.ob = p0.w;
  c.on = p1.x;
  c.so = p1.y;
  c.co = p1.z;
  c.dm = make_dequant_row(__int_as_float(p2.x), p2.y);
  c.dg = make_dequant_row(__int_as_float(p2.z), p2.w);
  c.roff = (size_t)c.lrow * (size_t)p1.w;  // p1.w = cols
  return c;
}

// next row of this CTA's static stride that is in the stable tier
__device__ __forceinline__ int next_stable(const LaunchArgs& a, int gr) {
  while (gr < a.total_rows && !(__ldg(&a.prep[gr].info) & I_STABLE)) gr += gridDim.x;
  return gr;
}

// m' = RN(RN(b2*m) + RN(c2*g)) for a pair: the products are FFMA2s with a RUNTIME -0
// addend (exactly RN(x*y) for every x, y), so ptxas has no FMUL to contract into the
// sum (it fuses FMUL2 + FADD2 into FFMA2 regardless of .rn, see qft_device.cuh).
__device__ __forceinline__ float2 mprime2(float2 m, float2 g, float2 b2, float2 c2, float2 nz) {
  return __fadd2_rn(__ffma2_rn(b2, m, nz), __ffma2_rn(c2, g, nz));
}

// any byte of the 4 words equal to 0 or qmax (b-bit codes: bits >= b are zero):
// byte in {0, qmax} <=> its low b bits are all equal <=> (x ^ x>>1) & K == 0 on the
// byte, K = bits 0..b-2; then the classic zero-byte test.  The flag word is exact for
// "some byte"; per-byte flags may include false positives above a flagged byte
// (harmless: flagged elements take the exact path).
__device__ __forceinline__ uint32_t cand_flags(uint32_t x, uint32_t K) {
  const uint32_t t = (x ^ (x >> 1)) & K;
  return (t - 0x01010101u) & ~t & 0x80808080u;
}
__device__ __forceinline__ uint32_t flags16(uint4 q, uint32_t K) {
  auto f4 = [&](uint32_t x) -> uint32_t {
    const uint32_t f = cand_flags(x, K) >> 7;  // bits 0, 8, 16, 24
    return (f | (f >> 7) | (f >> 14) | (f >> 21)) & 0xFu;
  };
  return f4(q.x) | (f4(q.y) << 4) | (f4(q.z) << 8) | (f4(q.w) << 12);
}

__device__ __forceinline__ uint32_t byte_of(const uint4& q, int e) {
  const int w = e >> 2;
  const uint32_t x = w == 0 ? q.x : (w == 1 ? q.y : (w == 2 ? q.z : q.w));
  return (x >> ((e & 3) * 8)) & 0xFFu;
}
__device__ __forceinline__ void set_byte(uint4& q, int e, uint32_t v) {
  const uint32_t sh = (uint32_t)(e & 3) * 8u;
  const uint32_t keep = ~(0xFFu << sh), put = (v & 0xFFu) << sh;
  const int w = e >> 2;
  q.x = (w == 0) ? ((q.x & keep) | put) : q.x;
  q.y = (w == 1) ? ((q.y & keep) | put) : q.y;
  q.z = (w == 2) ? ((q.z & keep) | put) : q.z;
  q.w = (w == 3) ? ((q.w & keep) | put) : q.w;
}

// exact w' of one dense element from its three codes (lion1: the reference's fp32
// order; dequantize as quantize.hpp:209)
__device__ __forceinline__ float exact_wprime(uint32_t qw, uint32_t qm, uint32_t qg,
                                              const DevTensor* T, int lrow, const RowCtx& c,
                                              const Hyper& h) {
  float w = dequant_exact(qw, __ldg(T->w_scale + lrow), __ldg(T->w_zp + lrow));
  float m = dequant_exact(qm, c.dm.s, c.dm.z);
  const float g = dequant_exact(qg, c.dg.s, c.dg.z);
  lion1(w, m, g, h);
  return w;
}

}  // namespace rs6

int rows_kernel_nt(int cols, int v) {
  const int nvec = (cols + 15) / 16;
  const int per = (nvec + v - 1) / v;
  return ((per + 31) / 32) * 32;
}

size_t rows_kernel_smem(int cols, int v, int oldcap) {
  const int nt = rows_kernel_nt(cols, v);
  rs6::Smem L{nt * v, oldcap, nt / 32};
  return (size_t)L.total();
}

template <int V>
__global__ void __launch_bounds__(512, 1) rows_kernel(const LaunchArgs a) {
  using namespace rs6;
  extern __shared__ __align__(16) uint8_t smem[];
  const int NT = blockDim.x, NW = NT >> 5;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const Smem L{NT * V, a.oldcap6, NW};
  const int qmax = (1 << a.bit_width) - 1;
  const uint32_t KC = (uint32_t)((1 << (a.bit_width - 1)) - 1) * 0x01010101u;
  const int in = a.flip, out = 1 - a.flip;
  const int cols = a.cols_p;  // uniform row length of the launch (multiple of 16)
  const int nvec = cols >> 4;
  Hyper h;
  h.lr = a.lr; h.b1 = a.b1; h.b2 = a.b2; h.wd = a.wd;
  h.c1 = __fsub_rn(1.0f, a.b1);
  h.c2 = __fsub_rn(1.0f, a.b2);
  const float2 B2 = f2(h.b2), C2 = f2(h.c2), NZ = f2(a.negzero);

  auto bits16 = [&](int b) { return reinterpret_cast<uint16_t*>(smem + L.o_bits(b)); };
  auto frank = [&](int b) { return reinterpret_cast<uint16_t*>(smem + L.o_frank(b)); };
  auto spval = [&](int b) { return reinterpret_cast<float*>(smem + L.o_spval(b)); };
  auto spcw = [&](int b) { return reinterpret_cast<uint32_t*>(smem + L.o_spcw(b)); };
  float4* part = reinterpret_cast<float4*>(smem + L.o_part());
  int2* seg = reinterpret_cast<int2*>(smem + L.o_seg());
  RowRes* res = reinterpret_cast<RowRes*>(smem + L.o_res());

  // sparse pass over the OLD outliers of row c into buffer b (threads t0.. of the CTA):
  // the exact w' (general Lion form), its class against the cached thresholds and its
  // code (quantize.hpp:274-285); bitmap + first-rank table for O(1) lookups
  auto sparse_pass = [&](const RowCtx& c, int b, int t0) {
    const DevTensor* T = a.tensors + c.tensor;
    const uint8_t* m_in = T->m_codes[in] + c.roff;
    const uint8_t* g_in = T->g_codes + c.roff;
    const float sw = __ldg(T->w_scale + c.lrow);
    const int32_t zw = __ldg(T->w_zp + c.lrow);
    const float tmin = __ldg(T->t_min + c.lrow), tmax = __ldg(T->t_max + c.lrow);
    uint32_t* bw = reinterpret_cast<uint32_t*>(bits16(b));
    uint16_t* fr = frank(b);
    float* sv = spval(b);
    uint32_t* sc = spcw(b);
    for (int i = t - t0; i < c.on; i += NT - t0) {
      const int col = __ldg(a.col_in + c.ob + i);
      atomicOr(&bw[col >> 5], 1u << (col & 31));
      const int vv = col >> 4;
      if (i == 0 || (__ldg(a.col_in + c.ob + i - 1) >> 4) != vv) fr[vv] = (uint16_t)i;
      float wv = __ldg(a.val_in + c.ob + i);
      float mv = dequant_exact(m_in[col], c.dm.s, c.dm.z);
      const float gv = dequant_exact(g_in[col], c.dg.s, c.dg.z);
      lion1(wv, mv, gv, h);
      const bool o = (wv < tmin) || (wv > tmax);
      const uint32_t code = o ? c.zpay : quant_exact(wv, sw, zw, qmax);
      sv[i] = wv;
      sc[i] = code | (o ? 0x100u : 0u);
    }
  };
  auto clear_bits = [&](int b) {
#pragma unroll
    for (int j = 0; j < V; ++j) bits16(b)[t + j * NT] = 0;
  };

  int gr = next_stable(a, blockIdx.x);
  if (gr >= a.total_rows) return;
  RowCtx cur = load_ctx(a, gr);
  uint4 cw[V], cm[V], cg[V];
  auto load_codes = [&](const RowCtx& c, uint4* wv, uint4* mv, uint4* gv) {
    const DevTensor* T = a.tensors + c.tensor;
    const uint4* w4 = reinterpret_cast<const uint4*>(T->w_codes[in] + c.roff);
    const uint4* m4 = reinterpret_cast<const uint4*>(T->m_codes[in] + c.roff);
    const uint4* g4 = reinterpret_cast<const uint4*>(T->g_codes + c.roff);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int v = t + j * NT;
      if (v < nvec) {
        wv[j] = __ldg(w4 + v);
        mv[j] = __ldg(m4 + v);
        gv[j] = __ldg(g4 + v);
      }
    }
  };
  load_codes(cur, cw, cm, cg);
  clear_bits(0);
  __syncthreads();
  sparse_pass(cur, 0, 0);
  __syncthreads();

  for (int it = 0;; ++it) {
    const int b = it % 3, bn = (it + 1) % 3;
    const int gn = next_stable(a, gr + gridDim.x);
    const bool has_next = gn < a.total_rows;
    RowCtx nxt;
    if (has_next) nxt = load_ctx(a, gn);
    clear_bits(bn);
    const DevTensor* T = a.tensors + cur.tensor;
    uint8_t* w_out = T->w_codes[out] + cur.roff;

    // ================================ phase 1 ================================
    float mp[V][16];
    uint32_t mask[V], o16[V];
    float mlo = __int_as_float(0x7f800000), mhi = __int_as_float(0xff800000);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int v = t + j * NT;
      mask[j] = 0;
      o16[j] = 0;
      if (v < nvec) {
        const uint32_t mw[4] = {cm[j].x, cm[j].y, cm[j].z, cm[j].w};
        const uint32_t gw[4] = {cg[j].x, cg[j].y, cg[j].z, cg[j].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float2 a0 = make_float2(magic_byte(mw[i], 0), magic_byte(mw[i], 1));
          float2 a1 = make_float2(magic_byte(mw[i], 2), magic_byte(mw[i], 3));
          float2 b0 = make_float2(magic_byte(gw[i], 0), magic_byte(gw[i], 1));
          float2 b1 = make_float2(magic_byte(gw[i], 2), magic_byte(gw[i], 3));
          a0 = mul2(add2(a0, f2(cur.dm.negc)), f2(cur.dm.s));
          a1 = mul2(add2(a1, f2(cur.dm.negc)), f2(cur.dm.s));
          b0 = mul2(add2(b0, f2(cur.dg.negc)), f2(cur.dg.s));
          b1 = mul2(add2(b1, f2(cur.dg.negc)), f2(cur.dg.s));
          const float2 r0 = mprime2(a0, b0, B2, C2, NZ);
          const float2 r1 = mprime2(a1, b1, B2, C2, NZ);
          mp[j][4 * i] = r0.x; mp[j][4 * i + 1] = r0.y;
          mp[j][4 * i + 2] = r1.x; mp[j][4 * i + 3] = r1.y;
        }
#pragma unroll
        for (int pp = 0; pp < 8; ++pp) {
          float tt;
          asm("min.f32 %0, %1, %2, %3;" : "=f"(tt) : "f"(mlo), "f"(mp[j][2 * pp]), "f"(mp[j][2 * pp + 1]));
          mlo = tt;
          asm("max.f32 %0, %1, %2, %3;" : "=f"(tt) : "f"(mhi), "f"(mp[j][2 * pp]), "f"(mp[j][2 * pp + 1]));
          mhi = tt;
        }
        // weight codes: pass through, except candidates (codes 0 / qmax) and old outliers
        uint4 wq = cw[j];
        const uint32_t any = (cand_flags(wq.x, KC) | cand_flags(wq.y, KC) |
                              cand_flags(wq.z, KC) | cand_flags(wq.w, KC));
        const uint32_t ob16 = bits16(b)[v];
        o16[j] = ob16;
        if (any | ob16) {
          uint32_t cmask = any ? (flags16(wq, KC) & ~ob16) : 0u;
          uint32_t msk = 0;
          if (cmask) {
            const uint4 q0 = wq;
            const float tmin = __ldg(T->t_min + cur.lrow), tmax = __ldg(T->t_max + cur.lrow);
            const float sw = __ldg(T->w_scale + cur.lrow);
            const int32_t zw = __ldg(T->w_zp + cur.lrow);
            while (cmask) {
              const int e = __ffs(cmask) - 1;
              cmask &= cmask - 1u;
              const float wv = exact_wprime(byte_of(q0, e), byte_of(cm[j], e), byte_of(cg[j], e), T,
                                            cur.lrow, cur, h);
              const bool o = (wv < tmin) || (wv > tmax);
              set_byte(wq, e, o ? cur.zpay : quant_exact(wv, sw, zw, qmax));
              msk |= (o ? 1u : 0u) << e;
            }
          }
          uint32_t om = ob16;
          while (om) {
            const int e = __ffs(om) - 1;
            om &= om - 1u;
            const int rank = frank(b)[v] + __popc(ob16 & ((1u << e) - 1u));
            const uint32_t c = spcw(b)[rank];
            set_byte(wq, e, c);
            msk |= ((c >> 8) & 1u) << e;
          }
          mask[j] = msk;
        }
        __stcs(reinterpret_cast<uint4*>(w_out) + v, wq);
      }
    }
    // prefetch the next row's codes (in flight during the barriers and phase 2)
    if (has_next) load_codes(nxt, cw, cm, cg);

    // warp partials: m' range, CSR counts (packed j=0 | j=1 << 16, prefix-scanned)
    {
      float wlo, whi;
      asm("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(wlo) : "f"(mlo));
      asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(whi) : "f"(mhi));
      mlo = wlo;
      mhi = whi;
    }
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < V; ++j) cnt |= (uint32_t)__popc(mask[j]) << (16 * j);
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t tt = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += tt;
    }
    const uint32_t excl = incl - cnt;
    if (lane == 31) part[wid] = make_float4(mlo, mhi, __uint_as_float(incl), 0.0f);
    __syncthreads();  // ---------------------------------------------------- A

    if (wid == 0) {
      // the row's m' range and CSR segment offsets (segment order: j-major, then warp)
      float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
      uint32_t c = 0;
      if (lane < NW) {
        const float4 pp = part[lane];
        lo = pp.x;
        hi = pp.y;
        c = __float_as_uint(pp.z);
      }
      asm("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(lo) : "f"(lo));
      asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(hi) : "f"(hi));
      uint32_t in0 = c & 0xFFFFu, in1 = c >> 16;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u0 = __shfl_up_sync(0xffffffffu, in0, d);
        const uint32_t u1 = __shfl_up_sync(0xffffffffu, in1, d);
        if (lane >= d) {
          in0 += u0;
          in1 += u1;
        }
      }
      const uint32_t tot0 = __shfl_sync(0xffffffffu, in0, 31);
      const uint32_t tot1 = __shfl_sync(0xffffffffu, in1, 31);
      if (lane < NW)
        seg[lane] = make_int2((int)(in0 - (c & 0xFFFFu)), (int)(tot0 + in1 - (c >> 16)));
      if (lane == 0) {
        float smv = 1.0f;
        int32_t zmv = 0;
        // stable rows have bounded, finite m' (k_step_prep), so lo <= hi
        affine_from_bounds(lo, hi, a.bit_width, smv, zmv);
        const QuantRow qm = make_quant_row(smv, zmv, a.bit_width);
        const bool qmf = qm.fast && code_unclamped(lo, smv, zmv) >= 0.0 &&
                         code_unclamped(hi, smv, zmv) <= (double)qmax;
        RowRes r;
        r.s = smv; r.inv = qm.inv_s; r.magic = qm.magic; r.thr = qm.thr;
        r.ylo = qm.ylo; r.yhi = qm.yhi; r.z = zmv; r.qmf = qmf ? 1 : 0;
        *res = r;
        T->m_scale[out][cur.lrow] = smv;
        T->m_zp[out][cur.lrow] = zmv;
        const int total = (int)(tot0 + tot1);
        T->cnt[out][cur.lrow] = total;
        if (total > cur.co) atomicOr(&a.hdr->overflow, 1u);
      }
      if (NW == 1 && has_next) sparse_pass(nxt, bn, 0);
    } else if (has_next) {
      sparse_pass(nxt, bn, 32);
    }
    __syncthreads();  // ---------------------------------------------------- B

    // ================================ phase 2 ================================
    {
      const RowRes r = *res;
      QuantRow qm;
      qm.s = r.s; qm.inv_s = r.inv; qm.magic = r.magic; qm.thr = r.thr;
      qm.ylo = r.ylo; qm.yhi = r.yhi; qm.z = r.z; qm.qmax = qmax; qm.fast = true;
      uint8_t* m_out = T->m_codes[out] + cur.roff;
      const int2 sg2 = seg[wid];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int v = t + j * NT;
        if (v < nvec) {
          uint32_t cq[4];
          bool ok;
          if (r.qmf) {
            float em = 0.0f;
#pragma unroll
            for (int q = 0; q < 4; ++q) cq[q] = quant4_e(&mp[j][4 * q], qm, em);
            ok = em < qm.thr;
          } else {
            QAcc qa = qacc_init();
#pragma unroll
            for (int q = 0; q < 4; ++q) cq[q] = quant4_nc(&mp[j][4 * q], qm, qa);
            ok = quant_vec_ok(qa, qm);
          }
          if (!ok) {
#pragma unroll
            for (int q = 0; q < 4; ++q) cq[q] = quant4_exact(&mp[j][4 * q], qm);
          }
          __stcs(reinterpret_cast<uint4*>(m_out) + v, make_uint4(cq[0], cq[1], cq[2], cq[3]));
          // CSR entries of this vector (columns ascending)
          uint32_t mm = mask[j];
          if (mm) {
            int pos = (j == 0 ? sg2.x : sg2.y) + (int)((excl >> (16 * j)) & 0xFFFFu);
            const uint8_t* w_in = T->w_codes[in] + cur.roff;
            const uint8_t* m_in = T->m_codes[in] + cur.roff;
            const uint8_t* g_in = T->g_codes + cur.roff;
            while (mm) {
              const int e = __ffs(mm) - 1;
              mm &= mm - 1u;
              const int col = v * 16 + e;
              float val;
              if (o16[j] & (1u << e)) {
                val = spval(b)[frank(b)[v] + __popc(o16[j] & ((1u << e) - 1u))];
              } else {
                val = exact_wprime(w_in[col], m_in[col], g_in[col], T, cur.lrow, cur, h);
              }
              if (pos < cur.co) {
                a.col_out[cur.so + pos] = col;
                a.val_out[cur.so + pos] = val;
              }
              ++pos;
            }
          }
        }
      }
    }
    if (!has_next) break;
    gr = gn;
    cur = nxt;
  }
}

// ---------------------------------------------------------------------------- prep
// One thread per row of the launch: the RowPrep record and the tier decision.
__global__ void k_step_prep(const LaunchArgs a, int stable_ok) {
  const int gr = blockIdx.x * blockDim.x + threadIdx.x;
  if (gr >= a.total_rows) return;
  // tensor of the row (binary search over the row bases)
  int lo = 0, hi = a.n_tensors - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a.tensors[mid].row_base <= gr) lo = mid;
    else hi = mid - 1;
  }
  const DevTensor& T = a.tensors[lo];
  const int r = gr - T.row_base;
  const int in = a.flip, out = 1 - a.flip;
  const int qmax = (1 << a.bit_width) - 1;
  const float sw = T.w_scale[r], tmin = T.t_min[r], tmax = T.t_max[r];
  const int32_t zw = T.w_zp[r];
  const float sm = T.m_scale[in][r];
  const int32_t zm = T.m_zp[in][r];
  const float sg = T.g_scale ? T.g_scale[r] : 0.0f;
  const int32_t zg = T.g_zp ? T.g_zp[r] : 0;
  const int32_t* rsi = T.rs[in];
  const int ob = rsi[r];
  const int cap_in = rsi[r + 1] - ob;
  const int on = T.cnt[in] ? min(T.cnt[in][r], cap_in) : cap_in;
  const int so = T.rs[out][r];
  const int co = T.rs[out][r + 1] - so;
  const int zpay = zw < 0 ? 0 : (zw > qmax ? qmax : zw);

  bool ok = stable_ok != 0 && on <= a.oldcap6;
  ok = ok && make_dequant_row(sw, zw).fast && make_dequant_row(sm, zm).fast &&
       make_dequant_row(sg, zg).fast;
  // positive, normal scales (so 1/s is finite and the dense values are bounded)
  ok = ok && sw >= 0x1.0p-126f && sw <= 0x1.0p100f && sm >= 0x1.0p-126f && sm <= 0x1.0p100f &&
       sg >= 0x1.0p-126f && sg <= 0x1.0p100f;
  if (ok) {
    const double K = (double)qmax + fabs((double)zw);
    // m' = b2*m + c2*g finite: |m|, |g| <= s*(qmax+|z|) <= 2^100 * 2^23, |b2|, |c2| <= 4
    const double c2 = (double)__fsub_rn(1.0f, a.b2);
    ok = (double)sm * ((double)qmax + fabs((double)zm)) <= 0x1.0p120 &&
         (double)sg * ((double)qmax + fabs((double)zg)) <= 0x1.0p120 &&
         fabs((double)a.b2) <= 4.0 && fabs(c2) <= 4.0;
    // thresholds map to the ends of the code range
    ok = ok && (tmin <= tmax) && code_unclamped(tmin, sw, zw) == 0.0 &&
         code_unclamped(tmax, sw, zw) == (double)qmax;
    // (*) the step cannot move a dense code: D/sw <= 0.5 - (K+2)*2^-21
    const double lr = fabs((double)a.lr), wd = fabs((double)a.wd);
    const double wmax = (double)sw * K * (1.0 + 0x1.0p-20);
    const double D = lr * (1.0 + wd * wmax) * (1.0 + 0x1.0p-20);
    ok = ok && isfinite(lr) && isfinite(wd) && D / (double)sw <= 0.5 - (K + 2.0) * 0x1.0p-21;
  }
  RowPrep p;
  p.info = (ok ? rs6::I_STABLE : 0u) | ((uint32_t)zpay << 8);
  p.tensor = lo;
  p.lrow = r;
  p.ob = ob;
  p.on = on;
  p.so = so;
  p.co = co;
  p.cols = T.cols;
  p.sm = sm;
  p.zm = zm;
  p.sg = sg;
  p.zg = zg;
  a.prep[gr] = p;
  if (!ok) {
    const int k = atomicAdd(a.xcount, 1);
    a.xlist[k] = RowBlock{lo, r, 1, 0};
  }
}

// ---------------------------------------------------------------------------- launch
template <int V>
static cudaError_t rows_launch_t(const LaunchArgs& a, int nt, size_t smem, cudaStream_t st) {
  auto k = rows_kernel<V>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, nt, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  long grid = (long)sms * per_sm;
  if (grid > a.total_rows) grid = a.total_rows;
  if (grid < 1) grid = 1;
  k<<<(unsigned)grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}

bool rows_kernel_eligible(int gk, int use_bulk, int uniform_cols) {
  return gk == G_U8 && use_bulk && uniform_cols > 0 && uniform_cols % 16 == 0 &&
         uniform_cols <= 16384;  // <= 512 threads at V = 2
}

int rows_kernel_oldcap(int cols) { return (cols / 16 + 31) & ~31; }

cudaError_t launch_rows_step(const LaunchArgs& a0, cudaStream_t st) {
  LaunchArgs a = a0;
  a.negzero = -0.0f;
  cudaError_t e = cudaMemsetAsync(a.xcount, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return e;
  const int pt = 256;
  const int stable_ok = a.use_bulk ? 1 : 0;
  k_step_prep<<<(a.total_rows + pt - 1) / pt, pt, 0, st>>>(a, stable_ok);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int V = 2;
  const int nt = rows_kernel_nt(a.cols_p, V);
  const size_t smem = rows_kernel_smem(a.cols_p, V, a.oldcap6);
  if ((e = rows_launch_t<2>(a, nt, smem, st)) != cudaSuccess) return e;
  // the general kernel over the device row list
  LaunchArgs x = a;
  x.blocks = a.xlist;
  x.n_blocks = a.total_rows;  // upper bound; the kernel reads the true count
  x.n_blocks_dev = a.xcount;
  return launch_step_kernel(G_U8, x, st);
}

}  // namespace qftk
