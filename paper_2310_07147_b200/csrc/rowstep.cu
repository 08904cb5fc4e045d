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
//   k_step_prep   one thread per row: the row's tier and a self-describing 128-byte
//                 record (RowPrep: per-row constants, CSR slot bounds, absolute row
//                 pointers); rows outside the stable tier are appended to a device row
//                 list for the general kernel.
//   rows_kernel   every STABLE row, one CTA per row, persistent over a static stride:
//                   TMA      thread 0 streams the NEXT row -- record, w | m | g codes,
//                            the old CSR slot -- into a 2-stage shared-memory ring
//                            (cp.async.bulk on an mbarrier), one row ahead.
//                   phase 1  each thread owns V=2 16-byte vectors: dequant m, g (PRMT
//                            magic numbers, FADD2/FMUL2) -> m' = b2*m + c2*g kept in
//                            registers; m' min/max (FMNMX3, CREDUX); weight codes pass
//                            through except boundary-code candidates; STG.128.
//                   barrier A  warp 0: the row's m' range -> affine_from_bounds (fp64),
//                            CSR segment offsets.  The other warps: the deferred output
//                            of the PREVIOUS row's old outliers (code bytes, CSR entries)
//                            and the sparse pass of the NEXT row (one thread per old
//                            outlier, reading the landed stage).
//                   barrier B  phase 2: quantize m' (range-proven fast quantizer),
//                            STG.128; per-vector CSR bases; new-outlier entries.
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
// exactly (fp32 reference order; the quantizer's fp64 formula or its proven fp32
// equivalent).  (*) is checked per row in fp64 (k_step_prep); at the paper's lr = 2e-5
// every LLaMA row satisfies it (sw ~ 4e-4 at 8 bits).  The bytes are the reference's
// either way: rows without the proof run the general kernel.
#include "qft_device.cuh"
#include "qft_internal.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace qftk {
using namespace qftd;

#ifndef QFT_STATIC_ROWS
#define QFT_STATIC_ROWS 0  // 1: static row assignment (A/B of the dynamic row claims)
#endif
#ifndef QFT_CLAIM_K
#define QFT_CLAIM_K 8  // rows per dynamic claim
#endif
#ifndef QFT_OC3
#define QFT_OC3 64  // old-outlier table of the 3-stage class: cols / QFT_OC3 entries
#endif

namespace rs6 {
constexpr uint32_t I_STABLE = 1u;
constexpr uint32_t I_GEN = 0x80u;  // the GEN tier: every code requantized in this kernel
constexpr int V = 2;  // 16-byte vectors per thread

// Per-CTA shared memory (runtime sizes).
//   stage[2]   record (128 B) | w codes | m codes | g codes | old cols | old values
//   bars[2]    the stages' mbarriers
//   buf[3]     sparse buffers (row k of the CTA uses buffer k % 3): a 16-byte header
//              (the row's w_out, so, co), per vector one u32 word -- bits 0..15 the OLD
//              outlier positions, bits 16..31 the OUTPUT outlier positions (old ones
//              that stay, new ones from the candidate path) -- and per old outlier its
//              w' value, code|class, column
//   vbase      CSR base of every vector with outputs (phase 2 -> next row's old_out)
//   part, seg, res  warp partials, CSR segment offsets, the m' quantizer
struct Smem {
  int nvec, oldcap, nw, cols, ns;  // ns: TMA stages (3 on the 128-thread class)
  __device__ __host__ int stage_bytes() const { return 128 + 3 * cols + 8 * oldcap; }
  __device__ __host__ int o_stage(int s) const { return s * stage_bytes(); }
  __device__ __host__ int o_bar() const { return ns * stage_bytes(); }
  __device__ __host__ int buf_bytes() const { return 16 + nvec * 4 + oldcap * 12; }
  __device__ __host__ int o_buf(int b) const { return o_bar() + 32 + b * buf_bytes(); }
  __device__ __host__ int o_vbase() const { return o_buf(3); }
  __device__ __host__ int o_part() const { return o_vbase() + nvec * 4; }
  __device__ __host__ int o_seg() const { return o_part() + nw * 16; }
  __device__ __host__ int o_res() const { return o_seg() + nw * 8; }
  __device__ __host__ int o_rowid() const { return o_res() + 32; }  // int[4]: row of each stage
  __device__ __host__ int total() const { return o_rowid() + 16; }
};

struct BufHdr {  // what the deferred output of a row needs after its stage is reused
  uint8_t* w_out;
  int32_t so, co;
};

struct RowRes {  // the row's m' quantizer, published by warp 0
  float s, inv, magic, thr;
  int32_t z, qmf, _p0, _p1;
};

// the fields the CTA needs to ISSUE a row's copies (loaded one row ahead)
struct RowHead {
  uint32_t info;
  int32_t ob, on;
  const uint8_t *w_in, *m_in, *g_in;
};
__device__ __forceinline__ RowHead load_head(const LaunchArgs& a, int gr) {
  RowHead h;
  const RowPrep* p = a.prep + gr;
  const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(p));
  const ulonglong2 q4 = __ldg(reinterpret_cast<const ulonglong2*>(p) + 4);
  const ulonglong2 q5 = __ldg(reinterpret_cast<const ulonglong2*>(p) + 5);
  h.info = q0.x;
  h.ob = (int32_t)q0.z;
  h.on = (int32_t)q0.w;
  h.w_in = reinterpret_cast<const uint8_t*>(q4.x);
  h.m_in = reinterpret_cast<const uint8_t*>(q4.y);
  h.g_in = reinterpret_cast<const uint8_t*>(q5.x);
  return h;
}

// m' = RN(RN(b2*m) + RN(c2*g)) for a pair: the products are FFMA2s with a RUNTIME -0
// addend (exactly RN(x*y) for every x, y), so ptxas has no FMUL to contract into the
// sum (it fuses FMUL2 + FADD2 into FFMA2 regardless of .rn, see qft_device.cuh).
__device__ __forceinline__ float2 mprime2(float2 m, float2 g, float2 b2, float2 c2, float2 nz) {
  return __fadd2_rn(__ffma2_rn(b2, m, nz), __ffma2_rn(c2, g, nz));
}

// byte in {0, qmax} of b-bit codes (bits >= b are zero) <=> its low b bits are all
// equal <=> (x ^ x>>1) & K == 0 on the byte, K = bits 0..b-2; then the classic
// zero-byte test.  Exact for "some byte"; per-byte flags may include false positives
// above a flagged byte (harmless: flagged elements take the exact path).
__device__ __forceinline__ uint32_t cand_flags(uint32_t x, uint32_t K) {
  const uint32_t t = (x ^ (x >> 1)) & K;
  return (t - 0x01010101u) & ~t & 0x80808080u;
}
// bytes equal to zero (flag exact for "some byte"; neighbours may be false positives)
__device__ __forceinline__ uint32_t zero_flags(uint32_t x) {
  return (x - 0x01010101u) & ~x & 0x80808080u;
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

// Rare exact paths out of line: their fp64 divides (and the divide's slow-path call)
// would otherwise set the kernel's register budget while the hot state is live.
__device__ __noinline__ uint32_t quant_exact_ni(float x, float s, int32_t z, int qmax) {
  return quant_exact(x, s, z, qmax);
}
__device__ __noinline__ void affine_ni(float lo, float hi, int bw, float* s, int32_t* z) {
  affine_from_bounds(lo, hi, bw, *s, *z);
}

// code of an INLIER weight of a stable row (its exact code lies in [0, qmax], proven
// by code(t_min) == 0 and code(t_max) == qmax): the fast quantizer with its tie proof,
// the reference's fp64 formula when the proof fails
__device__ __forceinline__ uint32_t quant_inlier(float x, float sw, int32_t zw, int bw) {
  const QuantRow q = make_quant_row(sw, zw, bw);
  const float y = __fmul_rn(x, q.inv_s);
  const float tt = __fadd_rn(y, q.magic);
  const float e = __fsub_rn(y, __fsub_rn(tt, q.magic));
  if (q.fast && fabsf(e) < q.thr && y > q.ylo - 0.5f && y < q.yhi + 0.5f)
    return __float_as_uint(tt) & 0xFFu;
  return quant_exact_ni(x, sw, zw, q.qmax);
}

// exact w' of one dense element from its three codes (lion1: the reference's fp32
// order; dequantize as quantize.hpp:209), the row's record in r
__device__ __forceinline__ float exact_wprime(uint32_t qw, uint32_t qm, uint32_t qg,
                                              const RowPrep& r, const Hyper& h) {
  float w = dequant_exact(qw, r.sw, r.zw);
  float m = dequant_exact(qm, r.sm, r.zm);
  const float g = dequant_exact(qg, r.sg, r.zg);
  lion1(w, m, g, h);
  return w;
}

// w' = w - lr*(sign(d) + wd*w) for a pair (lion_apply, optimizer.hpp:38) given d: with
// weight decay 0 the update is exactly -copysign(lr, d) or nothing (d == +-0; w is finite),
// else the general form in the reference's order (see lion2 in qft_device.cuh)
__device__ __forceinline__ float2 gen_lion(float2 w, float2 d, const Hyper& h, uint32_t nlr) {
  if (h.wd == 0.0f) {
    asm("{\n\t.reg .pred p;\n\t"
        "setp.gt.f32 p, %1, 0f00000000;\n\t"
        "@p add.rn.f32 %0, %0, %2;\n\t}"
        : "+f"(w.x)
        : "f"(fabsf(d.x)), "f"(neg_lr_sign(d.x, nlr)));
    asm("{\n\t.reg .pred p;\n\t"
        "setp.gt.f32 p, %1, 0f00000000;\n\t"
        "@p add.rn.f32 %0, %0, %2;\n\t}"
        : "+f"(w.y)
        : "f"(fabsf(d.y)), "f"(neg_lr_sign(d.y, nlr)));
    return w;
  }
  const float2 sg = make_float2(sign_of(d.x), sign_of(d.y));
  const float2 upd = mul2(f2(h.lr), sadd2(sg, mul2(f2(h.wd), w)));
  return sadd2(w, neg2(upd));
}

// A GEN-tier vector whose fast quantization came near a tie: every code of the 16 exactly
// (quant_exact32: the fp32 tie decision; out of line: rare)
__device__ __noinline__ void gen_vec_exact(uint4 cw, uint4 cm, uint4 cg, const RowPrep& R,
                                           const Hyper& h, int bw, uint32_t* cq,
                                           uint32_t& mask) {
  const int qmax = (1 << bw) - 1;
  const uint32_t zpay = (R.info >> 8) & 0xFFu;
  const float inv = __frcp_rn(R.sw);
  const float lim = fmaxf(fabsf((float)R.zw), fabsf((float)(qmax - R.zw))) + 2.0f;
  const bool x32 = R.sw >= 0x1.0p-100f && R.sw <= 0x1.0p125f && lim < 1048576.0f;
  const uint32_t ww[4] = {cw.x, cw.y, cw.z, cw.w};
  const uint32_t mw[4] = {cm.x, cm.y, cm.z, cm.w};
  const uint32_t gw[4] = {cg.x, cg.y, cg.z, cg.w};
  mask = 0;
  for (int i = 0; i < 4; ++i) {
    uint32_t c = 0;
    for (int e = 0; e < 4; ++e) {
      float w = dequant_exact((ww[i] >> (8 * e)) & 0xFFu, R.sw, R.zw);
      float m = dequant_exact((mw[i] >> (8 * e)) & 0xFFu, R.sm, R.zm);
      const float g = dequant_exact((gw[i] >> (8 * e)) & 0xFFu, R.sg, R.zg);
      lion1(w, m, g, h);
      const bool o = (w < R.tmin) || (w > R.tmax);
      if (o) mask |= 1u << (4 * i + e);
#if QFT_EXACT32
      c |= (o ? zpay : (x32 ? quant_exact32(w, R.sw, inv, R.zw, qmax)
                            : quant_exact(w, R.sw, R.zw, qmax))) << (8 * e);
#else
      c |= (o ? zpay : quant_exact(w, R.sw, R.zw, qmax)) << (8 * e);
#endif
    }
    cq[i] = c;
  }
}

}  // namespace rs6

int rows_kernel_nt(int cols) {
  const int nvec = (cols + 15) / 16;
  const int per = (nvec + rs6::V - 1) / rs6::V;
  return ((per + 31) / 32) * 32;
}

// TMA stages: 3 where the smem budget keeps 5 CTAs/SM (rows <= 4096 columns, old-outlier
// table cols/64: 64 entries at 4096 columns; rows with more old outliers take the
// general kernel), else 2 (table cols/16)
static int rows_kernel_ns(int cols) { return rows_kernel_nt(cols) <= 128 ? 3 : 2; }
int rows_kernel_oldcap(int cols) {
  return ((rows_kernel_ns(cols) == 3 ? cols / QFT_OC3 : cols / 16) + 31) & ~31;
}

size_t rows_kernel_smem(int cols, int oldcap) {
  const int nt = rows_kernel_nt(cols);
  rs6::Smem L{nt * rs6::V, oldcap, nt / 32, ((cols + 15) / 16) * 16, rows_kernel_ns(cols)};
  return (size_t)L.total();
}

#ifndef QFT_BW8
#define QFT_BW8 1
#endif
#ifndef QFT_BW34
#define QFT_BW34 1
#endif
// compile-time row geometry of a CCOLS-column instance (rows_kernel_nt / _oldcap)
__host__ __device__ constexpr int geom_nt(int cols) {
  return ((((cols + 15) / 16 + rs6::V - 1) / rs6::V + 31) / 32) * 32;
}
__host__ __device__ constexpr int geom_oldcap(int cols, int ns) {
  return ((ns >= 3 ? cols / QFT_OC3 : cols / 16) + 31) & ~31;
}

// FULL (2): every thread owns V whole vectors of the row (cols == blockDim.x * V * 16);
// FIRST (1): every thread's first vector is inside the row (nvec >= blockDim.x).  The
// per-vector bounds checks they cover vanish at compile time.
// CCOLS > 0: the launch's row length is the compile-time constant CCOLS (LLaMA widths)
// and its input CSR is slotted; BWC > 0: the bit width is the constant BWC
template <int MAXT, int MINB, int NS, int FULL, int CCOLS, int BWC, bool GEN>
__global__ void __launch_bounds__(MAXT, MINB) rows_kernel(const LaunchArgs a) {
  using namespace rs6;
  // the tier this instance runs (its row list holds only such rows; the flag is checked
  // again from the record)
  constexpr uint32_t I_ACT = GEN ? I_GEN : I_STABLE;
  extern __shared__ __align__(128) uint8_t smem[];
  // CCOLS: the row geometry is a compile-time constant (threads, columns, old-outlier
  // table), so every shared-memory offset folds
  constexpr bool CG = CCOLS > 0;
  const int NT = CG ? geom_nt(CCOLS) : (int)blockDim.x, NW = NT >> 5;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  // uniform row length of the launch (multiple of 16)
  const int cols = CG ? CCOLS : a.cols_p;
  const int nvec = cols >> 4;
  const Smem L{NT * V, CG ? geom_oldcap(CCOLS, NS) : a.oldcap6, NW, cols, NS};
  const int bw = BWC > 0 ? BWC : a.bit_width;
  const int qmax = (1 << bw) - 1;
  const uint32_t KC = (uint32_t)((1 << (bw - 1)) - 1) * 0x01010101u;
  const uint32_t QB = (uint32_t)qmax * 0x01010101u;
  const bool slotted = CG || a.slotted_in != 0;
  Hyper h;
  h.lr = a.lr; h.b1 = a.b1; h.b2 = a.b2; h.wd = a.wd;
  h.c1 = __fsub_rn(1.0f, a.b1);
  h.c2 = __fsub_rn(1.0f, a.b2);
  const float2 B2 = f2(h.b2), C2 = f2(h.c2), NZ = f2(a.negzero);
  const float2 B1 = f2(h.b1), C1 = f2(h.c1);
  const uint32_t nlr = __float_as_uint(-h.lr);
  const double rq = __drcp_rn((double)qmax);

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.o_bar());
  auto stage = [&](int s) { return smem + L.o_stage(s); };
  auto rec = [&](int s) { return reinterpret_cast<const RowPrep*>(stage(s)); };
  auto hdr = [&](int b) { return reinterpret_cast<BufHdr*>(smem + L.o_buf(b)); };
  auto words = [&](int b) { return reinterpret_cast<uint32_t*>(smem + L.o_buf(b) + 16); };
  auto spval = [&](int b) {
    return reinterpret_cast<float*>(smem + L.o_buf(b) + 16 + L.nvec * 4);
  };
  auto spcw = [&](int b) { return reinterpret_cast<uint32_t*>(spval(b) + L.oldcap); };
  auto spcol = [&](int b) { return reinterpret_cast<int32_t*>(spval(b) + 2 * L.oldcap); };
  int* vbase = reinterpret_cast<int*>(smem + L.o_vbase());
  float4* part = reinterpret_cast<float4*>(smem + L.o_part());
  int2* seg = reinterpret_cast<int2*>(smem + L.o_seg());
  RowRes* res = reinterpret_cast<RowRes*>(smem + L.o_res());
  volatile int* rowid = reinterpret_cast<volatile int*>(smem + L.o_rowid());

  // thread 0: the row's record, codes and old CSR slot into stage s (TMA bulk copies)
  auto issue_row = [&](int grow, const RowHead& hd, int s) {
    uint8_t* dst = stage(s);
    const uint32_t n = (uint32_t)cols;
    const uint32_t cb = (slotted && hd.on > 0) ? (uint32_t)((hd.on * 4 + 15) & ~15) : 0u;
    mbar_arrive_expect_tx(&bars[s], 128u + 3u * n + 2u * cb);
    bulk_g2s(dst, a.prep + grow, 128u, &bars[s]);
    bulk_g2s(dst + 128, hd.w_in, n, &bars[s]);
    bulk_g2s(dst + 128 + n, hd.m_in, n, &bars[s]);
    bulk_g2s(dst + 128 + 2 * n, hd.g_in, n, &bars[s]);
    if (cb) {
      bulk_g2s(dst + 128 + 3 * n, a.col_in + hd.ob, cb, &bars[s]);
      bulk_g2s(dst + 128 + 3 * n + 4 * L.oldcap, a.val_in + hd.ob, cb, &bars[s]);
    }
  };
  // Sparse pass over the OLD outliers of the row in stage s into buffer b (threads t0..
  // of the CTA): the exact w' (general Lion form), its class against the cached
  // thresholds and its code (quantize.hpp:274-285); marks bit e (old) and bit 16+e
  // (stays an outlier) of its vector's word.
  auto sparse_pass = [&](int s, int b, int t0, int t1) {  // threads [t0, t1)
    const RowPrep& r = *rec(s);
    const uint8_t* st = stage(s);
    const int32_t* cin = slotted ? reinterpret_cast<const int32_t*>(st + 128 + 3 * cols)
                                 : a.col_in + r.ob;
    const float* vin = slotted ? reinterpret_cast<const float*>(st + 128 + 3 * cols + 4 * L.oldcap)
                               : a.val_in + r.ob;
    const uint32_t zpay = (r.info >> 8) & 0xFFu;
    uint32_t* wd = words(b);
    if (t == t0) *hdr(b) = BufHdr{r.w_out, r.so, r.co};
    if (t < t0 || t >= t1) return;
    for (int i = t - t0; i < r.on; i += t1 - t0) {
      const int col = cin[i];
      float wv = vin[i];
      float mv = dequant_exact(st[128 + cols + col], r.sm, r.zm);
      const float gv = dequant_exact(st[128 + 2 * cols + col], r.sg, r.zg);
      lion1(wv, mv, gv, h);
      const bool o = (wv < r.tmin) || (wv > r.tmax);
      const uint32_t code = o ? zpay : quant_inlier(wv, r.sw, r.zw, bw);
      atomicOr(&wd[col >> 4], (1u << (col & 15)) | (o ? (0x10000u << (col & 15)) : 0u));
      spval(b)[i] = wv;
      spcw(b)[i] = code | (o ? 0x100u : 0u);
      spcol(b)[i] = col;
    }
  };
  // Deferred output of a row's old outliers (after its phase 2 published vbase): the
  // weight code byte over the payload left by the dense pass and, for those that stay
  // outliers, the CSR entry at its column-ordered position.
  auto old_out = [&](int b, int on, int t0, int t1) {  // threads [t0, t1)
    const BufHdr hd = *hdr(b);
    const uint32_t* wd = words(b);
    if (t < t0 || t >= t1) return;
    for (int i = t - t0; i < on; i += t1 - t0) {
      const uint32_t cw = spcw(b)[i];
      const int col = spcol(b)[i];
      hd.w_out[col] = (uint8_t)(cw & 0xFFu);
      if (cw & 0x100u) {
        const int v = col >> 4, e = col & 15;
        const int pos = vbase[v] + __popc((wd[v] >> 16) & ((1u << e) - 1u));
        if (pos < hd.co) {
          a.col_out[hd.so + pos] = col;
          a.val_out[hd.so + pos] = spval(b)[i];
        }
      }
    }
  };
  auto clear_words = [&](int b) {
#pragma unroll
    for (int j = 0; j < V; ++j) words(b)[t + j * NT] = 0u;
  };

  // ---------------------------------------------------------------- prologue
  // Rows are CLAIMED dynamically (one atomic per row on the launch's counter, zeroed by
  // k_step_prep), so CTAs that start late -- e.g. behind a concurrently running width
  // class -- simply take fewer rows.  The issuing thread claims two rows ahead of the one
  // it streams (the atomic's result is not needed until the next issue, and the row's
  // record head is loaded one issue ahead), writes the row index of every stage to
  // rowid[] before the stage's arrive, and arrives without data (a sentinel, rowid -1)
  // once the rows are exhausted.  Rows outside the stable tier still flow through the
  // pipeline (their record says so) but do no work here.
  const int TR = a.total_rows;
  // The issuing thread streams row it+NS-1 each iteration.  With 2 stages that is
  // thread 0 at the top of the iteration; with 3 it is the last warp's lane 0 inside
  // the barrier window, where that warp has no other work (off the phase-1 path).
  const int ti = (NS == 3 && NW > 1) ? NT - 32 : 0;
  // The launch iterates a ROW LIST (k_step_prep's list of this tier's rows, in nearly
  // ascending row order).  List positions are claimed in chunks of QFT_CLAIM_K; the
  // issuer runs three deep: position claimed -> row read from the list -> record head
  // loaded -> row streamed, each result consumed one issue after it was requested.
  RowHead hn{};   // issuing thread: the head of the row it streams next ...
  int nxt = TR;   // ... that row (>= TR: none)
  int nxt2 = TR;  // the row after it (claimed / read from the list one issue ahead)
  // Rows (the stable instance: every row of the launch; rows outside the stable tier flow
  // through without work) or list positions (the GEN instance: k_step_prep's list of GEN
  // rows) are claimed in chunks of QFT_CLAIM_K consecutive ones; the next chunk's atomic is
  // issued when the current one is taken, so its result is needed only K claims later.
  int sc = blockIdx.x;  // QFT_STATIC_ROWS: the static sequence blockIdx.x + k*gridDim.x
  int c_cur = 0, c_end = 0, c_pend = 0;
  int cnt_l = 0;  // GEN: the list length
  auto claim = [&]() -> int {
    if (QFT_STATIC_ROWS) {
      const int r = sc;
      sc += (int)gridDim.x;
      return r;
    }
    if (c_cur == c_end) {
      if (c_end == 0) c_pend = atomicAdd(a.rclaim, QFT_CLAIM_K);  // the first chunk
      c_cur = c_pend;
      c_end = c_pend + QFT_CLAIM_K;
      c_pend = atomicAdd(a.rclaim, QFT_CLAIM_K);
    }
    return c_cur++;
  };
  auto next_row = [&]() -> int {
    if constexpr (GEN) {
      const int pos = claim();
      return pos < cnt_l ? __ldg(a.rlist + pos) : TR;
    } else {
      return claim();
    }
  };
  auto issue_or_end = [&](int s) {
    if (nxt < TR) {
      rowid[s] = nxt;
      issue_row(nxt, hn, s);
    } else {
      rowid[s] = -1;
      mbar_arrive(&bars[s]);  // sentinel: completes the stage's phase without data
    }
    nxt = nxt2;
    if (nxt < TR) hn = load_head(a, nxt);
    nxt2 = next_row();
  };
  if (t == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  clear_words(0);
  __syncthreads();
  if (t == ti) {
    if constexpr (GEN) {
      cnt_l = *a.rcount;
      if (a.xseen && blockIdx.x == 0) {
        *reinterpret_cast<volatile int32_t*>(a.xseen) = cnt_l;
        // the stable rows k_step_prep counted (routed or not): next step's routing decision
        if (a.scount) reinterpret_cast<volatile int32_t*>(a.xseen)[1] = *a.scount;
      }
    }
    nxt = next_row();
    if (nxt < TR) hn = load_head(a, nxt);
    nxt2 = next_row();
    for (int i = 0; i < NS - 1; ++i) issue_or_end(i);
  }
  mbar_wait(&bars[0], 0u);
  int gr = rowid[0];
  if (gr < 0) return;  // no row for this CTA (its other stages hold sentinels too)
  if (rec(0)->info & I_ACT) sparse_pass(0, 0, 0, NT);
  int on_prev = (rec(0)->info & I_ACT) ? rec(0)->on : 0;
  __syncthreads();

  const int tw = NW > 1 ? 32 : 0;  // first thread of the deferred / sparse work
  int it = 0;
  for (;; ++it) {
    const int b = it % 3, bn = (it + 1) % 3, bp = (it + 2) % 3;
    const int s = it % NS, sn = (it + 1) % NS;
    auto issue_ahead = [&]() {
      if (t == ti) issue_or_end((it + NS - 1) % NS);
    };
    if (NS == 2) issue_ahead();
    clear_words(bn);
    mbar_wait(&bars[s], (uint32_t)((it / NS) & 1));
    const RowPrep& R = *rec(s);
    const bool stable = (R.info & I_ACT) != 0;  // (the GEN instance: "active")
    const uint8_t* st = stage(s);
    const float negc_m = R.negc_m, sm = R.sm, negc_g = R.negc_g, sg = R.sg;
    uint8_t* const m_out = R.m_out;
    // boundary codes 0 / qmax need the candidate path only if one of their tabulated
    // outcomes differs from "same code, inlier" (k_step_prep)
    const uint32_t need =
        (((R.cand & 0xFFFFFFu) != 0u || (R.info & (7u << 1)) != 0u) ? 1u : 0u) |
        ((((R.cand >> 24) & 0xFFu) != (uint32_t)qmax || (R.info >> 16) != ((uint32_t)qmax * 0x101u) ||
          (R.info & (7u << 4)) != 0u) ? 2u : 0u);
    const int so = R.so, co = R.co, on_cur = stable ? R.on : 0;
    // GEN tier: the row's weight dequant / quantizer constants and the payload value
    float gw_s = 0.0f, gw_negc = 0.0f, gw_z = 0.0f;
    QuantRow gw_q{};
    if constexpr (GEN) {
      gw_s = R.sw;
      gw_negc = -__fadd_rn(8388608.0f, (float)R.zw);
      gw_z = dequant_exact((R.info >> 8) & 0xFFu, R.sw, R.zw);
      gw_q = make_quant_row(R.sw, R.zw, bw);
    }

    // ================================ phase 1 ================================
    float mp[V][16];
    uint32_t nmask[V], out16[V];
    float mlo = __int_as_float(0x7f800000), mhi = __int_as_float(0xff800000);
    uint32_t cnt = 0;
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const int v = t + j * NT;
      nmask[j] = 0;
      out16[j] = 0;
      if (stable && (FULL == 2 || (FULL == 1 && j == 0) || v < nvec)) {
        const uint4 cwj = *reinterpret_cast<const uint4*>(st + 128 + v * 16);
        const uint4 cmj = *reinterpret_cast<const uint4*>(st + 128 + cols + v * 16);
        const uint4 cgj = *reinterpret_cast<const uint4*>(st + 128 + 2 * cols + v * 16);
        if constexpr (GEN) {
          // ---- the GEN tier: every dense weight through the reference arithmetic --
          // w = dequant (quantize.hpp:209), Lion (optimizer.hpp:33-40, fp32, separate
          // roundings), the outlier test against the cached thresholds and the code
          // (quantize.hpp:274-285) -- with the range-proven fast quantizer (the row's
          // thresholds map to codes 0 and qmax, so an inlier never needs the clip);
          // outliers take the payload value wz (its code is the payload, exactly)
          const uint32_t mw[4] = {cmj.x, cmj.y, cmj.z, cmj.w};
          const uint32_t gw[4] = {cgj.x, cgj.y, cgj.z, cgj.w};
          const uint32_t ww[4] = {cwj.x, cwj.y, cwj.z, cwj.w};
          uint32_t cq[4], mask = 0;
          float em = 0.0f;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float2 a0 = make_float2(magic_byte(mw[i], 0), magic_byte(mw[i], 1));
            float2 a1 = make_float2(magic_byte(mw[i], 2), magic_byte(mw[i], 3));
            float2 b0 = make_float2(magic_byte(gw[i], 0), magic_byte(gw[i], 1));
            float2 b1 = make_float2(magic_byte(gw[i], 2), magic_byte(gw[i], 3));
            float2 w0 = make_float2(magic_byte(ww[i], 0), magic_byte(ww[i], 1));
            float2 w1 = make_float2(magic_byte(ww[i], 2), magic_byte(ww[i], 3));
            a0 = mul2(add2(a0, f2(negc_m)), f2(sm));
            a1 = mul2(add2(a1, f2(negc_m)), f2(sm));
            b0 = mul2(add2(b0, f2(negc_g)), f2(sg));
            b1 = mul2(add2(b1, f2(negc_g)), f2(sg));
            w0 = mul2(add2(w0, f2(gw_negc)), f2(gw_s));
            w1 = mul2(add2(w1, f2(gw_negc)), f2(gw_s));
            const float2 r0 = mprime2(a0, b0, B2, C2, NZ);
            const float2 r1 = mprime2(a1, b1, B2, C2, NZ);
            mp[j][4 * i] = r0.x; mp[j][4 * i + 1] = r0.y;
            mp[j][4 * i + 2] = r1.x; mp[j][4 * i + 3] = r1.y;
            const float2 d0 = mprime2(a0, b0, B1, C1, NZ);  // d = RN(RN(b1 m) + RN(c1 g))
            const float2 d1 = mprime2(a1, b1, B1, C1, NZ);
            w0 = gen_lion(w0, d0, h, nlr);
            w1 = gen_lion(w1, d1, h, nlr);
            float q4[4];
            q4[0] = outlier_select(w0.x, R.tmin, R.tmax, gw_z, 1u << (4 * i), mask);
            q4[1] = outlier_select(w0.y, R.tmin, R.tmax, gw_z, 2u << (4 * i), mask);
            q4[2] = outlier_select(w1.x, R.tmin, R.tmax, gw_z, 4u << (4 * i), mask);
            q4[3] = outlier_select(w1.y, R.tmin, R.tmax, gw_z, 8u << (4 * i), mask);
            cq[i] = quant4_e(q4, gw_q, em);
          }
#pragma unroll
          for (int pp = 0; pp < 8; ++pp) {
            float tt;
            asm("min.f32 %0, %1, %2, %3;" : "=f"(tt) : "f"(mlo), "f"(mp[j][2 * pp]), "f"(mp[j][2 * pp + 1]));
            mlo = tt;
            asm("max.f32 %0, %1, %2, %3;" : "=f"(tt) : "f"(mhi), "f"(mp[j][2 * pp]), "f"(mp[j][2 * pp + 1]));
            mhi = tt;
          }
          if (!(em < gw_q.thr)) gen_vec_exact(cwj, cmj, cgj, R, h, bw, cq, mask);  // near a tie
          const uint32_t wrd = words(b)[v];
          // old-outlier positions: class and code come from the sparse pass (old_out)
          const uint32_t dn = mask & ~(wrd & 0xFFFFu);
          const uint32_t o16 = dn | (wrd >> 16);
          nmask[j] = dn;
          if (dn) atomicOr(&words(b)[v], dn << 16);
          out16[j] = o16;
          cnt |= (uint32_t)__popc(o16) << (16 * j);
          __stcs(reinterpret_cast<uint4*>(R.w_out) + v, make_uint4(cq[0], cq[1], cq[2], cq[3]));
        } else {
        const uint32_t mw[4] = {cmj.x, cmj.y, cmj.z, cmj.w};
        const uint32_t gw[4] = {cgj.x, cgj.y, cgj.z, cgj.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float2 a0 = make_float2(magic_byte(mw[i], 0), magic_byte(mw[i], 1));
          float2 a1 = make_float2(magic_byte(mw[i], 2), magic_byte(mw[i], 3));
          float2 b0 = make_float2(magic_byte(gw[i], 0), magic_byte(gw[i], 1));
          float2 b1 = make_float2(magic_byte(gw[i], 2), magic_byte(gw[i], 3));
          a0 = mul2(add2(a0, f2(negc_m)), f2(sm));
          a1 = mul2(add2(a1, f2(negc_m)), f2(sm));
          b0 = mul2(add2(b0, f2(negc_g)), f2(sg));
          b1 = mul2(add2(b1, f2(negc_g)), f2(sg));
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
        // weight codes pass through; candidates (codes 0 / qmax, not old outliers) get
        // the exact Lion step; old-outlier bytes are rewritten by old_out()
        uint4 wq = cwj;
        const uint32_t wrd = words(b)[v];
        // detect only the boundary codes whose step can change them (row-uniform)
        uint32_t any = 0;
        if (need == 3u) {
          any = cand_flags(wq.x, KC) | cand_flags(wq.y, KC) | cand_flags(wq.z, KC) |
                cand_flags(wq.w, KC);
        } else if (need == 1u) {
          any = zero_flags(wq.x) | zero_flags(wq.y) | zero_flags(wq.z) | zero_flags(wq.w);
        } else if (need == 2u) {
          any = zero_flags(wq.x ^ QB) | zero_flags(wq.y ^ QB) | zero_flags(wq.z ^ QB) |
                zero_flags(wq.w ^ QB);
        }
        uint32_t o16 = wrd >> 16;
        if (any) {
          uint32_t cmask = flags16(wq, KC) & ~(wrd & 0xFFFFu);
          if (cmask) {
            // a dense code-0 / code-qmax weight has one value per row, so its step has 3
            // possible outcomes (k_step_prep tabulates them): only sign(d) is needed,
            // d = b1*m + (1-b1)*g in the reference order (optimizer.hpp:36)
            const uint4 q0 = wq;
            uint32_t nm = 0;
            while (cmask) {
              const int e = __ffs(cmask) - 1;
              cmask &= cmask - 1u;
              const uint32_t c = byte_of(q0, e);
              // SWAR false positives and boundary codes the step cannot change: stable
              if (c == 0u ? !(need & 1u) : (c == (uint32_t)qmax ? !(need & 2u) : true)) continue;
              const float mv = __fmul_rn(__fadd_rn(magic_byte(byte_of(cmj, e), 0), negc_m), sm);
              const float gv = __fmul_rn(__fadd_rn(magic_byte(byte_of(cgj, e), 0), negc_g), sg);
              const float d = __fadd_rn(__fmul_rn(h.b1, mv), __fmul_rn(h.c1, gv));
              const int k = (c ? 3 : 0) + (d > 0.0f ? 2 : (d < 0.0f ? 0 : 1));
              const uint32_t code = k < 4 ? (R.cand >> (8 * k)) & 0xFFu
                                          : (R.info >> (16 + 8 * (k - 4))) & 0xFFu;
              set_byte(wq, e, code);
              nm |= ((R.info >> (1 + k)) & 1u) << e;
            }
            if (nm) {
              atomicOr(&words(b)[v], nm << 16);
              o16 |= nm;
              nmask[j] = nm;
            }
          }
        }
        out16[j] = o16;
        cnt |= (uint32_t)__popc(o16) << (16 * j);
        __stcs(reinterpret_cast<uint4*>(R.w_out) + v, wq);
        }  // stable tier
      }
    }

    // warp partials: m' range, CSR counts (packed j=0 | j=1 << 16, prefix-scanned)
    asm("redux.sync.min.f32 %0, %1, 0xffffffff;" : "=f"(mlo) : "f"(mlo));
    asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(mhi) : "f"(mhi));
    uint32_t incl = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t tt = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += tt;
    }
    const uint32_t excl = incl - cnt;
    if (lane == 31) part[wid] = make_float4(mlo, mhi, __uint_as_float(incl), 0.0f);
    __syncthreads();  // ---------------------------------------------------- A
    // the next row's index was stored before a CTA barrier (its issue precedes barrier A
    // of this iteration with 2 stages, barrier B of the previous one with 3)
    const int gn = rowid[sn];
    const bool has_next = gn >= 0;

    if (wid == 0) {
      if (stable) {
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
        // (the FMA-verified fast divide pays off where more warps wait on this chain:
        // the wide-row instances; measured same-run, slower on the 128-thread one)
        if (!(MAXT > 128 && affine_fast(lo, hi, (double)qmax, rq, smv, zmv)))
          affine_ni(lo, hi, bw, &smv, &zmv);
        const QuantRow qm = make_quant_row(smv, zmv, bw);
        // every m' lies in [lo, hi]: if their codes need no clip (proven with the fast
        // quantizer's own tie bound), no code of the row does
        float em = 0.0f;
        const float lh[4] = {lo, hi, lo, hi};
        (void)quant4_e(lh, qm, em);
        const float ylo = __fmul_rn(lo, qm.inv_s), yhi = __fmul_rn(hi, qm.inv_s);
        const bool qmf = qm.fast && em < qm.thr && ylo > qm.ylo - 0.5f && yhi < qm.yhi + 0.5f;
        RowRes rr;
        rr.s = smv; rr.inv = qm.inv_s; rr.magic = qm.magic; rr.thr = qm.thr;
        rr.z = zmv; rr.qmf = qmf ? 1 : 0;
        *res = rr;
        *R.m_scale_out = smv;
        *R.m_zp_out = zmv;
        const int total = (int)(tot0 + tot1);
        *R.cnt_out = total;
        if (total > co) {
          atomicOr(&a.hdr->overflow, 1u);
          if (a.oflag) *reinterpret_cast<volatile uint32_t*>(a.oflag) = 1u;
        }
      }
      }
      if (NW == 1) {
        if (NS == 3) issue_ahead();
        if (it > 0) old_out(bp, on_prev, 0, NT);
        if (has_next) {
          mbar_wait(&bars[sn], (uint32_t)(((it + 1) / NS) & 1));
          if (rec(sn)->info & I_ACT) sparse_pass(sn, bn, 0, NT);
        }
      }
    } else {
      if (NS == 3) issue_ahead();
      // The next row's sparse pass and the previous row's CSR output on disjoint warps,
      // so no warp runs both chains: on the 3-stage class the output takes the last
      // warp (which also issues the TMA)
      // (8+ warps: the output on the last 4, one iteration for ~100 old outliers)
      const int ts = (NS == 3 && NW >= 4) ? NT - 32 : (NW >= 8 ? NT - 128 : NT);
      if (it > 0) old_out(bp, on_prev, ts < NT ? ts : tw, NT);
      if (has_next && t < ts) {  // the next row's old outliers, from its landed stage
        mbar_wait(&bars[sn], (uint32_t)(((it + 1) / NS) & 1));
        if (rec(sn)->info & I_ACT) sparse_pass(sn, bn, tw, ts);
      }
    }
    __syncthreads();  // ---------------------------------------------------- B

    // ================================ phase 2 ================================
    // (the stage is not read after B: thread 0 refills it at the next row's start)
    if (stable) {
      const RowRes r = *res;
      QuantRow qm;
      qm.s = r.s; qm.inv_s = r.inv; qm.magic = r.magic; qm.thr = r.thr;
      qm.z = r.z; qm.qmax = qmax; qm.fast = true;
      qm.ylo = (float)(-r.z);
      qm.yhi = (float)(qmax - r.z);
      const int2 sg2 = seg[wid];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int v = t + j * NT;
        if (FULL == 2 || (FULL == 1 && j == 0) || v < nvec) {
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
          if (out16[j]) {
            const int vb = (j == 0 ? sg2.x : sg2.y) + (int)((excl >> (16 * j)) & 0xFFFFu);
            vbase[v] = vb;
            // new outliers (candidate path): CSR entries with the exact w'
            uint32_t nm = nmask[j];
            if (nm) {
              const RowPrep& G0 = a.prep[gr];  // global copy (the stage may be refilled)
              while (nm) {
                const int e = __ffs(nm) - 1;
                nm &= nm - 1u;
                const int col = v * 16 + e;
                const int pos = vb + __popc(out16[j] & ((1u << e) - 1u));
                const float val = exact_wprime(G0.w_in[col], G0.m_in[col], G0.g_in[col], G0, h);
                if (pos < co) {
                  a.col_out[so + pos] = col;
                  a.val_out[so + pos] = val;
                }
              }
            }
          }
        }
      }
    }
    on_prev = on_cur;
    if (!has_next) break;
    gr = gn;
  }
  // the last row's old outliers
  __syncthreads();
  old_out(it % 3, on_prev, 0, NT);
}

// ---------------------------------------------------------------------------- prep
// warp-aggregated append of the flagged lanes' values to a list (one atomic per warp, the
// lanes' order kept), so a list built by consecutive rows stays in nearly ascending order
template <typename T>
__device__ __forceinline__ void warp_append(bool flag, T val, T* list, int32_t* count) {
  const uint32_t m = __ballot_sync(0xffffffffu, flag);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (flag) list[base + __popc(m & ((1u << lane) - 1u))] = val;
}

// One thread per row of the launch: the RowPrep record and the row's TIER --
//   stable  (*) holds: no dense code can move (rows kernel, pass-through),
//   GEN     every other condition of the stable tier holds (fast dequant of w/m/g,
//           bounded scales, thresholds at codes 0 / qmax, the old outliers fit the
//           table): the GEN rows kernel requantizes every code,
//   general the rest: step_kernel.
// Each tier's rows are appended to its list (this step's flip); the other flip's
// counters and both row-claim counters are zeroed for the next step.
constexpr int PREP_T = 256;  // threads (rows) per prep block

__global__ void __launch_bounds__(PREP_T) k_step_prep(const LaunchArgs a, int stable_ok) {
  const int gr = blockIdx.x * PREP_T + threadIdx.x;
  if (gr == 0) {
    if (a.xclear) a.xclear[0] = a.xclear[1] = a.xclear[2] = a.xclear[3] = 0;
    if (a.rclaim) a.rclaim[0] = a.rclaim[1] = 0;
  }
  int tier = -1;  // -1: past the end
  int lo = 0, r = 0;
  if (gr < a.total_rows) {
    // tensor of the row (binary search over the row bases)
    int hi = a.n_tensors - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (a.tensors[mid].row_base <= gr) lo = mid;
      else hi = mid - 1;
    }
    const DevTensor& T = a.tensors[lo];
    r = gr - T.row_base;
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

    bool ok = stable_ok != 0 && on <= a.oldcap6 && T.cols == a.cols_p && T.cnt[out] != nullptr;
    ok = ok && make_dequant_row(sw, zw).fast && make_dequant_row(sm, zm).fast &&
         make_dequant_row(sg, zg).fast;
    // positive, normal scales (so 1/s is finite and the dense values are bounded)
    ok = ok && sw >= 0x1.0p-126f && sw <= 0x1.0p100f && sm >= 0x1.0p-126f && sm <= 0x1.0p100f &&
         sg >= 0x1.0p-126f && sg <= 0x1.0p100f;
    bool st = false;
    if (ok) {
      const double K = (double)qmax + fabs((double)zw);
      // m' = b2*m + c2*g finite: |m|, |g| <= s*(qmax+|z|) <= 2^120, |b2|, |c2| <= 4
      const double c2 = (double)__fsub_rn(1.0f, a.b2);
      ok = (double)sm * ((double)qmax + fabs((double)zm)) <= 0x1.0p120 &&
           (double)sg * ((double)qmax + fabs((double)zg)) <= 0x1.0p120 &&
           fabs((double)a.b2) <= 4.0 && fabs(c2) <= 4.0;
      // thresholds map to the ends of the code range
      ok = ok && (tmin <= tmax) && code_unclamped(tmin, sw, zw) == 0.0 &&
           code_unclamped(tmax, sw, zw) == (double)qmax;
      // D bounds |w' - w| (|sign(d)| <= 1, |w| <= Wmax): finite and small keeps w' finite
      const double lr = fabs((double)a.lr), wd = fabs((double)a.wd);
      const double wmax = (double)sw * K * (1.0 + 0x1.0p-20);
      const double D = lr * (1.0 + wd * wmax) * (1.0 + 0x1.0p-20);
      ok = ok && isfinite(lr) && isfinite(wd) && D <= 0x1.0p100 &&
           fabs((double)a.b1) <= 4.0 && fabs((double)__fsub_rn(1.0f, a.b1)) <= 4.0;
      // (*) the step cannot move a dense code: D/sw <= 0.5 - (K+2)*2^-21
      st = ok && D / (double)sw <= 0.5 - (K + 2.0) * 0x1.0p-21;
    }
    // stable_ok bit 1: few rows were stable last step, so this step runs no stable launch
    // and its stable rows join the GEN list (the GEN kernel requantizes every code: the
    // same bytes, the reference's arithmetic); they are still counted as stable
    if (st && a.scount) {
      const unsigned m = __activemask();
      const int leader = __ffs(m) - 1;
      if ((int)(threadIdx.x & 31) == leader) atomicAdd(a.scount, __popc(m));
    }
    const bool route = st && (stable_ok & 2) && a.gen_on;
    if (route) st = false;
    const bool gen = ok && !st && a.gen_on;
    tier = st ? 1 : (gen ? 2 : 0);
    RowPrep p;
    p.info = (st ? rs6::I_STABLE : 0u) | (gen ? rs6::I_GEN : 0u) | ((uint32_t)zpay << 8);
    p.cand = 0u;
    if (st) {
      // the candidate outcomes: w = dequant(B), w' = w - lr*(s + wd*w) for s = -1, 0, +1
      // (lion_apply, optimizer.hpp:38), then the class and code against the cached
      // thresholds exactly as the step computes them (quantize.hpp:274-285)
      for (int B = 0; B < 2; ++B) {
        const float w = dequant_exact(B ? (uint32_t)qmax : 0u, sw, zw);
        for (int S = 0; S < 3; ++S) {
          const float sg1 = (float)(S - 1);
          const float wn = __fsub_rn(w, __fmul_rn(a.lr, __fadd_rn(sg1, __fmul_rn(a.wd, w))));
          const bool o = (wn < tmin) || (wn > tmax);
          const uint32_t code = o ? (uint32_t)zpay : quant_exact(wn, sw, zw, qmax);
          const int k = 3 * B + S;
          if (o) p.info |= 1u << (1 + k);
          if (k < 4) p.cand |= code << (8 * k);
          else p.info |= code << (16 + 8 * (k - 4));
        }
      }
    }
    p.ob = ob;
    // the rows kernels copy a row's old CSR slot into the stage: general-tier rows
    // (whose slot may exceed the stage) get 0 -- the general kernel reads its own bounds
    p.on = (st || gen) ? on : 0;
    p.so = so;
    p.co = co;
    p.zw = zw;
    p.zm = zm;
    p.sm = sm;
    p.negc_m = make_dequant_row(sm, zm).negc;
    p.sg = sg;
    p.negc_g = make_dequant_row(sg, zg).negc;
    p.zg = zg;
    p.sw = sw;
    p.tmin = tmin;
    p.tmax = tmax;
    const size_t roff = (size_t)r * (size_t)T.cols;
    p.w_in = T.w_codes[in] + roff;
    p.m_in = T.m_codes[in] + roff;
    p.g_in = T.g_codes ? T.g_codes + roff : nullptr;
    p.w_out = T.w_codes[out] + roff;
    p.m_out = T.m_codes[out] + roff;
    p.m_scale_out = T.m_scale[out] + r;
    p.m_zp_out = T.m_zp[out] + r;
    p.cnt_out = T.cnt[out] ? T.cnt[out] + r : nullptr;
    a.prep[gr] = p;
  }
  // the GEN and general tiers' row lists (warp-aggregated appends: runs of consecutive
  // rows, one atomic per warp); the stable rows kernel walks every row of the launch
  warp_append<int32_t>(tier == 2, gr, a.glist, a.gcount);
  warp_append<RowBlock>(tier == 0, RowBlock{lo, r, 1, 0}, a.xlist, a.xcount);
}

// ---------------------------------------------------------------------------- launch
cudaError_t launch_k(const KLaunch& k, const LaunchArgs& a, cudaStream_t st) {
  LaunchArgs aa = a;
  void* args[] = {&aa};
  return cudaLaunchKernel(k.fn, dim3((unsigned)k.grid), dim3((unsigned)k.block), args, k.smem, st);
}
cudaError_t launch_k2(const KLaunch& k, const LaunchArgs& a, cudaStream_t st) {
  LaunchArgs aa = a;
  int a1 = k.arg1;
  void* args[] = {&aa, &a1};
  return cudaLaunchKernel(k.fn, dim3((unsigned)k.grid), dim3((unsigned)k.block), args, k.smem, st);
}

// QFT_ROWS_GRID caps a persistent grid (read once, when a plan resolves its launches):
// the tests use it so every CTA pipelines many rows
static long grid_cap() {
  const char* g = getenv("QFT_ROWS_GRID");
  return g ? std::max(1L, atol(g)) : 0L;
}

template <int MAXT, int MINB, int NS, int FULL = 0, int CCOLS = 0, int BWC = 0, bool GEN = false>
static cudaError_t rows_resolve_t(const LaunchArgs& a, int nt, size_t smem, KLaunch* out,
                                  int cap_per_sm) {
  auto k = rows_kernel<MAXT, MINB, NS, FULL, CCOLS, BWC, GEN>;
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
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, nt, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  if (cap_per_sm > 0 && per_sm > cap_per_sm) per_sm = cap_per_sm;
  long grid = (long)sms * per_sm;
  if (grid > a.total_rows) grid = a.total_rows;
  if (const long cap = grid_cap()) grid = std::min(grid, cap);
  if (grid < 1) grid = 1;
  out->fn = reinterpret_cast<const void*>(k);
  out->grid = (int)grid;
  out->block = nt;
  out->smem = smem;
  snprintf(out->name, sizeof(out->name), "rows_kernel<%d,%d,%d,%d,%d,%d%s>", MAXT, MINB, NS, FULL,
           CCOLS, BWC, GEN ? ",gen" : "");
  return cudaSuccess;
}

bool rows_kernel_eligible(int gk, int use_bulk, int uniform_cols) {
  return gk == G_U8 && use_bulk && uniform_cols > 0 && uniform_cols % 16 == 0 &&
         uniform_cols <= 16384 &&  // <= 512 threads at V = 2
         rows_kernel_smem(uniform_cols, rows_kernel_oldcap(uniform_cols)) <= 227 * 1024;
}

// register budget per width class (tuning: -DQFT_ROWS_MINB_S / _M)
#ifndef QFT_ROWS_MINB_S
#define QFT_ROWS_MINB_S 5  // rows of <= 4096 columns (<= 128 threads): 5 CTAs/SM
#endif
#ifndef QFT_ROWS_MINB_M
#define QFT_ROWS_MINB_M 2  // rows of <= 12288 columns (<= 384 threads)
#endif

// the rows-kernel instance of a launch (compile-time geometry for the LLaMA-2 widths
// 4096 / 11008 (7B) and 5120 / 13824 (13B), used only when the plan's table size is the
// one that geometry implies)
static cudaError_t rows_resolve(const LaunchArgs& a, KLaunch* out, int cps) {
  const int nt = rows_kernel_nt(a.cols_p);
  const size_t smem = rows_kernel_smem(a.cols_p, a.oldcap6);
  const int c = a.cols_p;
  auto geom_ok = [&](int cc, int ns) {
    return c == cc && a.oldcap6 == geom_oldcap(cc, ns) && a.slotted_in;
  };
  const bool b8 = QFT_BW8 && a.bit_width == 8;  // the 7B widths also get a constant width
  if (nt == 128 && geom_ok(4096, 3) && b8)
    return rows_resolve_t<128, QFT_ROWS_MINB_S, 3, 2, 4096, 8>(a, nt, smem, out, cps);
  if (nt == 128 && geom_ok(4096, 3))
    return rows_resolve_t<128, QFT_ROWS_MINB_S, 3, 2, 4096>(a, nt, smem, out, cps);
  if (geom_ok(11008, 2) && b8)
    return rows_resolve_t<384, QFT_ROWS_MINB_M, 2, 1, 11008, 8>(a, nt, smem, out, cps);
#if QFT_BW34
  // the down-projection sweep (configs[4]) also runs 3- and 4-bit codes
  if (geom_ok(11008, 2) && a.bit_width == 4)
    return rows_resolve_t<384, QFT_ROWS_MINB_M, 2, 1, 11008, 4>(a, nt, smem, out, cps);
  if (geom_ok(11008, 2) && a.bit_width == 3)
    return rows_resolve_t<384, QFT_ROWS_MINB_M, 2, 1, 11008, 3>(a, nt, smem, out, cps);
#endif
  if (geom_ok(11008, 2)) return rows_resolve_t<384, QFT_ROWS_MINB_M, 2, 1, 11008>(a, nt, smem, out, cps);
  if (geom_ok(5120, 2) && b8)
    return rows_resolve_t<384, QFT_ROWS_MINB_M, 2, 1, 5120, 8>(a, nt, smem, out, cps);
  if (geom_ok(5120, 2)) return rows_resolve_t<384, QFT_ROWS_MINB_M, 2, 1, 5120>(a, nt, smem, out, cps);
  if (geom_ok(13824, 2) && b8) return rows_resolve_t<512, 1, 2, 1, 13824, 8>(a, nt, smem, out, cps);
  if (geom_ok(13824, 2)) return rows_resolve_t<512, 1, 2, 1, 13824>(a, nt, smem, out, cps);
  if (nt <= 128) return rows_resolve_t<128, QFT_ROWS_MINB_S, 3>(a, nt, smem, out, cps);
  if (nt <= 384 && c / 16 >= nt) return rows_resolve_t<384, QFT_ROWS_MINB_M, 2, 1>(a, nt, smem, out, cps);
  if (nt <= 384) return rows_resolve_t<384, QFT_ROWS_MINB_M, 2>(a, nt, smem, out, cps);
  return rows_resolve_t<512, 1, 2>(a, nt, smem, out, cps);
}

#ifndef QFT_GEN_MINB_M
#define QFT_GEN_MINB_M QFT_ROWS_MINB_M  // GEN tier, 11008 columns (A/B: 1 = no spills)
#endif
#ifndef QFT_GEN_MINB_S
#define QFT_GEN_MINB_S 4  // GEN tier, rows of <= 4096 columns: 4 CTAs/SM (128 registers)
#endif
// the GEN-tier instance of a launch (compile-time geometry for the LLaMA-2-7B widths at
// 8 bits, generic otherwise)
static cudaError_t rows_resolve_gen(const LaunchArgs& a, KLaunch* out, int cps) {
  const int nt = rows_kernel_nt(a.cols_p);
  const size_t smem = rows_kernel_smem(a.cols_p, a.oldcap6);
  const int c = a.cols_p;
  auto geom_ok = [&](int cc, int ns) {
    return c == cc && a.oldcap6 == geom_oldcap(cc, ns) && a.slotted_in;
  };
  const bool b8 = QFT_BW8 && a.bit_width == 8;
  if (nt == 128 && geom_ok(4096, 3) && b8)
    return rows_resolve_t<128, QFT_GEN_MINB_S, 3, 2, 4096, 8, true>(a, nt, smem, out, cps);
  if (geom_ok(11008, 2) && b8)
    return rows_resolve_t<384, QFT_GEN_MINB_M, 2, 1, 11008, 8, true>(a, nt, smem, out, cps);
  if (nt <= 128) return rows_resolve_t<128, QFT_GEN_MINB_S, 3, 0, 0, 0, true>(a, nt, smem, out, cps);
  if (nt <= 384 && c / 16 >= nt)
    return rows_resolve_t<384, QFT_ROWS_MINB_M, 2, 1, 0, 0, true>(a, nt, smem, out, cps);
  if (nt <= 384) return rows_resolve_t<384, QFT_ROWS_MINB_M, 2, 0, 0, 0, true>(a, nt, smem, out, cps);
  return rows_resolve_t<512, 1, 2, 0, 0, 0, true>(a, nt, smem, out, cps);
}

// One step of a rows-path plan: k_step_prep (records + the device list of general-tier
// rows), the rows kernel over the stable tier, the general kernel over the list.  Every
// launch is resolved once per plan (RowsCache); the list counter of this flip was zeroed
// by the previous step's prep (a repeated flip -- a re-run after an overflow -- zeroes it
// here).
cudaError_t launch_rows_step(const LaunchArgs& a0, RowsCache& c, cudaStream_t st) {
  LaunchArgs a = a0;
  a.negzero = -0.0f;
  int32_t* cf = c.xcount + 4 * a.flip;  // this step's list counters
  a.xcount = cf;
  a.scount = cf + 1;
  a.gcount = cf + 2;
  a.xclear = c.xcount + 4 * (1 - a.flip);
  a.rclaim = c.xcount + 8;
  a.slist = c.slist;
  a.glist = c.glist;
  a.gen_on = c.gen_on;
  cudaError_t e;
  if (c.last_flip == a.flip && (e = cudaMemsetAsync(cf, 0, 4 * sizeof(int32_t), st)) != cudaSuccess)
    return e;
  c.last_flip = a.flip;
  // stable rows below 1/16 of the launch last step (seen_host[2], published by the GEN
  // kernel): route them into the GEN list and skip the stable launch, whose walk over
  // every row would cost a full read of the row records for a handful of rows
  const bool route = c.gen_on && c.route_on && c.seen_host &&
                     (long long)c.seen_host[2] * 16 < (long long)a.total_rows;
  const int nb = (a.total_rows + PREP_T - 1) / PREP_T;
  k_step_prep<<<nb, PREP_T, 0, st>>>(a, route ? 3 : 1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  c.routed = route;
  // the stable tier: the rows kernel walks every row of the launch
  LaunchArgs sa = a;
  sa.rlist = nullptr;
  sa.rcount = nullptr;
  sa.rclaim = c.xcount + 8;
  sa.xseen = nullptr;
  KLaunch& rk = c.rows[a.slotted_in ? 1 : 0];
  if (!rk.fn && (e = rows_resolve(sa, &rk, c.cap_per_sm)) != cudaSuccess) return e;
  if (!route && (e = launch_k(rk, sa, st)) != cudaSuccess) return e;
  // the GEN tier over its list (one CTA per SM when the list was empty last step: the
  // kernel covers any length)
  if (c.gen_on) {
    LaunchArgs ga = a;
    ga.rlist = c.glist;
    ga.rcount = a.gcount;
    ga.rclaim = c.xcount + 9;
    ga.xseen = c.seen_dev ? c.seen_dev + 1 : nullptr;
    KLaunch& gr = c.genrows[a.slotted_in ? 1 : 0];
    if (!gr.fn && (e = rows_resolve_gen(ga, &gr, c.cap_per_sm)) != cudaSuccess) return e;
    KLaunch g2 = gr;
    if (c.seen_host && c.seen_host[1] == 0 && c.sms > 0 && g2.grid > c.sms) g2.grid = c.sms;
    if ((e = launch_k(g2, ga, st)) != cudaSuccess) return e;
  }
  // the general kernel over the device row list
  LaunchArgs x = a;
  x.blocks = a.xlist;
  x.n_blocks = a.total_rows;  // upper bound; the kernel reads the true count
  x.n_blocks_dev = a.xcount;
  KLaunch& gk = c.gen[a.wd == 0.0f ? 1 : 0];
  if (!gk.fn && (e = resolve_step_kernel(G_U8, x, &gk)) != cudaSuccess) return e;
  x.xseen = c.seen_dev;
  if (c.seen_host && *c.seen_host == 0 && c.sms > 0 && gk.grid > c.sms) {
    KLaunch small = gk;  // the list was empty last step: a small grid (still covers any list)
    small.grid = c.sms;
    return launch_k(small, x, st);
  }
  return launch_k(gk, x, st);
}

}  // namespace qftk
