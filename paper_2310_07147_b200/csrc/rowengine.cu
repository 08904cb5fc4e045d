// rowengine.cu -- the fused per-row kernels of the QFT update path (sm_100a).
//
// One persistent, warp-specialised kernel template serves four modes:
//   MODE_STEP        fused quantized Lion step  == lion_step_quantized body,
//                    optimizer.hpp:103-118 (dequant g,m,w -> lion_apply ->
//                    quantize_state(m) -> requantize_weight(w))
//   MODE_DECOMPOSE   decompose_dense_sparse     (quantize.hpp:253-290)
//   MODE_RECON_F32   reconstruct                (quantize.hpp:331-338)
//   MODE_RECON_BF16  reconstruct -> bf16 for the next forward (network.hpp:208-211)
//
// CTA = 1 producer warp + 4 consumer warps; the unit of work is one ROW (one
// output channel: scales, zero points, thresholds, the m' min/max and the CSR
// segment are all row-local).
//
// Producer warp (STEP/RECON): walks a static list of row blocks (<= 32 rows of
// one tensor, round-robin over CTAs).  Per block its lanes load the 32 rows'
// metadata in parallel (params, thresholds, CSR slot bounds); per row it waits
// for a free stage, writes the row context and issues TMA 1-D bulk copies
// (cp.async.bulk -> SASS UBLKCP) of the row's w/m/g codes and of the row's old
// CSR slot (cols, values) into the stage, completion counted on the stage's
// mbarrier.  It runs up to S rows ahead of the consumers.
//
// Consumer warps (128 threads, one 16-byte vector = 16 elements per thread-step):
//   old-outlier bitmap from the staged slot; named barrier;
//   pass 1: dequant g,m,w (+old outlier patch) -> Lion (packed FP32x2 products,
//           scalar sums: see qft_device.cuh) -> classify / quantize w' -> dense
//           W codes straight to HBM (STG.128); m' kept in smem; m' row min/max;
//           new-outlier masks;
//   named barrier; m' params in fp64 (as the reference); pass 2 quantizes m';
//   CSR write into the row's own slot (ascending columns: warp ballot/popc and a
//   chunk-major prefix), slot count stored; overflow of a slot raises a flag and
//   the host re-plans the slots and re-runs from the intact ping-pong inputs.
// No row ever waits on another row.
//
// DECOMPOSE (init / threshold refresh only) writes the STRICT reference CSR
// directly: rows are taken by an atomic ticket and the row offsets come from a
// warp-wide decoupled look-back over per-row status words.
#include <cstdio>

#include "qft_device.cuh"
#include "qft_internal.h"

namespace qftk {
using namespace qftd;

constexpr int NCW = 4;             // consumer warps
constexpr int NCT = NCW * 32;      // consumer threads
constexpr int NT = NCT + 32;       // + producer warp
constexpr int OLDCAP = 256;        // old CSR entries staged in smem per stage
constexpr int NCH_MAX = 32;        // chunks of NCT*16 columns
constexpr int MAX_COLS = NCH_MAX * NCT * 16;  // 65536
constexpr int MAX_STAGES = 6;
constexpr int HDR = 256;           // stage header (row context) bytes

constexpr uint32_t FLAG_A = 1u, FLAG_P = 2u;
constexpr uint32_t VAL_MASK = (1u << 30) - 1u;

constexpr int BAR_C = 1;      // after pass 1 (row reduction)
constexpr int BAR_D = 2;      // decompose: row offset known
constexpr int BAR_G = 3;      // raw-gradient row reduction
constexpr int BAR_B0 = 4;     // old-outlier bitmap ready

struct StageCtx {
  int32_t row;        // >= 0 valid (decompose: launch-global row); -1 = no more work
  int32_t lrow;       // row inside its tensor
  int32_t cols;
  int32_t old_begin;  // arena index of the row's first old outlier
  int32_t old_n;
  int32_t old_staged; // old (col,val) list is TMA-staged in this stage
  int32_t is_last;    // lrow == rows-1 (decompose)
  int32_t zw, zm, zg, zpay;
  float sw, tmin, tmax, sm, sg;
  int32_t slot_out, cap_out;
  uint8_t* w_out;     // row pointers in HBM
  uint8_t* m_out;
  void* aux_out;      // reconstruct output row
  float* m_scale_out; // tensor arrays
  int32_t* m_zp_out;
  int32_t* cnt_out;
  int32_t* row_ptr_out;  // decompose (strict)
};
static_assert(sizeof(StageCtx) <= HDR, "ctx size");

__host__ __device__ inline int round16(int x) { return (x + 15) & ~15; }

__host__ __device__ inline int stage_data_bytes(int mode, int gk, int cp) {
  switch (mode) {
    case MODE_STEP: return 2 * cp + (gk == G_U8 ? cp : gk == G_F32 ? 4 * cp : 2 * cp);
    case MODE_DECOMPOSE: return 4 * cp;
    default: return cp;
  }
}
__host__ __device__ inline int old_bits_bytes(int cp) { return round16((cp + 31) / 32 * 4); }
__host__ __device__ inline int frank_bytes(int cp) { return round16((cp + 31) / 32 * 2); }
__host__ __device__ inline int stage_bytes(int mode, int gk, int cp) {
  const int old =
      (mode == MODE_DECOMPOSE) ? 0 : OLDCAP * 8 + old_bits_bytes(cp) + frank_bytes(cp);
  return HDR + old + stage_data_bytes(mode, gk, cp);
}
struct Tabs {
  float red_lo[2][NCW];
  float red_hi[2][NCW];
  int32_t red_nan[2][NCW];
  float gred_lo[2][NCW];
  float gred_hi[2][NCW];
  int32_t gred_nan[2][NCW];
  int32_t cnt[2][NCH_MAX][NCW];
  int32_t prefix[2];
  int32_t _pad[2];
};
__host__ __device__ inline int mprime_bytes(int cp) {
  return 4 * ((cp + NCT * 16 - 1) / (NCT * 16)) * (NCT * 16);
}
__host__ __device__ inline int consumer_bytes(int mode, int cp, bool mrec) {
  int b = (int)sizeof(Tabs);
  if (mode == MODE_STEP && !mrec) b += mprime_bytes(cp);
  if (mode == MODE_STEP || mode == MODE_DECOMPOSE) b += round16(cp / 16 * 2);  // masks
  return b;
}
size_t row_engine_smem(int mode, int gk, int cols_p, int stages, bool mrec) {
  return 128 /*barriers*/ + (size_t)stages * stage_bytes(mode, gk, cols_p) +
         consumer_bytes(mode, cols_p, mrec);
}
int row_engine_max_cols() { return MAX_COLS; }

// ----------------------------------------------------------------------------
// small helpers
// ----------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long pack_status(uint32_t epoch, uint32_t flag,
                                                          uint32_t v) {
  return ((unsigned long long)epoch << 32) | ((unsigned long long)flag << 30) | v;
}

// value of the old outlier at column `col` (its bit is set): the entry's rank in
// the row's sorted list is first_rank[word] + popc(lower bits of the word) -- O(1)
__device__ __forceinline__ float old_value(const uint32_t* bits, const uint16_t* frank,
                                           const float* ov, int staged, int old_begin, int col,
                                           const float* val_in) {
  const int w = col >> 5;
  const int r = (int)frank[w] + __popc(bits[w] & ((1u << (col & 31)) - 1u));
  return (staged && r < OLDCAP) ? ov[r] : val_in[old_begin + r];
}

__device__ __forceinline__ uint32_t bits16(const uint32_t* bits, int v) {
  return (bits[v >> 1] >> ((v & 1) * 16)) & 0xFFFFu;
}

// spread a 4-bit nibble to a byte mask (bit i -> byte i = 0xFF)
__device__ __forceinline__ uint32_t nib_to_bytemask(uint32_t nib) {
  return ((nib * 0x00204081u) & 0x01010101u) * 0xFFu;
}

template <int GK>
__device__ __forceinline__ float load_graw(const uint8_t* gdata, int idx) {
  if (GK == G_F32) return reinterpret_cast<const float*>(gdata)[idx];
  const uint16_t b = reinterpret_cast<const uint16_t*>(gdata)[idx];
  return __uint_as_float((uint32_t)b << 16);
}

__device__ __forceinline__ float dequant1(uint32_t code, const DequantRow& d) {
  return d.fast ? __fmul_rn(__fadd_rn(magic_byte(code, 0), d.negc), d.s)
                : dequant_exact(code, d.s, d.z);
}

// ----------------------------------------------------------------------------
// the kernel
// ----------------------------------------------------------------------------
template <int MODE, int GK, bool ALIGNED, bool WD0, bool MREC>
__global__ void __launch_bounds__(NT, QFT_MIN_CTAS) row_engine_kernel(const LaunchArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + MAX_STAGES;
  const int cp = a.cols_p;
  const int S = a.stages;
  const int sbytes = stage_bytes(MODE, GK, cp);
  uint8_t* stage0 = smem + 128;
  uint8_t* cons = stage0 + (size_t)S * sbytes;
  Tabs* tabs = reinterpret_cast<Tabs*>(cons);
  float* mprime = reinterpret_cast<float*>(cons + sizeof(Tabs));
  uint16_t* masks = reinterpret_cast<uint16_t*>(cons + sizeof(Tabs) +
                                                (MODE == MODE_STEP && !MREC ? mprime_bytes(cp)
                                                                            : 0));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int qmax = (1 << a.bit_width) - 1;
  constexpr bool kOld = (MODE != MODE_DECOMPOSE);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    mbar_fence_init();
  }
  __syncthreads();

  auto stage_ptr = [&](int s) { return stage0 + (size_t)s * sbytes; };
  auto ctx_of = [&](uint8_t* st) { return reinterpret_cast<StageCtx*>(st); };
  auto oldc_of = [&](uint8_t* st) { return reinterpret_cast<int32_t*>(st + HDR); };
  auto oldv_of = [&](uint8_t* st) { return reinterpret_cast<float*>(st + HDR + OLDCAP * 4); };
  auto oldb_of = [&](uint8_t* st) { return reinterpret_cast<uint32_t*>(st + HDR + OLDCAP * 8); };
  auto frank_of = [&](uint8_t* st) {
    return reinterpret_cast<uint16_t*>(st + HDR + OLDCAP * 8 + old_bits_bytes(cp));
  };
  auto data_of = [&](uint8_t* st) {
    return st + HDR + (kOld ? OLDCAP * 8 + old_bits_bytes(cp) + frank_bytes(cp) : 0);
  };

  if (warp == NCW) {
    // ============================ PRODUCER WARP =============================
    const int in = a.flip, out = 1 - a.flip;
    int it = 0;
    if (MODE == MODE_DECOMPOSE) {
      // dynamic tickets in global row order (the look-back needs them)
      for (;; ++it) {
        const int s = it % S;
        mbar_wait(&empty[s], ((uint32_t)(it / S) & 1u) ^ 1u);
        uint8_t* st = stage_ptr(s);
        StageCtx* cx = ctx_of(st);
        int row = 0;
        if (lane == 0) row = (int)atomicAdd(&a.hdr->ticket, 1u);
        row = __shfl_sync(0xffffffffu, row, 0);
        if (row >= a.total_rows) {
          if (lane == 0) {
            cx->row = -1;
            mbar_arrive(&full[s]);
          }
          break;
        }
        int lo = 0, hi = a.n_tensors - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (a.tensors[mid].row_base <= row) lo = mid; else hi = mid - 1;
        }
        const DevTensor& T = a.tensors[lo];
        const int lrow = row - T.row_base;
        const int cols = T.cols;
        const size_t roff = (size_t)lrow * (size_t)cols;
        const uint8_t* src = reinterpret_cast<const uint8_t*>(T.w_f32 + roff);
        if (lane == 0) {
          cx->row = row;
          cx->lrow = lrow;
          cx->cols = cols;
          cx->is_last = (lrow == T.rows - 1);
          const float sw = T.w_scale[lrow];
          const int32_t zw = T.w_zp[lrow];
          cx->sw = sw;
          cx->zw = zw;
          cx->zpay = zw < 0 ? 0 : (zw > qmax ? qmax : zw);
          cx->tmin = T.t_min[lrow];
          cx->tmax = T.t_max[lrow];
          cx->w_out = T.w_codes[1] + roff;
          cx->row_ptr_out = T.rs[1];
        }
        uint8_t* data = data_of(st);
        if (ALIGNED) {
          if (lane == 0) {
            mbar_expect_tx(&full[s], 4u * cols);
            bulk_g2s(data, src, 4u * cols, &full[s]);
          }
        } else {
          for (int i = lane; i < 4 * cols; i += 32) data[i] = src[i];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&full[s]);
      }
    } else {
      // static round-robin over row blocks; 32 rows' metadata loaded lane-parallel
      for (int blk = blockIdx.x; blk < a.n_blocks; blk += gridDim.x) {
        const RowBlock B = a.blocks[blk];
        const DevTensor* T = a.tensors + B.tensor;
        const int cols = T->cols;
        const bool act = lane < B.nrows;
        const int lrow_l = B.row0 + lane;
        float sw = 0.f, tmin = 0.f, tmax = 0.f, smv = 0.f, sgv = 0.f;
        int zw = 0, zm = 0, zg = 0, ob = 0, on = 0, so = 0, co = 0;
        if (act) {
          sw = T->w_scale[lrow_l];
          zw = T->w_zp[lrow_l];
          const int32_t* rs_in = T->rs[in];
          ob = rs_in[lrow_l];
          const int cap_in = rs_in[lrow_l + 1] - ob;
          // never read past the slot (a count above it means the previous step
          // overflowed and was not re-run; the host reports that state invalid)
          on = T->cnt[in] ? min(T->cnt[in][lrow_l], cap_in) : cap_in;
          if (MODE == MODE_STEP) {
            tmin = T->t_min[lrow_l];
            tmax = T->t_max[lrow_l];
            smv = T->m_scale[in][lrow_l];
            zm = T->m_zp[in][lrow_l];
            if (GK == G_U8) {
              sgv = T->g_scale[lrow_l];
              zg = T->g_zp[lrow_l];
            }
            so = T->rs[out][lrow_l];
            co = T->rs[out][lrow_l + 1] - so;
          }
        }
        // per-tensor pointers (lane 0; broadcast where the copy loop needs them)
        const uint8_t* w_in = nullptr;
        const uint8_t* m_in = nullptr;
        const uint8_t* g_in = nullptr;
        uint8_t* w_outp = nullptr;
        uint8_t* m_outp = nullptr;
        float* ms_out = nullptr;
        int32_t* mz_out = nullptr;
        int32_t* cnt_out = nullptr;
        void* aux = nullptr;
        if (lane == 0) {
          w_in = T->w_codes[in];
          if (MODE == MODE_STEP) {
            m_in = T->m_codes[in];
            g_in = (GK == G_U8) ? T->g_codes : reinterpret_cast<const uint8_t*>(T->g_raw);
            w_outp = T->w_codes[out];
            m_outp = T->m_codes[out];
            ms_out = T->m_scale[out];
            mz_out = T->m_zp[out];
            cnt_out = T->cnt[out];
          } else {
            aux = T->out;
          }
        }
        const int gel = (MODE != MODE_STEP) ? 0 : (GK == G_U8 ? 1 : GK == G_F32 ? 4 : 2);
        const int gbytes = gel * cols;
        const bool slotted = a.slotted_in != 0;
        for (int j = 0; j < B.nrows; ++j, ++it) {
          const int s = it % S;
          mbar_wait(&empty[s], ((uint32_t)(it / S) & 1u) ^ 1u);
          uint8_t* st = stage_ptr(s);
          StageCtx* cx = ctx_of(st);
          uint32_t* bits = oldb_of(st);
          for (int i = lane; i < (cp + 31) / 32; i += 32) bits[i] = 0u;
          if (lane == j) {
            cx->sw = sw;
            cx->zw = zw;
            cx->zpay = zw < 0 ? 0 : (zw > qmax ? qmax : zw);
            cx->old_begin = ob;
            cx->old_n = on;
            if (MODE == MODE_STEP) {
              cx->tmin = tmin;
              cx->tmax = tmax;
              cx->sm = smv;
              cx->zm = zm;
              cx->sg = sgv;
              cx->zg = zg;
              cx->slot_out = so;
              cx->cap_out = co;
            }
          }
          const int obj = __shfl_sync(0xffffffffu, ob, j);
          const int onj = __shfl_sync(0xffffffffu, on, j);
          const int lrow = B.row0 + j;
          const size_t roff = (size_t)lrow * (size_t)cols;
          const bool staged = ALIGNED && slotted && onj > 0 && ((obj & 3) == 0);
          const int nstage = staged ? min((onj + 3) & ~3, OLDCAP) : 0;
          uint8_t* data = data_of(st);
          if (lane == 0) {
            cx->row = lrow;
            cx->lrow = lrow;
            cx->cols = cols;
            cx->old_staged = staged ? 1 : 0;
            if (MODE == MODE_STEP) {
              cx->w_out = w_outp + roff;
              cx->m_out = m_outp + roff;
              cx->m_scale_out = ms_out;
              cx->m_zp_out = mz_out;
              cx->cnt_out = cnt_out;
            } else if (MODE == MODE_RECON_F32) {
              cx->aux_out = reinterpret_cast<float*>(aux) + roff;
            } else {
              cx->aux_out = reinterpret_cast<__nv_bfloat16*>(aux) + roff;
            }
          }
          if (!ALIGNED) {
            // generic path (rows not 16-byte aligned): the producer lanes copy
            const uint8_t* wsrc = reinterpret_cast<const uint8_t*>(
                                      __shfl_sync(0xffffffffu, (unsigned long long)w_in, 0)) +
                                  roff;
            for (int i = lane; i < cols; i += 32) data[i] = wsrc[i];
            if (MODE == MODE_STEP) {
              const uint8_t* msrc = reinterpret_cast<const uint8_t*>(
                                        __shfl_sync(0xffffffffu, (unsigned long long)m_in, 0)) +
                                    roff;
              const uint8_t* gsrc = reinterpret_cast<const uint8_t*>(
                                        __shfl_sync(0xffffffffu, (unsigned long long)g_in, 0)) +
                                    (size_t)gel * roff;
              for (int i = lane; i < cols; i += 32) data[cp + i] = msrc[i];
              for (int i = lane; i < gbytes; i += 32) data[2 * cp + i] = gsrc[i];
            }
          }
          __syncwarp();
          if (lane == 0) {
            uint32_t tx = 0;
            if (ALIGNED) tx += (MODE == MODE_STEP) ? (uint32_t)(2 * cols + gbytes) : (uint32_t)cols;
            tx += 8u * (uint32_t)nstage;
            if (tx) mbar_expect_tx(&full[s], tx);
            if (ALIGNED) {
              bulk_g2s(data, w_in + roff, cols, &full[s]);
              if (MODE == MODE_STEP) {
                bulk_g2s(data + cp, m_in + roff, cols, &full[s]);
                bulk_g2s(data + 2 * cp, g_in + (size_t)gel * roff, gbytes, &full[s]);
              }
            }
            if (nstage) {
              bulk_g2s(oldc_of(st), a.col_in + obj, 4u * nstage, &full[s]);
              bulk_g2s(oldv_of(st), a.val_in + obj, 4u * nstage, &full[s]);
            }
            mbar_arrive(&full[s]);
          }
        }
      }
      const int s = it % S;
      mbar_wait(&empty[s], ((uint32_t)(it / S) & 1u) ^ 1u);
      if (lane == 0) {
        ctx_of(stage_ptr(s))->row = -1;
        mbar_arrive(&full[s]);
      }
    }
  } else {
    // ============================ CONSUMER WARPS ============================
    const int ct = threadIdx.x;  // 0..127
    const int cw = warp;
    Hyper h;
    h.lr = a.lr; h.b1 = a.b1; h.b2 = a.b2; h.wd = a.wd;
    h.c1 = __fsub_rn(1.0f, a.b1);
    h.c2 = __fsub_rn(1.0f, a.b2);
    const uint32_t epoch = *(volatile uint32_t*)&a.hdr->epoch;

    for (int it = 0;; ++it) {
      const int s = it % S;
      const int par = it & 1;
      mbar_wait(&full[s], (uint32_t)(it / S) & 1u);
      uint8_t* st = stage_ptr(s);
      const StageCtx* cx = ctx_of(st);
      const int row = cx->row;
      if (row < 0) break;
      const int cols = cx->cols;
      const int nvec = (cols + 15) >> 4;
      const int nch = (nvec + NCT - 1) / NCT;
      const uint8_t* data = data_of(st);
      uint32_t* obits = oldb_of(st);
      uint16_t* frank = frank_of(st);
      const int32_t* ocols = oldc_of(st);
      const float* ovals = oldv_of(st);
      const int old_n = kOld ? cx->old_n : 0;
      const int old_begin = kOld ? cx->old_begin : 0;
      const int staged = kOld ? cx->old_staged : 0;
      const DequantRow dw = make_dequant_row(cx->sw, cx->zw);

      if (kOld) {
        // old-outlier bitmap of this row (the producer cleared it) and, for every
        // bitmap word holding an outlier, the rank of its first entry
        for (int i = ct; i < old_n; i += NCT) {
          const int col = (staged && i < OLDCAP) ? ocols[i] : a.col_in[old_begin + i];
          const int wd = col >> 5;
          atomicOr(&obits[wd], 1u << (col & 31));
          const int prev = (i == 0) ? -1
                           : ((staged && i - 1 < OLDCAP) ? ocols[i - 1]
                                                         : a.col_in[old_begin + i - 1]);
          if (i == 0 || (prev >> 5) != wd) frank[wd] = (uint16_t)i;
        }
        named_bar_sync(BAR_B0, NCT);
      }

      if (MODE == MODE_RECON_F32 || MODE == MODE_RECON_BF16) {
        for (int k = 0; k < nch; ++k) {
          const int v = k * NCT + ct;
          if (v >= nvec) break;
          const uint4 wq = *reinterpret_cast<const uint4*>(data + v * 16);
          float w[16];
          dequant4(wq.x, dw, w);
          dequant4(wq.y, dw, w + 4);
          dequant4(wq.z, dw, w + 8);
          dequant4(wq.w, dw, w + 12);
          const uint32_t o16 = bits16(obits, v);
          if (o16) {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (o16 & (1u << e))
                w[e] = old_value(obits, frank, ovals, staged, old_begin, v * 16 + e, a.val_in);
          }
          const int nvalid = min(16, cols - v * 16);
          if (MODE == MODE_RECON_F32) {
            float* o = reinterpret_cast<float*>(cx->aux_out) + v * 16;
            if (ALIGNED) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                reinterpret_cast<float4*>(o)[q] =
                    make_float4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
            } else {
              for (int e = 0; e < nvalid; ++e) o[e] = w[e];
            }
          } else {
            __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(cx->aux_out) + v * 16;
            uint32_t pk[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const __nv_bfloat162 b2 = __floats2bfloat162_rn(w[2 * q], w[2 * q + 1]);
              pk[q] = *reinterpret_cast<const uint32_t*>(&b2);
            }
            if (ALIGNED) {
              reinterpret_cast<uint4*>(o)[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
              reinterpret_cast<uint4*>(o)[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
            } else {
              for (int e = 0; e < nvalid; ++e)
                reinterpret_cast<uint16_t*>(o)[e] = (uint16_t)(pk[e >> 1] >> ((e & 1) * 16));
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        continue;
      }

      // ---------------- STEP / DECOMPOSE ----------------
      // dense params: stored (w_scale, w_zp) == affine_params_from_bounds(t_min, t_max)
      // (requantize_weight -> decompose_dense_sparse, quantize.hpp:264), an invariant
      // the host maintains because the params are only ever produced by decompose.
      const QuantRow qw = make_quant_row(cx->sw, cx->zw, a.bit_width);
      const float tmin = cx->tmin, tmax = cx->tmax;
      const uint32_t zpay4 = (uint32_t)cx->zpay * 0x01010101u;
      const uint32_t wz_bits = __float_as_uint(__fmul_rn(cx->sw, (float)(cx->zpay - cx->zw)));
      // dequantized w can only be non-finite if s*(qmax+|z|) overflows fp32
      const bool w_ovf = !(__fmul_rn(fabsf(cx->sw), (float)qmax + fabsf((float)cx->zw)) < 3.0e38f);
      DequantRow dm, dg;
      QuantRow qg;
      if (MODE == MODE_STEP) {
        dm = make_dequant_row(cx->sm, cx->zm);
        if (GK == G_U8) dg = make_dequant_row(cx->sg, cx->zg);
      }

      // ---- raw-gradient modes: fused quantize_state(g) -> dequantize(g) (gradflow.hpp:77)
      if (MODE == MODE_STEP && GK != G_U8) {
        float lo = __int_as_float(0x7f800000), hi = __int_as_float(0xff800000);
        int nan0 = 0;
        const uint8_t* gd = data + 2 * cp;
        for (int k = 0; k < nch; ++k) {
          const int v = k * NCT + ct;
          if (v < nvec) {
            const int nvalid = min(16, cols - v * 16);
            for (int e = 0; e < nvalid; ++e) {
              const float x = load_graw<GK>(gd, v * 16 + e);
              lo = fminf(lo, x);
              hi = fmaxf(hi, x);
            }
            if (v == 0 && isnan(load_graw<GK>(gd, 0))) nan0 = 1;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
          hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
          nan0 |= __shfl_xor_sync(0xffffffffu, nan0, o);
        }
        if (lane == 0) {
          tabs->gred_lo[par][cw] = lo;
          tabs->gred_hi[par][cw] = hi;
          tabs->gred_nan[par][cw] = nan0;
        }
        named_bar_sync(BAR_G, NCT);
        lo = tabs->gred_lo[par][0]; hi = tabs->gred_hi[par][0]; nan0 = tabs->gred_nan[par][0];
#pragma unroll
        for (int w2 = 1; w2 < NCW; ++w2) {
          lo = fminf(lo, tabs->gred_lo[par][w2]);
          hi = fmaxf(hi, tabs->gred_hi[par][w2]);
          nan0 |= tabs->gred_nan[par][w2];
        }
        if (nan0) lo = hi = __int_as_float(0x7fc00000);
        float sgv; int32_t zgv;
        if (!affine_from_bounds(lo, hi, a.bit_width, sgv, zgv)) {
          if (ct == 0) atomicOr(&a.hdr->err, ERR_GPARAMS);
          sgv = 1.0f; zgv = 0;
        }
        qg = make_quant_row(sgv, zgv, a.bit_width);
        dg = make_dequant_row(sgv, zgv);
      }

      float mlo = __int_as_float(0x7f800000), mhi = __int_as_float(0xff800000);
      int mnan0 = 0;

      // ================= pass 1 =================
      for (int k = 0; k < nch; ++k) {
        const int v = k * NCT + ct;
        uint32_t mask = 0;
        if (v < nvec) {
          const int nvalid = min(16, cols - v * 16);
          const uint32_t valid = nvalid >= 16 ? 0xFFFFu : ((1u << nvalid) - 1u);
          float w[16];
          if (MODE == MODE_DECOMPOSE) {
            const float4* src = reinterpret_cast<const float4*>(data + v * 64);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 f = src[q];
              w[4 * q] = f.x; w[4 * q + 1] = f.y; w[4 * q + 2] = f.z; w[4 * q + 3] = f.w;
            }
          } else {
            float m[16], g[16];
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
                graw[e] = (e < nvalid) ? load_graw<GK>(data + 2 * cp, v * 16 + e) : 0.0f;
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
            const uint32_t o16 = bits16(obits, v);
            bool wspecial = w_ovf;  // non-finite w must take the general Lion form
            if (o16) {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (o16 & (1u << e)) {
                  w[e] = old_value(obits, frank, ovals, staged, old_begin, v * 16 + e, a.val_in);
                  wspecial |= !isfinite(w[e]);
                }
            }
            if (WD0 && !wspecial) {
#pragma unroll
              for (int p = 0; p < 8; ++p) {
                float2 W = make_float2(w[2 * p], w[2 * p + 1]);
                float2 M = make_float2(m[2 * p], m[2 * p + 1]);
                lion2_wd0(W, M, make_float2(g[2 * p], g[2 * p + 1]), h);
                w[2 * p] = W.x; w[2 * p + 1] = W.y;
                m[2 * p] = M.x; m[2 * p + 1] = M.y;
              }
            } else {
#pragma unroll
              for (int p = 0; p < 8; ++p) {
                float2 W = make_float2(w[2 * p], w[2 * p + 1]);
                float2 M = make_float2(m[2 * p], m[2 * p + 1]);
                lion2(W, M, make_float2(g[2 * p], g[2 * p + 1]), h);
                w[2 * p] = W.x; w[2 * p + 1] = W.y;
                m[2 * p] = M.x; m[2 * p + 1] = M.y;
              }
            }
            if (v == 0 && isnan(m[0])) mnan0 = 1;
            if (valid != 0xFFFFu) {
#pragma unroll
              for (int e = 1; e < 16; ++e)
                if (!(valid & (1u << e))) m[e] = m[0];
            }
#pragma unroll
            for (int p = 0; p < 8; ++p) {
              float t;
              asm("min.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(mlo), "f"(m[2 * p]), "f"(m[2 * p + 1]));
              mlo = t;
              asm("max.f32 %0, %1, %2, %3;" : "=f"(t) : "f"(mhi), "f"(m[2 * p]), "f"(m[2 * p + 1]));
              mhi = t;
            }
            if (!MREC) {
              float4* mp = reinterpret_cast<float4*>(mprime);
#pragma unroll
              for (int q = 0; q < 4; ++q)
                mp[(k * 4 + q) * NCT + ct] =
                    make_float4(m[4 * q], m[4 * q + 1], m[4 * q + 2], m[4 * q + 3]);
            }
          }
          // ---- classify + quantize w'.  Outliers are replaced by wz = s*(zpay-z)
          // before quantizing, which quantizes exactly to the payload zpay
          // (decompose_dense_sparse stores clamp(z) under an outlier, quantize.hpp:279).
          float wq[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const uint32_t d = outside_mask(w[e], tmin, tmax);
            mask |= d & (1u << e);
            wq[e] = __uint_as_float((__float_as_uint(w[e]) & ~d) | (wz_bits & d));
          }
          mask &= valid;
          float em = 0.0f;
          uint32_t c[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) c[q] = quant4_fast(wq + 4 * q, qw, em);
          if (!qw.fast || !(em < qw.thr)) {
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] = quant4_exact(w + 4 * q, qw);
            if (mask) {
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const uint32_t bm = nib_to_bytemask((mask >> (4 * q)) & 0xFu);
                c[q] = (c[q] & ~bm) | (zpay4 & bm);
              }
            }
          }
          uint8_t* wo = cx->w_out + v * 16;
          if (ALIGNED) {
            *reinterpret_cast<uint4*>(wo) = make_uint4(c[0], c[1], c[2], c[3]);
          } else {
            for (int e = 0; e < nvalid; ++e) wo[e] = (uint8_t)(c[e >> 2] >> ((e & 3) * 8));
          }
          masks[v] = (uint16_t)mask;
        }
        const int wc = __reduce_add_sync(0xffffffffu, __popc(mask));
        if (lane == 0) tabs->cnt[par][k][cw] = wc;
      }

      // ================= row reduction =================
      if (MODE == MODE_STEP) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          mlo = fminf(mlo, __shfl_xor_sync(0xffffffffu, mlo, o));
          mhi = fmaxf(mhi, __shfl_xor_sync(0xffffffffu, mhi, o));
          mnan0 |= __shfl_xor_sync(0xffffffffu, mnan0, o);
        }
        if (lane == 0) {
          tabs->red_lo[par][cw] = mlo;
          tabs->red_hi[par][cw] = mhi;
          tabs->red_nan[par][cw] = mnan0;
        }
      }
      named_bar_sync(BAR_C, NCT);

      // chunk-major CSR offsets of this warp: lane l < nch holds the offset of
      // (chunk l, this warp) inside the row
      int tot_l = 0, mine_l = 0;
      if (lane < nch) {
#pragma unroll
        for (int w2 = 0; w2 < NCW; ++w2) {
          const int cv = tabs->cnt[par][lane][w2];
          tot_l += cv;
          if (w2 < cw) mine_l += cv;
        }
      }
      int incl_l = tot_l;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl_l, d);
        if (lane >= d) incl_l += t;
      }
      const int chunk_pref = incl_l - tot_l + mine_l;
      const int row_total = __shfl_sync(0xffffffffu, incl_l, nch - 1);

      QuantRow qm;
      if (MODE == MODE_STEP) {
        float lo = tabs->red_lo[par][0], hi = tabs->red_hi[par][0];
        int nan0 = tabs->red_nan[par][0];
#pragma unroll
        for (int w2 = 1; w2 < NCW; ++w2) {
          lo = fminf(lo, tabs->red_lo[par][w2]);
          hi = fmaxf(hi, tabs->red_hi[par][w2]);
          nan0 |= tabs->red_nan[par][w2];
        }
        if (nan0) lo = hi = __int_as_float(0x7fc00000);
        float smv; int32_t zmv;
        if (!affine_from_bounds(lo, hi, a.bit_width, smv, zmv)) {
          if (ct == 0) atomicOr(&a.hdr->err, ERR_MPARAMS);
          smv = 1.0f; zmv = 0;
        }
        qm = make_quant_row(smv, zmv, a.bit_width);
        if (ct == 0) {
          cx->m_scale_out[cx->lrow] = smv;
          cx->m_zp_out[cx->lrow] = zmv;
          cx->cnt_out[cx->lrow] = row_total;
          if (row_total > cx->cap_out) atomicOr(&a.hdr->overflow, 1u);
        }
      }

      int row_base_out = 0, row_cap = 0x7fffffff;
      if (MODE == MODE_STEP) {
        row_base_out = cx->slot_out;
        row_cap = cx->cap_out;
      }

      if (MODE == MODE_DECOMPOSE && cw == 0) {
        // ---- decoupled look-back over the per-row status words (strict CSR)
        const uint32_t total = (uint32_t)row_total;
        uint32_t excl = 0;
        if (row > 0) {
          if (lane == 0) st_relaxed_u64(a.status + row, pack_status(epoch, FLAG_A, total));
          int base = row - 1;
          while (true) {
            const int idx = base - lane;
            uint32_t flag = FLAG_P, val = 0;
            if (idx >= 0) {
              const unsigned long long wd = ld_relaxed_u64(a.status + idx);
              flag = ((uint32_t)(wd >> 32) == epoch) ? (uint32_t)(wd >> 30) & 3u : 0u;
              val = (uint32_t)wd & VAL_MASK;
            }
            const uint32_t pm = __ballot_sync(0xffffffffu, flag == FLAG_P);
            const uint32_t nm = __ballot_sync(0xffffffffu, flag == 0u);
            const int lim = pm ? __ffs(pm) - 1 : 31;
            const uint32_t need = (lim >= 31) ? 0xffffffffu : ((2u << lim) - 1u);
            if (nm & need) {
              __nanosleep(32);
              continue;
            }
            excl += __reduce_add_sync(0xffffffffu, lane <= lim ? val : 0u);
            if (pm) break;
            base -= 32;
          }
        }
        const uint32_t inclusive = excl + total;
        if (lane == 0) {
          st_relaxed_u64(a.status + row, pack_status(epoch, FLAG_P, inclusive & VAL_MASK));
          if (inclusive > VAL_MASK) atomicOr(&a.hdr->err, ERR_PREFIX);
          tabs->prefix[par] = (int32_t)excl;
          cx->row_ptr_out[cx->lrow] = (int32_t)excl;
          if (cx->is_last) cx->row_ptr_out[cx->lrow + 1] = (int32_t)inclusive;
          if (row == a.total_rows - 1) {
            a.hdr->total_nnz = (int64_t)inclusive;
            if ((int64_t)inclusive > a.cap_out) atomicOr(&a.hdr->overflow, 1u);
          }
        }
      }

      // ================= pass 2: quantize m' with the fresh row params =================
      if (MODE == MODE_STEP) {
        const float4* mp = reinterpret_cast<const float4*>(mprime);
        for (int k = 0; k < nch; ++k) {
          const int v = k * NCT + ct;
          if (v >= nvec) break;
          float m[16];
          if (MREC) {
            // recompute m' = b2*m + (1-b2)*g from the staged codes (same expression
            // as pass 1, so the same bits) instead of keeping a 4*cols smem buffer
            float g[16];
            const uint4 mq = *reinterpret_cast<const uint4*>(data + cp + v * 16);
            const uint4 gq = *reinterpret_cast<const uint4*>(data + 2 * cp + v * 16);
            dequant4(mq.x, dm, m); dequant4(mq.y, dm, m + 4);
            dequant4(mq.z, dm, m + 8); dequant4(mq.w, dm, m + 12);
            dequant4(gq.x, dg, g); dequant4(gq.y, dg, g + 4);
            dequant4(gq.z, dg, g + 8); dequant4(gq.w, dg, g + 12);
#pragma unroll
            for (int p = 0; p < 8; ++p) {
              const float2 M = sadd2(mul2(f2(h.b2), make_float2(m[2 * p], m[2 * p + 1])),
                                     mul2(f2(h.c2), make_float2(g[2 * p], g[2 * p + 1])));
              m[2 * p] = M.x;
              m[2 * p + 1] = M.y;
            }
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              const float4 f = mp[(k * 4 + q) * NCT + ct];
              m[4 * q] = f.x; m[4 * q + 1] = f.y; m[4 * q + 2] = f.z; m[4 * q + 3] = f.w;
            }
          }
          float em = 0.0f;
          uint32_t c[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) c[q] = quant4_fast(m + 4 * q, qm, em);
          if (!qm.fast || !(em < qm.thr)) {
#pragma unroll
            for (int q = 0; q < 4; ++q) c[q] = quant4_exact(m + 4 * q, qm);
          }
          uint8_t* mo = cx->m_out + v * 16;
          if (ALIGNED) {
            *reinterpret_cast<uint4*>(mo) = make_uint4(c[0], c[1], c[2], c[3]);
          } else {
            const int nvalid = min(16, cols - v * 16);
            for (int e = 0; e < nvalid; ++e) mo[e] = (uint8_t)(c[e >> 2] >> ((e & 3) * 8));
          }
        }
      }

      if (MODE == MODE_DECOMPOSE) {
        named_bar_sync(BAR_D, NCT);  // the row's offset from the look-back
        row_base_out = tabs->prefix[par];
      }

      // ================= CSR write (ascending columns) =================
      {
        const int64_t cap = (MODE == MODE_DECOMPOSE) ? a.cap_out : (int64_t)row_cap;
        for (int k = 0; k < nch; ++k) {
          const int pref_k = __shfl_sync(0xffffffffu, chunk_pref, k);
          if (tabs->cnt[par][k][cw] == 0) continue;  // warp-uniform
          const int v = k * NCT + ct;
          uint32_t mask = (v < nvec) ? (uint32_t)masks[v] : 0u;
          const int c = __popc(mask);
          int incl = c;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += t;
          }
          int pos = pref_k + incl - c;
          while (mask) {
            const int e = __ffs(mask) - 1;
            mask &= mask - 1u;
            const int col = v * 16 + e;
            float val;
            if (MODE == MODE_DECOMPOSE) {
              val = reinterpret_cast<const float*>(data)[col];
            } else {
              // recompute w' for this element exactly as pass 1 did (scalar, exact)
              float wv = dequant1(data[col], dw);
              if (bits16(obits, v) & (1u << e))
                wv = old_value(obits, frank, ovals, staged, old_begin, col, a.val_in);
              float mv = dequant1(data[cp + col], dm);
              float gv;
              if (GK == G_U8) {
                gv = dequant1(data[2 * cp + col], dg);
              } else {
                const float gr = load_graw<GK>(data + 2 * cp, col);
                gv = dequant1(quant_exact(gr, qg.s, qg.z, qg.qmax), dg);
              }
              lion1(wv, mv, gv, h);
              val = wv;
            }
            if (pos < cap) {
              const int64_t dst = (int64_t)row_base_out + pos;
              a.col_out[dst] = col;
              a.val_out[dst] = val;
            }
            ++pos;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }

  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t prev = atomicAdd(&a.hdr->done, 1u);
    if (prev == gridDim.x - 1) {
      a.hdr->ticket = 0u;
      a.hdr->done = 0u;
      a.hdr->epoch = a.hdr->epoch + 1u;
      __threadfence();
    }
  }
}

// ----------------------------------------------------------------------------
// host-side launcher
// ----------------------------------------------------------------------------
template <int MODE, int GK, bool AL, bool WD0, bool MREC = false>
static cudaError_t launch_t(const LaunchArgs& a, size_t smem, cudaStream_t st, int* grid_out) {
  auto k = row_engine_kernel<MODE, GK, AL, WD0, MREC>;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NT, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int grid = sms * per_sm;
  const int work = (MODE == MODE_DECOMPOSE) ? a.total_rows : a.n_blocks;
  if (grid > work) grid = work;
  if (grid < 1) grid = 1;
  k<<<grid, NT, smem, st>>>(a);
  if (grid_out) *grid_out = grid;
  return cudaGetLastError();
}

cudaError_t launch_row_engine(int mode, int gk, const LaunchArgs& a, cudaStream_t st,
                              int* grid_out) {
  const bool mrec = a.mrec && mode == MODE_STEP && gk == G_U8 && a.use_bulk;
  const size_t smem = row_engine_smem(mode, gk, a.cols_p, a.stages, mrec);
  const bool al = a.use_bulk != 0;
  const bool wd0 = (a.wd == 0.0f);
  if (mrec) {
    return wd0 ? launch_t<MODE_STEP, G_U8, true, true, true>(a, smem, st, grid_out)
               : launch_t<MODE_STEP, G_U8, true, false, true>(a, smem, st, grid_out);
  }
#define QFT_L(M, G)                                                              \
  if (wd0) return al ? launch_t<M, G, true, true>(a, smem, st, grid_out)        \
                     : launch_t<M, G, false, true>(a, smem, st, grid_out);      \
  return al ? launch_t<M, G, true, false>(a, smem, st, grid_out)                \
            : launch_t<M, G, false, false>(a, smem, st, grid_out)
#define QFT_L1(M)                                                                \
  return al ? launch_t<M, G_U8, true, false>(a, smem, st, grid_out)             \
            : launch_t<M, G_U8, false, false>(a, smem, st, grid_out)
  switch (mode) {
    case MODE_STEP:
      if (gk == G_U8) { QFT_L(MODE_STEP, G_U8); }
      if (gk == G_F32) { QFT_L(MODE_STEP, G_F32); }
      { QFT_L(MODE_STEP, G_BF16); }
    case MODE_DECOMPOSE: QFT_L1(MODE_DECOMPOSE);
    case MODE_RECON_F32: QFT_L1(MODE_RECON_F32);
    default: QFT_L1(MODE_RECON_BF16);
  }
#undef QFT_L
#undef QFT_L1
}

}  // namespace qftk
