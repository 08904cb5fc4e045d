// qft_internal.h -- host/device structures shared by the kernels and the C-ABI layer.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "qft_b200.h"

// CTAs per SM the row engine's register budget is sized for (launch bounds)
#ifndef QFT_MIN_CTAS
#define QFT_MIN_CTAS 3
#endif
// CTAs per SM the 128-thread step kernel is sized for
#ifndef QFT_STEP_MIN_CTAS
#define QFT_STEP_MIN_CTAS 4
#endif

namespace qftk {

// One tensor of a launch.
//
// CSR on the device is SLOTTED: row r of set k owns arena entries
// [rs[k][r], rs[k][r+1]) (a 16-byte aligned slot sized from its previous count
// plus slack) of which the first cnt[k][r] are used, columns ascending.  A step
// therefore needs no cross-row scan.  With cnt[k] == nullptr the arrays are a
// strict reference CSR (rs = row_ptr, count = rs[r+1]-rs[r]).
struct DevTensor {
  int32_t rows, cols;
  int32_t row_base, _pad;
  uint8_t* w_codes[2];
  int32_t* rs[2];
  int32_t* cnt[2];
  const float* w_scale;
  const int32_t* w_zp;
  const float* t_min;
  const float* t_max;
  uint8_t* m_codes[2];
  float* m_scale[2];
  int32_t* m_zp[2];
  const uint8_t* g_codes;
  const float* g_scale;
  const int32_t* g_zp;
  const void* g_raw;   // f32 or bf16 raw gradient (fused quantize_state)
  const float* w_f32;  // decompose input
  void* out;           // reconstruct output (f32 or bf16)
};

// A static unit of work: up to 32 consecutive rows of one tensor.
struct RowBlock {
  int32_t tensor, row0, nrows, _pad;
};
constexpr int kBlockRows = 8;  // step rows per work item (static round-robin over warps)

// Device header of a workspace.  `epoch` tags the decompose look-back status
// words so the status array never needs clearing; the last CTA of every launch
// bumps it and resets the ticket counter.
struct Header {
  uint32_t epoch;
  uint32_t ticket;
  uint32_t done;
  uint32_t overflow;
  uint32_t err;
  uint32_t _pad;
  int64_t total_nnz;
  int64_t _pad2[5];
};

enum GradKind : int { G_U8 = 0, G_F32 = 1, G_BF16 = 2 };

// error bits in Header::err
constexpr uint32_t ERR_MPARAMS = 1u;   // momentum min > max (NaN in column 0)
constexpr uint32_t ERR_GPARAMS = 2u;   // gradient min > max

struct LaunchArgs {
  DevTensor* tensors;
  const RowBlock* blocks;
  int32_t n_tensors;
  int32_t n_blocks;
  int32_t total_rows;
  int32_t flip;
  int32_t bit_width;
  float lr, b1, b2, wd;
  const int32_t* col_in;
  const float* val_in;
  int32_t* col_out;
  float* val_out;
  int64_t cap_out;    // decompose: arena capacity (strict CSR output)
  Header* hdr;
  unsigned long long* status;
  int32_t cols_p;     // max padded (x16) row length of the launch
  int32_t _pad0;
  int32_t use_bulk;   // TMA bulk copies (all rows 16-byte aligned)
  int32_t slotted_in; // input CSR is slotted (16-byte aligned slots)
  int32_t oldcap;     // step: old outliers per row handled by the sparse pass
  int32_t oldcap6;    // rows kernel: old outliers per row of its sparse table
  float negzero;      // -0.0f at run time (an FFMA2 addend ptxas cannot fold)
  struct RowPrep* prep;          // rows kernel: per-row records (k_step_prep)
  RowBlock* xlist;               // rows outside the stable tier (general kernel)
  int32_t* xcount;               // their number (device)
  const int32_t* n_blocks_dev;   // step_kernel: read the block count from the device
  int32_t* xclear;               // prep: the OTHER flip's row-list counter, zeroed for the next step
  uint32_t* oflag;               // mapped pinned overflow flag (host-visible without a sync)
  int32_t* xseen;                // step_kernel / GEN rows kernel: the list length it saw
                                 // (mapped pinned)
  int32_t* rclaim;               // prep: [2] row-claim counters (zeroed); rows kernel: its own
  int32_t* slist;                // prep: stable-tier rows (this step) ...
  int32_t* glist;                // ... and GEN-tier rows
  int32_t* scount;
  int32_t* gcount;
  const int32_t* rlist;          // rows kernel: the row list it iterates ...
  const int32_t* rcount;         // ... and its length (device)
  int32_t gen_on;                // prep: route rows that miss only (*) to the GEN tier
  int32_t epoch;                 // prep: this launch's look-back epoch
  unsigned long long* pstatus;   // prep: per-block look-back status words
};

// Per-row record of the rows kernel (128 B), written by k_step_prep every step and
// bulk-copied into shared memory with the row's codes: everything a row needs.
struct RowPrep {
  // info: bit 0 stable tier; bits 1..6 outlier flags of the candidate outcomes below;
  // bits 8..15 the outlier payload code clamp(z, 0, qmax); bits 16..31 outcomes 4, 5
  uint32_t info;
  // cand: the codes of the candidate outcomes 0..3 (a byte each).  Outcome 3*B + S is a
  // dense weight of code 0 (B=0) or qmax (B=1) after the Lion step with sign(d) < 0,
  // == 0, > 0 (S = 0, 1, 2): w' = w - lr*(sign(d) + wd*w) takes only these 3 values.
  uint32_t cand;
  int32_t ob, on;                // old CSR slot start / count
  int32_t so, co, zw, zm;        // new slot start / capacity, w / m zero points
  float sm, negc_m, sg, negc_g;  // m / g scale and -(2^23 + z) (the PRMT dequant form)
  int32_t zg;
  float sw, tmin, tmax;
  const uint8_t* w_in;           // row pointers of the step's inputs ...
  const uint8_t* m_in;
  const uint8_t* g_in;
  uint8_t* w_out;                // ... and outputs
  uint8_t* m_out;
  float* m_scale_out;            // &m_scale[out][row], &m_zp[out][row], &cnt[out][row]
  int32_t* m_zp_out;
  int32_t* cnt_out;
};
static_assert(sizeof(RowPrep) == 128, "RowPrep is one 128-byte record");

size_t step_kernel_smem(int gk, int cols_p, int oldcap);
cudaError_t launch_step_kernel(int gk, const LaunchArgs& a, cudaStream_t s);

// A resolved kernel launch (function, geometry, instance name), computed once per plan so
// the per-step host path is one cudaLaunchKernel per kernel (no attribute / occupancy
// queries, no environment reads).
struct KLaunch {
  const void* fn = nullptr;
  int grid = 0, block = 0;
  size_t smem = 0;
  int arg1 = 0;  // the kernel's second argument, for kernels taking (LaunchArgs, int)
  char name[96] = {0};
};
cudaError_t launch_k(const KLaunch& k, const LaunchArgs& a, cudaStream_t s);
cudaError_t launch_k2(const KLaunch& k, const LaunchArgs& a, cudaStream_t s);  // (a, k.arg1)
// the general step kernel's launch for grad kind gk (rows of a.n_blocks / the device list)
cudaError_t resolve_step_kernel(int gk, const LaunchArgs& a, KLaunch* out);

// per-plan launch cache of the rows path (rowstep.cu)
struct RowsCache {
  KLaunch rows[2];     // by slotted input (0/1)
  KLaunch gen[2];      // general kernel over the device list, by weight decay == 0 (0/1)
  int last_flip = -1;  // the flip of the previous step (a repeated flip re-zeroes its counter)
  // [16]: per flip f, [4f] general-list, [4f+1] stable-list, [4f+2] GEN-list counters,
  // [4f+3] the prep block ticket; [8] / [9] the stable / GEN rows kernels' claim counters
  int32_t* xcount = nullptr;
  int32_t* slist = nullptr;  // stable-tier / GEN-tier row lists (rows entries each)
  int32_t* glist = nullptr;
  KLaunch genrows[2];        // the GEN rows kernel, by slotted input (0/1)
  int gen_on = 1;
  int stable_allrows = 0;  // A/B: the stable kernel over every row (no list)
  int route_on = 1;        // QFT_NO_ROUTE=1 disables routing stable rows into the GEN list
  bool routed = false;     // the last step routed its stable rows (no stable launch)
  unsigned long long* pstatus = nullptr;  // prep look-back status words (one per block)
  int epoch = 0;
  // the general-tier row count the general kernel last saw (mapped pinned, read without a
  // sync): an empty list last time -> launch that kernel with one CTA per SM (it still
  // covers any list length, grid-stride)
  volatile int32_t* seen_host = nullptr;
  int32_t* seen_dev = nullptr;
  int sms = 0;
  int cap_per_sm = 0;  // rows kernel: resident CTAs per SM cap (0: occupancy maximum)
};

int step_kernel_max_cols();

// quantize_state of a raw (f32/bf16) gradient into the plan's u8 entry (gradquant.cu)
cudaError_t resolve_grad_quant(int gk, int max_cols, int total_rows, KLaunch* out);
// ... and the ZeRO-1 reduce-scatter fused with it: bf16 rows summed from npeer peer buffers
cudaError_t resolve_rs_grad_quant(int max_cols, int total_rows, KLaunch* out);
cudaError_t launch_rs_grad_quant(const KLaunch& k, const LaunchArgs& a, const int64_t* deltas,
                                 int npeer, cudaStream_t s);

// v6 rows kernel (rowstep.cu): prep + stable rows + step_kernel over the rest
bool rows_kernel_eligible(int gk, int use_bulk, int uniform_cols);
int rows_kernel_oldcap(int cols);
cudaError_t launch_rows_step(const LaunchArgs& a, RowsCache& c, cudaStream_t s);

// decomposition with given thresholds (decompose.cu)
cudaError_t decompose_codes(const float* w, int rows, int cols, const float* scale,
                            const int32_t* zp, const float* t_min, const float* t_max,
                            int bit_width, uint8_t* codes, int32_t* counts, cudaStream_t s);
cudaError_t decompose_csr(const float* w, int rows, int cols, const float* t_min,
                          const float* t_max, const int32_t* row_ptr, int32_t* col_idx,
                          float* values, cudaStream_t s);
cudaError_t csr_row_ptr(const int32_t* counts, int rows, int32_t* row_ptr, cudaStream_t s,
                        const int32_t* slot_start = nullptr);
// ZeRO-1 packed all-gather of slotted segments (csr.cu)
constexpr int QFT_PACK_MAXW = 8;
struct PackWidths {
  const int32_t* col_in[QFT_PACK_MAXW];
  const float* val_in[QFT_PACK_MAXW];
  int32_t* col_out[QFT_PACK_MAXW];
  float* val_out[QFT_PACK_MAXW];
  int64_t base[QFT_PACK_MAXW];
  int32_t first_chunk[QFT_PACK_MAXW];
};
cudaError_t csr_pack_plan_create(const qftc_pack_segment* segs, int nseg, int nwidth,
                                 cudaStream_t s, void** plan);
cudaError_t csr_pack_run(void* plan, const int32_t* row_start, const int32_t* row_count,
                         PackWidths P, int32_t* row_start_out, cudaStream_t s);
void csr_pack_plan_destroy(void* plan);
int csr_pack_nwidth(const void* plan);

// checkpoint CRC over device segments (crc32.cu); synchronises
cudaError_t crc32_device(const void* const* segs, const int64_t* lens, int n, uint32_t* crc_out,
                         cudaStream_t s);

// weight expansion (expand.cu): one launch per expand_max_tensors() tensors
int expand_max_tensors();
cudaError_t launch_expand(const qftc_expand_tensor* ts, int n, bool bf16, cudaStream_t s);
// tix[r][t] = the first used slot entry of row r whose column is >= t * tile_cols (t < tiles),
// tix[r][tiles] = the row's used end (dqgemm_t.cu, k_csr_tile_index)
cudaError_t launch_csr_tile_index(const int32_t* row_start, const int32_t* row_count,
                                  const int32_t* col, int rows, int tiles, int tile_cols,
                                  int32_t* tix, cudaStream_t st);
// the consumer GEMM with the weight dequantization fused into its operand producer
// (dqgemm.cu): y[M,N] = x[M,K] . W^T, x / y bf16, W a dense-and-sparse QFT weight;
// workspace: the per-(row, 32-column) CSR index
size_t dq_gemm_workspace_bytes(int N, int K);
cudaError_t launch_dq_gemm(const void* x, int M, int K, const uint8_t* codes, int N,
                           const float* scale, const int32_t* zp, const int32_t* row_start,
                           const int32_t* row_count, const int32_t* col, const float* val,
                           void* y, void* workspace, cudaStream_t s, bool build_index = true);
// re-plan slot capacities (csr.cu, k_replan_caps)
cudaError_t launch_replan_caps(const uint8_t* codes, int rows, int cols, int bit_width,
                               const int32_t* cnt_out, const int32_t* cnt_in, int lvl, int gmul,
                               int64_t* caps, cudaStream_t st);
// the backward's input gradient dX = dY . W with W dequantized in the operand producer
// (dqgemm_t.cu); workspace: the per-(row, column tile) CSR index
size_t dq_gemm_t_workspace_bytes(int O, int I);
cudaError_t launch_dq_gemm_t(const void* dy, int T, int O, const uint8_t* codes, int I,
                             const float* scale, const int32_t* zp, const int32_t* row_start,
                             const int32_t* row_count, const int32_t* col, const float* val,
                             void* dx, void* workspace, cudaStream_t st, bool build_index = true);
// the backward weight gradient with the sink's quantization in the GEMM epilogue (wgrad.cu):
// codes/scale/zp = quantize_state(dY^T . X [+ dequantize(entry)]); workspace: rows bounds,
// counters and the error word (its last uint32)
size_t wgrad_workspace_bytes(int O);
cudaError_t launch_wgrad_quant(const void* dy, const void* x, int T, int O, int I, int bw,
                               int accumulate, uint8_t* codes, float* scale, int32_t* zp,
                               float* g_out, double* norm_sq, void* workspace, uint32_t lbo,
                               uint32_t sbo, cudaStream_t st);
// opt-in checkpoint format extensions (ckptext.cu)
cudaError_t launch_pack_codes(const uint8_t* src, int rows, int cols, int bits, uint8_t* dst,
                              bool unpack, cudaStream_t s);
cudaError_t launch_mom_blocks(const uint8_t* codes, const float* scale, const int32_t* zp,
                              int rows, int cols, int bits, int block, uint8_t* out,
                              float* oscale, int32_t* ozp, bool from_blocks, uint32_t* err,
                              cudaStream_t s);
// an expand plan: the table uploaded once, any number of tensors per launch
cudaError_t expand_plan_create(const qftc_expand_tensor* ts, int n, bool bf16, cudaStream_t s,
                               void** out);
cudaError_t expand_plan_run(void* plan, cudaStream_t s);
void expand_plan_destroy(void* plan);

}  // namespace qftk
