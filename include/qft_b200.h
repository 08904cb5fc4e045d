/*
 * qft_b200.h -- C-ABI of the B200-native QFT model-state update path.
 *
 * This is the drop-in boundary for the reference's quantizer/optimizer API
 * (/root/reference/proj/include/qft/{quantize,optimizer,gradflow}.hpp).  Every
 * entry point below names the reference interface it replaces (file:line).
 * Signatures use plain pointers, sizes and a CUDA stream -- no torch or STL types.
 *
 * Memory: every array argument is DEVICE memory unless the name ends in _host.
 * Layout: row-major [rows x cols], row = output channel (tensor.hpp:13-16).
 *   codes       u8  [rows*cols]  one byte per element for any bit width <= 8
 *                                (quantize.hpp:41, :356)
 *   scale       f32 [rows]       per-channel scale (> 0)
 *   zero_point  i32 [rows]       unclipped (quantize.hpp:22-25)
 *   t_min,t_max f32 [rows]       cached dense thresholds (quantize.hpp:66)
 *   row_ptr     i32 [rows+1]     strict CSR, col_idx ascending within a row
 *   col_idx     i32 [nnz], values f32 [nnz]   (quantize.hpp:48-57)
 *
 * Errors: functions return QFTC_OK (0) or a negative status; qftc_last_error()
 * returns a thread-local message.  QFTC_EINVAL <-> std::invalid_argument and
 * QFTC_ERANGE <-> std::out_of_range of the reference, with the same validation
 * order, so the C++ shim (include/qft_b200/qft.hpp) rethrows the same types.
 *
 * Asynchrony: all work is enqueued on `stream`; functions that must return a
 * host-visible value (nnz, status) say "synchronises".  There is no CPU
 * fallback: without a CUDA device every compute call returns QFTC_ECUDA.
 */
#ifndef QFT_B200_H_
#define QFT_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* qftc_stream_t; /* == cudaStream_t */

enum {
  QFTC_OK = 0,
  QFTC_EINVAL = -1,    /* std::invalid_argument in the reference */
  QFTC_ERANGE = -2,    /* std::out_of_range in the reference      */
  QFTC_ECUDA = -3,     /* CUDA runtime error / no device           */
  QFTC_EOVERFLOW = -4, /* CSR output capacity exceeded (re-run with more) */
  QFTC_ENOTSUP = -5    /* shape outside what the kernels support   */
};

enum { QFTC_PERCENTILE = 0, QFTC_RANGE_FRACTION = 1 }; /* ThresholdKind, quantize.hpp:20 */
enum { QFTC_GRAD_U8 = 0, QFTC_GRAD_F32 = 1, QFTC_GRAD_BF16 = 2 };

const char* qftc_last_error(void);
int qftc_version(void);
/* largest row length (cols) the row kernels accept */
int qftc_max_cols(void);

/* ---------------------------------------------------------------- L0 / L1 */

/* channel_minmax  (tensor.hpp:133-148) */
int qftc_channel_minmax(const float* x, int rows, int cols, float* mins, float* maxs,
                        qftc_stream_t stream);

/* affine_params_from_bounds  (quantize.hpp:105-131).  Validation of min <= max
 * needs the data: this call synchronises and returns QFTC_EINVAL on violation. */
int qftc_affine_params_from_bounds(const float* mins, const float* maxs, int64_t n,
                                   int bit_width, float* scale, int32_t* zero_point,
                                   qftc_stream_t stream);

/* quantize with given params; channels is 1 or rows  (quantize.hpp:149-175) */
int qftc_quantize(const float* x, int rows, int cols, const float* scale,
                  const int32_t* zero_point, int channels, int bit_width, uint8_t* codes,
                  qftc_stream_t stream);

/* quantize_state, affine mode: fresh per-row params + quantize (quantize.hpp:189-193).
 * Fused row kernel: one HBM read of x.  Synchronises only if `check` != 0 (to
 * report a NaN-in-column-0 row as QFTC_EINVAL like the reference). */
int qftc_quantize_state(const float* x, int rows, int cols, int bit_width, uint8_t* codes,
                        float* scale, int32_t* zero_point, int check, qftc_stream_t stream);

/* accumulate (gradflow.hpp:52-58): the integer-form micro-batch gradient sum,
 * quantize_state(dequantize(acc) + g_new) with fresh per-row params and acc's bit
 * width, fused in one row kernel (the fp32 sum never reaches HBM).  May run in place
 * (codes_out == codes, ...).  Synchronises; a NaN in column 0 of the sum ->
 * QFTC_EINVAL (the reference's min > max). */
int qftc_accumulate_state(const uint8_t* codes, const float* scale, const int32_t* zero_point,
                          int rows, int cols, int bit_width, const float* g_new,
                          uint8_t* codes_out, float* scale_out, int32_t* zero_point_out,
                          qftc_stream_t stream);

/* dequantize  (quantize.hpp:195-212) -> f32, and the bf16 expansion (RNE of the f32) */
int qftc_dequantize(const uint8_t* codes, int rows, int cols, const float* scale,
                    const int32_t* zero_point, int channels, float* out, qftc_stream_t stream);
int qftc_dequantize_bf16(const uint8_t* codes, int rows, int cols, const float* scale,
                         const int32_t* zero_point, int channels, uint16_t* out,
                         qftc_stream_t stream);

/* compute_outlier_thresholds  (quantize.hpp:216-247): exact per-row order
 * statistics by radix select (percentile) or row range (range_fraction). */
int qftc_outlier_thresholds(const float* w, int rows, int cols, double fraction, int kind,
                            float* t_min, float* t_max, qftc_stream_t stream);

/* decompose_dense_sparse  (quantize.hpp:253-290).  Writes dense codes, the
 * threshold-derived params, row_ptr (rows+1) and up to `capacity` CSR entries.
 * The true nnz is row_ptr[rows]; if it exceeds capacity the call returns
 * QFTC_EOVERFLOW (synchronises) and can be re-run with larger buffers. */
int qftc_decompose_dense_sparse(const float* w, int rows, int cols, const float* t_min,
                                const float* t_max, int bit_width, uint8_t* codes, float* scale,
                                int32_t* zero_point, int32_t* row_ptr, int32_t* col_idx,
                                float* values, int64_t capacity, int64_t* nnz_host,
                                qftc_stream_t stream);

/* reconstruct  (quantize.hpp:331-338) -> f32, and -> bf16 for the next forward
 * (network.hpp:208-211 consumer).  row_ptr may hold absolute offsets into a shared
 * CSR arena (col_idx/values are indexed by row_ptr directly). */
int qftc_reconstruct(const uint8_t* codes, int rows, int cols, const float* scale,
                     const int32_t* zero_point, const int32_t* row_ptr, const int32_t* col_idx,
                     const float* values, float* out, qftc_stream_t stream);
int qftc_reconstruct_bf16(const uint8_t* codes, int rows, int cols, const float* scale,
                          const int32_t* zero_point, const int32_t* row_ptr,
                          const int32_t* col_idx, const float* values, uint16_t* out,
                          qftc_stream_t stream);

/* ---------------------------------------------------------------- L4: Lion */

/* LionHyper  (optimizer.hpp:15-21) */
typedef struct {
  float lr, beta1, beta2, weight_decay;
} qftc_lion_hyper;

/* One layer of lion_step_quantized (optimizer.hpp:85-120) for a grouped launch.
 * Ping-pong state: a step with flip=f reads set [f] and writes set [1-f]; the
 * caller swaps its view after the step.  The weight's dense params and
 * thresholds are fixed between refreshes (requantize_weight, quantize.hpp:318-329)
 * and are read-only here.
 *
 * Outliers live in a SLOTTED CSR on the device: row r of set k owns entries
 * [row_start[k][r], row_start[k][r+1]) of the plan's arena k (offsets absolute in
 * the arena, multiples of 4 so slots are 16-byte aligned), the first
 * row_count[k][r] of them used, columns ascending.  No row of a step depends on
 * another row.  A row whose new count exceeds its slot sets the overflow status;
 * the caller re-plans row_start[1-f] (qftc_csr_plan_slots on the returned counts)
 * and re-runs the step -- its inputs (set f) are intact.  The strict reference
 * CSR is produced by qftc_csr_compact.
 *
 * The gradient is the GradientStack entry (u8 codes + per-row params,
 * gradflow.hpp:77) or, for QFTC_GRAD_F32/BF16, the raw fp gradient that the
 * backward sink would quantize: the fused kernel applies quantize_state ->
 * dequantize to it exactly. */
typedef struct {
  int32_t rows, cols;
  uint8_t* w_codes[2];
  int32_t* row_start[2];
  int32_t* row_count[2];
  const float* w_scale;
  const int32_t* w_zero_point;
  const float* t_min;
  const float* t_max;
  uint8_t* m_codes[2];
  float* m_scale[2];
  int32_t* m_zero_point[2];
  const uint8_t* g_codes;
  const float* g_scale;
  const int32_t* g_zero_point;
  const void* g_raw;
} qftc_lion_tensor;

typedef struct qftc_plan qftc_plan; /* opaque */

/* Build a grouped step plan over n tensors (uploads descriptors, allocates the
 * look-back workspace; synchronises).  All tensors share bit_width and gradient
 * kind.  CSR arenas: col_idx[k]/values[k] with capacity[k] entries, k = 0, 1. */
int qftc_plan_create(qftc_plan** plan, const qftc_lion_tensor* tensors_host, int n,
                     int bit_width, int grad_kind, int32_t* col_idx[2], float* values[2],
                     const int64_t capacity[2], qftc_stream_t stream);
/* Re-point the CSR arenas (after growing them). */
int qftc_plan_set_arena(qftc_plan* plan, int32_t* col_idx[2], float* values[2],
                        const int64_t capacity[2]);
/* Enqueue one fused quantized Lion step over every row of every tensor
 * (dequant g,m,w -> Lion -> requant m (fresh params) -> requant w (cached
 * thresholds) + ordered CSR re-extraction), reading set [flip]. */
int qftc_plan_step(qftc_plan* plan, int flip, qftc_lion_hyper hyper, qftc_stream_t stream);
/* One step over several plans (e.g. a model's width classes) that run CONCURRENTLY:
 * plan i is enqueued on its own stream, forked from and joined back into `stream`
 * (events, no host synchronisation), in the order given -- pass the wide classes first
 * so their CTAs are resident before the dominant class fills the rest of the GPU (the
 * rows kernel claims rows dynamically, so a class's late CTAs just take fewer rows). */
int qftc_plans_step(qftc_plan* const* plans, int n, int flip, qftc_lion_hyper hyper,
                    qftc_stream_t stream);
/* The fused ZeRO-1 reduce-scatter: a bf16 raw-gradient plan reads
 * its rows of the summed gradient straight from npeer peer buffers over NVLink peer memory
 * (peer p's copy of a row lives at the plan's own gradient address + byte_deltas[p]), sums
 * them in fp32 in peer order and quantizes them (quantize_state) in the same pass; npeer 0
 * restores the local gradient.  CUDA IPC helpers map the peers' buffers: a handle of the
 * allocation holding ptr (+ ptr's offset in it), its mapping in this process, the unmap. */
int qftc_plan_set_peer_gradients(qftc_plan* plan, const int64_t* byte_deltas, int npeer);
int qftc_ipc_handle(const void* ptr, unsigned char handle[64], int64_t* offset);
int qftc_ipc_open(const unsigned char handle[64], void** base);
int qftc_ipc_close(void* base);
/* device -> device copy between (IPC-mapped) peer and local buffers (cudaMemcpyDefault) */
int qftc_copy_peer(void* dst, const void* src, size_t bytes, qftc_stream_t stream);
/* Cap the resident CTAs per SM of a plan's rows kernel (0: occupancy maximum), so a
 * concurrently stepped plan leaves room for another's CTAs. */
int qftc_plan_set_ctas_per_sm(qftc_plan* plan, int ctas_per_sm);
/* Synchronises; returns the new total nnz of the arena written by the last step
 * and QFTC_EOVERFLOW / QFTC_EINVAL if that step overflowed or hit a degenerate row. */
int qftc_plan_result(qftc_plan* plan, int64_t* nnz_total, qftc_stream_t stream);
/* number of kernel launches one qftc_plan_step enqueues (for accounting; a step that
 * routes its few stable rows into the GEN list -- fewer than 1/16 of the rows were stable
 * the step before -- skips the stable launch and enqueues one fewer) */
int qftc_plan_launches(const qftc_plan* plan);
/* the main kernel instance the last qftc_plan_step launched, e.g.
 * "rows_kernel<128,5,3,2,4096,8>" (MAXT, MINB, stages, FULL, compile-time columns, bit
 * width) or "step_kernel<gk,aligned,wd0>"; "" before the first step */
const char* qftc_plan_kernel_name(const qftc_plan* plan);
/* 1 if a step of this plan has overflowed a CSR slot and qftc_plan_result has not been
 * called since (a mapped host flag: no synchronisation, so a step still in flight may not
 * be reflected yet).  The overflowed step's output set is incomplete: re-plan the slots
 * and re-run it from its (intact) input set before stepping on. */
int qftc_plan_pending_overflow(const qftc_plan* plan);
/* rows of the last step in the stable tier (rows kernel) and the general tier (general
 * kernel); synchronises */
/* rows of the last step per tier: [0] stable (pass-through rows kernel), [1] GEN (rows
 * kernel requantizing every code; includes stable rows routed into the GEN list), [2]
 * general (step_kernel).  Synchronises. */
int qftc_plan_tiers(qftc_plan* plan, int64_t rows_out[3], qftc_stream_t stream);
int qftc_plan_tier_rows(qftc_plan* plan, int64_t* stable_rows, int64_t* general_rows,
                        qftc_stream_t stream);
int qftc_plan_destroy(qftc_plan* plan);

/* Single-tensor convenience: lion_step_quantized for one layer, out-of-place,
 * synchronous (reference semantics).  Returns the new nnz in *nnz_host. */
int qftc_lion_step(int rows, int cols, int bit_width, const uint8_t* g_codes,
                   const float* g_scale, const int32_t* g_zero_point, const uint8_t* m_codes,
                   const float* m_scale, const int32_t* m_zero_point, const uint8_t* w_codes,
                   const float* w_scale, const int32_t* w_zero_point, const float* t_min,
                   const float* t_max, const int32_t* row_ptr, const int32_t* col_idx,
                   const float* values, uint8_t* m_codes_out, float* m_scale_out,
                   int32_t* m_zero_point_out, uint8_t* w_codes_out, int32_t* row_ptr_out,
                   int32_t* col_idx_out, float* values_out, int64_t capacity,
                   qftc_lion_hyper hyper, int64_t* nnz_host, qftc_stream_t stream);

/* ---------------------------------------------------------------- slotted CSR */

/* Slot capacities for re-planning a slotted CSR after an overflow (the engine's
 * _replan): per row, want = count_out + (dense codes at 0 or 2^b-1 in `codes` -- the
 * elements a stable-tier step can turn into outliers), grow = max(count_out - count_in, 0),
 * caps[r] = want + want/4 + growth_mult*grow + want*level/4 + min(8 << 2 level, 64), rounded
 * up to a multiple of 4 (16-byte slots).  One pass over the codes, no synchronisation. */
int qftc_csr_replan_caps(const uint8_t* codes, int rows, int cols, int bit_width,
                         const int32_t* count_out, const int32_t* count_in, int level,
                         int growth_mult, int64_t* caps, qftc_stream_t stream);

/* row_start[0..rows] of 16-byte aligned slots with capacity count + count/4 + slack
 * (rounded up to 4 entries), counts taken from `counts` or, if NULL, from a
 * strict `row_ptr`.  Synchronises to return the arena size in *total_host. */
int qftc_csr_plan_slots(const int32_t* counts, const int32_t* row_ptr, int rows, int slack,
                        int32_t* row_start, int64_t* total_host, qftc_stream_t stream);
/* copy every row's entries from a slotted (src_count != NULL) or strict (src_count
 * == NULL: src_start is row_ptr) CSR to the slots dst_start of another arena. */
int qftc_csr_copy_rows(int rows, const int32_t* src_start, const int32_t* src_count,
                       const int32_t* src_col, const float* src_val, const int32_t* dst_start,
                       int32_t* dst_col, float* dst_val, int64_t dst_capacity,
                       qftc_stream_t stream);
/* ZeRO-1 all-gather of only the USED CSR entries.  A pack PLAN
 * describes nseg slotted segments (one per tensor row range): rows, width class (< nwidth
 * <= 8), the offset of its rows+1 slot starts in row_start and of its rows counts in
 * row_count (counts are clamped to their slots).  A run packs each class's used entries
 * densely -- classes independent, segments in table order -- from col_in[w] / val_in[w]
 * (the class's slotted arena) into col_out[w] / val_out[w] (capacity: the class's nnz)
 * and writes row_start_out (row_start's layout): the packed starts plus base[w], the
 * rank's offset inside the gathered arena, so receivers index the gathered entries
 * directly.  create uploads the chunk table and synchronises; run is asynchronous (three
 * launches for any number of segments); col_in..base are host arrays of nwidth entries. */
typedef struct qftc_pack_segment {
  int32_t rows, width;
  int64_t rs_off, cnt_off;
} qftc_pack_segment;
typedef struct qftc_csr_pack_plan qftc_csr_pack_plan;
int qftc_csr_pack_plan_create(qftc_csr_pack_plan** plan, const qftc_pack_segment* segments,
                              int nseg, int nwidth, qftc_stream_t stream);
int qftc_csr_pack_run(qftc_csr_pack_plan* plan, const int32_t* row_start,
                      const int32_t* row_count, const int32_t* const* col_in,
                      const float* const* val_in, int32_t* const* col_out,
                      float* const* val_out, const int64_t* base, int32_t* row_start_out,
                      qftc_stream_t stream);
int qftc_csr_pack_plan_destroy(qftc_csr_pack_plan* plan);
/* slotted -> strict reference CSR (SparseOutliers, quantize.hpp:48-57): row_ptr =
 * exclusive scan of the counts, entries gathered.  Synchronises for *nnz_host;
 * QFTC_EOVERFLOW if nnz > capacity. */
int qftc_csr_compact(int rows, const int32_t* row_start, const int32_t* row_count,
                     const int32_t* col_idx, const float* values, int32_t* row_ptr,
                     int32_t* col_out, float* val_out, int64_t capacity, int64_t* nnz_host,
                     qftc_stream_t stream);
/* reconstruct from a slotted CSR (out: f32, or bf16 if bf16 != 0) */
int qftc_reconstruct_slots(const uint8_t* codes, int rows, int cols, const float* scale,
                           const int32_t* zero_point, const int32_t* row_start,
                           const int32_t* row_count, const int32_t* col_idx,
                           const float* values, void* out, int bf16, qftc_stream_t stream);

/* Grouped weight expansion for the next forward (quantize.hpp:331-338 reconstruct of
 * every tensor of a model, network.hpp:208-211): one launch per up to 224 tensors, no
 * host synchronisation, no device allocation.  Each tensor: codes [rows, cols] u8, its
 * per-row scale/zero_point, its CSR as row_start (+ row_count for a slotted CSR; NULL
 * means strict, count = row_start[r+1]-row_start[r]) indexing col_idx/values, and out
 * [rows, cols] f32 or (bf16 != 0) bf16 bits, RNE of the f32 reconstruction. */
typedef struct qftc_expand_tensor {
  int32_t rows, cols;
  const uint8_t* codes;
  const float* scale;
  const int32_t* zero_point;
  const int32_t* row_start;
  const int32_t* row_count;
  const int32_t* col_idx;
  const float* values;
  void* out;
} qftc_expand_tensor;
int qftc_expand(const qftc_expand_tensor* tensors, int n_tensors, int bf16,
                qftc_stream_t stream);

/* The backward's input gradient with the dequantization fused into the operand producer
 * (backward weight operand; network.hpp:145 backward_core:
 * in_grad = matmul(out_grad, w), w = reconstruct(W), gradflow.hpp:78): dx[tokens,in] =
 * dy[tokens,out] . W for the dense-and-sparse W [out,in] (codes, per-row params, slotted CSR
 * with row_count or strict with row_count = NULL), dy / dx bf16 row-major.  The tensor cores
 * read bf16 RNE(reconstruct(W)) as an MN-major operand built in shared memory from the u8
 * codes.  workspace: qftc_dequant_gemm_t_workspace_bytes(out, in) device bytes (a per-row,
 * per-column-tile CSR index rebuilt by the call).  out % 64 == 0, in % 64 == 0; dy, codes, dx
 * 16-byte aligned. */
int64_t qftc_dequant_gemm_t_workspace_bytes(int out_features, int in_features);
/* The per-(row, 32-column) CSR slot index both GEMMs build into their workspace, built once
 * (qftc_dequant_gemm_workspace_bytes(rows, cols) == qftc_dequant_gemm_t_workspace_bytes(
 * rows, cols) bytes) and reused by the _prebuilt forms while the weight's CSR is unchanged
 * -- e.g. across the micro-batches between two optimizer steps. */
int qftc_dequant_gemm_index(const int32_t* row_start, const int32_t* row_count,
                            const int32_t* col_idx, int rows, int cols, void* index,
                            qftc_stream_t stream);
int qftc_dequant_gemm_prebuilt(const void* x_bf16, int m, int k, const uint8_t* codes, int n,
                               const float* scale, const int32_t* zero_point,
                               const int32_t* col_idx, const float* values, const void* index,
                               void* y_bf16, qftc_stream_t stream);
int qftc_dequant_gemm_t_prebuilt(const void* dy_bf16, int tokens, int out_features,
                                 const uint8_t* codes, int in_features, const float* scale,
                                 const int32_t* zero_point, const int32_t* col_idx,
                                 const float* values, const void* index, void* dx_bf16,
                                 qftc_stream_t stream);
int qftc_dequant_gemm_t(const void* dy_bf16, int tokens, int out_features, const uint8_t* codes,
                        int in_features, const float* scale, const int32_t* zero_point,
                        const int32_t* row_start, const int32_t* row_count,
                        const int32_t* col_idx, const float* values, void* dx_bf16,
                        void* workspace, qftc_stream_t stream);

/* The backward's weight gradient with the sink fused into the GEMM epilogue (SURVEY.md
 * §8(f) row 2; network.hpp:131-155 backward_core: wgrad = matmul(transpose(out_grad), in),
 * then the sink gradflow.hpp:70-84).  G[out,in] = dy[tokens,out]^T . x[tokens,in] (bf16
 * row-major activations, fp32 accumulation in TMEM) goes straight into the GradientStack
 * entry (codes [out,in] u8, scale [out], zero_point [out]):
 *   accumulate == 0: quantize_state(G, bit_width)                       (gradflow.hpp:77)
 *   accumulate == 1: quantize_state(dequantize(entry) + G), in place    (accumulate, :52-58)
 * The fp32 gradient never reaches HBM.  Optional: g_out [out,in] f32 receives the values
 * that were quantized (G, or the sum), norm_sq (device double) += sum(G^2) (backward_core's
 * norm, network.hpp:140).  workspace: qftc_wgrad_workspace_bytes(out) device bytes.
 * in % 64 == 0, out % 8 == 0; dy, x, codes, g_out 16-byte aligned; a row may span at most
 * one tile of 256 columns per SM (QFTC_ENOTSUP otherwise).  check != 0 synchronises and
 * reports a NaN in column 0 as QFTC_EINVAL (the reference's min > max). */
int64_t qftc_wgrad_workspace_bytes(int out_features);
int qftc_wgrad_quant(const void* dy_bf16, const void* x_bf16, int tokens, int out_features,
                     int in_features, int bit_width, int accumulate, uint8_t* codes, float* scale,
                     int32_t* zero_point, float* g_out, double* norm_sq, void* workspace,
                     int check, qftc_stream_t stream);

/* The forward consumer's GEMM with the dequantization fused into its operand producer
 * (network.hpp:113-129 forward_core: matmul(cur, transpose(w))):
 * y[m,n] = x[m,k] . W^T for a dense-and-sparse weight W [n,k] (codes, per-row params,
 * CSR -- slotted with row_count, or strict with row_count = NULL), x and y bf16 row-major.
 * The tensor cores read bf16 RNE(reconstruct(W)) built in shared memory from the u8
 * codes; W never exists in HBM.  k % 64 == 0; x, codes, y 16-byte aligned.  `workspace`
 * (qftc_dequant_gemm_workspace_bytes(n, k) bytes, device) receives the per-(row, 32-column)
 * index of the CSR slots that lets each producer thread load its outliers ahead. */
int64_t qftc_dequant_gemm_workspace_bytes(int n, int k);
int qftc_dequant_gemm(const void* x_bf16, int m, int k, const uint8_t* codes, int n,
                      const float* scale, const int32_t* zero_point, const int32_t* row_start,
                      const int32_t* row_count, const int32_t* col_idx, const float* values,
                      void* y_bf16, void* workspace, qftc_stream_t stream);

/* Opt-in QFTC format extensions (checkpoint.cpp:100-140 is the v1
 * layout they extend; the files carry version 0x8001, which the reference rejects):
 * b-bit codes (b in [2, 8]) bit-packed LSB-first per row, each row padded to a byte
 * (lossless), and the momentum re-quantized with one affine (scale, zero point) per
 * block of `block` elements of a row -- and back to the per-row form of quantize_state
 * (lossy).  The momentum conversions synchronise (they report min > max). */
int qftc_pack_codes(const uint8_t* codes, int rows, int cols, int bits, uint8_t* packed,
                    qftc_stream_t stream);
int qftc_unpack_codes(const uint8_t* packed, int rows, int cols, int bits, uint8_t* codes,
                      qftc_stream_t stream);
int qftc_momentum_to_blocks(const uint8_t* codes, const float* scale, const int32_t* zero_point,
                            int rows, int cols, int bit_width, int block, uint8_t* block_codes,
                            float* block_scale, int32_t* block_zero_point, qftc_stream_t stream);
int qftc_momentum_from_blocks(const uint8_t* block_codes, const float* block_scale,
                              const int32_t* block_zero_point, int rows, int cols, int bit_width,
                              int block, uint8_t* codes, float* scale, int32_t* zero_point,
                              qftc_stream_t stream);

/* An expand PLAN: the tensor table uploaded once (synchronises), then one launch per
 * run for any number of tensors -- e.g. the pieces of a ZeRO-1 all-gather (every rank's
 * rows of every tensor, read straight from the gathered shard-major buffers). */
typedef struct qftc_expand_plan qftc_expand_plan;
int qftc_expand_plan_create(qftc_expand_plan** plan, const qftc_expand_tensor* tensors,
                            int n_tensors, int bf16, qftc_stream_t stream);
int qftc_expand_plan_run(qftc_expand_plan* plan, qftc_stream_t stream);
int qftc_expand_plan_destroy(qftc_expand_plan* plan);

/* Pass-through mode (QuantMode::passthrough, quantize.hpp:17): lion_apply on raw
 * fp32 state, bitwise equal to lion_step_reference (optimizer.hpp:135-142). */
int qftc_lion_apply(float* w, float* m, const float* g, int64_t n, qftc_lion_hyper hyper,
                    qftc_stream_t stream);

/* ---------------------------------------------------------------- checkpoint CRC */

/* The QFTC v1 checkpoint checksum (checkpoint.cpp:20-33: CRC-32, reflected polynomial
 * 0xEDB88320, preset 0xFFFFFFFF, final complement) of the concatenation of n DEVICE
 * byte segments, computed on the GPU (save_checkpoint appends it, load_checkpoint
 * verifies it, checkpoint.cpp:134/:151-154).  Synchronises; *crc_out on the host. */
int qftc_crc32(const void* const* segments, const int64_t* lengths, int n, uint32_t* crc_out,
               qftc_stream_t stream);

/* ---------------------------------------------------------------- memory helpers
 * For FFI hosts (ctypes / cgo / JNI / pybind) that have no CUDA runtime of their
 * own: device allocation and stream-ordered copies. */
int qftc_device_alloc(void** ptr, size_t bytes);
int qftc_device_free(void* ptr);
int qftc_copy_to_device(void* dst, const void* src_host, size_t bytes, qftc_stream_t stream);
int qftc_copy_to_host(void* dst_host, const void* src, size_t bytes, qftc_stream_t stream);
int qftc_memset(void* dst, int value, size_t bytes, qftc_stream_t stream);
int qftc_stream_synchronize(qftc_stream_t stream);

/* ---------------------------------------------------------------- inputs */

/* Deterministic synthetic tensor, bit-identical to oracle/synth.c qo_synth. */
int qftc_synth(float* out, int64_t n, uint64_t seed, double sigma, double spike_p,
               qftc_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* QFT_B200_H_ */
