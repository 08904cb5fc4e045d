// qft_internal.h -- host/device structures shared by the kernels and the C-ABI layer.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "qft_b200.h"

namespace qftk {

// One tensor of a grouped launch, device copy of qftc_lion_tensor plus the row
// base of the tensor inside the launch's global row numbering.
struct DevTensor {
  int32_t rows, cols;
  int32_t row_base, _pad;
  uint8_t* w_codes[2];
  int32_t* row_ptr[2];
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

// Device header of a plan / scan workspace.  `epoch` tags look-back status
// words so the status array never needs clearing between launches; the last
// CTA of every launch bumps it and resets the ticket counter.
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

enum Mode : int { MODE_STEP = 0, MODE_DECOMPOSE = 1, MODE_RECON_F32 = 2, MODE_RECON_BF16 = 3 };
enum GradKind : int { G_U8 = 0, G_F32 = 1, G_BF16 = 2 };

// error bits in Header::err
constexpr uint32_t ERR_MPARAMS = 1u;   // momentum min > max (NaN in column 0)
constexpr uint32_t ERR_GPARAMS = 2u;   // gradient min > max
constexpr uint32_t ERR_PREFIX = 4u;    // nnz prefix exceeded 2^30

struct LaunchArgs {
  DevTensor* tensors;
  int32_t n_tensors;
  int32_t total_rows;
  int32_t flip;
  int32_t bit_width;
  float lr, b1, b2, wd;
  const int32_t* col_in;
  const float* val_in;
  int32_t* col_out;
  float* val_out;
  int64_t cap_out;
  Header* hdr;
  unsigned long long* status;
  int32_t cols_p;     // max padded (x16) row length of the launch
  int32_t stages;
  int32_t use_bulk;   // TMA bulk copies (all rows 16-byte aligned)
  int32_t _pad;
};

// launch helpers (rowengine.cu)
size_t row_engine_smem(int mode, int gkind, int cols_p, int stages);
cudaError_t launch_row_engine(int mode, int gkind, const LaunchArgs& a, cudaStream_t s,
                              int* grid_out);
int row_engine_max_cols();

}  // namespace qftk
