#!/bin/bash
export QFT_DQ_PAIR=1
bash tools/ab_gemm.sh tma_np tma_np_nof ldg_np ldg_np_nof
