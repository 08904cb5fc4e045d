#!/bin/bash
export QFT_DQ_PAIR=1
for v in tma_h4 ldg_h4; do QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so timeout -s KILL 200 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -1; done
bash tools/ab_gemm.sh tma tma_h4 ldg_h4 tma_h4_np
