#!/bin/bash
timeout -s KILL 240 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -2
QFT_B200_LIB=$PWD/tools/_variants/tma/libqft_b200.so timeout -s KILL 240 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -1
QFT_DQ_PAIR=1 bash tools/ab_gemm.sh tma tma_np ldg_np
echo "---- single"
QFT_DQ_PAIR=0 bash tools/ab_gemm.sh tma
