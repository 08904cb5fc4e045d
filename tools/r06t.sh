#!/bin/bash
QFT_B200_LIB=$PWD/tools/_variants/onef/libqft_b200.so timeout -s KILL 300 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -1
bash tools/ab_gemm.sh onef
bash tools/ab_gemm.sh onef
