#!/bin/bash
timeout -s KILL 240 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -1
QFT_B200_LIB=$PWD/tools/_variants/h4/libqft_b200.so timeout -s KILL 240 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -1
QFT_DQ_PAIR=1 bash tools/ab_gemm.sh h4 np h4np
QFT_DQ_PAIR=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dq_gemm_pair|k_csr_tile" -c 4 python tools/gemm_probe.py 2>&1 | grep -E "k_|gpu__time" | head -8
