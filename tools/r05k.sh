#!/bin/bash
timeout -s KILL 240 python -m pytest -x -q tests/test_gpu_dqgemm.py tests/test_gpu_wgrad.py 2>&1 | tail -2
for p in 1 0; do echo "pair=$p"; QFT_DQ_PAIR=$p bash tools/ab_gemm.sh; done
