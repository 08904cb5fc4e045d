#!/bin/bash
# dgrad (transposed dequant operand) first contact + wgrad/dqgemm regression + gemm bench
timeout 300 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -15
timeout 300 python -m pytest -x -q tests/test_gpu_wgrad.py 2>&1 | tail -2
timeout 300 python bench.py --mode gemm 2>&1 | tail -1
