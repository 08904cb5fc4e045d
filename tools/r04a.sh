#!/bin/bash
# wgrad first contact: the fused-sink GEMM tests (default descriptor strides, then swapped)
timeout 300 python -m pytest -x -q tests/test_gpu_wgrad.py 2>&1 | tail -25
echo "== swapped LBO/SBO"
QFT_WG_LBO=1024 QFT_WG_SBO=8192 timeout 120 python -m pytest -x -q tests/test_gpu_wgrad.py -k "push and 128-256-64" 2>&1 | tail -5
echo "== dqgemm (refactor)"
timeout 300 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -2
echo "== bench wgrad"
timeout 300 python bench.py --mode wgrad 2>&1 | tail -2
