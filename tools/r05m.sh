#!/bin/bash
timeout -s KILL 240 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -3
for p in 1 0; do echo "pair=$p"; QFT_DQ_PAIR=$p bash tools/ab_gemm.sh np; done
QFT_DQ_PAIR=1 timeout 300 python bench.py --mode gemm 2>&1 | tail -1 > gpurun_out/r05m_gemm.json
