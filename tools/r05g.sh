#!/bin/bash
# CTA-pair GEMM, producers loading codes from global (LDG): parity, then locate the limit
timeout -s KILL 240 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -2
export QFT_DQ_PAIR=1
bash tools/ab_gemm.sh tma clrel noprod noprod_nox noprod_nomma nomma
echo "---- single CTA"
QFT_DQ_PAIR=0 bash tools/ab_gemm.sh tma noprod noprod_nox noprod_nomma nomma
