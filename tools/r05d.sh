#!/bin/bash
# CTA-pair GEMM: locate the limit (no producers / no X loads / no MMAs), arrive semantics
timeout -s KILL 240 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -2
export QFT_DQ_PAIR=1
bash tools/ab_gemm.sh clrel noprod noprod_nox noprod_nomma nox
echo "---- single CTA"
QFT_DQ_PAIR=0 bash tools/ab_gemm.sh noprod noprod_nox noprod_nomma nox
