#!/bin/bash
# ncu --set full of the CTA-pair GEMM (default + no-producer) and the single-CTA one
export QFT_DQ_PAIR=1
ncu --set full --import-source on --clock-control none -k regex:"k_dq_gemm" -s 1 -c 1 -o gpurun_out/r05c_pair python bench.py --mode gemm > /dev/null 2>&1
QFT_B200_LIB=$PWD/tools/_variants/noprod/libqft_b200.so ncu --set full --clock-control none -k regex:"k_dq_gemm" -s 1 -c 1 -o gpurun_out/r05c_pair_noprod python bench.py --mode gemm > /dev/null 2>&1
QFT_DQ_PAIR=0 QFT_B200_LIB=$PWD/tools/_variants/noprod/libqft_b200.so ncu --set full --clock-control none -k regex:"k_dq_gemm" -s 1 -c 1 -o gpurun_out/r05c_single_noprod python bench.py --mode gemm > /dev/null 2>&1
ls gpurun_out
