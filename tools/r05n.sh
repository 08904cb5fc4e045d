#!/bin/bash
QFT_DQ_PAIR=1 ncu --set full --import-source on --clock-control none -k regex:"k_dq_gemm_pair|k_csr_tile" -c 2 -o gpurun_out/r05n_pair python tools/gemm_probe.py > /dev/null 2>&1
ls gpurun_out | grep r05n
