#!/bin/bash
for p in 0 1; do
  for v in skel skel_c8 c8 c8w4; do
  QFT_DQ_PAIR=$p TAG="pair=$p $v" QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so timeout -s KILL 120 python tools/gemm_k_probe.py
  done
done
