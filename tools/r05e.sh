#!/bin/bash
for p in 0 1; do
  QFT_DQ_PAIR=$p TAG="pair=$p default" python tools/gemm_k_probe.py
  QFT_DQ_PAIR=$p TAG="pair=$p noprod_nomma" QFT_B200_LIB=$PWD/tools/_variants/noprod_nomma/libqft_b200.so python tools/gemm_k_probe.py
done
