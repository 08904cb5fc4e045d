#!/bin/bash
for v in "" noepi; do
  if [ -n "$v" ]; then export QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so; fi
  echo "== ${v:-default}"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dq_gemm_pair" python tools/gemm_k_probe.py 2>&1 | grep -E "gpu__time" | awk 'NR%23==1'
done
