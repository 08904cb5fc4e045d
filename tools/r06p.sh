#!/bin/bash
timeout -s KILL 300 python -m pytest -x -q tests/test_gpu_dqgemm.py tests/test_gpu_wgrad.py 2>&1 | tail -1
for v in "" v4; do
  if [ -n "$v" ]; then export QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so; fi
  echo "== ${v:-v8}"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dq_gemm_pair" python tools/gemm_k_probe.py 2>&1 | grep -E "gpu__time" | awk 'NR%23==1'
done
unset QFT_B200_LIB
bash tools/ab_gemm.sh v4
