#!/bin/bash
# parity of the fused GEMM for the default build and tools/_variants/*
for v in default "$@"; do
  if [ "$v" = default ]; then unset QFT_B200_LIB; else export QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so; fi
  echo "== $v"; timeout 300 python -m pytest tests/test_gpu_dqgemm.py -m gpu -q 2>&1 | tail -1
done
