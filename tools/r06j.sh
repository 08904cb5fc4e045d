#!/bin/bash
timeout -s KILL 600 python -m pytest -x -q tests/test_gpu_rawgrad.py tests/test_gpu_zero1_fused.py 2>&1 | tail -1
QFT_B200_LIB=$PWD/tools/_variants/mag/libqft_b200.so timeout -s KILL 600 python -m pytest -x -q tests/test_gpu_rawgrad.py tests/test_gpu_zero1_fused.py 2>&1 | tail -1
for v in new mag new mag; do
  if [ $v = mag ]; then L=$PWD/tools/_variants/mag/libqft_b200.so; else L=; fi
  echo "== $v"; QFT_B200_LIB=$L timeout 300 python tools/bf16_probe.py --steps 5 2>&1 | tail -1 | cut -c1-80
done
