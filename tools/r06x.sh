#!/bin/bash
QFT_B200_LIB=$PWD/tools/_variants/w4096/libqft_b200.so timeout -s KILL 600 python -m pytest -x -q tests/test_gpu_rawgrad.py 2>&1 | tail -1
for v in "" w4096 "" w4096; do
  if [ -n "$v" ]; then export QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so; else unset QFT_B200_LIB; fi
  echo "== ${v:-default}"; timeout 300 python tools/bf16_probe.py --steps 5 2>&1 | tail -1 | cut -c1-60
done
