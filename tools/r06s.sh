#!/bin/bash
# branch-free exact quantizer in the GEN tier: parity (GEN tests, raw gradients, engine depth) + A/B
timeout -s KILL 900 python -m pytest -x -q tests/test_gpu_parity.py tests/test_gpu_engine_depth.py tests/test_gpu_rawgrad.py tests/test_stable_tier.py 2>&1 | tail -2
for v in "" genold; do
  if [ -n "$v" ]; then export QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so; else unset QFT_B200_LIB; fi
  echo "== ${v:-genbf}"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rows_kernel" -s 8 -c 4 python tools/lr_probe.py --steps 1 --warmup 3 2>&1 | grep -E "gpu__time" | sed 's/  */ /g'
done
unset QFT_B200_LIB
timeout 300 python tools/lr_probe.py --steps 5 2>&1 | tail -1 | cut -c1-120
