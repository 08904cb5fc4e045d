#!/bin/bash
# GEN-tier occupancy A/B at lr 2.2e-4 (steady steps; launch list of one step)
for v in "" gm1 "" gm1; do
  if [ -n "$v" ]; then export QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so; else unset QFT_B200_LIB; fi
  echo "== ${v:-default}"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"rows_kernel" -s 8 -c 4 python tools/lr_probe.py --steps 1 --warmup 3 2>&1 | grep -E "gpu__time" | sed 's/  */ /g'
done
