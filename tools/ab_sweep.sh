#!/bin/bash
# A/B the default library against variants on the configs[4] sweep (min/max Gparams/s).
for v in default "$@"; do
  if [ "$v" = default ]; then unset QFT_B200_LIB; else export QFT_B200_LIB=tools/_variants/$v/libqft_b200.so; fi
  echo "== $v"; timeout 600 python bench.py --mode sweep --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print([(r['bit_width'], r['outlier_fraction'], round(r['gparams_s'],1)) for r in d['rows']])"
done
