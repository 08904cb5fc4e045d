#!/bin/bash
# A/B the default library against tuning variants on the 7B bench (no e2e/cpu legs).
for v in default "$@"; do
  if [ "$v" = default ]; then unset QFT_B200_LIB; else export QFT_B200_LIB=tools/_variants/$v/libqft_b200.so; fi
  echo "== $v"; timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['per_launch_ms'], d['roofline']['frac'])"
done
