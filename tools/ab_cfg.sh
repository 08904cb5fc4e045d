#!/bin/bash
# A/B step-kernel shapes via QFT_STEP_CFG="oldcap" (old-outlier table per warp) on the 7B bench.
for c in default "$@"; do
  if [ "$c" = default ]; then unset QFT_STEP_CFG; else export QFT_STEP_CFG=$c; fi
  echo "== cfg $c"; timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['per_launch_ms'].items()}, round(d['roofline']['frac'],3))"
done
