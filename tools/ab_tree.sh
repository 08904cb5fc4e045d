#!/bin/bash
# A/B the working tree against full source trees under tools/_variants/src_* (their own
# python + library), on the 7B bench (no e2e/cpu legs).
ROOT=$(pwd)
for v in default "$@"; do
  if [ "$v" = default ]; then d=$ROOT; else d=$ROOT/tools/_variants/$v; fi
  echo "== $v"; (cd $d && timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['per_launch_ms'], d['roofline']['frac'])")
done
