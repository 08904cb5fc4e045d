#!/bin/bash
# parity of the rows kernel + A/B bench of env variants: bash tools/gpu_ab.sh "ENV1" "ENV2" ...
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stable_tier or trajectory or engine or edge" 2>&1 | tail -3
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'Gp/s', d['per_launch_ms'], 'frac', round(d['roofline']['frac'],3))"
done
