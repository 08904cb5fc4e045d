#!/bin/bash
# A/B env-var configurations on the 7B bench: bash tools/ab_env.sh "A=1" "B=2 C=3" ...
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'Gp/s', d['per_launch_ms'], 'frac', round(d['roofline']['frac'],3))"
done
