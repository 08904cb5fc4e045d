#!/bin/bash
# A/B of environment switches on the 7B bench: ./tools/ab_env2.sh "NAME VAR=V ..." ...
run() { echo "== $1"; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-side 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['per_class_serial_ms'].items()}, round(d['roofline']['frac'],4), d['clocks']['reasons'])"; }
for spec in "$@"; do run $spec; done
