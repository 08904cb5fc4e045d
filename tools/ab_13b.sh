#!/bin/bash
# A/B of library variants on bench --mode 13b (step + gathered expansion).
run() { echo "== $1"; shift; env "$@" timeout 900 python bench.py --mode 13b --steps 5 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['step_ms'],3), round(d['dequant_ms'],3), round(d['dequant_frac_of_hbm'],4))"; }
run default
for v in "$@"; do run $v QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so; done
