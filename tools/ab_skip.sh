#!/bin/bash
# A/B of library variants on the 7B bench including the lr=2.2e-4 side run.
run() { echo "== $1"; shift; env "$@" timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d.get('side_lr_2.2e-4',{}); print(round(d['value'],1), round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d['clocks']['reasons'], 'lr2.2e-4:', round(s.get('ms_per_step',0),3), s.get('tier_rows'), s.get('replans_in_timed_steps'))"; }
run default
for v in "$@"; do run $v QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so; done
run default_again
