#!/bin/bash
# A/B of the width-class concurrency and the dynamic row claims on the 7B bench.
run() { echo "== $1"; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-side 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['per_class_serial_ms'].items()}, round(d['roofline']['frac'],4), d['clocks']['reasons'])"; }
run concurrent_cap1 QFT_WIDE_CTAS=1
run concurrent_cap2 QFT_WIDE_CTAS=2
run concurrent_nocap QFT_WIDE_CTAS=0
run serial_dynamic QFT_SERIAL_GROUPS=1
run serial_static QFT_SERIAL_GROUPS=1 QFT_B200_LIB=tools/_variants/static/libqft_b200.so
run concurrent_static_cap1 QFT_B200_LIB=tools/_variants/static/libqft_b200.so
run concurrent_cap1_again QFT_WIDE_CTAS=1
run serial_static_again QFT_SERIAL_GROUPS=1 QFT_B200_LIB=tools/_variants/static/libqft_b200.so
