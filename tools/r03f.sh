#!/bin/bash
timeout 2400 python -m pytest -q -x tests -m gpu 2>&1 | tail -2
run() { echo "== $1"; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-side 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d['clocks']['reasons'])"; }
run default; run fp64exact QFT_B200_LIB=$PWD/tools/_variants/fp64exact/libqft_b200.so; run default
for v in default fp64exact; do L=""; [ $v != default ] && L="QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so"
  echo "== bf16 $v"; env $L timeout 600 python tools/bf16_probe.py --steps 5 2>&1 | tail -1 | cut -c1-120
  echo "== lr $v"; env $L timeout 600 python tools/lr_probe.py --steps 5 2>&1 | tail -1 | cut -c1-250; done
./tools/gemm_check.sh bn128h2 bn128h4
./tools/ab_gemm.sh bn128h2 bn128h4
