#!/bin/bash
# A/B of fused-GEMM variants (tools/_variants/*) on bench --mode gemm.
run() { echo "== $1"; shift; env "$@" timeout 600 python bench.py --mode gemm 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(r['proj'], round(r['fused_ms'],3), round(r['fused_tflops'])) for r in d['rows']]"; }
run default
for v in "$@"; do run $v QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so; done
