#!/bin/bash
# weight-gradient GEMM: a grid of whole row blocks (QFT_WG_ALIGN=1) vs all SMs
QFT_WG_ALIGN=1 timeout -s KILL 300 python -m pytest -x -q tests/test_gpu_wgrad.py 2>&1 | tail -1
for a in 0 1 0 1; do QFT_WG_ALIGN=$a timeout 300 python bench.py --mode wgrad 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('align=$a', [(r['proj'], round(r['fused_ms'],4), round(r['fused_accumulate_ms'],4), round(r['cublas_f32_plus_quantize_state_ms'],4)) for r in d['rows']])"; done
