#!/bin/bash
# CTA-pair (cta_group::2) dequant GEMM: first contact (parity) + same-box A/B vs single CTA
timeout -s KILL 240 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -15
for p in 0 1; do QFT_DQ_PAIR=$p timeout -s KILL 240 python bench.py --mode gemm 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for r in d['rows']: print('pair=$p', r['proj'], round(r['fused_ms'],4), round(r['fused_tflops'],1), 'exp+cublas', round(r['expand_plus_cublas_ms'],4), 'cublas', round(r['cublas_tflops'],1))"; done
