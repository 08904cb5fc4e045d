#!/bin/bash
timeout -s KILL 300 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -4
for p in 1 0; do QFT_DQ_PAIR=$p timeout 300 python bench.py --mode gemm 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for r in d['rows']: print('pair=$p', r['proj'], 'fwd', round(r['fused_tflops']), 'dx', round(r['backward_dx_fused_tflops']), round(r['backward_dx_fused_ms'],4), 'exp+cublas dx', round(r['backward_dx_expand_plus_cublas_ms'],4))"; done
