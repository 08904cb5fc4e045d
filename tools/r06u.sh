#!/bin/bash
timeout -s KILL 300 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -1
timeout 300 python bench.py --mode gemm 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for r in d['rows']: print(r['proj'], 'fwd', round(r['fused_tflops']), round(r['fused_ms'],4), 'rebuild', round(r['fused_with_index_rebuild_ms'],4), 'idx', round(r['csr_index_ms'],4), 'exp+cub', round(r['expand_plus_cublas_ms'],4), 'dx', round(r['backward_dx_fused_tflops']), round(r['backward_dx_fused_ms'],4), 'rebuild', round(r['backward_dx_fused_with_index_rebuild_ms'],4), round(r['backward_dx_expand_plus_cublas_ms'],4))"
