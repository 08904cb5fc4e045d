#!/bin/bash
timeout -s KILL 300 python -m pytest -x -q tests/test_gpu_dqgemm.py tests/test_gpu_wgrad.py 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dq_gemm_pair" python tools/gemm_k_probe.py 2>&1 | grep -E "gpu__time" | awk 'NR%23==1'
timeout 300 python bench.py --mode gemm 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for r in d['rows']: print(r['proj'], 'fwd', round(r['fused_tflops']), round(r['fused_ms'],4), 'exp+cublas', round(r['expand_plus_cublas_ms'],4), 'dx', round(r['backward_dx_fused_tflops']), round(r['backward_dx_fused_ms'],4), round(r['backward_dx_expand_plus_cublas_ms'],4))"
