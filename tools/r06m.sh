#!/bin/bash
timeout -s KILL 300 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -1
for v in new pu1; do
  if [ $v = pu1 ]; then L=$PWD/tools/_variants/pu1/libqft_b200.so; else L=; fi
  QFT_B200_LIB=$L timeout 300 python bench.py --mode gemm 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for r in d['rows']: print('$v', r['proj'], 'fwd', round(r['fused_tflops']), 'dx', round(r['backward_dx_fused_tflops']))"
done
