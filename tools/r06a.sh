#!/bin/bash
# branch-free exact gradient quantizer: parity (raw gradients, ZeRO-1 fused, GEN, engine) + A/B
timeout -s KILL 600 python -m pytest -x -q tests/test_gpu_rawgrad.py tests/test_gpu_zero1_fused.py tests/test_gpu_engine_depth.py 2>&1 | tail -2
QFT_B200_LIB=$PWD/tools/_variants/gqold/libqft_b200.so timeout -s KILL 300 python -m pytest -x -q tests/test_gpu_rawgrad.py 2>&1 | tail -1
for v in new old; do
  if [ $v = old ]; then export QFT_B200_LIB=$PWD/tools/_variants/gqold/libqft_b200.so; fi
  echo "== $v"; timeout 300 python tools/bf16_probe.py --steps 5 2>&1 | tail -1
  timeout 300 python bench.py --mode 13b --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('13b step', d['step_ms'], d['step_frac_of_hbm'])"
done
