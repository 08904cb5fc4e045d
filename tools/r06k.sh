#!/bin/bash
# warp-per-row bf16 gradient quantizer: parity + A/B against the CTA ring kernel
timeout -s KILL 900 python -m pytest -x -q tests/test_gpu_rawgrad.py tests/test_gpu_zero1_fused.py tests/test_gpu_engine_depth.py 2>&1 | tail -2
for v in warp cta warp cta; do
  if [ $v = cta ]; then L=$PWD/tools/_variants/gqcta/libqft_b200.so; else L=; fi
  echo "== $v"; QFT_B200_LIB=$L timeout 300 python tools/bf16_probe.py --steps 5 2>&1 | tail -1 | cut -c1-100
done
timeout 300 python bench.py --mode 13b --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('13b step', d['step_ms'], d['step_frac_of_hbm'])"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_grad_quant" -s 2 -c 2 python tools/bf16_probe.py --steps 1 --warmup 2 2>&1 | grep -E "k_grad|duration|bytes_" | head -8
