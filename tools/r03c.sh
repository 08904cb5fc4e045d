#!/bin/bash
timeout 1200 python -m pytest -q -x tests/test_gpu_engine_depth.py tests/test_gpu_parity.py tests/test_gpu_gen_tier.py 2>&1 | tail -3
echo "== lr"; timeout 600 python tools/lr_probe.py --steps 5 2>&1 | tail -1
echo "== lr again"; timeout 600 python tools/lr_probe.py --steps 5 --warmup 6 2>&1 | tail -1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"rows_kernel<384" -s 1 -c 1 -o gpurun_out/r03c_r11008 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-side > gpurun_out/r03c_ncu.log 2>&1
tail -2 gpurun_out/r03c_ncu.log
