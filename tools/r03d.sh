#!/bin/bash
timeout 1500 python -m pytest -q -x tests/test_gpu_engine_depth.py tests/test_gpu_gen_tier.py tests/test_gpu_rawgrad.py tests/test_gpu_zero1_fused.py 2>&1 | tail -3
echo "== drift"; timeout 600 python tools/drift_probe.py 2 2>&1 | tail -12
for v in default gqclamp default; do echo "== bf16 $v"; if [ $v = default ]; then L=""; else L="QFT_B200_LIB=$PWD/tools/_variants/$v/libqft_b200.so"; fi; env $L timeout 600 python tools/bf16_probe.py --steps 5 2>&1 | tail -1 | cut -c1-400; done
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:rows_kernel<\(int\)384.*\(bool\)0' -s 1 -c 1 -o gpurun_out/r03d_r11008 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-side > gpurun_out/r03d_ncu.log 2>&1
tail -2 gpurun_out/r03d_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_grad_quant' -s 2 -c 1 -o gpurun_out/r03d_gq python tools/bf16_probe.py --steps 1 --warmup 2 > gpurun_out/r03d_gq.log 2>&1
tail -2 gpurun_out/r03d_gq.log
