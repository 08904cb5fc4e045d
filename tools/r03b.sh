#!/bin/bash
timeout 900 python -m pytest -q -x tests/test_gpu_csr_pack.py tests/test_gpu_zero1_fused.py tests/test_gpu_zero1_expand.py 2>&1 | tail -3
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py tests/test_gpu_engine_depth.py -k "zero1 or Zero1" 2>&1 | tail -2
for pk in 1 0; do echo "== packed $pk"; QFT_ZERO1_PACKED=$pk timeout 600 python bench.py --zero1 --no-e2e --no-cpu --no-side 2>&1 | python tools/zero1_show.py; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_chunk|k_pack|k_grad|rows_kernel|k_step_prep" --csv --log-file gpurun_out/r03b_zero1.csv python bench.py --zero1 --no-e2e --no-cpu --no-side --steps 2 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"rows_kernel" -s 6 -c 1 -o gpurun_out/r03b_gen python tools/lr_probe.py --steps 1 --warmup 3 > gpurun_out/r03b_gen.log 2>&1
tail -3 gpurun_out/r03b_gen.log
