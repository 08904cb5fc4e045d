#!/bin/bash
# One GPU call collecting the round's evidence into gpurun_out/$1_*: tests, smoke, bench
# lines (default + reference arm, zero1 at N=1, sweep, 13b, gemm), the bf16-gradient and
# large-lr probes, the launch list of the default bench and ncu --set full captures of the
# rows kernels, the gradient quantizer, the expansion kernel and the fused GEMM.
T=$1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${T}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python bench.py --impl reference > gpurun_out/${T}_bench_ref.json 2>&1
python bench.py --zero1 --no-e2e --no-cpu --no-side > gpurun_out/${T}_zero1.json 2>&1
python bench.py --mode sweep --steps 5 > gpurun_out/${T}_sweep.json 2>&1
python bench.py --mode 13b --steps 5 > gpurun_out/${T}_13b.json 2>&1
python bench.py --mode gemm > gpurun_out/${T}_gemm.json 2>&1
python bench.py --mode wgrad > gpurun_out/${T}_wgrad.json 2>&1
python tools/bf16_probe.py --steps 5 > gpurun_out/${T}_bf16.json 2>&1
python tools/lr_probe.py --steps 5 > gpurun_out/${T}_lr.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_step_prep|rows_kernel|step_kernel" --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-side > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"rows_kernel" -s 2 -c 2 -o gpurun_out/${T}_rows python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-side > /dev/null 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k 'regex:rows_kernel<\(int\)384.*\(bool\)0' -s 1 -c 1 -o gpurun_out/${T}_r11008 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-side > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_grad_quant" -s 2 -c 2 -o gpurun_out/${T}_gq python tools/bf16_probe.py --steps 1 --warmup 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"rows_kernel" -s 6 -c 1 -o gpurun_out/${T}_gen python tools/lr_probe.py --steps 1 --warmup 3 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_dq_gemm" -s 1 -c 1 -o gpurun_out/${T}_gemm python bench.py --mode gemm > /dev/null 2>&1
tail -2 gpurun_out/${T}_pytest.log; cat gpurun_out/${T}_smoke.log | tail -1
