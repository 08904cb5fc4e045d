#!/bin/bash
# One GPU round trip: parity tests, bench, ncu launch list + full capture of the step kernel.
# usage (under gpurun): bash tools/gpu_round.sh TAG [tests|notests]
TAG=${1:-r01}
mkdir -p gpurun_out
if [ "${2:-tests}" = "tests" ]; then
  timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -4
fi
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --kernel-name-base mangled -k regex:step_kernel --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch_$TAG.out 2>&1
tail -1 gpurun_out/ncu_launch_$TAG.out
# every kernel of the same command (setup + warmup + timed), duration only: the step's share
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_all_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_all_$TAG.out 2>&1
tail -1 gpurun_out/ncu_all_$TAG.out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:step_kernel -s 6 -c 2 -o gpurun_out/prof_$TAG \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full_$TAG.out 2>&1
tail -1 gpurun_out/ncu_full_$TAG.out
