#!/bin/bash
# One GPU round trip: parity tests, bench (all legs), sweep and 13B modes, ncu launch list
# of a step + full captures of the rows kernel (both width classes).
# usage (under gpurun): bash tools/gpu_round.sh TAG [tests|notests]
TAG=${1:-r01}
mkdir -p gpurun_out
if [ "${2:-tests}" = "tests" ]; then
  timeout 1200 python -m pytest tests/ -q -m gpu -x > gpurun_out/pytest_$TAG.log 2>&1; tail -1 gpurun_out/pytest_$TAG.log
fi
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -2 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 900 python bench.py --mode sweep --steps 5 --warmup 3 --no-cpu > gpurun_out/sweep_$TAG.json 2> gpurun_out/sweep_$TAG.err
timeout 900 python bench.py --mode 13b --steps 5 --warmup 3 --no-cpu > gpurun_out/b13_$TAG.json 2> gpurun_out/b13_$TAG.err
# every kernel of one bench command (setup + warmup + 2 timed steps), duration + DRAM bytes
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_all_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_all_$TAG.out 2>&1
tail -1 gpurun_out/ncu_all_$TAG.out
# full capture: one rows_kernel launch of each width class (4096, 11008)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:rows_kernel -s 4 -c 2 -o gpurun_out/prof_$TAG \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full_$TAG.out 2>&1
tail -1 gpurun_out/ncu_full_$TAG.out
