#!/bin/bash
# ncu capture of the rows kernel (full set, one launch) + launch list of one bench step
TAG=${1:-r01q}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:rows_kernel -s 4 -c 1 -o gpurun_out/prof_$TAG \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_full_$TAG.out 2>&1
tail -2 gpurun_out/ncu_full_$TAG.out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch_$TAG.out 2>&1
tail -1 gpurun_out/ncu_launch_$TAG.out
