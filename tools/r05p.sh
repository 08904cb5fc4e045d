#!/bin/bash
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r05p_bf16_launches.csv python tools/bf16_probe.py --steps 1 --warmup 1 > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/r05p_bf16_launches.csv 2>&1 | tail -20
