#!/bin/bash
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"rows_kernel|k_step_prep|step_kernel|k_replan|k_csr" --csv --log-file gpurun_out/r06d_lr_launches.csv python tools/lr_probe.py --steps 2 --warmup 3 > /dev/null 2>&1
tail -30 gpurun_out/r06d_lr_launches.csv | cut -c1-220
