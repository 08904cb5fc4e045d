#!/bin/bash
ncu --set full --import-source on --clock-control none -k regex:"k_grad_quant" -s 2 -c 2 -o gpurun_out/r06b_gq python tools/bf16_probe.py --steps 1 --warmup 2 > /dev/null 2>&1
ls gpurun_out | grep r06b
