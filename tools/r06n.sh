#!/bin/bash
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_dq_gemm_pair" python tools/gemm_k_probe.py 2>&1 | grep -E "gpu__time" | awk 'NR%23==1'
