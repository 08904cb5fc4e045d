#!/bin/bash
timeout 600 python tools/replan_time.py 2>&1 | tail -12
timeout -s KILL 900 python -m pytest -x -q tests/test_gpu_engine_depth.py tests/test_gpu_parity.py tests/test_zero1_gloo.py tests/test_gpu_zero1_expand.py 2>&1 | tail -2
timeout 300 python tools/lr_probe.py --steps 5 2>&1 | tail -1
