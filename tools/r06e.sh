#!/bin/bash
timeout -s KILL 600 python -m pytest -x -q tests/test_gpu_rawgrad.py tests/test_gpu_zero1_fused.py 2>&1 | tail -1
timeout 300 python tools/bf16_probe.py --steps 5 2>&1 | tail -1
timeout 300 python bench.py --mode 13b --steps 5 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('13b step', d['step_ms'], d['step_frac_of_hbm'])"
