#!/bin/bash
timeout 1200 python -m pytest -q -x tests/test_gpu_engine_depth.py tests/test_gpu_parity.py tests/test_gpu_gen_tier.py 2>&1 | tail -2
echo "== drift"; timeout 600 python tools/drift_probe.py 2 2>&1 | tail -12
echo "== lr"; timeout 600 python tools/lr_probe.py --steps 5 2>&1 | tail -1 | cut -c1-300
echo "== lr"; timeout 600 python tools/lr_probe.py --steps 5 --warmup 8 2>&1 | tail -1 | cut -c1-300
