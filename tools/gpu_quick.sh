#!/bin/bash
# quick GPU check: rows-kernel parity, full GPU suite, one bench line
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "stable_tier" 2>&1 | tail -15
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -15
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
tail -3 gpurun_out/bench_q.err; cat gpurun_out/bench_q.json
