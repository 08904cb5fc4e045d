#!/bin/bash
timeout -s KILL 300 python -m pytest -x -q tests/test_gpu_dqgemm.py 2>&1 | tail -15
