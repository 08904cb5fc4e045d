"""Probe: the 7B state stepped at a large lr (bench.side_lr) alone, for ncu."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=3)
args = ap.parse_args()
import paper_2310_07147_b200 as q  # noqa: E402
from paper_2310_07147_b200.shapes import llama2_7b  # noqa: E402
hbm, _ = bench.peaks()
st = bench.build_state(llama2_7b(), q, 1234)
print(json.dumps(bench.side_lr(st, args, torch.cuda.current_stream(), 34.86e9, hbm)))
