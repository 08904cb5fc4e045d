#!/bin/bash
# Golden QFTC v1 checkpoints from the REAL reference (oracle/ckpt_golden.cpp compiled with
# the reference's checkpoint.cpp by `make -C oracle ckpt`); needs /root/reference, so run
# it here, not on the GPU box.  Writes tests/golden/ckpt_*_{a,b}.qftc and ckpt_*_g.bin.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
make -C "$HERE/../../oracle" ckpt
"$HERE/../../oracle/_ref/ckpt_golden" "$HERE"
