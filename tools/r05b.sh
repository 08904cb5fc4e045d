#!/bin/bash
# CTA-pair dequant GEMM A/B: wait modes and the no-producer pipeline bound
export QFT_DQ_PAIR=1
bash tools/ab_gemm.sh pw1 noprod noprod_pw1
QFT_DQ_PAIR=0 bash tools/ab_gemm.sh noprod
