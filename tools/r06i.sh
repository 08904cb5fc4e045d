#!/bin/bash
QFT_DQ_PAIR=1 bash tools/ab_gemm.sh pw1
QFT_DQ_PAIR=1 bash tools/ab_gemm.sh pw1
