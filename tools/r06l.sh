#!/bin/bash
QFT_DQ_PAIR=1 bash tools/ab_gemm.sh pu2 pu4
