#!/bin/bash
# forward GEMM ring depths (X / W operand / codes) A/B
bash tools/ab_gemm.sh p3w6 p3w5c6 p4w3c6
