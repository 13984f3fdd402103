#!/bin/bash
# Round-2 (second part) ncu captures after the Gram-form gradient: the c1
# pass kernel (local Gram iterations), the c3 Gram product (128 x 64 DMMA
# tiles of Q, EPI_DERIV: k_gemm_big<0, 1>) and the c5 pass kernel (streaming
# Gram tiles).  One GPU; outputs under gpurun_out/.
set -x
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_pass -s 4 -c 1 \
    -o $O/ncu_pass_c1_r02 python tools/certify_long.py c1 > $O/ncu_pass_c1_r02.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_big -s 40 -c 6 \
    -o $O/ncu_gram_c3 python tools/certify_long.py c3 --limit 3 > $O/ncu_gram_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pass -s 20 -c 1 \
    -o $O/ncu_pass_c5_r02 python tools/certify_long.py c5 > $O/ncu_pass_c5_r02.log 2>&1
