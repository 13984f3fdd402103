#!/bin/bash
# ncu --set full of the dominant kernel at the other bench configs (c1, c5:
# k_pass; c4: k_gemm_big NN + TN); summarised as CLASS@CONFIG entries.
O=gpurun_out
ncu --set full --clock-control none -k regex:k_pass -s 3 -c 1 \
    -o $O/ncu_pass_c1 python tools/profile_solve.py c1 > $O/ncu_pass_c1.log 2>&1
ncu --set full --clock-control none -k regex:k_pass -s 3 -c 1 \
    -o $O/ncu_pass_c5 python tools/profile_solve.py c5 > $O/ncu_pass_c5.log 2>&1
ncu --set full --clock-control none -k regex:k_gemm_big -s 40 -c 2 \
    -o $O/ncu_gemm_big_c4 python tools/profile_solve.py c4 --limit 20 > $O/ncu_gemm_c4.log 2>&1
