#!/bin/bash
# ncu --set full captures of the dominant kernels (one launch each) + launch lists.
# Run on the GPU box from the repo root; outputs under gpurun_out/.
set -x
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_pass -s 5 -c 1 \
    -o $O/ncu_pass_c2 python tools/profile_solve.py c2 > $O/ncu_pass_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_reopt_cluster -s 5 -c 1 \
    -o $O/ncu_reopt_c2 python tools/profile_solve.py c2 > $O/ncu_reopt_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_big -s 20 -c 2 \
    -o $O/ncu_gemm_big_c3 python tools/profile_solve.py c3 --limit 8 > $O/ncu_gemm_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_branch_write -s 3 -c 1 \
    -o $O/ncu_branch_c5 python tools/profile_solve.py c5 > $O/ncu_branch_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $O/launches_c2.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/launches_c2.log 2>&1
