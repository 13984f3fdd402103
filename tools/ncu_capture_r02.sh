#!/bin/bash
# Round-2 ncu captures (one GPU; outputs under gpurun_out/): the kernels that
# changed or were unprofiled -- the TMA-staged 128x64 DMMA GEMM with split-K
# TN at c4, the tcgen05 kind::i8 emulated-FP64 GEMM at c4 (BNBG_OZAKI=1), the
# shared-memory-slice re-opt at c4 -- and the c2 bench launch list.
set -x
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_gemm_big -s 6 -c 2 \
    -o $O/ncu_gemm_big_c4 python tools/certify_long.py c4 --limit 4 > $O/ncu_gemm_big_c4.log 2>&1
BNBG_OZAKI=1 ncu --set full --clock-control none --import-source on -k regex:k_ozaki_gemm -s 6 -c 2 \
    -o $O/ncu_ozaki_c4 python tools/certify_long.py c4 --limit 4 > $O/ncu_ozaki_c4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_reopt_cluster_smem -s 1 -c 1 \
    -o $O/ncu_reopt_smem_c4 python tools/certify_long.py c4 --limit 4 > $O/ncu_reopt_smem_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $O/launches_c2_r02.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-secondary > $O/launches_c2_r02.log 2>&1
