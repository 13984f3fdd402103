#!/bin/bash
# Round-2 ncu captures (one GPU; outputs under gpurun_out/): the kernels that
# changed or were unprofiled -- the TMA-staged 128x64 DMMA GEMM with split-K
# TN, the tcgen05 kind::i8 emulated-FP64 GEMM (BNBG_OZAKI=1), the
# shared-memory-slice re-opt at c4 -- and the c2 bench launch list.
# c3 reaches m_a >= 100 (standalone 128x64 kernels) within its first second;
# c4 needs ~10 s to reach 64-node passes.
set -x
O=gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_gemm_big -s 20 -c 2 \
    -o $O/ncu_gemm_big_c3 python tools/certify_long.py c3 --limit 3 > $O/ncu_gemm_big_c3.log 2>&1
BNBG_OZAKI=1 ncu --set full --clock-control none --import-source on -k regex:k_ozaki_gemm -s 20 -c 2 \
    -o $O/ncu_ozaki_c3 python tools/certify_long.py c3 --limit 3 > $O/ncu_ozaki_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_big -s 4 -c 2 \
    -o $O/ncu_gemm_big_c4 python tools/certify_long.py c4 --limit 14 > $O/ncu_gemm_big_c4.log 2>&1
BNBG_OZAKI=1 ncu --set full --clock-control none --import-source on -k regex:k_ozaki_gemm -s 4 -c 2 \
    -o $O/ncu_ozaki_c4 python tools/certify_long.py c4 --limit 14 > $O/ncu_ozaki_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $O/launches_c2_r02.csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-secondary > $O/launches_c2_r02.log 2>&1
