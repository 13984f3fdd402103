#!/bin/bash
# ncu --set full of the HBM-side kernels (packer, prox, compaction, branch) -- one launch each.
O=gpurun_out
for spec in "k_pack_pool:c3:5" "k_prox_fista:c3:50" "k_compact:c3:20" "k_branch_scan:c3:5" "k_branch_write:c3:5" "k_eval:c3:10"; do
  IFS=: read kern cfg skip <<< "$spec"
  ncu --set full --clock-control none -k regex:$kern -s $skip -c 1 -o $O/ncu_${kern}_${cfg} \
      python tools/profile_solve.py $cfg --limit 6 > $O/ncu_${kern}.log 2>&1
done
