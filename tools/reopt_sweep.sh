#!/bin/bash
# reopt cluster-size sweep on c2 (prints the kernel-class times per certify)
for cs in 0 1 2 4 8; do
  if [ $cs = 0 ]; then unset BNBG_REOPT_CS; else export BNBG_REOPT_CS=$cs; fi
  echo "== BNBG_REOPT_CS=$cs"; python tools/pass_phases.py c2 2>&1 | head -4
done
