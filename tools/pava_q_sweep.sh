#!/bin/bash
# PAVA walk variants (built under build/var/): prox / PAVA sub-phases on c1, c2, c3
for lib in build/var/lib_q1.so build/var/lib_rq1.so build/var/lib_rq2.so paper_2605_22188_b200/libbnbg.so; do
  [ -f "$lib" ] || continue
  for c in c1 c2; do echo "== $lib $c"; BNBG_LIB_PATH=$PWD/$lib python tools/pass_phases.py $c | grep -E "^c|prox|pava \(|kernel pass"; done
  echo "== $lib c3"; BNBG_LIB_PATH=$PWD/$lib python tools/pass_phases.py c3 --limit 3 | grep -E "^c3|pava \(|prox sub"
done
