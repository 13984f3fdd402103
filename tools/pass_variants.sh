#!/bin/bash
# pass-kernel variants on c2 / c1 (phase profile per variant)
for cfg in c2 c1; do
  echo "#### $cfg default"; python tools/pass_phases.py $cfg 2>&1
  echo "#### $cfg BNBG_COLCACHE=0"; BNBG_COLCACHE=0 python tools/pass_phases.py $cfg 2>&1
done
echo "#### c2 BNBG_RESIDENT=0"; BNBG_RESIDENT=0 python tools/pass_phases.py c2 2>&1
