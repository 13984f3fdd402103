#!/bin/bash
# A/B of engine switches on the bench line: ab_env.sh CONFIG STEPS "ENV1" "ENV2" ...
# prints ms_per_step (device) and e2e time-to-certify per variant, twice each
cfg=$1; steps=$2; shift 2
for rep in 1 2; do
  for v in "$@"; do
    out=$(env $v python bench.py --config $cfg --steps $steps --warmup 3 --no-cpu-baseline --no-secondary 2>/dev/null | grep '^{')
    echo "$cfg [$v] $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("%.3f ms  e2e %.3f ms  nodes %d" % (d["ms_per_step"], 1e3*d["e2e"]["time_to_certify_s"], d["result"]["nodes_per_certify"]))')"
  done
done
