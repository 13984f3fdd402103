#!/bin/bash
# A/B of engine switches at a time limit: ab_limit.sh CONFIG LIMIT "ENV1" "ENV2" ...
# prints nodes/s and the kernel-class times (one timed step, one warm-up; not a bench value)
cfg=$1; lim=$2; shift 2
for v in "$@"; do
  out=$(env $v python bench.py --config $cfg --steps 1 --warmup 1 --time-limit $lim --no-cpu-baseline --no-secondary 2>/dev/null | grep '^{')
  echo "$cfg [$v] $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["result"]; print("%.1f nodes/s  %s nodes  %.2f s  status %s  kernels %s" % (d["value"], r["nodes_per_certify"], d["ms_per_step"]/1e3, r["status"], {k: round(v) for k, v in d["roofline"]["kernel_ms"].items()}))')"
done
