#!/bin/bash
for v in 1e30 4e9 1e9; do
  for c in c4 c3; do
    BNBG_PERSIST_MAXFLOPS=$v timeout 900 python bench.py --config $c --no-cpu-baseline --time-limit 15 --steps 1 --warmup 1 > gpurun_out/ps.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/ps.json').read().strip().splitlines()[-1]); print('$c maxflops=$v', round(d['value'],1), d['config']['nodes_per_certify'], {k: round(v) for k, v in d['roofline']['kernel_ms'].items()})"
  done
done
