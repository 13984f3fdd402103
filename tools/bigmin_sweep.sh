#!/bin/bash
# c4 (and c3) nodes/s vs the active width from which the 128x64 GEMM tiles are used
for v in 64 24 16; do
  BNBG_BIGGEMM=$v timeout 900 python bench.py --config c4 --no-cpu-baseline --time-limit 20 --steps 1 --warmup 1 > gpurun_out/bm.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/bm.json').read().strip().splitlines()[-1]); print('c4 big>=$v', round(d['value'],1), d['config']['nodes_per_certify'], d['roofline']['kernel_ms'])"
done
