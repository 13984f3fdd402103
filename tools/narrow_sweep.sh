#!/bin/bash
for cfg in "default:64:paper_2605_22188_b200/libbnbg.so" "bn64from24:24:build/var/lib_narrow0.so" "bn64from16:16:build/var/lib_narrow0.so"; do
  IFS=: read name bm lib <<< "$cfg"
  BNBG_LIB_PATH=$PWD/$lib BNBG_BIGGEMM=$bm BNBG_PERSIST_MAXFLOPS=1e30 timeout 900 python bench.py --config c4 --no-cpu-baseline --time-limit 15 --steps 1 --warmup 1 > gpurun_out/ns.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/ns.json').read().strip().splitlines()[-1]); print('$name', round(d['value'],1), d['config']['nodes_per_certify'], {k: round(v) for k, v in d['roofline']['kernel_ms'].items()})"
done
