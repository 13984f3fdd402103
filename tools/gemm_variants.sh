#!/bin/bash
# c3 GEMM throughput of big-tile variants (BK/NS) built under build/var/
for lib in paper_2605_22188_b200/libbnbg.so build/var/lib_bk32ns2.so build/var/lib_bk32ns3.so; do
  [ -f "$lib" ] || continue
  BNBG_LIB_PATH=$PWD/$lib timeout 300 python bench.py --config c3 --no-cpu-baseline --time-limit 10 --steps 1 --warmup 1 > gpurun_out/gv.json 2>/dev/null
  python - "$lib" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/gv.json").read().strip().splitlines()[-1])
r = d["roofline"]
print(sys.argv[1], "nodes/s", round(d["value"], 1), r["kernel"], "TF/s", round(r["achieved"], 2), r["kernel_ms"])
PY
done
