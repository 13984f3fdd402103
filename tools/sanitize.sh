#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (every device code path once,
# small instances).  Outputs gpurun_out/r02b_sanitize_<tool>.log and a summary.
O=gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --print-limit 20 python tools/sanitize_run.py all > $O/r02b_sanitize_memcheck.log 2>&1
for m in resident gemm ozaki reopt errors; do
  timeout 600 $CS --tool racecheck --print-limit 20 python tools/sanitize_run.py $m > $O/r02b_sanitize_racecheck_$m.log 2>&1
done
timeout 900 $CS --tool synccheck --print-limit 20 python tools/sanitize_run.py all > $O/r02b_sanitize_synccheck.log 2>&1
timeout 600 $CS --tool initcheck --print-limit 20 python tools/sanitize_run.py resident > $O/r02b_sanitize_initcheck.log 2>&1
grep -H "ERROR SUMMARY\|sanitize_run done\|RACECHECK SUMMARY\|Traceback" $O/r02b_sanitize_*.log
