#!/bin/bash
# Round-end measurement set (run on the GPU box from the repo root).
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q > $O/final_pytest.log 2>&1; echo "rc=$?" >> $O/final_pytest.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.log 2>&1; echo "rc=$?" >> $O/final_smoke.log
timeout 600 python bench.py > $O/final_bench_c2.json 2> $O/final_bench_c2.err
for c in c1 c5; do timeout 300 python bench.py --config $c --no-cpu-baseline > $O/final_bench_$c.json 2>/dev/null; done
timeout 300 python bench.py --config c3 --no-cpu-baseline --time-limit 20 --steps 1 --warmup 1 > $O/final_bench_c3.json 2>/dev/null
timeout 900 python bench.py --config c4 --no-cpu-baseline --time-limit 30 --steps 1 --warmup 1 > $O/final_bench_c4.json 2>/dev/null
timeout 300 python tools/pass_phases.py c2 > $O/final_phases_c2.txt 2>&1
