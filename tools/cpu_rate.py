"""CPU reference-port nodes/s on a BASELINE config within a time limit (the
bench's cpu_baseline leg for configs other than c2).

python tools/cpu_rate.py c3 [--limit SECONDS]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402  (test infrastructure: the CPU baseline)
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
limit = float(sys.argv[sys.argv.index("--limit") + 1]) if "--limit" in sys.argv else 120.0
n, p, k, rho, loss, desc = CONFIGS[name]
O.build()
threads = os.cpu_count() or 1
blas = O.use_openblas(threads)
inst = O.generate(n, p, k, rho, loss, 5.0, 0, 2.0, 1.0)
t0 = time.perf_counter()
c = O.solve(inst, O.solver_cfg(workers=threads, time_limit=limit))
wall = time.perf_counter() - t0
print(json.dumps({"config": name, "kind": "port", "cores": threads, "openblas": blas,
                  "seconds": wall, "nodes": c.nodes_processed,
                  "nodes_per_s": c.nodes_processed / wall, "status": c.status,
                  "gap_percent": c.gap_percent}), flush=True)
