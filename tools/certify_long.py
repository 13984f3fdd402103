"""One certify of a BASELINE config with a time limit; prints a JSON line
(status, time, nodes, nodes/s, gap, bound, value, support) with the
nvidia-smi clock record of the run (bench.ClockSampler: median SM clock,
max clock, throttle reasons seen).

python tools/certify_long.py c3 [--limit SECONDS]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_22188_b200 as P  # noqa: E402
from bench import CONFIGS, ClockSampler  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
limit = float(sys.argv[sys.argv.index("--limit") + 1]) if "--limit" in sys.argv else float("inf")
n, p, k, rho, loss, desc = CONFIGS[name]
inst, _ = P.generate_synthetic(P.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss, seed=0))
with P.Engine(inst) as eng:
    sampler = ClockSampler(0)
    sampler.start()
    t0 = time.perf_counter()
    cert = eng.solve(P.SolverConfig(time_limit=limit))
    wall = time.perf_counter() - t0
    clocks = sampler.stop()
print(json.dumps({"config": name, "workload": desc, "status": cert.status, "seconds": wall,
                  "nodes": cert.nodes_processed, "nodes_per_s": cert.nodes_processed / wall,
                  "lb_batches": cert.lb_batches, "gap_percent": cert.gap_percent,
                  "lower_bound": cert.lower_bound, "optimal_value": cert.optimal_value,
                  "support": cert.support, "relax_iterations": cert.relax_iterations,
                  "node_iterations": cert.node_iterations, "clocks": clocks}), flush=True)
