"""One certified solve of a bench config (for ncu launch lists / full captures).

python tools/profile_solve.py [c1|c2|c3|c4|c5] [--warm] [--limit SECONDS]
(c5 runs collect_rashomon with epsilon 0.01)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_22188_b200 as P  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, p, k, rho, loss, _ = CONFIGS[name]
inst, _ = P.generate_synthetic(P.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss, seed=0))
limit = float(sys.argv[sys.argv.index("--limit") + 1]) if "--limit" in sys.argv else float("inf")
cfg = P.SolverConfig(time_limit=limit)
with P.Engine(inst) as eng:
    run = ((lambda: eng.collect_rashomon(cfg, P.RashomonConfig(epsilon=0.01)).certificate)
           if name == "c5" else (lambda: eng.solve(cfg)))
    if "--warm" in sys.argv:
        run()
    cert = run()
    print(name, cert.optimal_value, cert.support, cert.nodes_processed, cert.profile)
