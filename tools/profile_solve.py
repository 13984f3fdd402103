"""One certified solve of a bench config (for ncu launch lists / full captures).

python tools/profile_solve.py [c1|c2|c3] [--warm]
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
with P.Engine(inst) as eng:
    if "--warm" in sys.argv:
        eng.solve()
    cert = eng.solve()
    print(name, cert.optimal_value, cert.support, cert.nodes_processed, cert.profile)
