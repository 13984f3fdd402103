"""Generates tests/golden/rashomon_c5.json: the oracle's Rashomon pool for
BASELINE config c5 (squared loss n=2000 p=500 k=8 rho=0.7, epsilon 0.01, no
cap) -- the reference algorithm restated in oracle/ (CPU, OpenBLAS).  Takes
about a quarter of an hour on 8 cores.

Usage: python tests/golden/make_golden_c5.py
"""
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from oracle import oracle as O  # noqa: E402
from make_golden import fnv1a  # noqa: E402


def main():
    O.build()
    threads = os.cpu_count() or 1
    O.use_openblas(threads)
    inst = O.generate(2000, 500, 8, 0.7, O.SQUARED, 5.0, 0, 2.0, 1.0)
    t0 = time.time()
    cert, pool = O.collect_rashomon(inst, O.solver_cfg(workers=threads), epsilon=0.01, cap=-1)
    out = dict(fingerprint=fnv1a(inst.xflat(), inst.y), epsilon=0.01,
               optimal_value=cert.optimal_value, support=cert.support,
               nodes=cert.nodes_processed, seconds=time.time() - t0,
               pool=[dict(sequence=list(map(int, s)), objective=float(o)) for s, _, o in pool])
    with open(os.path.join(HERE, "rashomon_c5.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(len(pool), "models", cert.optimal_value, cert.nodes_processed, out["seconds"])


if __name__ == "__main__":
    main()
