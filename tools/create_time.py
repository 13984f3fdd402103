"""Engine creation time per config (median of 9), for the library in BNBG_LIB_PATH."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_22188_b200 as P  # noqa: E402
from bench import CONFIGS  # noqa: E402

for name in sys.argv[1:] or ["c1", "c2"]:
    n, p, k, rho, loss, _ = CONFIGS[name]
    inst, _ = P.generate_synthetic(P.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss, seed=0))
    ts, L = [], None
    for _ in range(9):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e = P.Engine(inst)
        t1 = time.perf_counter()
        L = e.smoothness()
        e.close()
        ts.append(1e3 * (t1 - t0))
    ts.sort()
    print(f"{name}: create median {ts[4]:.2f} ms (min {ts[0]:.2f}), L = {L!r}")
