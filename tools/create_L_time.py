import os, sys, time
sys.path.insert(0, '.')
import paper_2605_22188_b200 as P
from bench import CONFIGS
for name in ('c1', 'c2', 'c3', 'c4'):
    n, p, k, rho, loss, _ = CONFIGS[name]
    inst, _ = P.generate_synthetic(P.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss, seed=0))
    for rep in range(3):
        t0 = time.perf_counter(); e = P.Engine(inst); t1 = time.perf_counter(); L = e.smoothness(); e.close()
        t2 = time.perf_counter(); e = P.Engine(inst, smoothness=L); t3 = time.perf_counter(); e.close()
        print(name, 'create', round(1e3*(t1-t0), 2), 'ms; with L given', round(1e3*(t3-t2), 2), 'ms', flush=True)
