import time, sys, os
sys.path.insert(0, os.getcwd())
import paper_2605_22188_b200 as P
inst, _ = P.generate_synthetic(P.GeneratorSpec(n=2000, p=500, k=8, correlation=0.7, loss=1, seed=0))
for i in range(4):
    t0 = time.perf_counter(); e = P.Engine(inst); t1 = time.perf_counter(); e.close(); t2 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms destroy {1e3*(t2-t1):.2f} ms")
