"""Engine creation cost breakdown (c2): power iteration, X upload, pageable vs pinned."""
import time, numpy as np, torch
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_22188_b200 as P
from bench import CONFIGS
n, p, k, rho, loss, _ = CONFIGS["c2"]
inst, _ = P.generate_synthetic(P.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss, seed=0))
e = P.Engine(inst); L = e.smoothness(); e.close()
xf = inst.xflat()
for label, kw in (("default", {}), ("L given", {"smoothness": L})):
    ts = []
    for _ in range(8):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        e = P.Engine(inst, **kw); t1 = time.perf_counter(); e.close(); ts.append(t1 - t0)
    print(label, "create ms", [round(1e3 * t, 2) for t in ts])
t0 = time.perf_counter(); xf2 = inst.xflat(); t1 = time.perf_counter()
print("xflat ms", round(1e3 * (t1 - t0), 3), type(xf2), getattr(xf2, 'flags', None) and xf2.flags['C_CONTIGUOUS'])
buf = torch.empty(n * p, dtype=torch.float64, device="cuda")
src = torch.from_numpy(np.ascontiguousarray(xf))
for pin in (False, True):
    s = src.pin_memory() if pin else src
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter(); buf.copy_(s); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print("h2d 8MB pinned" if pin else "h2d 8MB pageable", [round(1e3 * t, 3) for t in ts])
