"""Phase wall times of the persistent pass kernel for one certify.

BNBG_PASS_PROF=1 python tools/pass_phases.py [c1|c2|c3]
"""
import os
import sys
import time

os.environ.setdefault("BNBG_PASS_PROF", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_22188_b200 as P  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, p, k, rho, loss, _ = CONFIGS[name]
inst, _ = P.generate_synthetic(P.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss, seed=0))
with P.Engine(inst) as eng:
    eng.solve()
    before = eng.pass_profile()
    eng.set_timing(True)
    s0 = eng.kernel_stats()
    t0 = time.perf_counter()
    cert = eng.solve()
    wall = time.perf_counter() - t0
    s1 = eng.kernel_stats()
    after = eng.pass_profile()
    its = cert.relax_iterations
    evals = max(1, its // 10)
    print(f"{name}: {cert.nodes_processed} nodes, {cert.lb_batches} passes, {its} iterations, "
          f"{cert.node_iterations} node-iterations (avg active {cert.node_iterations / max(its, 1):.1f}), "
          f"wall {wall * 1e3:.1f} ms")
    for kc in s1:
        d = [a - b for a, b in zip(s1[kc], s0[kc])]
        if d[2]:
            print(f"  kernel {kc:10s} {d[0]:9.3f} ms  {int(d[2]):6d} launches")
    tot = 0.0
    for ph in after:
        ms = after[ph] - before.get(ph, 0.0)
        tot += ms
        per = ms / its * 1e3 if ph in ("xv", "xtr", "prox") else ms / evals * 1e3
        print(f"  phase {ph:10s} {ms:9.3f} ms  {per:8.2f} us per {'iteration' if ph in ('xv', 'xtr', 'prox') else 'evaluation'}")
    print(f"  phases total {tot:.3f} ms")
