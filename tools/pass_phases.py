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
limit = float(sys.argv[sys.argv.index("--limit") + 1]) if "--limit" in sys.argv else float("inf")
n, p, k, rho, loss, _ = CONFIGS[name]
inst, _ = P.generate_synthetic(P.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss, seed=0))
with P.Engine(inst) as eng:
    cfg = P.SolverConfig(time_limit=limit)
    eng.solve(cfg)
    before = eng.pass_profile()
    eng.set_timing(True)
    s0 = eng.kernel_stats()
    t0 = time.perf_counter()
    cert = eng.solve(cfg)
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
        tot += 0.0 if ph.endswith("_work") else ms
        if ph.endswith("_work"):
            continue
        w = after.get(ph + "_work", 0.0) - before.get(ph + "_work", 0.0)
        cnt = its if ph in ("xv", "xtr", "prox") else evals
        print(f"  phase {ph:10s} {ms:9.3f} ms  {ms / cnt * 1e3:8.2f} us per "
              f"{'iteration' if cnt == its else 'evaluation'}  (CTA 0 work {w / cnt * 1e3:6.2f} us, "
              f"barrier wait {(ms - w) / cnt * 1e3:6.2f} us)")
    print(f"  phases total {tot:.3f} ms")
    raw = eng.pass_profile_raw()
    its_all = max(1, its)
    names = ("load+sort", "pava", "scatter", "end barrier")
    print("  prox sub-phases (CTA 0, per iteration): " +
          ", ".join(f"{nm} {raw[16 + i] / its_all / 1e3 / 2:.2f} us" for i, nm in enumerate(names)))
    walks = max(1.0, raw[31])
    print(f"  pava (CTA 0): {raw[31] / its_all / 2:.2f} walks per iteration, scan "
          f"{raw[28] / walks / 1e3:.2f} us, walk {raw[29] / walks / 1e3:.2f} us, "
          f"{raw[30] / walks:.1f} warp steps per walk")
    tn = ("colmap+issue", "load wait", "mma", "reduce+epilogue")
    for nm, base in (("NN", 20), ("TN", 24)):
        print(f"  {nm} resident tile sub-phases (CTA 0, per iteration incl. evals): " +
              ", ".join(f"{t} {raw[base + i] / its_all / 1e3 / 2:.2f} us" for i, t in enumerate(tn)))
