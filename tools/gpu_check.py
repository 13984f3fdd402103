"""Quick device-vs-oracle diagnostic (prints max differences per entry point).

Run on the GPU box:  python tools/gpu_check.py
"""
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
import paper_2605_22188_b200 as P  # noqa: E402


def rnd_states(rng, p, m, k):
    st = np.zeros((p, m), dtype=np.uint8)
    kb = []
    for b in range(m):
        perm = rng.permutation(p)
        n1 = rng.integers(0, min(k, p))
        n0 = rng.integers(0, max(1, p - n1 - 1))
        st[perm[:n1], b] = 1
        st[perm[n1:n1 + n0], b] = 2
        kb.append(max(0, k - n1))
    return st, kb


def main():
    O.build()
    rng = np.random.default_rng(0)
    # prox_step
    for p, m, k in [(6, 8, 3), (64, 32, 5), (100, 16, 5), (500, 16, 8), (2000, 4, 10)]:
        U = rng.normal(size=(p, m)) * rng.choice([0.1, 1, 5], size=(1, m))
        st, kb = rnd_states(rng, p, m, k)
        eta, lam, M = 0.05, 1.0, 2.0
        out = P.prox_step(U, eta, lam, st, kb, M)
        rho = 1 / (2 * eta * lam)
        ref = np.stack([O.prox_step_column(U[:, b], st[:, b], kb[b], rho, M) for b in range(m)], 1)
        zero_mismatch = int(((out == 0) != (ref == 0)).sum())
        print(f"prox_step p={p} m={m}: maxabs={np.abs(out - ref).max():.3e} zero_mismatch={zero_mismatch}")
        cp = P.batched_conjugate_prox(U * rho, st, kb, rho, M)
        cref = np.stack([O.conjugate_prox_column(U[:, b] * rho, st[:, b], kb[b], rho, M) for b in range(m)], 1)
        print(f"  conj_prox maxabs={np.abs(cp - cref).max():.3e}")
        gv = P.g_value(out, st, kb, M)
        gref = np.array([O.g_value(out[:, b], st[:, b], kb[b], M) for b in range(m)])
        print(f"  g_value maxrel={np.nanmax(np.abs(gv - gref) / np.maximum(1, np.abs(gref))):.3e} inf_match={np.array_equal(np.isinf(gv), np.isinf(gref))}")
        gc = P.g_conjugate_value(U, st, kb, M)
        gcref = np.array([O.g_conjugate(U[:, b], st[:, b], kb[b], M) for b in range(m)])
        print(f"  g_conj maxrel={np.abs(gc - gcref).max() / max(1, np.abs(gcref).max()):.3e}")
    # engine on c1
    inst = O.generate(1000, 100, 5, 0.5, O.SQUARED)
    pin = P.ProblemInstance(inst.X, inst.y, P.LossKind.SQUARED, 5, 2.0, 1.0)
    eng = P.Engine(pin)
    L_o = O.smoothness(O.SQUARED, inst.X)
    print(f"smoothness dev={eng.smoothness():.17g} oracle={L_o:.17g} rel={abs(eng.smoothness()-L_o)/L_o:.2e}")
    for trans in (False, True):
        K = inst.n if trans else inst.p
        B = rng.normal(size=(K, 37))
        C = eng.gemm(B, trans)
        ref = (inst.X.T @ B) if trans else (inst.X @ B)
        print(f"gemm trans={trans}: maxrel={np.abs(C - ref).max() / np.abs(ref).max():.3e}")
    # relax root + random batch
    p = inst.p
    st, kb = rnd_states(rng, p, 12, 5)
    st[:, 0] = 0
    kb[0] = 5
    warm = np.zeros((p, 12))
    cfg = P.RelaxConfig(smoothness=L_o)
    t = time.time()
    res = eng.solve_batch_relaxation((st, kb, warm), cfg, math.inf)
    print("relax dev time", time.time() - t)
    ob, obnd, ost, oit = O.relax_batch(inst, st, kb, warm, math.inf, O.relax_cfg(smoothness=L_o))
    print("relax bounds rel diff", np.abs(res.bounds - obnd) / np.maximum(1, np.abs(obnd)))
    print("status dev", res.status.tolist(), "or", ost.tolist())
    print("iters dev", res.iterations.tolist(), "or", oit.tolist())
    print("beta maxabs", np.abs(res.beta - ob).max())
    # reopt
    sups = [[19, 39, 59], [1, 2, 3, 4, 5], [], [99]]
    r = eng.reoptimize_supports(sups)
    oc, oo = O.reoptimize(inst, sups, L_o)
    print("reopt obj rel", [abs(a - b) / abs(b) for a, b in zip(r.objectives, oo)])
    # full solve c1
    t = time.time()
    cert = eng.solve(P.SolverConfig())
    print("solve c1 dev", time.time() - t, cert.optimal_value, cert.support, cert.nodes_processed,
          cert.lb_batches, cert.profile)
    oc = O.solve(inst, O.solver_cfg(workers=8))
    print("solve c1 orc", oc.optimal_value, oc.support, oc.nodes_processed, oc.lb_batches)
    # logistic c2
    inst2 = O.generate(2000, 500, 8, 0.7, O.LOGISTIC)
    pin2 = P.ProblemInstance(inst2.X, inst2.y, P.LossKind.LOGISTIC, 8, 2.0, 1.0)
    t = time.time()
    cert2 = P.solve(pin2)
    print("solve c2 dev", time.time() - t, cert2.optimal_value, cert2.support, cert2.nodes_processed,
          cert2.lb_batches, cert2.relax_iterations, cert2.profile)


if __name__ == "__main__":
    main()
