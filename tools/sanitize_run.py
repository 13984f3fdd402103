"""Small workload that drives every device code path once, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

  - persistent pass kernel, resident mode (X in shared memory) and streaming
    mode (BNBG_RESIDENT=0), with the spin grid barrier (pass_kernel.cuh);
  - standalone kernels (BNBG_PERSISTENT=0): narrow split-K GEMMs, prox,
    eval, compaction;
  - the 128 x 64 GEMM with TMA-staged X tiles and split-K TN (m >= 64);
  - the tcgen05 kind::i8 emulated-FP64 GEMM (BNBG_OZAKI=1), 32- and 64-column
    tiles, NN with the l' epilogue inside a relaxation;
  - re-opt kernels: cluster (st.async / mbarrier exchange), Gram (squared),
    shared-memory slices (large n);
  - packer, round/select, branch write, node pool, Rashomon;
  - the NaN-key path of the prox (numeric_error) that memcheck flagged in r01;
  - round-2 variants: squared loss with the Gram-form gradient (local
    iterations for p <= 128, streaming Q tiles, the 128 x 64 tiles of Q with
    its TMA descriptor), the X form (BNBG_GRAM=0), and the logistic pass
    kernel as one 16-CTA cluster or as the 148-CTA grid.

Usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py [mode]
mode: all (default) | resident | streaming | standalone | gemm | ozaki | reopt | errors | variants
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_22188_b200 as P  # noqa: E402


def inst(n, p, k, rho, loss, seed=1):
    return P.generate_synthetic(P.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss,
                                                seed=seed))[0]


def solves():
    for loss in (0, 1):
        c = P.solve(inst(200, 40, 4, 0.8, loss), P.SolverConfig(batch_size=8))
        print("solve", loss, c.status, c.nodes_processed, c.support, flush=True)
    r = P.collect_rashomon(inst(60, 16, 3, 0.8, 0), rconfig=P.RashomonConfig(epsilon=0.2))
    print("rashomon", len(r.pool), flush=True)


def gemm():
    i = inst(600, 300, 5, 0.5, 0)
    rng = np.random.default_rng(0)
    with P.Engine(i) as eng:
        for m in (64, 130):
            for trans in (False, True):
                B = rng.normal(size=(i.n() if trans else i.p(), m))
                ref = i.X.T @ B if trans else i.X @ B
                out = eng.gemm(B, trans)
                assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()
        nodes = [P.root_node(i.p(), i.k) for _ in range(70)]
        for b, nd in enumerate(nodes):
            nd.fixed_zero = [b % i.p()]
        res = eng.solve_batch_relaxation(nodes, P.RelaxConfig(max_iterations=30))
        print("wide batch", len(res.bounds), flush=True)


def ozaki(flag="1"):
    os.environ["BNBG_OZAKI"] = flag
    try:
        gemm()
    finally:
        os.environ.pop("BNBG_OZAKI")


def reopt():
    for n, loss in ((300, 1), (300, 0), (30000, 1)):
        i = inst(n, 40, 8, 0.5, loss)
        with P.Engine(i) as eng:
            r = eng.reoptimize_supports([[1, 5, 9], list(range(8)), [3], list(range(0, 40, 3))])
            print("reopt", n, loss, [round(o, 6) for o in r.objectives], flush=True)


def errors():
    i = inst(100, 20, 3, 0.5, 0)
    with P.Engine(i) as eng:
        w = np.zeros(20)
        w[3] = math.nan
        nd = P.root_node(20, 3)
        nd.warm_start = w
        try:
            eng.solve_batch_relaxation([nd])
        except P.NumericError as e:
            print("numeric_error ok:", e, flush=True)
    U = np.full((20, 2), math.nan)
    st = np.zeros((20, 2), dtype=np.uint8)
    try:
        P.prox_step(U, 0.1, 1.0, st, [3, 3], 2.0)
    except Exception as e:  # noqa: BLE001
        print("prox on NaN:", type(e).__name__, flush=True)


def variants():
    for env in ({"BNBG_GRAM_LOCAL": "0"}, {"BNBG_GRAM": "0"}, {"BNBG_CLUSTER_PASS": "0"}):
        os.environ.update(env)
        try:
            print("variant", env, flush=True)
            solves()
        finally:
            for v in env:
                os.environ.pop(v)
    i = inst(600, 300, 5, 0.5, 0)  # Gram product on 128 x 64 tiles of Q (p >= 132)
    os.environ["BNBG_PERSISTENT"] = "0"
    try:
        with P.Engine(i) as eng:
            nodes = [P.root_node(i.p(), i.k) for _ in range(70)]
            for b, nd in enumerate(nodes):
                nd.fixed_zero = [b % i.p()]
            res = eng.solve_batch_relaxation(nodes, P.RelaxConfig(max_iterations=30))
            print("gram wide batch", len(res.bounds), flush=True)
    finally:
        os.environ.pop("BNBG_PERSISTENT")


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "all"
    if mode in ("all", "resident"):
        solves()
    if mode in ("all", "streaming"):
        os.environ["BNBG_RESIDENT"] = "0"
        solves()
        os.environ.pop("BNBG_RESIDENT")
    if mode in ("all", "standalone"):
        os.environ["BNBG_PERSISTENT"] = "0"
        solves()
        os.environ.pop("BNBG_PERSISTENT")
    if mode in ("all", "gemm"):
        ozaki("0")  # DMMA with TMA-staged tiles
    if mode in ("all", "ozaki"):
        ozaki()
    if mode in ("all", "reopt"):
        reopt()
    if mode in ("all", "errors"):
        errors()
    if mode in ("all", "variants"):
        variants()
    print("sanitize_run done", flush=True)


if __name__ == "__main__":
    main()
