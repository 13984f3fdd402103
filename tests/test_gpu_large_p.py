"""p beyond one CTA's shared memory (p > 7 680; the paper's largest instances
reach p = 16 000).  The column kernels (prox + FISTA, bound
evaluation, rounding / branch selection) then keep a node's sort keys,
indices and scans in a global-memory slice per CTA instead of shared memory
(Engine: colstride_); the persistent pass kernel is off.  Same arithmetic,
so the oracle comparisons are as tight as at small p."""
import math

import numpy as np
import pytest

from tests.test_gpu_kernels import _engine, rnd_batch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("p,m,k", [(8200, 3, 5), (16000, 2, 12)])
def test_prox_and_g_large_p_match_oracle(bnb, orc, p, m, k):
    rng = np.random.default_rng(p)
    st, kb = rnd_batch(rng, p, m, k, all_free_first=True)
    U = rng.normal(size=(p, m)) * 0.3
    out = bnb.prox_step(U, 0.01, 1.0, st, kb, 2.0)
    rho = 1.0 / (2.0 * 0.01 * 1.0)
    for b in range(m):
        ref = orc.prox_step_column(U[:, b], st[:, b], kb[b], rho, 2.0)
        np.testing.assert_array_equal(out[:, b] == 0.0, ref == 0.0)  # exact-zero pattern
        np.testing.assert_allclose(out[:, b], ref, rtol=1e-12, atol=1e-14)
    g = bnb.g_value(out, st, kb, 2.0)
    gc = bnb.g_conjugate_value(U, st, kb, 2.0)
    for b in range(m):
        assert abs(g[b] - orc.g_value(out[:, b], st[:, b], kb[b], 2.0)) <= 1e-12 * max(1.0, abs(g[b]))
        assert abs(gc[b] - orc.g_conjugate(U[:, b], st[:, b], kb[b], 2.0)) <= 1e-12 * max(1.0, abs(gc[b]))


@pytest.mark.parametrize("loss", [0, 1])
def test_relax_and_solve_large_p(bnb, orc, loss):
    """n = 60, p = 8 200: a relaxation batch (status, iterations, bounds,
    iterates) equals the oracle's, and so do the first three passes of a
    solve (batches, evaluation counts, bounds, incumbent)."""
    n, p, k = 60, 8200, 2
    inst, eng = _engine(bnb, orc, n, p, k, 0.5, loss, seed=4)
    rng = np.random.default_rng(loss)
    st, kb = rnd_batch(rng, p, 3, k, all_free_first=True)
    warm = np.zeros((p, 3))
    L = orc.smoothness(loss, inst.X)
    res = eng.solve_batch_relaxation((st, kb, warm), bnb.RelaxConfig(smoothness=L, max_iterations=40),
                                     math.inf)
    ob, obnd, ost, oit = orc.relax_batch(inst, st, kb, warm, math.inf,
                                         orc.relax_cfg(smoothness=L, max_iterations=40))
    np.testing.assert_allclose(res.bounds, obnd, rtol=1e-6, atol=1e-6)
    assert res.status.tolist() == ost.tolist() and res.iterations.tolist() == oit.tolist()
    np.testing.assert_allclose(res.beta, ob, rtol=1e-6, atol=1e-7)
    # the first three passes of a solve (batches of 4) trace the oracle's
    def passes(run):
        out, cur = [], {}

        def dual(j0, j1, v):
            cur.setdefault((tuple(j0), tuple(j1)), []).append(v)

        def boundary(lb, ub):
            out.append((dict(cur), lb, ub))
            cur.clear()

        run(dual, boundary)
        return out[:3]

    # the same smoothness constant on both sides: with p >> n the power
    # iteration's 1e-4 stopping test (losses.hpp:104-107) can stop a round
    # apart on the two sides, and a different step gives a different
    # (equally valid) trajectory
    dev = passes(lambda d, b: eng.solve(
        bnb.SolverConfig(batch_size=4, time_limit=3.0, relax=bnb.RelaxConfig(smoothness=L)),
        bnb.DebugHooks(on_dual_bound=lambda nd, v: d(nd.fixed_zero, nd.fixed_one, v),
                       on_batch_boundary=b)))
    ref = passes(lambda d, b: orc.solve(
        inst, orc.solver_cfg(batch_size=4, time_limit=20.0, relax={"smoothness": L}),
        on_dual_bound=d, on_batch_boundary=b))
    assert len(dev) == len(ref) == 3
    for (dn, dlb, dub), (rn, rlb, rub) in zip(dev, ref):
        assert list(dn) == list(rn)
        for key in rn:
            assert len(dn[key]) == len(rn[key])
            np.testing.assert_allclose(dn[key], rn[key], rtol=1e-6, atol=1e-6)
        assert abs(dlb - rlb) <= 1e-6 * max(1.0, abs(rlb)) and abs(dub - rub) <= 1e-6 * max(1.0, abs(rub))
