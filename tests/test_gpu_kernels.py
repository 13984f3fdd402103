"""Device kernels vs the CPU oracle, through the C-ABI (libbnbg.so).

Tolerances: index/rank work (supports, branch variable, exact zeros, status,
iteration counts) must be identical; prox outputs are required bit-equal where
the oracle is (same rank order and formula) and within 1e-12 otherwise;
GEMM/reduction outputs within 1e-12 relative (FP64, different association).
"""
import json
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rnd_batch(rng, p, m, k, all_free_first=False):
    st = np.zeros((p, m), dtype=np.uint8)
    kb = []
    for b in range(m):
        perm = rng.permutation(p)
        n1 = 0 if (all_free_first and b == 0) else int(rng.integers(0, min(k, p)))
        n0 = 0 if (all_free_first and b == 0) else int(rng.integers(0, max(1, p - n1 - 1)))
        st[perm[:n1], b] = 1
        st[perm[n1:n1 + n0], b] = 2
        kb.append(max(0, k - n1))
    return st, kb


@pytest.mark.parametrize("p,m,k", [(1, 1, 1), (2, 3, 1), (6, 8, 3), (64, 32, 5), (100, 16, 5),
                                   (500, 16, 8), (777, 5, 12), (2000, 4, 10), (5000, 2, 15)])
def test_prox_step_matches_oracle(bnb, orc, p, m, k):
    rng = np.random.default_rng(p * 131 + m)
    U = rng.normal(size=(p, m)) * rng.choice([0.05, 1.0, 8.0], size=(1, m))
    U[rng.random(size=(p, m)) < 0.05] = 0.0  # exact zeros
    st, kb = rnd_batch(rng, p, m, k)
    for eta in (0.002, 0.3):
        out = bnb.prox_step(U, eta, 1.0, st, kb, 2.0)
        rho = 1.0 / (2 * eta)
        ref = np.stack([orc.prox_step_column(U[:, b], st[:, b], kb[b], rho, 2.0)
                        for b in range(m)], 1)
        assert np.array_equal(out == 0.0, ref == 0.0)  # exact zeros (prox_kernel.hpp:262-272)
        np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("shape", ["plateau", "ramp", "ties", "heads_out_of_box"])
@pytest.mark.parametrize("p,k", [(100, 5), (500, 8), (2000, 15)])
def test_prox_long_pava_walks(bnb, orc, shape, p, k):
    """Key layouts that drive the PAVA walk through long right runs (more
    than one 64-state step), alternating left/right moves across the 2-D
    window, exact ties (rank order by index) and head values outside the box."""
    rng = np.random.default_rng(p + k)
    m = 4
    if shape == "plateau":
        U = 1.0 + 1e-3 * rng.normal(size=(p, m))
    elif shape == "ramp":
        U = np.linspace(3.0, 0.5, p)[:, None] * (1.0 + 1e-6 * rng.normal(size=(p, m)))
    elif shape == "ties":
        U = rng.choice([0.7, 0.7, 0.69, 0.5], size=(p, m))
    else:
        U = rng.normal(size=(p, m)) * 0.2
        U[:k, :] = 9.0 + rng.random(size=(k, m))
    U *= rng.choice([-1.0, 1.0], size=(p, m))
    st = np.zeros((p, m), dtype=np.uint8)
    st[rng.permutation(p)[: p // 10], 1] = 2  # fixed-zero coordinates in one column
    st[0, 2] = 1                              # one fixed-one coordinate
    kb = [k, k, k - 1, 1]
    for eta in (0.05, 0.5):
        out = bnb.prox_step(U, eta, 1.0, st, kb, 2.0)
        rho = 1.0 / (2 * eta)
        ref = np.stack([orc.prox_step_column(U[:, b], st[:, b], kb[b], rho, 2.0)
                        for b in range(m)], 1)
        assert np.array_equal(out == 0.0, ref == 0.0)
        np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)


def test_prox_golden_vectors(bnb):
    """Committed oracle vectors (tests/golden/prox_vectors.json)."""
    with open(os.path.join(GOLDEN, "prox_vectors.json")) as f:
        vecs = json.load(f)
    for v in vecs:
        u = np.array(v["u"])[:, None]
        st = np.array(v["state"], dtype=np.uint8)[:, None]
        eta = 1.0 / (2.0 * v["rho"])
        out = bnb.prox_step(u, eta, 1.0, st, [v["kbar"]], v["M"])[:, 0]
        np.testing.assert_allclose(out, v["prox"], rtol=1e-12, atol=1e-12)
        g = bnb.g_value(out, st[:, 0], v["kbar"], v["M"])[0]
        assert (math.isinf(g) and math.isinf(v["g"])) or abs(g - v["g"]) <= 1e-12 * max(1, abs(g))
        gc = bnb.g_conjugate_value(np.array(v["u"]), st[:, 0], v["kbar"], v["M"])[0]
        assert abs(gc - v["gconj"]) <= 1e-12 * max(1, abs(gc))


def test_conjugate_prox_spec_vectors_and_batch(bnb, orc):
    out = bnb.batched_conjugate_prox(np.array([[0.5], [2.0], [-0.3]]), np.zeros((3, 1)), [1], 1.0,
                                     1.0)
    np.testing.assert_allclose(out[:, 0], [0.5, 1.0, -0.3], atol=1e-12)
    out = bnb.batched_conjugate_prox(np.array([[1.0], [1.2]]), np.zeros((2, 1)), [1], 1.0, 2.0)
    np.testing.assert_allclose(out[:, 0], [11 / 15, 11 / 15], atol=1e-9)
    rng = np.random.default_rng(9)
    # acceptance #4: random batches p <= 64, m <= 32 vs per-column sequential
    for _ in range(30):
        p, m = int(rng.integers(1, 65)), int(rng.integers(1, 33))
        U = rng.normal(size=(p, m)) * 3
        st, kb = rnd_batch(rng, p, m, int(rng.integers(1, p + 1)))
        w, M = float(rng.choice([0.3, 2.0, 30.0])), float(rng.choice([0.5, 2.0]))
        out = bnb.batched_conjugate_prox(U, st, kb, w, M)
        ref = np.stack([orc.conjugate_prox_column(U[:, b], st[:, b], kb[b], w, M)
                        for b in range(m)], 1)
        np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)
        same = bnb.batched_conjugate_prox(np.repeat(U[:, :1], 3, 1), np.repeat(st[:, :1], 3, 1),
                                          [kb[0]] * 3, w, M)
        assert np.array_equal(same[:, 0], same[:, 1]) and np.array_equal(same[:, 1], same[:, 2])


@pytest.mark.parametrize("p,m", [(4, 4), (50, 20), (500, 12), (3000, 3)])
def test_g_and_gconj_match_oracle(bnb, orc, p, m):
    rng = np.random.default_rng(p + 7)
    st, kb = rnd_batch(rng, p, m, 6)
    U = rng.normal(size=(p, m))
    beta = bnb.prox_step(U, 0.05, 1.0, st, kb, 2.0)  # feasible points
    beta[:, -1] = U[:, -1] * 5                        # and an infeasible one
    g = bnb.g_value(beta, st, kb, 2.0)
    gr = np.array([orc.g_value(beta[:, b], st[:, b], kb[b], 2.0) for b in range(m)])
    assert np.array_equal(np.isinf(g), np.isinf(gr))
    fin = np.isfinite(gr)
    np.testing.assert_allclose(g[fin], gr[fin], rtol=1e-12, atol=1e-14)
    gc = bnb.g_conjugate_value(U, st, kb, 2.0)
    gcr = np.array([orc.g_conjugate(U[:, b], st[:, b], kb[b], 2.0) for b in range(m)])
    np.testing.assert_allclose(gc, gcr, rtol=1e-12)
    assert bnb.g_value(np.array([2, 1, 0.5, 0.25]), np.zeros(4), 2, 2.0)[0] == 3.53125


def _engine(bnb, orc, n, p, k, rho, loss, seed=0):
    inst = orc.generate(n, p, k, rho, loss, 5.0, seed)
    pin = bnb.ProblemInstance(inst.X, inst.y, loss, k, 2.0, 1.0)
    return inst, bnb.Engine(pin)


@pytest.mark.parametrize("n,p,k,rho,loss", [(1000, 100, 5, 0.5, 0), (2000, 500, 8, 0.7, 1),
                                            (30, 12, 3, 0.9, 1), (60, 8200, 2, 0.5, 0),
                                            (5000, 2000, 10, 0.9, 0)])
def test_smoothness_bit_identical_to_oracle(bnb, orc, n, p, k, rho, loss):
    """losses.hpp:86-112 on the device in the oracle's sequential order (no
    FMA): the smoothness constant -- hence the step 1/L of every relaxation
    and re-optimisation -- equals oracle.c's bit for bit."""
    inst, eng = _engine(bnb, orc, n, p, k, rho, loss)
    assert eng.smoothness() == orc.smoothness(loss, inst.X)


def test_smoothness_and_gemm(bnb, orc):
    inst, eng = _engine(bnb, orc, 1000, 100, 5, 0.5, 0)
    L = orc.smoothness(0, inst.X)
    assert eng.smoothness() == L
    rng = np.random.default_rng(3)
    for m in (1, 7, 8, 9, 16, 33, 300):
        for trans in (False, True):
            B = rng.normal(size=(inst.n if trans else inst.p, m))
            ref = inst.X.T @ B if trans else inst.X @ B
            out = eng.gemm(B, trans)
            assert np.abs(out - ref).max() <= 1e-12 * np.abs(ref).max()
    assert abs(bnb.smoothness_constant(0, np.eye(2)) - 1.01) < 1e-12
    assert abs(bnb.smoothness_constant(1, np.diag([3.0])) - 1.01 * 9 / 4) < 1e-12


def test_round_select_exact(bnb, orc):
    inst, eng = _engine(bnb, orc, 200, 60, 6, 0.5, 0)
    rng = np.random.default_rng(5)
    m = 24
    nodes, betas = [], []
    for b in range(m):
        perm = rng.permutation(60)
        n1 = int(rng.integers(0, 5))
        n0 = int(rng.integers(0, 30))
        nd = bnb.NodeState(list(perm[n1:n1 + n0]), list(perm[:n1]), np.zeros(60))
        beta = rng.normal(size=60)
        beta[rng.random(60) < 0.3] = 0.0
        beta[perm[0]] = beta[perm[1]]  # ties
        beta[nd.states() == 2] = 0.0
        nodes.append(nd)
        betas.append(beta)
    B = np.stack(betas, 1)
    sup = eng.round_support_batch(B, nodes)
    jb = eng.select_branch_variable_batch(B, nodes)
    for b, nd in enumerate(nodes):
        st = nd.states()
        ref = orc.round_support(B[:, b], st, nd.fixed_one, max(0, 6 - len(nd.fixed_one)))
        assert sup[b] == ref
        assert jb[b] == orc.select_branch(B[:, b], st)
    assert eng.select_branch_variable(np.array([0.1, -3.0, 0.2] + [0] * 57),
                                      bnb.NodeState([], [], np.zeros(60))) == 1


@pytest.mark.parametrize("loss", [0, 1])
def test_reopt_matches_oracle(bnb, orc, loss):
    inst, eng = _engine(bnb, orc, 500, 40, 6, 0.7, loss)
    rng = np.random.default_rng(11)
    sups = [[], [3], list(range(6)), [39, 0, 17], list(rng.choice(40, 6, replace=False))]
    r = eng.reoptimize_supports(sups)
    oc, oo = orc.reoptimize(inst, sups, orc.smoothness(loss, inst.X))
    for a, b in zip(r.objectives, oo):
        assert abs(a - b) <= 1e-9 * max(1, abs(b))
    for a, b in zip(r.coefficients, oc):
        np.testing.assert_allclose(a, b, rtol=1e-6, atol=1e-8)


@pytest.mark.parametrize("n,sizes", [(2000, [3, 8, 5]),        # registers, 8-wide
                                     (3000, [12, 9, 16]),      # registers, 16-wide
                                     (5000, [12, 15, 10]),     # large n: per-CTA gather form
                                     (9000, [7, 3])])
def test_reopt_cluster_paths_match_oracle(bnb, orc, n, sizes):
    """Logistic re-optimisation through each kernel variant (cluster register
    slices while a support's rows fit 8 CTAs' registers, else the gather form)."""
    p = 40
    inst, eng = _engine(bnb, orc, n, p, 16, 0.7, 1)
    rng = np.random.default_rng(n)
    sups = [list(rng.choice(p, q, replace=False)) for q in sizes]
    r = eng.reoptimize_supports(sups)
    oc, oo = orc.reoptimize(inst, sups, orc.smoothness(1, inst.X))
    for a, b in zip(r.objectives, oo):
        assert abs(a - b) <= 1e-9 * max(1, abs(b))
    for a, b in zip(r.coefficients, oc):
        np.testing.assert_allclose(a, b, rtol=1e-6, atol=1e-8)


@pytest.mark.parametrize("loss,n,p,k,m", [(0, 1000, 100, 5, 12), (1, 2000, 500, 8, 6),
                                          (0, 300, 64, 4, 40), (1, 150, 30, 3, 9)])
def test_relax_batch_matches_oracle(bnb, orc, loss, n, p, k, m):
    inst, eng = _engine(bnb, orc, n, p, k, 0.7, loss, seed=3)
    rng = np.random.default_rng(n + p)
    st, kb = rnd_batch(rng, p, m, k, all_free_first=True)
    warm = np.zeros((p, m))
    L = orc.smoothness(loss, inst.X)
    for thr in (math.inf, None):
        if thr is None:  # a finite threshold between the bounds so some columns prune
            _, bd, _, _ = orc.relax_batch(inst, st, kb, warm, math.inf,
                                          orc.relax_cfg(smoothness=L, max_iterations=50))
            srt = np.sort(bd)
            thr = float(0.5 * (srt[m // 2] + srt[m // 2 - 1])) if m > 1 else float(srt[0] - 1)
        trace_d, trace_o = [], []
        res = eng.solve_batch_relaxation((st, kb, warm), bnb.RelaxConfig(smoothness=L), thr,
                                         dual_trace=lambda b, v: trace_d.append((b, v)))
        ob, obnd, ost, oit = orc.relax_batch(inst, st, kb, warm, thr, orc.relax_cfg(smoothness=L),
                                             trace=lambda b, v: trace_o.append((b, v)))
        np.testing.assert_allclose(res.bounds, obnd, rtol=1e-6, atol=1e-6)
        assert res.status.tolist() == ost.tolist()
        assert res.iterations.tolist() == oit.tolist()
        np.testing.assert_allclose(res.beta, ob, rtol=1e-6, atol=1e-7)
        assert [b for b, _ in trace_d] == [b for b, _ in trace_o]
        np.testing.assert_allclose([v for _, v in trace_d], [v for _, v in trace_o], rtol=1e-6,
                                   atol=1e-6)


@pytest.mark.parametrize("loss,n,p,k,m,its", [
    (0, 200, 40, 4, 300, 40),     # m > 2 x SMs: multi-kernel path, 128 x 64 register-tiled GEMM
    (1, 240, 60, 5, 320, 30),
    (0, 1200, 1100, 6, 5, 30),    # p in (1024, 2048]: 8-wide register column sort
    (1, 900, 1500, 7, 4, 20),
])
def test_relax_batch_wide_and_large_p(bnb, orc, loss, n, p, k, m, its):
    """Parity of the c3/c4 code paths at oracle-affordable sizes (capped iterations)."""
    inst, eng = _engine(bnb, orc, n, p, k, 0.7, loss, seed=5)
    rng = np.random.default_rng(n * p + m)
    st, kb = rnd_batch(rng, p, m, k, all_free_first=True)
    warm = np.zeros((p, m))
    L = orc.smoothness(loss, inst.X)
    res = eng.solve_batch_relaxation((st, kb, warm),
                                     bnb.RelaxConfig(smoothness=L, max_iterations=its), math.inf)
    ob, obnd, ost, oit = orc.relax_batch(inst, st, kb, warm, math.inf,
                                         orc.relax_cfg(smoothness=L, max_iterations=its))
    np.testing.assert_allclose(res.bounds, obnd, rtol=1e-6, atol=1e-6)
    assert res.status.tolist() == ost.tolist()
    assert res.iterations.tolist() == oit.tolist()
    np.testing.assert_allclose(res.beta, ob, rtol=1e-6, atol=1e-7)


def test_relax_frozen_columns_bit_stable_and_batch_of_one(bnb, orc):
    """batch-of-m equals m independent single-node solves."""
    inst, eng = _engine(bnb, orc, 400, 50, 4, 0.6, 0, seed=5)
    rng = np.random.default_rng(1)
    st, kb = rnd_batch(rng, 50, 6, 4, all_free_first=True)
    warm = np.zeros((50, 6))
    full = eng.solve_batch_relaxation((st, kb, warm))
    for b in range(6):
        one = eng.solve_batch_relaxation((st[:, b:b + 1], [kb[b]], warm[:, b:b + 1]))
        assert np.array_equal(one.beta[:, 0], full.beta[:, b])
        assert one.bounds[0] == full.bounds[b] and one.iterations[0] == full.iterations[b]


def test_errors(bnb, orc):
    inst, eng = _engine(bnb, orc, 50, 10, 3, 0.5, 0)
    with pytest.raises(bnb.InputError):
        eng.solve_batch_relaxation([])
    with pytest.raises(bnb.InputError):
        bnb.prox_step(np.ones((3, 1)), -1.0, 1.0, np.zeros((3, 1)), [1], 1.0)
    with pytest.raises(bnb.LogicError):
        eng.select_branch_variable(np.ones(10), bnb.NodeState(list(range(10)), [], np.zeros(10)))
    warm = np.zeros((10, 1))
    warm[2, 0] = np.nan
    with pytest.raises(bnb.NumericError):
        eng.solve_batch_relaxation((np.zeros((10, 1)), [3], warm))


@pytest.mark.parametrize("cluster", ["1", "0"])
@pytest.mark.parametrize("loss,m", [(0, 5), (1, 16), (0, 20)])
def test_relax_one_cluster_pass_kernel(bnb, orc, monkeypatch, cluster, loss, m):
    """c1-sized X (n=1000, p=100) fits one 16-CTA cluster: batches of up to 16
    columns run the pass kernel as ONE cluster (64-row resident NN tiles,
    cluster barriers); BNBG_CLUSTER_PASS=0 forces the 148-CTA grid-barrier
    kernel.  Both match the oracle (m = 20 takes the grid kernel either way)."""
    monkeypatch.setenv("BNBG_CLUSTER_PASS", cluster)
    inst, eng = _engine(bnb, orc, 1000, 100, 5, 0.5, loss, seed=11)
    rng = np.random.default_rng(m * 7 + loss)
    st, kb = rnd_batch(rng, 100, m, 5, all_free_first=True)
    warm = np.zeros((100, m))
    L = orc.smoothness(loss, inst.X)
    res = eng.solve_batch_relaxation((st, kb, warm), bnb.RelaxConfig(smoothness=L), math.inf)
    ob, obnd, ost, oit = orc.relax_batch(inst, st, kb, warm, math.inf, orc.relax_cfg(smoothness=L))
    np.testing.assert_allclose(res.bounds, obnd, rtol=1e-6, atol=1e-6)
    assert res.status.tolist() == ost.tolist()
    assert res.iterations.tolist() == oit.tolist()
    np.testing.assert_allclose(res.beta, ob, rtol=1e-6, atol=1e-7)


def test_c1_certificate_same_with_and_without_cluster_pass(bnb, monkeypatch):
    """c1 (BASELINE configs[0]) certified by the one-cluster pass kernel and by
    the grid kernel: the reference's support, objective and node count."""
    inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=1000, p=100, k=5, correlation=0.5,
                                                       loss=bnb.LossKind.SQUARED, seed=0))
    certs = {}
    for cluster in ("1", "0"):
        monkeypatch.setenv("BNBG_CLUSTER_PASS", cluster)
        certs[cluster] = bnb.solve(inst, bnb.SolverConfig())
    for c in certs.values():
        assert c.status == "optimal" and c.support == [19, 39, 59, 79, 99]
        assert c.nodes_processed == 43
        assert abs(c.optimal_value - 6562.563358901953) <= 1e-9 * 6562.6


@pytest.mark.parametrize("gram", ["1", "0"])
@pytest.mark.parametrize("n,p,m,its", [(1000, 100, 12, 2000),   # persistent pass kernel
                                       (200, 40, 300, 40),      # m > 2 x SMs: standalone kernels
                                       (2000, 500, 70, 60)])    # 128 x 64 tiles of Q (p >= 132)
def test_relax_gram_form_matches_oracle(bnb, orc, monkeypatch, gram, n, p, m, its):
    """Squared loss, p <= n: the iteration gradient is Q V - c with Q = X'X,
    c = X'y formed once (BNBG_GRAM=0: X'(X V - y) as the reference writes it,
    relaxation.hpp:82-104).  Bounds, status, iteration counts and the iterates
    match the oracle either way; the evaluations use X in both."""
    monkeypatch.setenv("BNBG_GRAM", gram)
    inst, eng = _engine(bnb, orc, n, p, 5, 0.7, 0, seed=13)
    rng = np.random.default_rng(n + m)
    st, kb = rnd_batch(rng, p, m, 5, all_free_first=True)
    warm = np.zeros((p, m))
    L = orc.smoothness(0, inst.X)
    cfg = dict(smoothness=L, max_iterations=its)
    res = eng.solve_batch_relaxation((st, kb, warm), bnb.RelaxConfig(**cfg), math.inf)
    ob, obnd, ost, oit = orc.relax_batch(inst, st, kb, warm, math.inf, orc.relax_cfg(**cfg))
    np.testing.assert_allclose(res.bounds, obnd, rtol=1e-6, atol=1e-6)
    assert res.status.tolist() == ost.tolist()
    assert res.iterations.tolist() == oit.tolist()
    np.testing.assert_allclose(res.beta, ob, rtol=1e-6, atol=1e-7)
