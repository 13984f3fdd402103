"""SPEC.md:802-815 acceptance criteria at the spec's scale, on the device.

#1 and #11 are in test_gpu_solve.py; #5, #7 and #9 are CPU-side (oracle /
host I/O) or out of scope (partitioned_eval).  Here:

  #2  safe bounds: every dual bound the device emits is <= the node's true
      optimum, zero violations over >= 1e5 recorded bounds;
  #3  Theorem 1: device g(beta) equals direct minimisation over the
      z-polytope (budget-equation bisection) within 1e-6
      on 10^3 random feasible draws with p <= 10; tau sandwich exact
      (SPEC.md:807);
  #4  batched prox: device batched_conjugate_prox equals the per-column
      sequential computation within 1e-12 on 10^3 random batches (p <= 64,
      m <= 32); both equal a brute-force grid oracle within 1e-4 for p <= 4
      (SPEC.md:808);
  #6  Rashomon completeness on 50 enumeration instances, eps = 0.1, uncapped
      and cap N = 5;
  #8  batching speedup: a squared instance that needs >= 2000 nodes
      certifies at batch 256 in <= 1/3 of the batch-1 time (the
      spec's "e.g. n = p = 300" instance needs > 150 000 nodes on this
      generator, too many for a batch-1 run in a test, so n = 150, p = 80,
      k = 6, rho = 0.9: ~12 000 nodes);
  #10 profiling coherence: component seconds within 5% of total wall time,
      lb/reopt batch counters present;
  and the packer's Fig. 2 batch.
"""
import math
import time

import numpy as np
import pytest

from tests._enum import all_support_values, node_optimum

pytestmark = pytest.mark.gpu

ENUM = [(loss, seed) for loss in (0, 1) for seed in range(50)]


@pytest.fixture(scope="module")
def enum_instances(bnb):
    """The 100 SPEC #1 instances with every support's value (enumeration)."""
    out = []
    for loss, seed in ENUM:
        inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=30, p=12, k=3, correlation=0.9,
                                                           loss=loss, seed=seed))
        out.append((loss, seed, inst, all_support_values(inst.X, inst.y, loss, 3, 2.0, 1.0)))
    return out


def test_acceptance2_safe_bounds_1e5(bnb, enum_instances):
    """#2: >= 1e5 device bounds, none above the node's true optimum."""
    total, bad = 0, []
    for loss, seed, inst, vals in enum_instances:
        cache = {}
        events = []
        with bnb.Engine(inst) as eng:
            for cfg in (bnb.SolverConfig(prune_slack=0.0, batch_size=1,
                                         relax=bnb.RelaxConfig(check_interval=1)),
                        bnb.SolverConfig(prune_slack=0.0, relax=bnb.RelaxConfig(check_interval=1))):
                cert = eng.solve(cfg, bnb.DebugHooks(on_dual_bound=lambda nd, v: events.append(
                    (tuple(sorted(nd.fixed_zero)), tuple(sorted(nd.fixed_one)), v))))
                assert cert.status == "optimal"
        for z, o, psi in events:
            key = (z, o)
            if key not in cache:
                cache[key] = node_optimum(vals, z, o)
            opt = cache[key]
            if psi > opt + 1e-9 * max(1.0, abs(opt)):
                bad.append((loss, seed, key, psi, opt))
        total += len(events)
    print(f"#2: {total} device lower bounds checked against enumerated node optima")
    assert not bad, bad[:5]
    assert total >= 100_000


def _g_bisection(beta, st, kbar, M):
    """g(beta) = min over the node's z-polytope of 1/2 sum beta_j^2 / z_j
    (Appendix B.1): z_J0 = 0, z_J1 = 1, free z in [0, 1] with
    sum z <= kbar and |beta_j| <= M z_j.  Binding case: tau from the budget
    equation sum_f min(1, |beta_j| / tau) = kbar by bisection; z_j = min(1, |beta_j|/tau)."""
    tol = M * (1 + 1e-9)
    if np.any(beta[st == 2] != 0):
        return math.inf
    if np.any(np.abs(beta[st != 2]) > tol):
        return math.inf
    base = 0.5 * float(np.sum(beta[st == 1] ** 2))
    a = np.abs(beta[st == 0])
    if kbar <= 0:
        return math.inf if np.any(a != 0) else base
    if np.count_nonzero(a) <= kbar:
        return base + 0.5 * float(np.sum(a ** 2))
    if np.sum(np.minimum(1.0, a / M)) > kbar * (1 + 1e-12):
        return math.inf  # tau would exceed M: outside the relaxation's domain
    lo, hi = 0.0, M
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if np.sum(np.minimum(1.0, a / mid)) > kbar:
            lo = mid
        else:
            hi = mid
    tau = hi
    z = np.minimum(1.0, a / tau)
    nz = a > 0
    return base + 0.5 * float(np.sum(a[nz] ** 2 / z[nz]))


def test_acceptance3_theorem1_recovery(bnb, orc_any):
    """#3: 1e3 random feasible draws, p <= 10: device g == bisection within 1e-6;
    the recovered tau satisfies |beta_(s)| >= tau >= |beta_(s+1)| exactly."""
    rng = np.random.default_rng(3)
    draws = []
    while len(draws) < 1000:
        p = int(rng.integers(2, 11))
        st = rng.choice([0, 0, 0, 1, 2], size=p).astype(np.uint8)
        nf = int(np.sum(st == 0))
        k = int(rng.integers(1, p + 1))
        kbar = k - int(np.sum(st == 1))
        if kbar < 1 or nf == 0:
            continue
        M = float(rng.uniform(0.5, 3.0))
        beta = rng.normal(size=p) * rng.choice([0.2, 1.0, 3.0])
        beta[st == 2] = 0.0
        beta[rng.random(p) < 0.2] = 0.0
        beta = np.clip(beta, -M, M)
        free = st == 0
        s = np.sum(np.abs(beta[free])) / M
        if s > kbar:  # feasible for the relaxation: sum_f |beta| / M <= kbar
            beta[free] *= kbar / s * (1 - 1e-9)
        draws.append((beta, st, kbar, M))
    got = []
    for beta, st, kbar, M in draws:
        got.append(bnb.g_value(beta, st, kbar, M)[0])
    binding = 0
    for (beta, st, kbar, M), g in zip(draws, got):
        want = _g_bisection(beta, st, kbar, M)
        assert math.isfinite(want) and math.isfinite(g)
        assert abs(g - want) <= 1e-6 * max(1.0, abs(want)), (beta, st, kbar, M, g, want)
        z, tau, cap = orc_any.recover(beta, st, kbar, M)
        a = np.sort(np.abs(beta[st == 0]))[::-1]
        if np.count_nonzero(a) > kbar:
            binding += 1
            upper = math.inf if cap == 0 else a[cap - 1]
            assert upper >= tau >= a[cap], (a, cap, tau)  # primal_heuristics.hpp:90
    assert binding >= 200


def _huber(q, M):
    q = np.abs(q)
    return np.where(q <= M, 0.5 * q * q, M * q - 0.5 * M * M)


def _argmin_1d(f, lo, hi, iters=64):
    """Ternary search of a convex function, vectorised over coordinates."""
    for _ in range(iters):
        a = lo + (hi - lo) / 3
        b = hi - (hi - lo) / 3
        left = f(a) <= f(b)
        hi = np.where(left, b, hi)
        lo = np.where(left, lo, a)
    return 0.5 * (lo + hi)


def _grid_prox(x, st, kbar, w, M):
    """Brute-force oracle of prox_{w g*}(x), g* = sum_J1 H_M + TopSum_kbar H_M
    over the free set (prox_kernel.hpp:351-370), built only from 1-D convex
    searches: TopSum_k(h) = min_{t >= 0} k t + sum max(0, h - t), so for a
    fixed t the problem separates per coordinate, and the partial minimum is
    convex in t.  J0 is unpenalised (v = x)."""
    x = np.asarray(x, dtype=np.float64)
    v = x.copy()
    span = np.abs(x) + 1.0
    one = st == 1
    if one.any():
        xo = x[one]
        v[one] = _argmin_1d(lambda u: 0.5 * (u - xo) ** 2 + w * _huber(u, M), -span[one],
                            span[one])
    free = st == 0
    if free.any() and kbar > 0:
        xf, sf = x[free], span[free]

        def inner(t):
            return _argmin_1d(lambda u: 0.5 * (u - xf) ** 2 + w * np.maximum(0.0, _huber(u, M) - t),
                              -sf, sf)

        def outer(t):
            u = inner(t)
            return kbar * w * t + float(np.sum(0.5 * (u - xf) ** 2
                                               + w * np.maximum(0.0, _huber(u, M) - t)))

        lo, hi = 0.0, float(np.max(_huber(xf, M))) + 1.0
        for _ in range(64):
            a, b = lo + (hi - lo) / 3, hi - (hi - lo) / 3
            if outer(a) <= outer(b):
                hi = b
            else:
                lo = a
        v[free] = inner(0.5 * (lo + hi))
    return v


def test_acceptance4_batched_prox(bnb, orc):
    """#4: 1e3 random batches (p <= 64, m <= 32): device batch == per-column
    sequential within 1e-12; p <= 4 columns == grid oracle within 1e-4."""
    rng = np.random.default_rng(4)
    grid_checked = 0
    for it in range(1000):
        p = int(rng.integers(1, 65)) if it % 10 else int(rng.integers(1, 5))
        m = int(rng.integers(1, 33))
        st = rng.choice([0, 0, 0, 1, 2], size=(p, m)).astype(np.uint8)
        kbar = rng.integers(0, p + 1, size=m).tolist()
        w, M = float(rng.uniform(0.1, 5.0)), float(rng.uniform(0.5, 3.0))
        U = rng.normal(size=(p, m)) * rng.choice([0.1, 1.0, 4.0])
        dev = bnb.batched_conjugate_prox(U, st, kbar, w, M)
        for b in range(m):
            seq = orc.conjugate_prox_column(U[:, b], st[:, b], kbar[b], w, M)
            np.testing.assert_allclose(dev[:, b], seq, rtol=1e-12, atol=1e-12)
            if p <= 4 and grid_checked < 120 and b < 2:
                v = _grid_prox(U[:, b], st[:, b], kbar[b], w, M)
                np.testing.assert_allclose(dev[:, b], v, atol=1e-4)
                grid_checked += 1
    assert grid_checked >= 100


def test_acceptance6_rashomon_50_instances(bnb, enum_instances):
    """#6 at spec scale: 50 enumeration instances (25 per loss), eps = 0.1:
    pool == enumerated eps-Rashomon set; cap 5 == the 5 smallest values."""
    eps = 0.1
    count = 0
    for loss, seed, inst, vals in enum_instances:
        if seed >= 25:
            continue
        vstar = min(vals.values())
        tau = (1 + eps) * vstar
        res = bnb.collect_rashomon(inst, rconfig=bnb.RashomonConfig(epsilon=eps))
        got = {tuple(sorted(s)) for s, _, _ in res.pool}
        want_k = {S for S, v in vals.items() if len(S) == 3 and v <= tau}
        sound = {S for S, v in vals.items() if v <= tau}
        ambiguous = {S for S, v in vals.items() if abs(v - tau) <= 1e-6 * abs(tau)}
        assert want_k - ambiguous <= got, (loss, seed)
        assert got - ambiguous <= sound, (loss, seed)
        res5 = bnb.collect_rashomon(inst, rconfig=bnb.RashomonConfig(epsilon=eps, cap=5))
        best5 = sorted(v for S, v in vals.items() if len(S) == 3 and v <= tau)[:5]
        np.testing.assert_allclose(sorted(o for _, _, o in res5.pool), best5, rtol=1e-6)
        count += 1
    assert count == 50


def test_acceptance8_batching_speedup(bnb):
    """#8: n = 150, p = 80, k = 6, rho = 0.9, squared (>= 2000 nodes; see the
    module docstring): batch 256 certifies in <= 1/3 of the batch-1 wall time,
    both at gap 0 with the same support."""
    inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=150, p=80, k=6, correlation=0.9,
                                                       loss=0, seed=0))
    with bnb.Engine(inst) as eng:
        eng.solve(bnb.SolverConfig(batch_size=256, time_limit=2.0))  # warm-up
        t0 = time.perf_counter()
        c256 = eng.solve(bnb.SolverConfig(batch_size=256))
        t256 = time.perf_counter() - t0
        t0 = time.perf_counter()
        c1 = eng.solve(bnb.SolverConfig(batch_size=1))
        t1 = time.perf_counter() - t0
    print(f"#8: batch 1 {t1:.2f} s ({c1.nodes_processed} nodes), batch 256 {t256:.2f} s "
          f"({c256.nodes_processed} nodes): {t1 / t256:.1f}x")
    assert c1.status == c256.status == "optimal"
    assert c1.gap_percent == c256.gap_percent == 0.0
    assert c1.support == c256.support
    assert max(c1.nodes_processed, c256.nodes_processed) >= 2000
    assert t256 <= t1 / 3


def test_acceptance10_profiling_coherence(bnb, enum_instances):
    """#10: lower_bound + reoptimization + transfer + branch_generate seconds
    within 5% of total_seconds, on the acceptance runs that take >= 20 ms
    (below that the 5% is under the clock's resolution of host bookkeeping):
    c2, and batch-1 / auto certifies of c1 and two correlated instances; the
    batch counters are set."""
    runs = []
    for loss, seed, inst, _ in enum_instances[::10]:
        runs.append(bnb.solve(inst, bnb.SolverConfig(batch_size=1)))
    for n, p, k, rho, loss, batch in [(1000, 100, 5, 0.5, 0, 0), (2000, 500, 8, 0.7, 1, 0),
                                      (150, 80, 6, 0.9, 0, 0), (100, 60, 5, 0.9, 0, 1),
                                      (1000, 100, 5, 0.5, 0, 1)]:
        inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=n, p=p, k=k, correlation=rho,
                                                           loss=loss, seed=0))
        runs.append(bnb.solve(inst, bnb.SolverConfig(batch_size=batch)))
    checked = 0
    for c in runs:
        pr = c.profile
        parts = (pr.lower_bound_seconds + pr.reoptimization_seconds + pr.transfer_seconds
                 + pr.branch_generate_seconds)
        assert c.lb_batches > 0 and c.reopt_batches > 0
        assert parts <= pr.total_seconds * 1.0001
        if pr.total_seconds >= 0.02:
            assert parts >= 0.95 * pr.total_seconds, (parts, pr.total_seconds)
            checked += 1
    assert checked >= 4


def test_packer_fig2_batch(bnb):
    """PAPER.md:382-427 Fig. 2: p = 6, m = 3, k = 3 (1-based in the figure).
    N1: J0 {5}, J1 {2}; N2: J0 {2,6}, J1 {1,4}; N3: J0 {3}, J1 {}.  The device
    packer (BatchMeta::from_nodes, prox_kernel.hpp:52-90) must give the
    figure's free sets {1,3,4,6}, {3,5}, {1,2,4,5,6}, reduced budgets 2, 1, 3,
    and the sentinel pattern of K^pad; the prox over that batch equals the
    oracle's column by column."""
    rng = np.random.default_rng(0)
    inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=20, p=6, k=3, correlation=0.5, seed=1))
    one = lambda s: [j - 1 for j in s]  # noqa: E731
    nodes = [bnb.NodeState(fixed_zero=one([5]), fixed_one=one([2]), warm_start=np.zeros(6)),
             bnb.NodeState(fixed_zero=one([2, 6]), fixed_one=one([1, 4]), warm_start=np.zeros(6)),
             bnb.NodeState(fixed_zero=one([3]), fixed_one=[], warm_start=np.zeros(6))]
    with bnb.Engine(inst) as eng:
        state, kbar, free = eng.pack_batch(nodes)
    want_free = [one([1, 3, 4, 6]), one([3, 5]), one([1, 2, 4, 5, 6])]
    for b in range(3):
        assert sorted(np.flatnonzero(state[:, b] == 0).tolist()) == want_free[b]
        assert sorted(np.flatnonzero(state[:, b] == 2).tolist()) == sorted(nodes[b].fixed_zero)
        assert sorted(np.flatnonzero(state[:, b] == 1).tolist()) == sorted(nodes[b].fixed_one)
    assert kbar == [2, 1, 3] and free == [4, 2, 5]
    # K^pad: |u| on the free rows, -inf (lowest) elsewhere -- the figure's matrix
    kpad_finite = state == 0
    assert kpad_finite.tolist() == [[True, False, True], [False, False, True],
                                    [True, True, False], [True, False, True],
                                    [False, True, True], [True, False, True]]
    U = rng.normal(size=(6, 3))
    dev = bnb.batched_conjugate_prox(U, state, kbar, 1.0, 2.0)
    from oracle import oracle as O
    for b in range(3):
        np.testing.assert_allclose(dev[:, b], O.conjugate_prox_column(U[:, b], state[:, b],
                                                                      kbar[b], 1.0, 2.0),
                                   rtol=1e-12, atol=1e-12)
