"""Pins the CPU oracle (oracle/oracle.c) to the reference's known answers.

The reference ships no test code; its known-answer vectors live in SPEC.md
(cited per test).  These run on CPU only.
"""
import math

import numpy as np
import pytest


def test_losses_known_answers(orc_any):
    O = orc_any
    assert O.loss_value(O.SQUARED, 3.0, 3.0) == 0.0
    assert abs(O.loss_value(O.LOGISTIC, 0.0, 1.0) - math.log(2)) < 1e-12
    assert abs(O.loss_value(O.LOGISTIC, 2.0, -1.0) - 2.126928) < 1e-6
    assert O.loss_derivative(O.SQUARED, 1.0, 1.0) == 0.0
    assert O.loss_derivative(O.LOGISTIC, 0.0, 1.0) == -0.5
    assert abs(O.loss_derivative(O.LOGISTIC, 1.0, 1.0) + 0.268941) < 1e-6
    assert O.loss_conjugate(O.SQUARED, 0.0, 5.0) == 0.0
    assert abs(O.loss_conjugate(O.LOGISTIC, -0.5, 1.0) + math.log(2)) < 1e-12
    assert O.loss_conjugate(O.LOGISTIC, 0.1, 1.0) == math.inf
    # overflow safety at |s| = 1e4
    for s in (1e4, -1e4):
        assert math.isfinite(O.loss_value(O.LOGISTIC, s, 1.0))
        assert math.isfinite(O.loss_derivative(O.LOGISTIC, s, -1.0))


def test_fenchel_young_and_finite_differences(orc_any):
    O = orc_any
    rng = np.random.default_rng(1)
    for loss in (O.SQUARED, O.LOGISTIC):
        for _ in range(2000):
            s = rng.normal() * 3
            y = rng.choice([-1.0, 1.0]) if loss == O.LOGISTIC else rng.normal()
            z = O.loss_derivative(loss, s, y)
            fy = O.loss_value(loss, s, y) + O.loss_conjugate(loss, z, y) - z * s
            assert abs(fy) <= 1e-9
            h = 1e-5
            fd = (O.loss_value(loss, s + h, y) - O.loss_value(loss, s - h, y)) / (2 * h)
            assert abs(fd - z) <= 1e-6 * max(1.0, abs(z))


def test_smoothness_known_answers(orc_any):
    O = orc_any
    assert abs(O.smoothness(O.SQUARED, np.eye(2)) - 1.01) < 1e-12
    assert abs(O.smoothness(O.LOGISTIC, np.diag([3.0])) - 1.01 * 9 / 4) < 1e-12
    rng = np.random.default_rng(2)
    X = rng.normal(size=(10, 5))
    smax2 = np.linalg.svd(X, compute_uv=False)[0] ** 2
    assert abs(O.smoothness(O.SQUARED, X) / 1.01 - smax2) <= 0.01 * smax2
    assert O.smoothness(O.SQUARED, np.zeros((3, 2))) == 1e-12                # losses.hpp:103


def test_prox_known_answers(orc_any):
    O = orc_any
    assert O.prox_huber(3.0, 0.0, 2.0) == 3.0
    assert O.prox_huber(1.0, 1.0, 2.0) == 0.5
    assert O.prox_huber(10.0, 1.0, 2.0) == 8.0
    out = O.conjugate_prox_column([0.5, 2.0, -0.3], None, 1, 1.0, 1.0)
    np.testing.assert_allclose(out, [0.5, 1.0, -0.3], atol=1e-12)
    out = O.conjugate_prox_column([1.0, 1.2], None, 1, 1.0, 2.0)
    np.testing.assert_allclose(out, [0.733333333333, 0.733333333333], atol=1e-9)
    assert np.all(O.prox_step_column(np.zeros(5), None, 2, 3.0, 2.0) == 0)
    st = np.full(4, O.ZERO, dtype=np.uint8)
    assert np.all(O.prox_step_column(np.ones(4), st, 4, 3.0, 2.0) == 0)


def test_g_and_recovery_known_answers(orc_any):
    O = orc_any
    assert O.g_value(np.zeros(4), None, 2, 2.0) == 0.0
    assert abs(O.g_value([2, 1, 0.5, 0.25], None, 2, 2.0) - 3.53125) < 1e-12
    st = np.array([O.ONE, O.FREE, O.FREE], dtype=np.uint8)
    assert abs(O.g_conjugate([3.0, 0.5, 2.0], st, 1, 1.0) - 4.0) < 1e-12
    assert O.g_conjugate(np.zeros(3), None, 2, 1.0) == 0.0
    z, tau, cap = O.recover([2, 1, 0.5, 0.25], None, 2, 2.0)
    assert cap == 1 and abs(tau - 1.75) < 1e-12
    np.testing.assert_allclose(z, [1, 4 / 7, 2 / 7, 1 / 7], atol=1e-12)
    assert O.select_branch([0.1, -3.0, 0.2], None) == 1                      # SPEC.md:325 (1-based 2)


def test_boundary_seeded_pava_equals_generic(orc_any):
    """boundary-seeded PAVA == generic full-scan PAVA."""
    O = orc_any
    rng = np.random.default_rng(3)
    for _ in range(400):
        p = int(rng.integers(2, 40))
        x = rng.normal(size=p) * rng.choice([0.3, 1.0, 4.0])
        st = rng.choice([O.FREE, O.FREE, O.FREE, O.ONE, O.ZERO], size=p).astype(np.uint8)
        kbar = int(rng.integers(0, p + 1))
        w = float(rng.choice([0.2, 1.0, 7.0]))
        M = float(rng.choice([0.5, 2.0]))
        a = O.conjugate_prox_column(x, st, kbar, w, M)
        b = O.conjugate_prox_column(x, st, kbar, w, M, generic=True)
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)


def test_prox_step_feasible_and_optimal(orc_any):
    """SPEC.md:136 feasibility and the variational inequality of SPEC.md:165."""
    O = orc_any
    rng = np.random.default_rng(4)
    for _ in range(60):
        p = int(rng.integers(3, 9))
        u = rng.normal(size=p) * 2
        st = rng.choice([O.FREE, O.FREE, O.ONE, O.ZERO], size=p).astype(np.uint8)
        n1 = int((st == O.ONE).sum())
        kbar = max(0, int(rng.integers(1, p)) - n1)
        eta, lam, M = 0.3, 1.0, 1.5
        rho = 1.0 / (2 * eta * lam)
        b = O.prox_step_column(u, st, kbar, rho, M)
        assert np.all(b[st == O.ZERO] == 0)
        assert np.all(np.abs(b) <= M * (1 + 1e-12))
        assert np.abs(b[st == O.FREE]).sum() / M <= kbar + 1e-9

        def obj(beta):
            g = O.g_value(beta, st, kbar, M)
            return 0.5 * np.sum((beta - u) ** 2) + eta * 2 * lam * g

        f0 = obj(b)
        assert math.isfinite(f0)
        for _ in range(100):
            d = rng.normal(size=p)
            d[st == O.ZERO] = 0
            f1 = obj(b + 1e-4 * d)
            if math.isfinite(f1):
                assert f1 >= f0 - 1e-8


def test_generator_and_auto_batch(orc_any):
    O = orc_any
    inst = O.generate(1000, 100, 5, 0.5, O.SQUARED)
    assert inst.support == [19, 39, 59, 79, 99]                              # problem.hpp:101-107
    inst2 = O.generate(1000, 100, 5, 0.5, O.SQUARED)
    assert np.array_equal(inst.X, inst2.X) and np.array_equal(inst.y, inst2.y)  # reproducible
    lg = O.generate(200, 20, 4, 0.7, O.LOGISTIC)
    assert set(np.unique(lg.y)) <= {-1.0, 1.0}
    assert lg.support == [4, 9, 14, 19]
    # auto batch sizes of SURVEY 8(a) a20 at the 1 GiB default
    B = 1 << 30
    assert O.auto_batch_size(B, 1000, 100, 5, O.SQUARED) == 32768
    assert O.auto_batch_size(B, 2000, 500, 8, O.LOGISTIC) == 8192
    assert O.auto_batch_size(B, 5000, 2000, 10, O.SQUARED) == 4096
    assert O.auto_batch_size(B, 20000, 5000, 15, O.LOGISTIC) == 1024
    assert O.auto_batch_size(B, 2000, 500, 8, O.SQUARED) == 16384
    assert O.auto_batch_size(10, 100, 100, 5, O.SQUARED) == 1                # floor


def test_reopt_normal_equations(orc_any):
    """support = all p, huge M, tiny lambda2 -> least squares."""
    O = orc_any
    rng = np.random.default_rng(5)
    X = rng.normal(size=(40, 3))
    y = X @ np.array([1.0, -2.0, 0.5]) + 0.01 * rng.normal(size=40)
    inst = O.Instance(np.asfortranarray(X), y, O.SQUARED, 3, 100.0, 1e-9)
    coefs, objs = O.reoptimize(inst, [[0, 1, 2], []])
    grad = X.T @ (X @ coefs[0] - y)
    assert np.linalg.norm(grad) <= 1e-4
    assert abs(objs[1] - 0.5 * np.sum(y ** 2)) < 1e-9


def test_solve_zero_response(orc_any):
    """y = 0 -> value 0."""
    O = orc_any
    rng = np.random.default_rng(6)
    inst = O.Instance(np.asfortranarray(rng.normal(size=(20, 6))), np.zeros(20), O.SQUARED, 2,
                      2.0, 1.0)
    cert = O.solve(inst)
    assert cert.optimal_value == 0.0 and cert.status == "optimal"
