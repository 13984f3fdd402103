"""SPEC.md:802-815 acceptance criteria run on the CPU oracle (pins the checker)."""
import json
import math
import os

import numpy as np
import pytest

from tests._enum import all_support_values, node_optimum
from tests.golden.make_golden import fnv1a

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _enum_cases():
    with open(os.path.join(GOLDEN, "enum_optima.json")) as f:
        return json.load(f)


def test_acceptance1_exactness_vs_enumeration(orc_any):
    """#1: 50 seeded instances per loss, value within 1e-6, gap 0."""
    O = orc_any
    for case in _enum_cases():
        inst = O.generate(30, 12, 3, 0.9, case["loss"], 5.0, case["seed"], 2.0, 1.0)
        assert fnv1a(inst.xflat(), inst.y) == case["fingerprint"]
        cert = O.solve(inst)
        assert cert.status == "optimal" and cert.gap_percent == 0.0
        assert abs(cert.optimal_value - case["optimum"]) <= 1e-6 * max(1.0, abs(case["optimum"]))
        assert cert.support == case["support"]


def test_acceptance2_safe_bounds(orc_any):
    """#2: every traced dual bound <= the node's true optimum."""
    O = orc_any
    total = 0
    for loss in (O.SQUARED, O.LOGISTIC):
        for seed in range(4):
            inst = O.generate(30, 12, 3, 0.9, loss, 5.0, seed, 2.0, 1.0)
            vals = all_support_values(inst.X, inst.y, loss, 3, 2.0, 1.0)
            cache = {}
            bad = []

            def hook(j0, j1, psi):
                key = (tuple(sorted(j0)), tuple(sorted(j1)))
                if key not in cache:
                    cache[key] = node_optimum(vals, j0, j1)
                opt = cache[key]
                if psi > opt + 1e-9 * max(1.0, abs(opt)):
                    bad.append((key, psi, opt))

            counter = []
            O.solve(inst, O.solver_cfg(prune_slack=0.0),
                    on_dual_bound=lambda a, b, c: (counter.append(1), hook(a, b, c)))
            total += len(counter)
            assert not bad, bad[:3]
    assert total > 500


def test_acceptance6_rashomon_completeness(orc_any):
    """#6: pool == enumerated epsilon-Rashomon set (size-k supports), and cap N=5."""
    O = orc_any
    eps = 0.1
    for loss in (O.SQUARED, O.LOGISTIC):
        for seed in range(3):
            inst = O.generate(30, 12, 3, 0.9, loss, 5.0, seed, 2.0, 1.0)
            vals = all_support_values(inst.X, inst.y, loss, 3, 2.0, 1.0)
            vstar = min(vals.values())
            tau = (1 + eps) * vstar
            cert, pool = O.collect_rashomon(inst, epsilon=eps)
            assert abs(cert.optimal_value - vstar) <= 1e-6 * max(1, abs(vstar))
            got = {tuple(sorted(s)) for s, _, _ in pool}
            # complete on size-k supports, sound on every size <= k (smaller
            # supports appear only when a node's free set is exhausted)
            want_k = {S for S, v in vals.items() if len(S) == 3 and v <= tau}
            sound = {S for S, v in vals.items() if v <= tau}
            ambiguous = {S for S, v in vals.items() if abs(v - tau) <= 1e-6 * abs(tau)}
            assert want_k - ambiguous <= got
            assert got - ambiguous <= sound
            cert5, pool5 = O.collect_rashomon(inst, epsilon=eps, cap=5)
            best5 = sorted(v for S, v in vals.items() if len(S) == 3 and v <= tau)[:5]
            np.testing.assert_allclose(sorted(o for _, _, o in pool5), best5, rtol=1e-6)


def test_acceptance11_determinism_across_workers(orc_any):
    O = orc_any
    inst = O.generate(200, 40, 4, 0.8, O.LOGISTIC, 5.0, 7, 2.0, 1.0)
    a = O.solve(inst, O.solver_cfg(workers=1))
    b = O.solve(inst, O.solver_cfg(workers=4))
    assert a.optimal_value == b.optimal_value and a.support == b.support
    assert a.coefficients == b.coefficients and a.nodes_processed == b.nodes_processed
