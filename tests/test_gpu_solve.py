"""End-to-end certified solves on the device vs the golden fixtures and the
oracle (SPEC.md:802-815 acceptance criteria #1, #2, #6, #11).

Bar (BASELINE.json north_star): the same certified support bit-exactly, the
optimal objective and every lower bound within 1e-6 relative.
"""
import json
import math
import os

import numpy as np
import pytest

from tests._enum import all_support_values, node_optimum

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
REL = 1e-6


def _load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def _inst(bnb, n, p, k, rho, loss, seed=0):
    inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=n, p=p, k=k, correlation=rho, loss=loss,
                                                       seed=seed))
    return inst


def test_acceptance1_exactness_on_device(bnb):
    """#1: 50 seeded enumerable instances per loss; value within 1e-6, gap 0,
    support equal to the enumeration argmin."""
    from tests.golden.make_golden import fnv1a
    for case in _load("enum_optima.json"):
        inst = _inst(bnb, 30, 12, 3, 0.9, case["loss"], case["seed"])
        assert fnv1a(inst.xflat(), inst.y) == case["fingerprint"]
        inst.M, inst.lambda2 = 2.0, 1.0
        cert = bnb.solve(inst)
        assert cert.status == "optimal" and cert.gap_percent == 0.0
        assert abs(cert.optimal_value - case["optimum"]) <= REL * max(1.0, abs(case["optimum"]))
        assert cert.support == case["support"], (case, cert)


@pytest.mark.parametrize("name,spec", [("c1", (1000, 100, 5, 0.5, 0)),
                                       ("c2", (2000, 500, 8, 0.7, 1))])
def test_config_certificates_match_oracle(bnb, name, spec):
    """c1/c2 certificates vs the oracle's (tests/golden/certificates.json)."""
    from tests.golden.make_golden import fnv1a
    ref = _load("certificates.json")[name]
    inst = _inst(bnb, *spec)
    assert fnv1a(inst.xflat(), inst.y) == ref["fingerprint"]
    cert = bnb.solve(inst)
    assert cert.status == "optimal"
    assert cert.support == ref["support"]
    assert abs(cert.optimal_value - ref["optimal_value"]) <= REL * abs(ref["optimal_value"])
    np.testing.assert_allclose(cert.coefficients, ref["coefficients"], rtol=1e-6, atol=1e-7)
    assert cert.nodes_processed == ref["nodes"]


def test_certificates_match_oracle_small(bnb, orc):
    for key, ref in _load("certificates.json").items():
        if not key.startswith("enum_"):
            continue
        _, loss, seed = key.split("_")
        inst = _inst(bnb, 30, 12, 3, 0.9, int(loss), int(seed))
        cert = bnb.solve(inst)
        assert cert.support == ref["support"]
        assert abs(cert.optimal_value - ref["optimal_value"]) <= REL * max(1, abs(ref["optimal_value"]))
        assert cert.nodes_processed == ref["nodes"]


def test_acceptance2_safe_bounds_on_device(bnb):
    """#2: every dual bound traced on the device <= the node's true optimum."""
    total = 0
    for loss in (0, 1):
        for seed in range(10):
            inst = _inst(bnb, 30, 12, 3, 0.9, loss, seed)
            inst.M, inst.lambda2 = 2.0, 1.0
            vals = all_support_values(inst.X, inst.y, loss, 3, 2.0, 1.0)
            cache, bad, count = {}, [], [0]

            def on_dual(node, psi):
                count[0] += 1
                key = (tuple(sorted(node.fixed_zero)), tuple(sorted(node.fixed_one)))
                if key not in cache:
                    cache[key] = node_optimum(vals, node.fixed_zero, node.fixed_one)
                if psi > cache[key] + 1e-9 * max(1.0, abs(cache[key])):
                    bad.append((key, psi, cache[key]))

            bnb.solve(inst, bnb.SolverConfig(prune_slack=0.0), bnb.DebugHooks(on_dual_bound=on_dual))
            total += count[0]
            assert not bad, bad[:3]
    assert total > 1000


def test_dual_trace_matches_oracle(bnb, orc):
    """Every lower bound within 1e-6: the device's traced bound sequence equals
    the oracle's, node by node, on a solve with many passes."""
    for loss in (0, 1):
        inst = _inst(bnb, 200, 40, 4, 0.8, loss, 7)
        oi = orc.generate(200, 40, 4, 0.8, loss, 5.0, 7)
        dev, ref = [], []
        bnb.solve(inst, bnb.SolverConfig(batch_size=16),
                  bnb.DebugHooks(on_dual_bound=lambda nd, v: dev.append(
                      (tuple(nd.fixed_zero), tuple(nd.fixed_one), v))))
        orc.solve(oi, orc.solver_cfg(batch_size=16),
                  on_dual_bound=lambda j0, j1, v: ref.append((tuple(j0), tuple(j1), v)))
        assert [d[:2] for d in dev] == [r[:2] for r in ref]
        np.testing.assert_allclose([d[2] for d in dev], [r[2] for r in ref], rtol=REL, atol=REL)


def test_acceptance6_rashomon_matches_oracle(bnb, orc):
    """#6 on the device: pool equals the oracle pool set-for-set (objectives 1e-6)."""
    for loss in (0, 1):
        for seed in range(3):
            inst = _inst(bnb, 30, 12, 3, 0.9, loss, seed)
            inst.M, inst.lambda2 = 2.0, 1.0
            oi = orc.generate(30, 12, 3, 0.9, loss, 5.0, seed)
            for cap in (-1, 5):
                res = bnb.collect_rashomon(inst, rconfig=bnb.RashomonConfig(epsilon=0.1, cap=cap))
                ocert, opool = orc.collect_rashomon(oi, epsilon=0.1, cap=cap)
                assert [s for s, _, _ in res.pool] == [s for s, _, _ in opool]
                np.testing.assert_allclose([o for _, _, o in res.pool],
                                           [o for _, _, o in opool], rtol=REL)
                assert res.certificate.support == ocert.support


def test_acceptance11_determinism(bnb):
    inst = _inst(bnb, 300, 60, 5, 0.8, 1, 3)
    a = bnb.solve(inst)
    b = bnb.solve(inst)
    assert a.optimal_value == b.optimal_value and a.support == b.support
    assert np.array_equal(a.coefficients, b.coefficients)
    assert a.nodes_processed == b.nodes_processed and a.lb_batches == b.lb_batches


def test_zero_response_and_time_limit(bnb):
    rng = np.random.default_rng(6)
    inst = bnb.ProblemInstance(rng.normal(size=(20, 6)), np.zeros(20), 0, 2, 2.0, 1.0)
    cert = bnb.solve(inst)
    assert cert.optimal_value == 0.0 and cert.status == "optimal"
    big = _inst(bnb, 300, 80, 8, 0.9, 0, 1)
    c = bnb.solve(big, bnb.SolverConfig(time_limit=0.0))
    assert c.status == "time_limit" and c.gap_percent == 100.0


def test_c_client_certifies_like_python(bnb, tmp_path):
    """The plain-C client (examples/solve_c.c) through the C-ABI gives the same
    certificate as the Python mirror."""
    import json
    import subprocess
    from tests.test_boundary_cpu import _build_c_client
    exe = _build_c_client(tmp_path)
    out = subprocess.run([str(exe), "300", "60", "5", "0.8", "1", "3"], capture_output=True,
                         text=True, check=True).stdout
    got = json.loads(out.strip().splitlines()[-1])
    inst = _inst(bnb, 300, 60, 5, 0.8, 1, 3)
    ref = bnb.solve(inst)
    assert got["support"] == ref.support and got["status"] == 0
    assert got["optimal_value"] == ref.optimal_value and got["nodes"] == ref.nodes_processed


def test_config_c5_rashomon_matches_oracle(bnb):
    """BASELINE c5 (Rashomon set, epsilon 0.01, squared n=2000 p=500 k=8) vs the
    oracle's pool (tests/golden/rashomon_c5.json, make_golden_c5.py)."""
    ref = _load("rashomon_c5.json")
    inst = _inst(bnb, 2000, 500, 8, 0.7, 0, 0)
    res = bnb.collect_rashomon(inst, rconfig=bnb.RashomonConfig(epsilon=ref["epsilon"]))
    cert = res.certificate
    assert cert.support == ref["support"]
    assert abs(cert.optimal_value - ref["optimal_value"]) <= REL * abs(ref["optimal_value"])
    assert cert.nodes_processed == ref["nodes"]
    assert [s for s, _, _ in res.pool] == [m["sequence"] for m in ref["pool"]]
    np.testing.assert_allclose([o for _, _, o in res.pool], [m["objective"] for m in ref["pool"]],
                               rtol=REL)


@pytest.mark.parametrize("n,p,k,rho", [(7, 3, 1, 0.3), (33, 17, 17, 0.5), (50, 1, 1, 0.0),
                                       (101, 33, 5, 0.9), (15, 9, 4, 0.7)])
@pytest.mark.parametrize("loss", [0, 1])
def test_edge_shapes_match_oracle(bnb, orc, n, p, k, rho, loss):
    """Odd n and p (unaligned rows, padded tiles), k = p, p = 1, n < 16."""
    inst = _inst(bnb, n, p, k, rho, loss, seed=n + p)
    oi = orc.generate(n, p, k, rho, loss, 5.0, n + p)
    cert = bnb.solve(inst)
    ref = orc.solve(oi)
    assert cert.status == "optimal" and cert.support == ref.support
    assert abs(cert.optimal_value - ref.optimal_value) <= REL * max(1.0, abs(ref.optimal_value))
    assert cert.nodes_processed == ref.nodes_processed
