"""The reference itself, compiled here (oracle/_ref): CPU checks.

oracle/ref/ builds the unmodified bnbglm headers (/root/reference/proj/include)
through an Eigen-subset shim into oracle/_ref/libbnbref.so, exporting
oracle.h's C API, and compiles the reference-side adapter
(include/bnbglm_b200.hpp) against the same headers.  These tests pin
oracle/oracle.c (the restatement every other test uses as its checker) to the
reference's own outputs: certificates, node counts and enumeration optima.
The SPEC known-answer and acceptance tests (test_oracle_*.py) also run on both
backends through the `orc_any` fixture.
"""
import ctypes
import json
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def ref(orc):
    if not orc.ref_available():
        pytest.fail("oracle/_ref/libbnbref.so missing: build() compiles it where "
                    "/root/reference exists")
    return orc


def test_ref_exports_the_oracle_api(ref):
    """libbnbref.so answers every orc_* entry point oracle.py binds."""
    hdr = open(os.path.join(ROOT, "oracle", "oracle.h")).read()
    names = set(re.findall(r"\b(orc_[a-z0-9_]+)\s*\(", hdr))
    py = open(os.path.join(ROOT, "oracle", "oracle.py")).read()
    bound = {n for n in names if f"L.{n}." in py}
    lib = ctypes.CDLL(ref.REF_LIB_PATH)
    missing = [n for n in sorted(bound) if not hasattr(lib, n)]
    assert not missing, missing


def test_reference_generator_agrees_to_rounding(ref):
    """problem.hpp:70-132 run by the reference (LLT through the shim) vs the
    closed-form AR(1) factor of oracle.c / the product: same support, X and y
    equal to a few ulps (the instance bytes every leg uses are oracle.c's)."""
    for n, p, k, rho, loss in [(30, 12, 3, 0.9, 0), (1000, 100, 5, 0.5, 0), (400, 60, 4, 0.7, 1)]:
        a = ref.generate(n, p, k, rho, loss)
        b = ref.generate(n, p, k, rho, loss, reference_generator=True)
        assert list(a.support) == list(b.support)
        assert np.abs(a.X - b.X).max() <= 1e-13
        if loss == 0:
            assert np.abs(a.y - b.y).max() <= 1e-12
        else:
            assert (a.y == b.y).mean() > 0.99  # labels may flip only at sigma == u ties


def _certs(ref, inst, **cfg):
    out = {}
    for be in ("c", "ref"):
        with ref.backend(be):
            out[be] = ref.solve(inst, ref.solver_cfg(**cfg))
    return out["c"], out["ref"]


def test_oracle_equals_reference_c1(ref):
    """BASELINE c1 (squared n=1000 p=100 k=5 rho=0.5): certificate, node and
    pass counts identical; objective within 1e-12."""
    inst = ref.generate(1000, 100, 5, 0.5, 0, 5.0, 0, 2.0, 1.0)
    c, r = _certs(ref, inst)
    assert r.status == c.status == "optimal"
    assert r.support == c.support == [19, 39, 59, 79, 99]
    assert r.nodes_processed == c.nodes_processed and r.lb_batches == c.lb_batches
    assert abs(r.optimal_value - c.optimal_value) <= 1e-12 * abs(r.optimal_value)
    np.testing.assert_allclose(r.coefficients, c.coefficients, rtol=1e-10, atol=1e-12)


def test_oracle_equals_reference_dual_trace(ref):
    """The whole dual-bound trace of a many-pass solve (DebugHooks,
    bnb_engine.hpp:183-187): same nodes in the same order, psi within 1e-9."""
    for loss in (0, 1):
        inst = ref.generate(200, 40, 4, 0.8, loss, 5.0, 7, 2.0, 1.0)
        tr = {}
        for be in ("c", "ref"):
            ev = []
            with ref.backend(be):
                ref.solve(inst, ref.solver_cfg(batch_size=16),
                          on_dual_bound=lambda j0, j1, v: ev.append((tuple(j0), tuple(j1), v)),
                          on_batch_boundary=lambda lb, ub: ev.append(("b", lb, ub)))
            tr[be] = ev
        assert [e[:2] if e[0] != "b" else "b" for e in tr["c"]] == \
               [e[:2] if e[0] != "b" else "b" for e in tr["ref"]]
        np.testing.assert_allclose([e[2] for e in tr["c"]], [e[2] for e in tr["ref"]],
                                   rtol=1e-9, atol=1e-9)


def test_oracle_equals_reference_enumeration_instances(ref):
    """The 100 SPEC acceptance #1 instances (n=30 p=12 k=3 rho=0.9, 50 seeds x
    2 losses): both backends certify the enumerated optimum with the same
    support and node count."""
    with open(os.path.join(GOLDEN, "enum_optima.json")) as f:
        cases = json.load(f)
    assert len(cases) == 100
    for case in cases:
        inst = ref.generate(30, 12, 3, 0.9, case["loss"], 5.0, case["seed"], 2.0, 1.0)
        c, r = _certs(ref, inst)
        assert r.support == c.support == case["support"], case["seed"]
        assert r.nodes_processed == c.nodes_processed
        assert abs(r.optimal_value - c.optimal_value) <= 1e-12 * max(1.0, abs(c.optimal_value))


def test_oracle_equals_reference_rashomon(ref):
    """collect_rashomon (rashomon.hpp:149-218): same pool, same order."""
    inst = ref.generate(60, 16, 3, 0.8, 0, 5.0, 3, 2.0, 1.0)
    pools = {}
    for be in ("c", "ref"):
        with ref.backend(be):
            pools[be] = ref.collect_rashomon(inst, epsilon=0.2)
    (cc, cp), (rc, rp) = pools["c"], pools["ref"]
    assert [s for s, _, _ in cp] == [s for s, _, _ in rp] and len(cp) > 3
    np.testing.assert_allclose([o for _, _, o in cp], [o for _, _, o in rp], rtol=1e-12)
    assert cc.nodes_processed == rc.nodes_processed


def test_oracle_equals_reference_prox_columns(ref):
    """prox_step_column / g / g* on seeded random columns (prox_kernel.hpp):
    the restatement is bit-identical to the reference."""
    rng = np.random.default_rng(5)
    for _ in range(200):
        p = int(rng.integers(1, 80))
        st = rng.choice([0, 0, 0, 1, 2], size=p).astype(np.uint8)
        kbar = int(rng.integers(0, p + 1))
        u = rng.normal(size=p) * rng.choice([0.1, 1.0, 5.0])
        rho, M = float(rng.uniform(0.5, 50)), float(rng.uniform(0.5, 3))
        vals = {}
        for be in ("c", "ref"):
            with ref.backend(be):
                vals[be] = (ref.prox_step_column(u, st, kbar, rho, M),
                            ref.g_value(u, st, kbar, M), ref.g_conjugate(u, st, kbar, M))
        np.testing.assert_array_equal(vals["c"][0], vals["ref"][0])
        assert vals["c"][1] == vals["ref"][1] or (np.isinf(vals["c"][1]) and np.isinf(vals["ref"][1]))
        assert abs(vals["c"][2] - vals["ref"][2]) <= 1e-12 * max(1.0, abs(vals["c"][2]))


def test_adapter_compiles_against_reference_headers(ref):
    """include/bnbglm_b200.hpp (the reference-side adapter)
    compiled with the unmodified reference headers and linked with libbnbg.so;
    on CPU it must map errors to the reference's exception types."""
    exe = os.path.join(ROOT, "oracle", "_ref", "adapter_check")
    assert os.path.exists(exe), "build() compiles oracle/_ref/adapter_check"
    r = subprocess.run([exe, "errors"], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0 and "errors ok" in r.stdout, r.stdout + r.stderr
