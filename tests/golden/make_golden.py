"""Generates the committed golden fixtures under tests/golden/ (run on CPU).

  enum_optima.json   SPEC.md:805 acceptance #1 instances (n=30, p=12, k=3,
                     rho=0.9, M=2, lambda2=1, seeds 0..49, both losses): the
                     enumeration-oracle optimum v* and argmin support, plus the
                     FNV-1a fingerprint of the generated X, y bytes
                     (serialize.hpp:149-161 convention).
  certificates.json  oracle certificates (value, support, coefficients, nodes)
                     for c1 and the enumerable instances of seeds 0..9.
  prox_vectors.json  oracle prox_step / g / g* outputs on seeded random columns.

Usage: python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import oracle as O  # noqa: E402
from _enum import all_support_values  # noqa: E402


def fnv1a(*arrays):
    h = 0xcbf29ce484222325
    for a in arrays:
        for byte in np.ascontiguousarray(a).tobytes():
            h ^= byte
            h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def enum_instance(seed, loss):
    return O.generate(30, 12, 3, 0.9, loss, 5.0, seed, 2.0, 1.0)


def main():
    O.build()
    enum = []
    for loss in (O.SQUARED, O.LOGISTIC):
        for seed in range(50):
            inst = enum_instance(seed, loss)
            vals = all_support_values(inst.X, inst.y, loss, 3, 2.0, 1.0)
            best = min(vals, key=vals.get)
            enum.append(dict(loss=loss, seed=seed, fingerprint=fnv1a(inst.xflat(), inst.y),
                             optimum=vals[best], support=list(best)))
            print(loss, seed, vals[best], best, flush=True)
    with open(os.path.join(HERE, "enum_optima.json"), "w") as f:
        json.dump(enum, f, indent=1)

    certs = {}
    c1 = O.generate(1000, 100, 5, 0.5, O.SQUARED)
    c = O.solve(c1)
    certs["c1"] = dict(fingerprint=fnv1a(c1.xflat(), c1.y), optimal_value=c.optimal_value,
                       support=c.support, coefficients=c.coefficients,
                       nodes=c.nodes_processed, lb_batches=c.lb_batches)
    O.use_openblas(0)
    c2 = O.generate(2000, 500, 8, 0.7, O.LOGISTIC)
    c = O.solve(c2, O.solver_cfg(workers=os.cpu_count()))
    certs["c2"] = dict(fingerprint=fnv1a(c2.xflat(), c2.y), optimal_value=c.optimal_value,
                       support=c.support, coefficients=c.coefficients,
                       nodes=c.nodes_processed, lb_batches=c.lb_batches)
    for loss in (O.SQUARED, O.LOGISTIC):
        for seed in range(10):
            inst = enum_instance(seed, loss)
            c = O.solve(inst)
            certs[f"enum_{loss}_{seed}"] = dict(
                fingerprint=fnv1a(inst.xflat(), inst.y), optimal_value=c.optimal_value,
                support=c.support, coefficients=c.coefficients, nodes=c.nodes_processed)
    with open(os.path.join(HERE, "certificates.json"), "w") as f:
        json.dump(certs, f, indent=1)

    rng = np.random.default_rng(20261017)
    vecs = []
    for p, kb_max in [(6, 3), (17, 5), (64, 8), (100, 5)]:
        for _ in range(6):
            u = (rng.normal(size=p) * rng.choice([0.2, 1.0, 5.0])).tolist()
            st = rng.choice([0, 0, 0, 1, 2], size=p).astype(np.uint8)
            kbar = int(rng.integers(0, kb_max + 1))
            rho, M = float(rng.choice([0.5, 3.0, 40.0])), float(rng.choice([1.0, 2.0]))
            out = O.prox_step_column(np.array(u), st, kbar, rho, M)
            vecs.append(dict(u=u, state=st.tolist(), kbar=kbar, rho=rho, M=M, prox=out.tolist(),
                             g=O.g_value(out, st, kbar, M),
                             gconj=O.g_conjugate(np.array(u), st, kbar, M)))
    with open(os.path.join(HERE, "prox_vectors.json"), "w") as f:
        json.dump(vecs, f, indent=1)


if __name__ == "__main__":
    main()
