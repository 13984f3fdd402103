"""The 128 x 64 register-tiled DMMA GEMM (gemm_big.cuh) with TMA-staged X
tiles and split-K for the TN product, against numpy fp64 and against the
same kernel with cp.async staging (BNBG_TMA=0): staging must not change a
single bit (the arithmetic is identical), and split-K slabs summed in order
must agree with the unsplit product to rounding."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p", [(3000, 1000), (5000, 2000), (20000, 600), (1998, 702)])
def test_big_gemm_tma_and_split_k(bnb, n, p):
    inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=n, p=p, k=5, correlation=0.5, seed=2))
    rng = np.random.default_rng(n + p)
    cases = []
    for m in (64, 100, 300):
        for trans in (False, True):
            B = rng.normal(size=(n if trans else p, m))
            cases.append((m, trans, B))
    outs = {}
    os.environ["BNBG_OZAKI"] = "0"  # the DMMA kernels (the emulated path: test_gpu_ozaki.py)
    try:
        for tma in ("1", "0"):
            os.environ["BNBG_TMA"] = tma
            with bnb.Engine(inst) as eng:
                outs[tma] = [eng.gemm(B, trans) for _, trans, B in cases]
    finally:
        os.environ.pop("BNBG_TMA", None)
        os.environ.pop("BNBG_OZAKI", None)
    for (m, trans, B), a, b in zip(cases, outs["1"], outs["0"]):
        ref = inst.X.T @ B if trans else inst.X @ B
        assert np.abs(a - ref).max() <= 1e-12 * np.abs(ref).max(), (m, trans)
        np.testing.assert_array_equal(a, b)
