"""The tcgen05 (kind::i8, TMEM) emulated-FP64 TN product G = X' R
(csrc/ozaki.cuh; on by default, BNBG_OZAKI=0 disables): 8 signed 8-bit digits per operand with a
power-of-two scale per row / column, exact int32 digit products on the
tensor cores, FP64 recombination.  Checked against numpy fp64 and against the
DMMA kernel: the emulation error bound is ~2^-55 * n * max|x| * max|r| per
element, far inside the 1e-12 relative bar used here."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p", [(3000, 1000), (20000, 600), (1998, 702), (5000, 2000)])
def test_ozaki_tn_matches_fp64(bnb, n, p):
    inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=n, p=p, k=5, correlation=0.5, seed=3))
    rng = np.random.default_rng(n)
    cases = []
    for trans in (True, False):
        for m in (20, 33, 64, 100, 300):
            B = rng.normal(size=(n if trans else p, m)) * rng.choice([1e-3, 1.0, 50.0])
            if m == 100:
                B[:, 7] = 0.0  # an all-zero column (exponent 0, all digits 0)
            cases.append((trans, B))
    out = {}
    for flag in ("1", "0"):
        os.environ["BNBG_OZAKI"] = flag
        try:
            with bnb.Engine(inst) as eng:
                out[flag] = [eng.gemm(B, trans) for trans, B in cases]
        finally:
            del os.environ["BNBG_OZAKI"]
    for (trans, B), oz, dm in zip(cases, out["1"], out["0"]):
        ref = inst.X.T @ B if trans else inst.X @ B
        scale = np.abs(ref).max()
        assert np.abs(oz - ref).max() <= 1e-12 * scale, (trans, B.shape)
        assert np.abs(oz - dm).max() <= 1e-12 * scale
        if B.shape[1] == 100:
            assert np.all(oz[:, 7] == 0.0)
