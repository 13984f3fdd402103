"""The reference-side adapter on the B200 (include/bnbglm_b200.hpp).

oracle/_ref/adapter_check is the adapter compiled against the UNMODIFIED
reference headers (build() does this where /root/reference exists; the
binary travels with the snapshot).  In `solve` mode it runs the reference's
own bnbglm::solve on the CPU and bnbglm::b200::solve on the GPU on the same
generate_synthetic instance, plus solve_batch_relaxation on the root node
through both, and exits 0 only if supports match and values/bounds agree
within 1e-6 (north_star's bar).
"""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "adapter_check")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,p,k,rho,loss", [(200, 40, 4, 0.8, 0), (200, 40, 4, 0.8, 1),
                                            (1000, 100, 5, 0.5, 0)])
def test_adapter_solve_equals_reference(n, p, k, rho, loss):
    assert os.path.exists(EXE), "oracle/_ref/adapter_check not built"
    r = subprocess.run([EXE, "solve", str(n), str(p), str(k), str(rho), str(loss)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["support_equal"] and out["value_rel"] <= 1e-6
    assert out["root_bound_rel"] <= 1e-6 and out["root_status_equal"]
    assert out["root_iters"][0] == out["root_iters"][1]
    assert out["ref_nodes"] == out["dev_nodes"]
