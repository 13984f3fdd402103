"""CPU checks of the drop-in boundary: libbnbg.so loads, exports every symbol
declared in include/bnbg.h, and its host-only entry points (generator,
validation, auto batch size) agree with the oracle.  No device calls."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "bnbg.h")).read()
    return sorted(set(re.findall(r"\b(bnbg_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(bnb):
    lib = C.CDLL(bnb.lib_path())
    declared = _declared_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(bnb._L.EXPORTS) == declared


def test_library_is_sm100a(bnb):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", bnb.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("loss", [0, 1])
@pytest.mark.parametrize("n,p,k,rho", [(100, 20, 3, 0.5), (57, 31, 4, 0.0), (40, 12, 3, 0.9)])
def test_generator_bit_identical_to_oracle(bnb, orc, loss, n, p, k, rho):
    inst, sup = bnb.generate_synthetic(bnb.GeneratorSpec(n=n, p=p, k=k, correlation=rho,
                                                         loss=loss, seed=11))
    o = orc.generate(n, p, k, rho, loss, 5.0, 11)
    assert sup == o.support
    assert np.array_equal(inst.X, o.X) and np.array_equal(inst.y, o.y)


def test_auto_batch_size_matches_reference(bnb, orc):
    for args in [(1 << 30, 1000, 100, 5, 0), (1 << 30, 2000, 500, 8, 1), (1 << 30, 5000, 2000, 10, 0),
                 (1 << 30, 20000, 5000, 15, 1), (12345, 50, 50, 3, 1), (1 << 33, 10, 10, 2, 0)]:
        assert bnb.auto_batch_size(*args) == orc.auto_batch_size(*args)
    with pytest.raises(bnb.InputError):
        bnb.auto_batch_size(0, 10, 10, 2, 0)


def test_validate_errors(bnb):
    X = np.ones((4, 3))
    y = np.ones(4)
    bnb.validate(bnb.ProblemInstance(X, y, 0, 2, 1.0, 1.0))
    for bad in [dict(k=0), dict(k=4), dict(M=0.0), dict(lambda2=-1.0)]:
        kw = dict(loss=0, k=2, M=1.0, lambda2=1.0)
        kw.update(bad)
        with pytest.raises(bnb.InputError):
            bnb.validate(bnb.ProblemInstance(X, y, **kw))
    with pytest.raises(bnb.InputError):
        bnb.validate(bnb.ProblemInstance(X, np.array([1.0, 0.0, 1.0, -1.0]), 1, 2, 1.0, 1.0))
    Xn = X.copy()
    Xn[0, 0] = np.nan
    with pytest.raises(bnb.InputError):
        bnb.validate(bnb.ProblemInstance(Xn, y, 0, 2, 1.0, 1.0))
    with pytest.raises(bnb.InputError):
        bnb.generate_synthetic(bnb.GeneratorSpec(n=10, p=5, k=6))
    with pytest.raises(bnb.InputError):
        bnb.generate_synthetic(bnb.GeneratorSpec(n=10, p=5, k=2, correlation=1.0))


def test_product_does_not_import_oracle():
    """The product path must never route through oracle/ (no import, include or link)."""
    pkg = os.path.join(ROOT, "paper_2605_22188_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")) or fn == "Makefile":
                text = open(os.path.join(dirpath, fn)).read()
                assert "import oracle" not in text and "from oracle" not in text
                assert "oracle.h" not in text and "liboracle" not in text


def _build_c_client(tmp_path):
    exe = tmp_path / "solve_c"
    cmd = ["gcc", "-std=c99", "-Wall", "-Werror", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "solve_c.c"), "-L",
           os.path.join(ROOT, "paper_2605_22188_b200"), "-lbnbg",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2605_22188_b200"), "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_header_is_plain_c_and_links(tmp_path):
    """include/bnbg.h compiles as C99 and a C client links against libbnbg.so
    (the C-ABI boundary: no C++ types, no exceptions)."""
    assert _build_c_client(tmp_path).exists()
