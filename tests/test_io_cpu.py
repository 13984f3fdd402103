"""Instance and certificate I/O (problem.hpp:166-288, serialize.hpp:22-161)."""
import json
import math

import numpy as np
import pytest

from paper_2605_22188_b200 import io as bio


def test_format_double_matches_to_chars():
    cases = {0.1: "0.1", 100.0: "100", -2.5: "-2.5", 1e-05: "1e-05", 1e22: "1e+22",
             123456789012345680.0: "123456789012345680", 0.0: "0", 5e-324: "5e-324",
             1.7976931348623157e308: "1.7976931348623157e+308", 0.001: "0.001",
             1234.5: "1234.5", 1e16: "1e+16", 12345678.0: "12345678"}
    for v, want in cases.items():
        assert bio.format_double(v) == want, (v, bio.format_double(v), want)
    rng = np.random.default_rng(0)
    for v in rng.normal(size=2000) * 10.0 ** rng.integers(-30, 30, size=2000):
        assert float(bio.format_double(v)) == v  # shortest form round-trips


def test_csv_roundtrip_bit_exact_and_header(bnb, tmp_path):
    inst, _ = bnb.generate_synthetic(bnb.GeneratorSpec(n=40, p=7, k=3, correlation=0.6, loss=1,
                                                       seed=4))
    path = str(tmp_path / "inst.csv")
    bio.save_csv(path, inst.X, inst.y)
    with open(path) as f:
        assert f.readline() == "x1,x2,x3,x4,x5,x6,x7,y\n"
    names = []
    back = bio.load_csv(path, "y", bnb.LossKind.LOGISTIC, k=3, feature_names=names)
    assert names == [f"x{j}" for j in range(1, 8)]
    assert np.array_equal(back.X, inst.X) and np.array_equal(back.y, inst.y)
    # response in the middle, CRLF line ends, spaces around cells
    with open(path, "w") as f:
        f.write("a,resp,b\r\n 1.5 ,1,\t2\r\n-3,-1,4e-3\r\n\r\n")
    got = bio.load_csv(path, "resp", bnb.LossKind.LOGISTIC)
    assert got.X.tolist() == [[1.5, 2.0], [-3.0, 0.004]] and got.y.tolist() == [1.0, -1.0]


@pytest.mark.parametrize("text,err", [("", "empty file"), ("a,b\n", "no data rows"),
                                      ("a,b\n1,2,3\n", "row 2 has 3 cells"),
                                      ("a,b\n1,x\n", "row 2, column 2"),
                                      ("a,b\n1,+2\n", "row 2, column 2"),
                                      ("a,c\n1,2\n", "missing response column"),
                                      ("b\n1\n", "no feature columns")])
def test_csv_parse_errors(tmp_path, text, err):
    path = str(tmp_path / "bad.csv")
    with open(path, "w") as f:
        f.write(text)
    with pytest.raises(bio.ParseError, match=err):
        bio.load_csv(path, "b", 0)


def test_csv_input_errors(bnb, tmp_path):
    path = str(tmp_path / "x.csv")
    with open(path, "w") as f:
        f.write("a,y\n1,0.5\n")
    with pytest.raises(bnb.InputError):  # logistic labels must be +-1
        bio.load_csv(path, "y", bnb.LossKind.LOGISTIC)
    with open(path, "w") as f:
        f.write("a,y\ninf,1\n")
    with pytest.raises(bnb.InputError):  # non-finite values
        bio.load_csv(path, "y", bnb.LossKind.SQUARED)
    with pytest.raises(bnb.InputError):
        bio.load_csv(str(tmp_path / "missing.csv"), "y", 0)


def test_certificate_json_schema(bnb):
    cert = bnb.Certificate(optimal_value=1.25, support=[0, 4], coefficients=np.array([0.5, -1.0]),
                           gap_percent=0.0, lower_bound=1.25, nodes_processed=7, lb_batches=3,
                           reopt_batches=3, batch_size_used=64,
                           profile=bnb.ComponentProfile(0.5, 0.25, 0.0, 0.25, 1.0),
                           status="optimal")
    d = bio.certificate_to_json(cert)
    assert d["support"] == [1, 5] and d["schema_version"] == "1" and "profile" not in d
    assert d["batches"] == {"lower_bound": 3, "reoptimization": 3, "batch_size": 64}
    d2 = bio.certificate_to_json(cert, include_profile=True)
    assert d2["profile"]["lower_bound_percent"] == 50.0
    s = bio.dump_json(d)
    assert json.loads(s) == d and " " not in s and s.index('"batches"') < s.index('"coefficients"')


def test_fnv1a_fingerprint(tmp_path):
    assert bio.fnv1a(b"") == 0xcbf29ce484222325
    assert bio.fnv1a(b"a") == 0xaf63dc4c8601ec8c
    assert bio.fnv1a(b"foobar") == 0x85944171f73967e8
    path = tmp_path / "f.bin"
    path.write_bytes(b"foobar")
    assert bio.file_fingerprint(str(path)) == 0x85944171f73967e8


def test_certificate_json_time_limit_zero(bnb):
    """A time_limit=0 certificate (no incumbent, root unprocessed): nlohmann
    writes the non-finite optimal_value / lower_bound as null."""
    cert = bnb.Certificate(optimal_value=math.inf, support=[], coefficients=np.array([]),
                           gap_percent=100.0, lower_bound=-math.inf, nodes_processed=0,
                           lb_batches=0, reopt_batches=0, batch_size_used=8192,
                           profile=bnb.ComponentProfile(0.0, 0.0, 0.0, 0.0, 0.0),
                           status="time_limit")
    s = bio.dump_json(bio.certificate_to_json(cert))
    d = json.loads(s)
    assert d["optimal_value"] is None and d["lower_bound"] is None
    assert "Infinity" not in s and "NaN" not in s
