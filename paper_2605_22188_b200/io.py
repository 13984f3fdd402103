"""Instance and certificate I/O of the reference: CSV
instances (problem.hpp:166-288), certificate JSON (serialize.hpp:22-64) and
the FNV-1a input fingerprint (serialize.hpp:149-161).  Host-side, off the
node-processing path; kept so a user's files and reports stay byte-compatible.
"""
from __future__ import annotations

import json
import math
from typing import List, Optional

import numpy as np

SCHEMA_VERSION = "1"  # serialize.hpp:22


class ParseError(RuntimeError):
    """errors.hpp parse_error: malformed input file; names the row/column."""


def format_double(v: float) -> str:
    """std::to_chars(double) shortest round-trip form (problem.hpp:200-204):
    the shorter of fixed and scientific notation, fixed on a tie."""
    v = float(v)
    if math.isnan(v) or math.isinf(v):
        return repr(v)
    r = repr(v)  # shortest round-trip digits
    mant, _, exp = r.partition("e")
    digits = mant.replace("-", "").replace(".", "").lstrip("0") or "0"
    e10 = (int(exp) if exp else 0)
    # decimal exponent of the leading digit
    if "." in mant:
        ip, fp = mant.replace("-", "").split(".")
    else:
        ip, fp = mant.replace("-", ""), ""
    if ip.strip("0"):
        lead = len(ip.lstrip("0")) - 1 + e10
    else:
        lead = -(len(fp) - len(fp.lstrip("0")) + 1) + e10
    digits = digits.rstrip("0") or "0"
    sign = "-" if v < 0 or (v == 0 and math.copysign(1.0, v) < 0) else ""
    nd = len(digits)
    # scientific: d[.ddd]e[+-]XX (at least two exponent digits)
    sci = digits[0] + ("." + digits[1:] if nd > 1 else "") + "e" + ("-" if lead < 0 else "+") + \
        f"{abs(lead):02d}"
    # fixed
    if lead >= 0:
        if nd <= lead + 1:
            fix = digits + "0" * (lead + 1 - nd)
        else:
            fix = digits[:lead + 1] + "." + digits[lead + 1:]
    else:
        fix = "0." + "0" * (-lead - 1) + digits
    if digits == "0":
        fix, sci = "0", "0e+00"
    return sign + (fix if len(fix) <= len(sci) else sci)


def _split_csv_line(line: str) -> List[str]:
    """problem.hpp:174-181: plain comma split; a trailing comma adds an empty cell."""
    if line == "":
        return []
    return line.split(",")


def _parse_cell(cell: str, row: int, col: int) -> float:
    """problem.hpp:183-197: trims spaces/tabs (and a trailing CR), then parses
    the whole cell as a double."""
    s = cell.strip(" \t").rstrip(" \t\r")
    try:
        # std::from_chars: no leading '+', no digit separators; inf/nan are
        # numbers (load_csv rejects them afterwards as non-finite)
        if s == "" or s.startswith("+") or "_" in s or s != s.strip():
            raise ValueError
        return float(s)
    except ValueError:
        raise ParseError(f"csv: non-numeric cell at row {row}, column {col}") from None


def load_csv(path: str, response_column: str, loss: int, k: int = 1, M: float = 1.0,
             lambda2: float = 1.0, feature_names: Optional[list] = None):
    """problem.hpp:208-260 load_csv: the named response column becomes y, the
    remaining columns the features in header order; constraint parameters are
    supplied separately."""
    from . import InputError, LossKind, ProblemInstance
    try:
        f = open(path, "r", newline="")
    except OSError:
        raise InputError(f"csv: cannot open {path}") from None
    with f:
        lines = f.read().split("\n")
    if not lines or (len(lines) == 1 and lines[0] == ""):
        raise ParseError(f"csv: empty file {path}")
    header = _split_csv_line(lines[0].rstrip("\r"))
    try:
        ri = header.index(response_column)
    except ValueError:
        raise ParseError(f"csv: missing response column '{response_column}'") from None
    rows = []
    for number, line in enumerate(lines[1:], start=2):
        line = line.rstrip("\r")
        if line == "":
            continue
        cells = _split_csv_line(line)
        if len(cells) != len(header):
            raise ParseError(f"csv: row {number} has {len(cells)} cells, expected {len(header)}")
        rows.append([_parse_cell(c, number, j + 1) for j, c in enumerate(cells)])
    if not rows:
        raise ParseError(f"csv: no data rows in {path}")
    A = np.array(rows, dtype=np.float64)
    if A.shape[1] - 1 < 1:
        raise ParseError(f"csv: no feature columns in {path}")
    keep = [j for j in range(A.shape[1]) if j != ri]
    if feature_names is not None:
        feature_names[:] = [header[j] for j in keep]
    X, y = A[:, keep], A[:, ri]
    if loss == LossKind.LOGISTIC and not np.all((y == 1.0) | (y == -1.0)):
        raise InputError("logistic label must be -1 or +1")
    if not (np.all(np.isfinite(X)) and np.all(np.isfinite(y))):
        raise InputError(f"csv: non-finite values in {path}")
    return ProblemInstance(X, y, loss, k, M, lambda2)


def save_csv(path: str, X: np.ndarray, y: np.ndarray, response_column: str = "y") -> None:
    """problem.hpp:265-286 save_csv: x1..xp then the response; shortest
    round-trip doubles, so save/load is bit-exact."""
    from . import InputError
    X = np.asarray(X, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    n, p = X.shape
    parts = [",".join(f"x{j + 1}" for j in range(p)) + "," + response_column + "\n"]
    for i in range(n):
        parts.append("".join(format_double(X[i, j]) + "," for j in range(p)) +
                     format_double(y[i]) + "\n")
    try:
        with open(path, "w", newline="") as f:
            f.write("".join(parts))
    except OSError:
        raise InputError(f"csv: cannot write {path}") from None


def profile_to_json(profile) -> dict:
    """serialize.hpp:24-37."""
    total = profile.total_seconds

    def pct(v):
        return 100.0 * v / total if total > 0.0 else 0.0
    return {
        "lower_bound_seconds": profile.lower_bound_seconds,
        "reoptimization_seconds": profile.reoptimization_seconds,
        "transfer_seconds": profile.transfer_seconds,
        "branch_generate_seconds": profile.branch_generate_seconds,
        "total_seconds": total,
        "lower_bound_percent": pct(profile.lower_bound_seconds),
        "reoptimization_percent": pct(profile.reoptimization_seconds),
        "transfer_percent": pct(profile.transfer_seconds),
        "branch_generate_percent": pct(profile.branch_generate_seconds),
    }


def certificate_to_json(cert, include_profile: bool = False) -> dict:
    """serialize.hpp:40-64: 1-based support, keys as in the reference."""
    out = {
        "schema_version": SCHEMA_VERSION,
        "optimal_value": cert.optimal_value,
        "support": [j + 1 for j in cert.support],
        "coefficients": [float(c) for c in cert.coefficients],
        "gap_percent": cert.gap_percent,
        "lower_bound": cert.lower_bound,
        "nodes": cert.nodes_processed,
        "batches": {"lower_bound": cert.lb_batches, "reoptimization": cert.reopt_batches,
                    "batch_size": cert.batch_size_used},
        "status": cert.status,
    }
    if include_profile:
        out["profile"] = profile_to_json(cert.profile)
    return out


def _finite_or_null(obj):
    """nlohmann::json writes non-finite doubles as null (e.g. optimal_value of
    a time-limited run with no incumbent, lower_bound of an unprocessed root)."""
    if isinstance(obj, float):
        return obj if math.isfinite(obj) else None
    if isinstance(obj, dict):
        return {k: _finite_or_null(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_finite_or_null(v) for v in obj]
    return obj


def dump_json(obj) -> str:
    """nlohmann::json::dump() layout: keys sorted, no whitespace, non-finite
    numbers as null (allow_nan=False catches any that slip through)."""
    return json.dumps(_finite_or_null(obj), sort_keys=True, separators=(",", ":"),
                      allow_nan=False)


def fnv1a(data: bytes) -> int:
    """64-bit FNV-1a (serialize.hpp:149-161)."""
    h = 0xcbf29ce484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def file_fingerprint(path: str) -> int:
    """serialize.hpp:149-161: FNV-1a over the raw bytes of a file."""
    from . import InputError
    try:
        with open(path, "rb") as f:
            return fnv1a(f.read())
    except OSError:
        raise InputError(f"cannot read {path}") from None
