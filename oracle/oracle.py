"""ctypes wrapper over oracle/_build/liboracle.so -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU reference.  The product (paper_2605_22188_b200) never imports
it.  See oracle.h for the reference file:line each entry point restates.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
# The reference itself (its headers compiled through the Eigen-subset shim,
# oracle/ref/), exporting the same orc_* C API: backend "ref".
REF_LIB_PATH = os.path.join(_HERE, "_ref", "libbnbref.so")
_libs = {}
_backend = "c"

SQUARED, LOGISTIC = 0, 1
FREE, ONE, ZERO = 0, 1, 2
PRUNABLE, CONVERGED, CAPPED = 0, 1, 2


def build() -> str:
    """Compile the oracle (gcc, seconds) and, where /root/reference exists,
    the reference itself into oracle/_ref (g++, ~15 s)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    subprocess.run(["make", "-s", "-C", os.path.join(_HERE, "ref")], check=True)
    return _LIB_PATH


def ref_available() -> bool:
    """True when oracle/_ref/libbnbref.so (the compiled reference) exists."""
    return os.path.exists(REF_LIB_PATH)


def set_backend(name: str) -> str:
    """Select which library answers every call: "c" (oracle.c, the
    restatement) or "ref" (the reference headers compiled via the shim).
    Returns the previous backend."""
    global _backend
    if name not in ("c", "ref"):
        raise ValueError(name)
    if name == "ref" and not ref_available():
        raise FileNotFoundError(REF_LIB_PATH)
    prev, _backend = _backend, name
    return prev


class backend:
    """Context manager: ``with backend("ref"): ...``"""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        self.prev = set_backend(self.name)
        return self

    def __exit__(self, *exc):
        set_backend(self.prev)


class RelaxCfg(C.Structure):
    _fields_ = [("max_iterations", C.c_int), ("gap_tolerance", C.c_double),
                ("check_interval", C.c_int), ("acceleration", C.c_int),
                ("smoothness", C.c_double), ("workers", C.c_int)]


class SolverCfg(C.Structure):
    _fields_ = [("batch_size", C.c_int), ("memory_budget", C.c_uint64),
                ("time_limit", C.c_double), ("prune_slack", C.c_double),
                ("relax", RelaxCfg), ("workers", C.c_int)]


class _Cert(C.Structure):
    _fields_ = [("optimal_value", C.c_double), ("support_len", C.c_int),
                ("support", C.POINTER(C.c_int)), ("coefficients", C.POINTER(C.c_double)),
                ("gap_percent", C.c_double), ("lower_bound", C.c_double),
                ("nodes_processed", C.c_longlong), ("lb_batches", C.c_longlong),
                ("reopt_batches", C.c_longlong), ("batch_size_used", C.c_int),
                ("prof_lower_bound", C.c_double), ("prof_reoptimization", C.c_double),
                ("prof_transfer", C.c_double), ("prof_branch_generate", C.c_double),
                ("prof_total", C.c_double), ("status", C.c_int), ("err_column", C.c_int)]


TRACE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.c_double)
DUAL_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.POINTER(C.c_int), C.c_int,
                        C.POINTER(C.c_int), C.c_double)
BOUNDARY_HOOK = C.CFUNCTYPE(None, C.c_void_p, C.c_double, C.c_double)

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_up = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


def lib():
    if _backend not in _libs:
        path = _LIB_PATH if _backend == "c" else REF_LIB_PATH
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        d, i, u64, vp = C.c_double, C.c_int, C.c_uint64, C.c_void_p
        L.orc_loss_value.restype = d
        L.orc_loss_value.argtypes = [i, d, d]
        L.orc_loss_derivative.restype = d
        L.orc_loss_derivative.argtypes = [i, d, d]
        L.orc_loss_conjugate.restype = d
        L.orc_loss_conjugate.argtypes = [i, d, d]
        L.orc_smoothness.restype = d
        L.orc_smoothness.argtypes = [i, _dp, i, i]
        L.orc_generate.argtypes = [i, i, i, d, i, d, u64, _dp, _dp, _ip]
        L.orc_validate.argtypes = [_dp, _dp, i, i, i, i, d, d]
        L.orc_huber.restype = d
        L.orc_huber.argtypes = [d, d]
        L.orc_prox_huber.restype = d
        L.orc_prox_huber.argtypes = [d, d, d]
        L.orc_prox_step_column.argtypes = [_dp, _up, i, i, d, d, _dp]
        L.orc_conjugate_prox_column.argtypes = [_dp, _up, i, i, d, d, _dp]
        L.orc_conjugate_prox_column_generic.argtypes = [_dp, _up, i, i, d, d, _dp]
        L.orc_g_value.restype = d
        L.orc_g_value.argtypes = [_dp, _up, i, i, d]
        L.orc_g_conjugate.restype = d
        L.orc_g_conjugate.argtypes = [_dp, _up, i, i, d]
        L.orc_recover.argtypes = [_dp, _up, i, i, d, _dp, C.POINTER(d), C.POINTER(i)]
        L.orc_relax_cfg_default.argtypes = [C.POINTER(RelaxCfg)]
        L.orc_solver_cfg_default.argtypes = [C.POINTER(SolverCfg)]
        L.orc_relax_batch.argtypes = [_dp, _dp, i, i, i, d, d, C.POINTER(RelaxCfg), d, i,
                                      _up, _ip, _dp, _dp, _dp, _ip, _ip, TRACE_FN, vp,
                                      C.POINTER(i)]
        L.orc_round_support.argtypes = [_dp, _up, i, _ip, i, i, _ip]
        L.orc_select_branch.argtypes = [_dp, _up, i]
        L.orc_reoptimize.argtypes = [_dp, _dp, i, i, i, d, d, d, i, _ip, _ip, i, _dp, _dp]
        L.orc_auto_batch_size.argtypes = [u64, i, i, i, i]
        L.orc_solve.argtypes = [_dp, _dp, i, i, i, i, d, d, C.POINTER(SolverCfg),
                                C.POINTER(_Cert), DUAL_HOOK, BOUNDARY_HOOK, vp]
        L.orc_collect_rashomon.argtypes = [_dp, _dp, i, i, i, i, d, d, C.POINTER(SolverCfg),
                                           d, C.c_longlong, C.POINTER(_Cert),
                                           C.POINTER(vp)]
        L.orc_pool_size.argtypes = [vp]
        L.orc_pool_record.argtypes = [vp, i, _ip, _dp, C.POINTER(d)]
        L.orc_pool_free.argtypes = [vp]
        L.orc_use_openblas.argtypes = [C.c_char_p, i]
        _libs[_backend] = L
    return _libs[_backend]


def use_openblas(threads: int = 0) -> bool:
    """Route the oracle's GEMMs through numpy's bundled OpenBLAS (timing legs)."""
    import glob
    libs = glob.glob(os.path.join(os.path.dirname(np.__file__), "..", "numpy.libs",
                                  "libscipy_openblas64_*.so"))
    for path in libs:
        if lib().orc_use_openblas(path.encode(), threads):
            return True
    return False


# ------------------------------------------------------------------ scalars
def loss_value(loss, s, y):
    return lib().orc_loss_value(loss, s, y)


def loss_derivative(loss, s, y):
    return lib().orc_loss_derivative(loss, s, y)


def loss_conjugate(loss, z, y):
    return lib().orc_loss_conjugate(loss, z, y)


def huber(q, M):
    return lib().orc_huber(q, M)


def prox_huber(x, w, M):
    return lib().orc_prox_huber(x, w, M)


def smoothness(loss, X):
    X = np.asfortranarray(X, dtype=np.float64)
    n, p = X.shape
    return lib().orc_smoothness(loss, X.ravel(order="F"), n, p)


# ------------------------------------------------------------------ problem
@dataclass
class Instance:
    X: np.ndarray  # n x p, Fortran order
    y: np.ndarray
    loss: int
    k: int
    M: float = 2.0
    lambda2: float = 1.0
    support: Optional[List[int]] = None

    @property
    def n(self):
        return self.X.shape[0]

    @property
    def p(self):
        return self.X.shape[1]

    def xflat(self):
        return np.asfortranarray(self.X).ravel(order="F")


def generate(n, p, k, rho, loss, snr=5.0, seed=0, M=2.0, lambda2=1.0,
             reference_generator=False) -> Instance:
    """problem.hpp:70-132 generate_synthetic.

    The instance fixture is always oracle.c's restatement (AR(1) Cholesky
    factor in closed form), whose bytes equal the product's generator
    (tests/test_io_cpu.py), whatever the backend: every leg then sees the
    same X, y.  reference_generator=True runs the reference's own
    generate_synthetic (oracle/_ref; LLT through the shim), which agrees to
    rounding (tests/test_ref_cpu.py)."""
    X = np.zeros(n * p, dtype=np.float64)
    y = np.zeros(n, dtype=np.float64)
    sup = np.zeros(k, dtype=np.int32)
    with backend("ref" if reference_generator else "c"):
        rc = lib().orc_generate(n, p, k, rho, loss, snr, seed, X, y, sup)
    if rc != 0:
        raise ValueError("generator: invalid spec")
    return Instance(X.reshape(p, n).T, y, loss, k, M, lambda2, sup.tolist())


# ------------------------------------------------------------------ prox
def _st(st, p):
    if st is None:
        return np.zeros(p, dtype=np.uint8)
    return np.ascontiguousarray(st, dtype=np.uint8)


def prox_step_column(u, st, kbar, rho, M):
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros_like(u)
    lib().orc_prox_step_column(u, _st(st, len(u)), len(u), kbar, rho, M, out)
    return out


def conjugate_prox_column(x, st, kbar, w, M, generic=False):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    f = lib().orc_conjugate_prox_column_generic if generic else lib().orc_conjugate_prox_column
    f(x, _st(st, len(x)), len(x), kbar, w, M, out)
    return out


def g_value(beta, st, kbar, M):
    beta = np.ascontiguousarray(beta, dtype=np.float64)
    return lib().orc_g_value(beta, _st(st, len(beta)), len(beta), kbar, M)


def g_conjugate(q, st, kbar, M):
    q = np.ascontiguousarray(q, dtype=np.float64)
    return lib().orc_g_conjugate(q, _st(st, len(q)), len(q), kbar, M)


def recover(beta, st, kbar, M):
    beta = np.ascontiguousarray(beta, dtype=np.float64)
    z = np.zeros_like(beta)
    tau = C.c_double()
    cap = C.c_int()
    ok = lib().orc_recover(beta, _st(st, len(beta)), len(beta), kbar, M, z, C.byref(tau),
                           C.byref(cap))
    if not ok:
        raise ValueError("recover_indicators: beta infeasible for node domain")
    return z, tau.value, cap.value


def round_support(beta, st, fixed_one, kbar):
    beta = np.ascontiguousarray(beta, dtype=np.float64)
    p = len(beta)
    one = np.ascontiguousarray(list(fixed_one) or [0], dtype=np.int32)
    out = np.zeros(p + 1, dtype=np.int32)
    ln = lib().orc_round_support(beta, _st(st, p), p, one, len(fixed_one), kbar, out)
    return out[:ln].tolist()


def select_branch(beta, st):
    beta = np.ascontiguousarray(beta, dtype=np.float64)
    j = lib().orc_select_branch(beta, _st(st, len(beta)), len(beta))
    if j < 0:
        raise RuntimeError("select_branch_variable: no free coordinate")
    return j


def reoptimize(inst: Instance, supports: Sequence[Sequence[int]], smoothness_value=0.0,
               workers=1):
    offsets = np.zeros(len(supports) + 1, dtype=np.int32)
    for t, s in enumerate(supports):
        offsets[t + 1] = offsets[t] + len(s)
    idx = np.ascontiguousarray([j for s in supports for j in s] or [0], dtype=np.int32)
    coef = np.zeros(max(1, int(offsets[-1])), dtype=np.float64)
    obj = np.zeros(max(1, len(supports)), dtype=np.float64)
    lib().orc_reoptimize(inst.xflat(), inst.y, inst.n, inst.p, inst.loss, inst.M,
                         inst.lambda2, smoothness_value, len(supports), offsets, idx, workers,
                         coef, obj)
    return ([coef[offsets[t]:offsets[t + 1]].copy() for t in range(len(supports))],
            obj[:len(supports)].tolist())


# ------------------------------------------------------------------ relaxation
def relax_cfg(**kw) -> RelaxCfg:
    c = RelaxCfg()
    lib().orc_relax_cfg_default(C.byref(c))
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def relax_batch(inst: Instance, state: np.ndarray, kbar: Sequence[int], warm: np.ndarray,
                prune_threshold: float, cfg: Optional[RelaxCfg] = None,
                trace: Optional[Callable[[int, float], None]] = None):
    """relaxation.hpp:163-255.  state/warm are p x m (column per node)."""
    cfg = cfg or relax_cfg()
    p, m = warm.shape
    st = np.ascontiguousarray(np.asarray(state, dtype=np.uint8).T)  # m x p rows = columns
    wm = np.ascontiguousarray(np.asarray(warm, dtype=np.float64).T)
    beta = np.zeros((m, p), dtype=np.float64)
    bounds = np.zeros(m, dtype=np.float64)
    status = np.zeros(m, dtype=np.int32)
    iters = np.zeros(m, dtype=np.int32)
    err = C.c_int(-1)
    cb = TRACE_FN(lambda _u, b, psi: trace(b, psi)) if trace else TRACE_FN()
    rc = lib().orc_relax_batch(inst.xflat(), inst.y, inst.n, inst.p, inst.loss, inst.M,
                               inst.lambda2, C.byref(cfg), prune_threshold, m, st.ravel(),
                               np.ascontiguousarray(kbar, dtype=np.int32), wm.ravel(),
                               beta.ravel(), bounds, status, iters, cb, None, C.byref(err))
    if rc == 1:
        raise ValueError("solve_batch_relaxation: empty batch")
    if rc == 2:
        raise FloatingPointError(f"relaxation: non-finite iterate in column {err.value}")
    return beta.T.copy(), bounds, status, iters


# ------------------------------------------------------------------ engine
def solver_cfg(**kw) -> SolverCfg:
    c = SolverCfg()
    lib().orc_solver_cfg_default(C.byref(c))
    for k, v in kw.items():
        if k == "relax":
            for kk, vv in v.items():
                setattr(c.relax, kk, vv)
        else:
            setattr(c, k, v)
    return c


@dataclass
class Certificate:
    optimal_value: float
    support: List[int]
    coefficients: List[float]
    gap_percent: float
    lower_bound: float
    nodes_processed: int
    lb_batches: int
    reopt_batches: int
    batch_size_used: int
    profile: dict
    status: str


def _cert_buffers(k):
    sup = (C.c_int * (k + 1))()
    coef = (C.c_double * (k + 1))()
    cert = _Cert()
    cert.support = C.cast(sup, C.POINTER(C.c_int))
    cert.coefficients = C.cast(coef, C.POINTER(C.c_double))
    return cert, sup, coef


def _to_cert(cert) -> Certificate:
    L = cert.support_len
    return Certificate(
        cert.optimal_value, [cert.support[t] for t in range(L)],
        [cert.coefficients[t] for t in range(L)], cert.gap_percent, cert.lower_bound,
        cert.nodes_processed, cert.lb_batches, cert.reopt_batches, cert.batch_size_used,
        dict(lower_bound_seconds=cert.prof_lower_bound,
             reoptimization_seconds=cert.prof_reoptimization,
             transfer_seconds=cert.prof_transfer,
             branch_generate_seconds=cert.prof_branch_generate,
             total_seconds=cert.prof_total),
        "optimal" if cert.status == 0 else "time_limit")


def solve(inst: Instance, cfg: Optional[SolverCfg] = None, on_dual_bound=None,
          on_batch_boundary=None) -> Certificate:
    """bnb_engine.hpp:299-309."""
    cfg = cfg or solver_cfg()
    cert, _s, _c = _cert_buffers(inst.k)
    dh = (DUAL_HOOK(lambda _u, n0, j0, n1, j1, psi: on_dual_bound(
        [j0[t] for t in range(n0)], [j1[t] for t in range(n1)], psi))
          if on_dual_bound else DUAL_HOOK())
    bh = (BOUNDARY_HOOK(lambda _u, lb, ub: on_batch_boundary(lb, ub))
          if on_batch_boundary else BOUNDARY_HOOK())
    rc = lib().orc_solve(inst.xflat(), inst.y, inst.n, inst.p, inst.loss, inst.k, inst.M,
                         inst.lambda2, C.byref(cfg), C.byref(cert), dh, bh, None)
    if rc == 1:
        raise ValueError("invalid instance")
    if rc == 2:
        raise FloatingPointError(f"non-finite iterate in column {cert.err_column}")
    if rc == 3:
        raise RuntimeError("logic error")
    return _to_cert(cert)


def collect_rashomon(inst: Instance, cfg: Optional[SolverCfg] = None, epsilon=0.0, cap=-1):
    """rashomon.hpp:149-218; returns (certificate, [(sequence, coefs, objective)])."""
    cfg = cfg or solver_cfg()
    cert, _s, _c = _cert_buffers(inst.k)
    pool = C.c_void_p()
    rc = lib().orc_collect_rashomon(inst.xflat(), inst.y, inst.n, inst.p, inst.loss, inst.k,
                                    inst.M, inst.lambda2, C.byref(cfg), epsilon, cap,
                                    C.byref(cert), C.byref(pool))
    recs = []
    try:
        if rc != 0:
            raise RuntimeError(f"rashomon failed rc={rc}")
        seq = np.zeros(inst.k + 1, dtype=np.int32)
        coef = np.zeros(inst.k + 1, dtype=np.float64)
        obj = C.c_double()
        for t in range(lib().orc_pool_size(pool)):
            ln = lib().orc_pool_record(pool, t, seq, coef, C.byref(obj))
            recs.append((seq[:ln].tolist(), coef[:ln].copy(), obj.value))
    finally:
        lib().orc_pool_free(pool)
    return _to_cert(cert), recs


def auto_batch_size(budget, n, p, k, loss):
    return lib().orc_auto_batch_size(budget, n, p, k, loss)
